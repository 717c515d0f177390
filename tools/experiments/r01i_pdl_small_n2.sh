# PDL on the small-message kernels only: parity at n=2, C3 1 KiB..64 MiB (graph <= 1 MiB), bench N=2
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/i_multi2.log 2>&1; echo multi=$?; tail -1 gpurun_out/i_multi2.log
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
SMALL=$(python -c "print(','.join(str(1024<<k) for k in range(0,11,2)))")
MID=$(python -c "print(','.join(str(1024<<k) for k in range(11,17)))")
timeout 300 $R --master-port 29721 tools/sweep.py --dtype bf16 --sizes $SMALL --algos auto --graph --out gpurun_out/i_c3.jsonl > gpurun_out/i_c3.log 2>&1; echo small=$?
timeout 300 $R --master-port 29722 tools/sweep.py --dtype bf16 --sizes $MID --algos auto --out gpurun_out/i_c3.jsonl >> gpurun_out/i_c3.log 2>&1; echo mid=$?
timeout 300 $R --master-port 29723 tools/sweep.py --dtype bf16 --sizes $SMALL --algos auto --out gpurun_out/i_c3_eager.jsonl >> gpurun_out/i_c3.log 2>&1; echo smalleager=$?
HFR_PDL=0 timeout 300 $R --master-port 29724 tools/sweep.py --dtype bf16 --sizes $SMALL --algos auto --out gpurun_out/i_c3_eager_nopdl.jsonl >> gpurun_out/i_c3.log 2>&1; echo smalleager0=$?
python - <<'PY'
import json
for f in ("i_c3", "i_c3_eager", "i_c3_eager_nopdl"):
    rows = [json.loads(l) for l in open(f"gpurun_out/{f}.jsonl")]
    print(f, [(r["bytes"] >> 10, round(r["us"], 2), r["graph"]) for r in rows])
PY

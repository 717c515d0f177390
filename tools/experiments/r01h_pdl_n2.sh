# programmatic dependent launch A/B at n=2: parity (multi-GPU test), C3 sweep graphs <=1 MiB + eager, bench N=2
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/h_multi2.log 2>&1; echo multi=$?; tail -1 gpurun_out/h_multi2.log
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
SMALL=$(python -c "print(','.join(str(1024<<k) for k in range(0,11,2)))")
MID=$(python -c "print(','.join(str(1024<<k) for k in range(11,17)))")
for pdl in 1 0; do
  HFR_PDL=$pdl timeout 300 $R --master-port 2962$pdl tools/sweep.py --dtype bf16 --sizes $SMALL --algos auto --graph --out gpurun_out/h_c3_pdl$pdl.jsonl > gpurun_out/h_c3_$pdl.log 2>&1; echo small$pdl=$?
  HFR_PDL=$pdl timeout 300 $R --master-port 2963$pdl tools/sweep.py --dtype bf16 --sizes $MID --algos auto --out gpurun_out/h_c3_pdl$pdl.jsonl >> gpurun_out/h_c3_$pdl.log 2>&1; echo mid$pdl=$?
  HFR_PDL=$pdl timeout 300 $R --master-port 2964$pdl bench.py --gpus 2 --steps 20 --warmup 5 --no-variants --no-e2e > gpurun_out/h_bench_pdl$pdl.log 2>&1; echo bench$pdl=$?
done
python - <<'PY'
import json
for pdl in (1, 0):
    rows = [json.loads(l) for l in open(f"gpurun_out/h_c3_pdl{pdl}.jsonl")]
    print("pdl", pdl, [(r["bytes"] >> 10, round(r["us"], 2), r["graph"]) for r in rows])
    for l in open(f"gpurun_out/h_bench_pdl{pdl}.log"):
        if l.startswith("{"):
            d = json.loads(l); print("  bench", round(d["value"], 1), round(d["ms_per_step"] * 1e3, 1), "us")
PY

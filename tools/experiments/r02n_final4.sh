# round 2: final-binary evidence on a 4-GPU box — multi-process parity n=4 and n=2 (per-rank verdicts),
# bench N=4 and N=2, NVLink probe n=4 incl. TMA modes, C3 bf16 sweep AUTO vs NCCL at n=4
set -x
python -c "import __graft_entry__ as g; g.build()"
python -c "import bench; print(bench.source_sha())"
HFR_MULTI_OUT=gpurun_out/r02n_multi timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -rA > gpurun_out/r02n_multigpu_n4.log 2>&1; echo multi4=$?
tail -2 gpurun_out/r02n_multigpu_n4.log
CUDA_VISIBLE_DEVICES=0,1 HFR_MULTI_OUT=gpurun_out/r02n_multi timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -rA > gpurun_out/r02n_multigpu_n2.log 2>&1; echo multi2=$?
tail -2 gpurun_out/r02n_multigpu_n2.log
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $R --nproc-per-node 4 --master-port 29801 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r02n_bench_n4.log 2>&1; echo bench4=$?
grep '^{' gpurun_out/r02n_bench_n4.log | head -c 900; echo
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $R --nproc-per-node 2 --master-port 29802 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r02n_bench_n2.log 2>&1; echo bench2=$?
grep '^{' gpurun_out/r02n_bench_n2.log | head -c 900; echo
timeout 300 tools/p2p_probe 4 256 148 512 > gpurun_out/r02n_probe_n4.txt 2>&1; echo probe=$?
cat gpurun_out/r02n_probe_n4.txt
timeout 900 $R --nproc-per-node 4 --master-port 29803 tools/sweep.py --dtype bf16 --algos auto --nccl --sizes 1024,16384,262144,1048576,4194304,16777216,67108864,268435456,1073741824 --out gpurun_out/r02n_c3_n4.jsonl > gpurun_out/r02n_c3.log 2>&1; echo c3=$?
python - <<'PY'
import json
rows = {}
for l in open("gpurun_out/r02n_c3_n4.jsonl"):
    d = json.loads(l); rows.setdefault(d["bytes"], {})[d["impl"]] = d
for b, r in sorted(rows.items()):
    h, n = r.get("hfr"), r.get("nccl")
    print(b, "hfr us %.1f busbw %.1f" % (h["us"], h["busbw"]) if h else "-", "| nccl us %.1f busbw %.1f" % (n["us"], n["busbw"]) if n else "-")
PY

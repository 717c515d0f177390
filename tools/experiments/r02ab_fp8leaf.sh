# round 2: FP8 DBT leaves send raw values — parity + perf at n=4 (4-GPU box)
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_virtual.py -x -q -k "fp8 or e4m3 or e5m2 or tree_staging or tree_many" > gpurun_out/r02ab_tests.log 2>&1; echo tests=$?
tail -2 gpurun_out/r02ab_tests.log
timeout 600 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/r02ab_multi.log 2>&1; echo multi=$?
tail -1 gpurun_out/r02ab_multi.log
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for dt in e4m3 bf16; do
timeout 600 $R --master-port 29970 tools/sweep.py --dtype $dt --algos dbt,pair_dbt --sizes 67108864,1073741824 --out gpurun_out/r02ab_n4.jsonl > gpurun_out/r02ab_$dt.log 2>&1; echo $dt=$?
done
python - <<'PY'
import json
for l in open("gpurun_out/r02ab_n4.jsonl"):
    d = json.loads(l); print(d["dtype"], d["bytes"], d["algo"], round(d["busbw"], 1))
PY

timeout 900 python -m pytest tests/test_gpu_virtual.py -x -q -k "dbt" > gpurun_out/t4_v.log 2>&1; echo v=$?; grep -E "passed|FAILED|failed" gpurun_out/t4_v.log | tail -2
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/t4_m.log 2>&1; echo m=$?; grep -E "passed|FAILED|failed" gpurun_out/t4_m.log | tail -2
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 2 4; do
timeout 600 $R --nproc-per-node $N --master-port $((31000+N)) tools/sweep.py --sizes $((186<<20)) --algos dbt,pair_dbt --chunks 16384,32768,65536 --out gpurun_out/t4.jsonl > /dev/null 2>&1
timeout 600 $R --nproc-per-node $N --master-port $((31010+N)) tools/sweep.py --dtype bf16 --sizes $((1<<30)) --algos dbt,pair_dbt --out gpurun_out/t4.jsonl > /dev/null 2>&1
done
python -c "
import json
for l in open('gpurun_out/t4.jsonl'):
    x=json.loads(l); print(x['n'], x['dtype'], x['algo'], x['chunk'], x['bytes'], round(x['us'],1), round(x['busbw'],1))"

timeout 900 python -m pytest tests/test_gpu_virtual.py -x -q -k "pair or fuzz" > gpurun_out/pr_v.log 2>&1; echo v=$?; grep -E "passed|FAILED|failed" gpurun_out/pr_v.log | tail -2
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/pr_m.log 2>&1; echo m=$?; grep -E "passed|FAILED|failed" gpurun_out/pr_m.log | tail -2
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 2 4; do
timeout 600 $R --nproc-per-node $N --master-port $((31300+N)) tools/sweep.py --sizes $((186<<20)) --algos pair_dbt,dbt --chunks 16384,32768,65536 --out gpurun_out/pr.jsonl > /dev/null 2>&1
timeout 600 $R --nproc-per-node $N --master-port $((31310+N)) tools/sweep.py --dtype bf16 --sizes $((1<<30)) --algos pair_dbt --chunks 16384,32768,65536 --out gpurun_out/pr.jsonl > /dev/null 2>&1
done
python -c "
import json
for l in open('gpurun_out/pr.jsonl'):
    x=json.loads(l); print(x['n'], x['dtype'], x['algo'], x['chunk'], round(x['busbw'],1))"

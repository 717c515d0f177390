HFR_TMA_STORE=1 timeout 900 python -m pytest tests/test_gpu_virtual.py -x -q -k "(parity_sizes and flat) or (collectives and reduce_scatter) or (graph and flat)" > gpurun_out/ts_v.log 2>&1; echo v=$?; grep -E "passed|FAILED|failed|rror" gpurun_out/ts_v.log | tail -3
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for b in 1 0; do
HFR_TMA_STORE=$b timeout 300 python tools/sweep.py --virtual 8 --sizes $((186<<20)) --algos flat --out gpurun_out/ts_$b.jsonl > /dev/null 2>&1
for N in 2 4; do
HFR_TMA_STORE=$b timeout 600 $R --nproc-per-node $N --master-port $((30700+N+10*b)) tools/sweep.py --sizes $((186<<20)) --algos flat --out gpurun_out/ts_$b.jsonl > /dev/null 2>&1
HFR_TMA_STORE=$b timeout 600 $R --nproc-per-node $N --master-port $((30720+N+10*b)) tools/sweep.py --dtype bf16 --sizes $((1<<30)) --algos flat --out gpurun_out/ts_$b.jsonl > /dev/null 2>&1
done; done
HFR_TMA_STORE=1 timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/ts_m.log 2>&1; echo m=$?; grep -E "passed|FAILED|failed" gpurun_out/ts_m.log | tail -2
for b in 1 0; do python -c "
import json
for l in open('gpurun_out/ts_$b.jsonl'):
    x=json.loads(l); print('bulkstore=$b', x['n'], x['virtual'], x['dtype'], x['bytes'], round(x['us'],1), round(x['busbw'],1))"; done

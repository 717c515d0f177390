HFR_FLAT_TMA=1 timeout 900 python -m pytest tests/test_gpu_virtual.py -x -q -k "(parity_sizes and flat) or (collectives and reduce_scatter) or (c2_full and flat) or (graph and flat)" > gpurun_out/tma_v.log 2>&1; echo v=$?; grep -E "passed|FAILED|failed|rror" gpurun_out/tma_v.log | tail -5
for t in 1 0; do
HFR_FLAT_TMA=$t timeout 600 python tools/sweep.py --virtual 8 --sizes $((186<<20)) --algos flat --out gpurun_out/tma_$t.jsonl > /dev/null 2>&1
HFR_FLAT_TMA=$t timeout 600 python tools/sweep.py --virtual 4 --sizes $((186<<20)) --algos flat --out gpurun_out/tma_$t.jsonl > /dev/null 2>&1
done
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
HFR_FLAT_TMA=1 timeout 300 $R --nproc-per-node 2 --master-port 30501 tools/sweep.py --sizes $((1<<20)) --algos flat --out gpurun_out/tma_probe.jsonl > gpurun_out/tma_probe.log 2>&1; echo probe=$?; tail -3 gpurun_out/tma_probe.log
if [ -s gpurun_out/tma_probe.jsonl ]; then
for t in 1 0; do for N in 2 4; do
HFR_FLAT_TMA=$t timeout 600 $R --nproc-per-node $N --master-port $((30510+N+10*t)) tools/sweep.py --sizes $((186<<20)) --algos flat --out gpurun_out/tma_$t.jsonl > /dev/null 2>&1
HFR_FLAT_TMA=$t timeout 600 $R --nproc-per-node $N --master-port $((30530+N+10*t)) tools/sweep.py --dtype bf16 --sizes $((1<<30)) --algos flat --out gpurun_out/tma_$t.jsonl > /dev/null 2>&1
done; done
fi
for t in 1 0; do python -c "
import json
for l in open('gpurun_out/tma_$t.jsonl'):
    x=json.loads(l); print('tma=$t', x['n'], x['virtual'], x['dtype'], x['bytes'], round(x['us'],1), round(x['busbw'],1))"; done

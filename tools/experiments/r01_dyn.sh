timeout 900 python -m pytest tests/test_gpu_virtual.py -x -q -k "flat or collectives or graph" > gpurun_out/dy_v.log 2>&1; echo v=$?; grep -E "passed|FAILED" gpurun_out/dy_v.log | tail -3
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for d in 1 0; do
HFR_DYN_TILES=$d timeout 600 python tools/sweep.py --virtual 8 --sizes $((186<<20)) --algos flat --out gpurun_out/dy_$d.jsonl > /dev/null 2>&1
HFR_DYN_TILES=$d timeout 600 python tools/sweep.py --virtual 8 --sizes $((186<<20)) --algos flat --out gpurun_out/dy_$d.jsonl > /dev/null 2>&1
for N in 2 4; do
HFR_DYN_TILES=$d timeout 600 $R --nproc-per-node $N --master-port $((30300+N+10*d)) tools/sweep.py --sizes $((186<<20)) --algos flat --out gpurun_out/dy_$d.jsonl > /dev/null 2>&1
HFR_DYN_TILES=$d timeout 600 $R --nproc-per-node $N --master-port $((30320+N+10*d)) tools/sweep.py --dtype bf16 --sizes $((1<<30)) --algos flat --out gpurun_out/dy_$d.jsonl > /dev/null 2>&1
done; done
for d in 1 0; do python -c "
import json
for l in open('gpurun_out/dy_$d.jsonl'):
    x=json.loads(l); print('dyn=$d', x['n'], x['virtual'], x['dtype'], x['bytes'], round(x['us'],1), round(x['busbw'],1))"; done

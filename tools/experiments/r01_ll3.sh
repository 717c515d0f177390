timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/l3_pytest.log 2>&1; echo pytest=$?; grep -E "passed|FAILED|failed" gpurun_out/l3_pytest.log | tail -3
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
SZ=$(python -c "print(','.join(str(1024<<k) for k in range(0,14)))")
timeout 900 $R --nproc-per-node 4 --master-port 31421 tools/sweep.py --graph --iters 50 --dtype bf16 --sizes $SZ --algos auto --nccl --out gpurun_out/l3.jsonl > /dev/null 2>gpurun_out/l3.err; echo sw=$?
python -c "
import json
by={}
for l in open('gpurun_out/l3.jsonl'):
    d=json.loads(l); k=d['impl'] if d['impl']=='nccl' else d['algo']; by.setdefault(d['bytes'],{})[k]=round(d['us'],1)
for b in sorted(by): print(b, by[b])"

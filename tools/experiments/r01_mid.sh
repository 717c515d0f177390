R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
SZ=$(python -c "print(','.join(str(1024<<k) for k in range(6,16)))")
timeout 900 $R --nproc-per-node 4 --master-port 31401 tools/sweep.py --graph --iters 50 --dtype bf16 --sizes $SZ --algos auto,flat --nccl --out gpurun_out/mid_n4.jsonl > /dev/null 2>gpurun_out/mid.err; echo sw=$?
python -c "
import json
by={}
for l in open('gpurun_out/mid_n4.jsonl'):
    d=json.loads(l); k=d['impl'] if d['impl']=='nccl' else d['algo']; by.setdefault(d['bytes'],{})[k]=(round(d['us'],1), round(d['busbw'],1))
for b in sorted(by): print(b, by[b])"

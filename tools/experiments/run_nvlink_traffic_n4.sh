mkdir -p gpurun_out
nvidia-smi nvlink -s -i 0 > gpurun_out/nvlink_status.txt 2>&1
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512"
timeout 300 $T tools/nvlink_traffic.py 2> gpurun_out/nvlink_traffic_n4.err | grep "^{" > gpurun_out/nvlink_traffic_n4.jsonl; echo rc=$?
tail -5 gpurun_out/nvlink_traffic_n4.err
python -c "
import json
for l in open('gpurun_out/nvlink_traffic_n4.jsonl'):
    d=json.loads(l)
    if 'per_allreduce_bytes' in d:
        p=d['per_allreduce_bytes']; print(d['schedule'], d['rank'], {k:(None if v is None else round(v/d['bytes_per_rank'],3)) for k,v in p.items() if 'packets' not in k})
    else: print(d)
"

R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
i=0
for cfg in "flat 32 1 128" "flat 64 1 128" "flat 48 1 128" "flat 24 1 256" "flat 96 1 128" "nvls 48 1 128"; do
set -- $cfg; i=$((i+1))
timeout 900 $R --nproc-per-node 4 --master-port $((30410+i)) tools/ddp_overlap.py --algo $1 --max-ctas $2 --gate $3 --threads $4 2>gpurun_out/ddp4_$i.err | grep '^{' > gpurun_out/ddp4_$i.json
python -c "
import json; d=json.load(open('gpurun_out/ddp4_$i.json'))
print('$cfg', {k:round(d[k],3) for k in ('T_bwd_ms','T_comm_ms','T_both_ms','overlap','bwd_slowdown','comm_busbw')})" || tail -3 gpurun_out/ddp4_$i.err
done

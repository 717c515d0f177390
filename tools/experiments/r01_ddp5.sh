R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
i=0
for cfg in "flat 32 1 128" "flat 24 1 128" "flat 40 1 128" "flat 32 0 128"; do
set -- $cfg; i=$((i+1))
timeout 900 $R --nproc-per-node 4 --master-port $((30420+i)) tools/ddp_overlap.py --algo $1 --max-ctas $2 --gate $3 --threads $4 --reps 5 2>gpurun_out/ddp5_$i.err | grep '^{' > gpurun_out/ddp5_$i.json
python -c "
import json; d=json.load(open('gpurun_out/ddp5_$i.json'))
print('$cfg', {k:round(d[k],3) for k in ('T_bwd_ms','T_comm_ms','T_both_ms','overlap','bwd_slowdown','comm_busbw')}, [round(x*1e3,1) for x in d['reps']['bwd']], [round(x*1e3,1) for x in d['reps']['both']])" || tail -3 gpurun_out/ddp5_$i.err
done

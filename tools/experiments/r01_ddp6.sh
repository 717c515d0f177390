R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
i=0
for cfg in "32 128 1" "32 128 2" "16 256 2" "24 128 1"; do
set -- $cfg; i=$((i+1))
timeout 900 $R --nproc-per-node 4 --master-port $((30800+i)) tools/ddp_overlap.py --algo flat --max-ctas $1 --threads $2 --staging $3 --gate 1 --reps 5 2>gpurun_out/ddp6_$i.err | grep '^{' > gpurun_out/ddp6_$i.json
python -c "
import json; d=json.load(open('gpurun_out/ddp6_$i.json'))
print('$cfg', {k:round(d[k],3) for k in ('T_bwd_ms','T_comm_ms','T_both_ms','overlap','bwd_slowdown','comm_busbw')})" || tail -3 gpurun_out/ddp6_$i.err
done

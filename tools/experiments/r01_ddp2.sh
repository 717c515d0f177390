R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
i=0
for cfg in "flat 2 1" "flat 4 1" "flat 6 1" "nvls 4 1" "nvls 8 1" "nvls 16 1"; do
set -- $cfg; i=$((i+1))
timeout 900 $R --nproc-per-node 4 --master-port $((30010+i)) tools/ddp_overlap.py --algo $1 --max-ctas $2 --gate $3 2>gpurun_out/ddp2_$i.err | grep '^{' > gpurun_out/ddp2_$i.json
python -c "
import json; d=json.load(open('gpurun_out/ddp2_$i.json'))
print('$cfg', {k:round(d[k],3) for k in ('T_bwd_ms','T_comm_ms','T_both_ms','overlap','bwd_slowdown','comm_busbw')}, d['clocks']['both']['sm_mhz'], d['clocks']['bwd']['sm_mhz'])" || tail -3 gpurun_out/ddp2_$i.err
done

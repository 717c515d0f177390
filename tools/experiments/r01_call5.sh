bash tools/ncu_profile.sh
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $R --nproc-per-node 4 --master-port 29981 tools/ddp_overlap.py --max-ctas 8 --gate 1 --reps 5 2>/dev/null | grep '^{' > gpurun_out/ddp_clk.json
python -c "
import json; d=json.load(open('gpurun_out/ddp_clk.json'))
print({k:d[k] for k in ('T_bwd_ms','T_comm_ms','T_both_ms','overlap','bwd_slowdown')}); print(json.dumps(d['clocks']))"

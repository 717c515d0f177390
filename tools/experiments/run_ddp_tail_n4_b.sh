mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 tools/ddp_overlap.py"
F="--gate 1 --threads 128 --staging 1"
i=0
for args in "--max-ctas 32 $F --tail 0" "--max-ctas 32 $F --tail 1" "--max-ctas 40 $F --tail 1" "--max-ctas 24 $F --tail 1" \
            "--algo nvls --max-ctas 16 --gate 1 --tail 0" "--algo nvls --max-ctas 16 --gate 1 --tail 1 --tail-algo nvls" \
            "--algo nvls --max-ctas 8 --gate 1 --tail 1 --tail-algo nvls" "--algo nvls --max-ctas 24 --gate 1 --tail 1 --tail-algo nvls" \
            "--max-ctas 32 $F --tail 1"; do
  i=$((i+1)); timeout 200 $T $args > gpurun_out/ddpb_$i.log 2>&1; echo "$i rc=$?"
done
grep -h '^{' gpurun_out/ddpb_*.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['algo'],d['max_ctas'],d['tail'],'ov',round(d['overlap'],3),'pair',round(d['overlap_paired_median'],3),'min',round(d['overlap_min'],3),'slow',round(d['bwd_slowdown'],3),round(d['T_bwd_ms'],1),round(d['T_comm_ms'],1),round(d['T_both_ms'],1), d['clocks']['all']['sm_mhz'])"

# C5 DDP overlap with the final binary (1-CTA/SM tail default), 15 interleaved reps
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29811 tools/ddp_overlap.py"
timeout 200 $T --max-ctas 32 --gate 1 --threads 128 --staging 1 --tail 1 > gpurun_out/kddp_1.log 2>&1; echo flat=$?
timeout 200 $T --algo nvls --max-ctas 16 --gate 1 --tail 1 --tail-algo nvls > gpurun_out/kddp_2.log 2>&1; echo nvls=$?
grep -h '^{' gpurun_out/kddp_*.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['algo'],d['max_ctas'],d['tail'],'ov',round(d['overlap'],3),'pair',round(d['overlap_paired_median'],3),'min',round(d['overlap_min'],3),'slow',round(d['bwd_slowdown'],3),round(d['T_bwd_ms'],1),round(d['T_comm_ms'],1),round(d['T_both_ms'],1))"

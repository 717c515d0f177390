mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 tools/ddp_overlap.py"
C="--max-ctas 32 --gate 1 --threads 128 --staging 1"
timeout 150 $T $C --tail 0 > gpurun_out/ddp_a.log 2>&1; echo a=$?
timeout 150 $T $C --tail 1 > gpurun_out/ddp_b.log 2>&1; echo b=$?
timeout 150 $T --max-ctas 24 --gate 1 --threads 128 --staging 1 --tail 1 > gpurun_out/ddp_c.log 2>&1; echo c=$?
timeout 150 $T --max-ctas 16 --gate 1 --threads 128 --staging 1 --tail 1 > gpurun_out/ddp_d.log 2>&1; echo d=$?
timeout 150 $T --algo nvls --max-ctas 16 --gate 1 --tail 1 --tail-algo nvls > gpurun_out/ddp_e.log 2>&1; echo e=$?
timeout 400 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/multi4.log 2>&1; echo multi=$?
grep -h '^{' gpurun_out/ddp_*.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['algo'],d['max_ctas'],d['tail'],round(d['overlap'],3),round(d['overlap_paired_median'],3),round(d['bwd_slowdown'],3),round(d['T_bwd_ms'],1),round(d['T_comm_ms'],1),round(d['T_both_ms'],1))"
tail -3 gpurun_out/multi4.log

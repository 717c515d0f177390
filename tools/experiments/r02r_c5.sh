# round 2: C5 DDP, 32 CTAs x 128 vs 32 x 256 threads (register staging, stream gate, full-width tail), 3 runs each, interleaved
set -x
python -c "import __graft_entry__ as g; g.build()"
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
T="tools/ddp_overlap.py"
for i in 1 2 3; do
timeout 300 $R --master-port $((29840+i)) $T --max-ctas 32 --gate 1 --threads 128 --staging 1 --tail 1 2>/dev/null | grep '^{' > gpurun_out/r02r_t128_$i.json; echo t128_$i=$?
timeout 300 $R --master-port $((29850+i)) $T --max-ctas 32 --gate 1 --threads 256 --staging 1 --tail 1 2>/dev/null | grep '^{' > gpurun_out/r02r_t256_$i.json; echo t256_$i=$?
done
timeout 300 $R --master-port 29861 $T --max-ctas 24 --gate 1 --threads 256 --staging 1 --tail 1 2>/dev/null | grep '^{' > gpurun_out/r02r_c24t256.json; echo c24=$?
timeout 300 $R --master-port 29862 $T --max-ctas 40 --gate 1 --threads 256 --staging 1 --tail 1 2>/dev/null | grep '^{' > gpurun_out/r02r_c40t256.json; echo c40=$?
timeout 300 $R --master-port 29863 $T --max-ctas 32 --gate 1 --threads 512 --staging 1 --tail 1 2>/dev/null | grep '^{' > gpurun_out/r02r_c32t512.json; echo c32t512=$?
cat gpurun_out/r02r_*.json | python -c "
import sys,json
for l in sys.stdin:
    if not l.strip(): continue
    d=json.loads(l); print(d['max_ctas'],d['threads'],'ov',round(d['overlap'],3),'vsfull',round(d['overlap_vs_full'],3),'min',round(d['overlap_min'],3),'slow',round(d['bwd_slowdown'],3),'bwd',round(d['T_bwd_ms'],1),'comm',round(d['T_comm_ms'],1),'both',round(d['T_both_ms'],1),'full',round(d['T_comm_full_ms'],1))"

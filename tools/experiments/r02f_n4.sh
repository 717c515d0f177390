# round 2, 4-GPU box: NVLS+FLAT link-sharing probe, C5 DDP overlap (3x the
# round-1 config + TMA-staged variants, with the full-width T_comm), trees at n=4
set -x
python -c "import __graft_entry__ as g; g.build()"
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 600 $R --master-port 29641 tools/hybrid_probe.py --out gpurun_out/r02f_hybrid_n4.jsonl > gpurun_out/r02f_hybrid_f32.log 2>&1; echo hy1=$?
timeout 600 $R --master-port 29642 tools/hybrid_probe.py --dtype bf16 --bytes 1073741824 --out gpurun_out/r02f_hybrid_n4.jsonl > gpurun_out/r02f_hybrid_bf16.log 2>&1; echo hy2=$?
cat gpurun_out/r02f_hybrid_n4.jsonl
T="tools/ddp_overlap.py"
for i in 1 2 3; do
timeout 300 $R --master-port $((29650+i)) $T --max-ctas 32 --gate 1 --threads 128 --staging 1 --tail 1 2>gpurun_out/r02f_ddp_base$i.err | grep '^{' > gpurun_out/r02f_ddp_base$i.json; echo base$i=$?
done
timeout 300 $R --master-port 29661 $T --max-ctas 16 --gate 1 --staging 2 --tail 1 2>gpurun_out/r02f_ddp_tma16.err | grep '^{' > gpurun_out/r02f_ddp_tma16.json; echo tma16=$?
timeout 300 $R --master-port 29662 $T --max-ctas 32 --gate 1 --staging 2 --tail 1 2>gpurun_out/r02f_ddp_tma32.err | grep '^{' > gpurun_out/r02f_ddp_tma32.json; echo tma32=$?
timeout 300 $R --master-port 29663 $T --max-ctas 24 --gate 1 --threads 128 --staging 1 --tail 1 2>gpurun_out/r02f_ddp_reg24.err | grep '^{' > gpurun_out/r02f_ddp_reg24.json; echo reg24=$?
cat gpurun_out/r02f_ddp_*.json | python -c "
import sys,json
for l in sys.stdin:
    if not l.strip(): continue
    d=json.loads(l); print(d['max_ctas'],d['flat_staging'],d['threads'],'ov',round(d['overlap'],3),'vsfull',round(d['overlap_vs_full'],3),'min',round(d['overlap_min'],3),'slow',round(d['bwd_slowdown'],3),round(d['T_bwd_ms'],1),round(d['T_comm_ms'],1),round(d['T_both_ms'],1),round(d['T_comm_full_ms'],1))"
timeout 600 $R --master-port 29671 tools/sweep.py --algos dbt,pair_dbt --tree-staging 1,2 --sizes 195035136 --out gpurun_out/r02f_trees_n4.jsonl > gpurun_out/r02f_sweep_trees.log 2>&1; echo trees=$?
timeout 600 $R --master-port 29672 tools/sweep.py --dtype bf16 --algos dbt,pair_dbt --tree-staging 1,2 --sizes 1073741824 --out gpurun_out/r02f_trees_n4.jsonl > gpurun_out/r02f_sweep_trees2.log 2>&1; echo trees2=$?
cat gpurun_out/r02f_trees_n4.jsonl | cut -c1-300

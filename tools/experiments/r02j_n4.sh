# round 2, 4-GPU box: tree parity (in-place outputs) + n=2/n=4 tree sweeps, NVLS+FLAT link-sharing probe,
# C5 DDP overlap (3x round-1 config + TMA-staged variants, with the full-width T_comm)
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_virtual.py -x -q -k "tree_staging or tree_many or (parity_sizes and dbt) or (parity_fp8 and dbt) or c2_full_size or (distributions and dbt)" > gpurun_out/r02j_tree_tests.log 2>&1; echo trees=$?
tail -3 gpurun_out/r02j_tree_tests.log
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $R2 --master-port 29741 tools/sweep.py --algos dbt,pair_dbt --tree-staging 1,2 --tree-sync 0,40 --sizes 195035136 --out gpurun_out/r02j_trees.jsonl > gpurun_out/r02j_s1.log 2>&1; echo s1=$?
timeout 600 $R --master-port 29742 tools/sweep.py --algos dbt,pair_dbt --tree-staging 1,2 --tree-sync 0,40 --sizes 195035136 --out gpurun_out/r02j_trees.jsonl > gpurun_out/r02j_s2.log 2>&1; echo s2=$?
timeout 600 $R --master-port 29743 tools/sweep.py --dtype bf16 --algos dbt,pair_dbt --tree-staging 1,2 --sizes 1073741824 --out gpurun_out/r02j_trees.jsonl > gpurun_out/r02j_s3.log 2>&1; echo s3=$?
python - <<'PY'
import json
for l in open("gpurun_out/r02j_trees.jsonl"):
    d = json.loads(l); print(d["n"], d["dtype"], d["algo"], "staging", d["tree_staging"], "sync", d.get("tree_sync"), round(d["busbw"], 1))
PY
CUDA_VISIBLE_DEVICES=0,1 timeout 300 $R2 --master-port 29744 tools/tree_trace.py --algo dbt --chunk 32768 --ctas 0 --staging 2 --out gpurun_out/r02j_tr > gpurun_out/r02j_tr.log 2>&1; echo tr=$?
grep '^{' gpurun_out/r02j_tr.log
python tools/tree_trace.py --analyze gpurun_out/r02j_tr > gpurun_out/r02j_tr.json; rm -rf gpurun_out/r02j_tr
timeout 600 $R --master-port 29745 tools/hybrid_probe.py --out gpurun_out/r02j_hybrid_n4.jsonl > gpurun_out/r02j_hybrid_f32.log 2>&1; echo hy1=$?
timeout 600 $R --master-port 29746 tools/hybrid_probe.py --dtype bf16 --bytes 1073741824 --out gpurun_out/r02j_hybrid_n4.jsonl > gpurun_out/r02j_hybrid_bf16.log 2>&1; echo hy2=$?
cat gpurun_out/r02j_hybrid_n4.jsonl
T="tools/ddp_overlap.py"
for i in 1 2 3; do
timeout 300 $R --master-port $((29750+i)) $T --max-ctas 32 --gate 1 --threads 128 --staging 1 --tail 1 2>gpurun_out/r02j_ddp_base$i.err | grep '^{' > gpurun_out/r02j_ddp_base$i.json; echo base$i=$?
done
timeout 300 $R --master-port 29761 $T --max-ctas 16 --gate 1 --staging 2 --tail 1 2>gpurun_out/r02j_ddp_tma16.err | grep '^{' > gpurun_out/r02j_ddp_tma16.json; echo tma16=$?
timeout 300 $R --master-port 29762 $T --max-ctas 32 --gate 1 --staging 2 --tail 1 2>gpurun_out/r02j_ddp_tma32.err | grep '^{' > gpurun_out/r02j_ddp_tma32.json; echo tma32=$?
timeout 300 $R --master-port 29763 $T --max-ctas 24 --gate 1 --threads 128 --staging 1 --tail 1 2>gpurun_out/r02j_ddp_reg24.err | grep '^{' > gpurun_out/r02j_ddp_reg24.json; echo reg24=$?
cat gpurun_out/r02j_ddp_*.json | python -c "
import sys,json
for l in sys.stdin:
    if not l.strip(): continue
    d=json.loads(l); print(d['max_ctas'],d['flat_staging'],d['threads'],'ov',round(d['overlap'],3),'vsfull',round(d['overlap_vs_full'],3),'min',round(d['overlap_min'],3),'slow',round(d['bwd_slowdown'],3),round(d['T_bwd_ms'],1),round(d['T_comm_ms'],1),round(d['T_both_ms'],1),round(d['T_comm_full_ms'],1))"
tail -3 gpurun_out/r02j_ddp_base1.err

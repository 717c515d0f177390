# round 2: TMA tree kernel with role-sized stage rings, D groups in flight, no per-tile system fence (2-GPU box)
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_virtual.py -x -q -k "tree_staging or tree_many or (parity_sizes and dbt) or (parity_fp8 and dbt) or c2_full_size" > gpurun_out/r02h_tree_tests.log 2>&1; echo trees=$?
tail -4 gpurun_out/r02h_tree_tests.log
timeout 600 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/r02h_multi.log 2>&1; echo multi=$?
tail -3 gpurun_out/r02h_multi.log
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 600 $R --master-port 29721 tools/sweep.py --algos dbt,pair_dbt --tree-staging 1,2 --tree-sync 0,2 --sizes 195035136 --out gpurun_out/r02h_trees_n2.jsonl > gpurun_out/r02h_sweep.log 2>&1; echo sweep=$?
timeout 600 $R --master-port 29722 tools/sweep.py --dtype bf16 --algos dbt,pair_dbt --tree-staging 1,2 --sizes 1073741824,67108864 --out gpurun_out/r02h_trees_n2.jsonl > gpurun_out/r02h_sweep2.log 2>&1; echo sweep2=$?
timeout 600 $R --master-port 29723 tools/sweep.py --algos dbt,pair_dbt --tree-staging 2 --chunks 8192,16384,32768,65536,131072 --sizes 195035136 --out gpurun_out/r02h_trees_n2.jsonl > gpurun_out/r02h_sweep3.log 2>&1; echo sweep3=$?
python - <<'PY'
import json
for l in open("gpurun_out/r02h_trees_n2.jsonl"):
    d = json.loads(l); print(d["dtype"], d["bytes"], d["algo"], d["chunk"], d["tree_staging"], d.get("tree_sync"), round(d["busbw"], 1))
PY
timeout 300 $R --master-port 29724 tools/tree_trace.py --algo dbt --chunk 32768 --ctas 0 --staging 2 --out gpurun_out/r02h_tr > gpurun_out/r02h_tr.log 2>&1; echo tr=$?
grep '^{' gpurun_out/r02h_tr.log
python tools/tree_trace.py --analyze gpurun_out/r02h_tr > gpurun_out/r02h_tr.json; rm -rf gpurun_out/r02h_tr; head -c 2500 gpurun_out/r02h_tr.json
# ncu on rank 0 without torchrun (plain env:// rendezvous, rank 0 hosts the store)
export MASTER_ADDR=127.0.0.1 MASTER_PORT=29790 WORLD_SIZE=2
RANK=1 LOCAL_RANK=1 timeout 200 python -u tools/ncu_debug.py > gpurun_out/r02h_dbg_r1.log 2>&1 &
RANK=0 LOCAL_RANK=0 timeout 200 ncu --target-processes application-only -k regex:hfr_flat -s 3 -c 1 --metrics nvltx__bytes.sum,nvlrx__bytes.sum --csv --log-file gpurun_out/r02h_ncu_dbg.csv python -u tools/ncu_debug.py > gpurun_out/r02h_dbg_r0.log 2>&1; echo ncudbg=$?
wait
cat gpurun_out/r02h_dbg_r1.log gpurun_out/r02h_dbg_r0.log | grep -v "^\s" | head -40; cat gpurun_out/r02h_ncu_dbg.csv

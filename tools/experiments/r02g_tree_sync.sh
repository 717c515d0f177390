# round 2: TMA tree kernel — where the time goes (trace) and fence variants (2-GPU box); ncu stall debug
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_virtual.py -x -q -k "tree_staging" > gpurun_out/r02g_tree_tests.log 2>&1; echo trees=$?
tail -4 gpurun_out/r02g_tree_tests.log
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for sy in 0 1 3 7; do
timeout 300 $R --master-port $((29700+sy)) tools/tree_trace.py --algo dbt --chunk 32768 --ctas 0 --staging 2 --sync $sy --out gpurun_out/r02g_tr_s$sy > gpurun_out/r02g_tr_s$sy.log 2>&1; echo tr$sy=$?
grep '^{' gpurun_out/r02g_tr_s$sy.log
python tools/tree_trace.py --analyze gpurun_out/r02g_tr_s$sy > gpurun_out/r02g_tr_s$sy.json; head -c 1500 gpurun_out/r02g_tr_s$sy.json
done
timeout 300 $R --master-port 29710 tools/tree_trace.py --algo dbt --chunk 16384 --ctas 0 --staging 1 --out gpurun_out/r02g_tr_reg > gpurun_out/r02g_tr_reg.log 2>&1; echo trreg=$?
grep '^{' gpurun_out/r02g_tr_reg.log
python tools/tree_trace.py --analyze gpurun_out/r02g_tr_reg > gpurun_out/r02g_tr_reg.json
timeout 600 $R --master-port 29711 tools/sweep.py --algos dbt,pair_dbt --tree-staging 2 --tree-sync 0,1,2,3,6,7 --sizes 195035136 --out gpurun_out/r02g_sync_n2.jsonl > gpurun_out/r02g_sweep.log 2>&1; echo sweep=$?
cut -c1-330 gpurun_out/r02g_sync_n2.jsonl
timeout 180 $R --master-port 29712 --no-python bash -c 'if [ "$LOCAL_RANK" = 0 ]; then exec ncu --target-processes application-only -k regex:hfr_flat -s 3 -c 1 --metrics gpu__time_duration.sum --csv --log-file gpurun_out/r02g_ncu_dbg.csv python -u tools/ncu_debug.py; else exec python -u tools/ncu_debug.py; fi' > gpurun_out/r02g_ncu_dbg.log 2>&1; echo ncudbg=$?
grep -v "^\s" gpurun_out/r02g_ncu_dbg.log | head -40

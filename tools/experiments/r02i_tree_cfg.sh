# round 2: TMA tree kernel geometry sweep at n=2 (smem budget / tile / CTAs), role-split trace
set -x
python -c "import __graft_entry__ as g; g.build()"
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 $R --master-port 29731 tools/sweep.py --algos dbt,pair_dbt --tree-staging 2 --tree-sync 0,2,8,40,72,16,48 --ctas 0,148,296 --sizes 195035136 --out gpurun_out/r02i_cfg_n2.jsonl > gpurun_out/r02i_sweep.log 2>&1; echo sweep=$?
timeout 600 $R --master-port 29732 tools/sweep.py --dtype bf16 --algos dbt,pair_dbt --tree-staging 2 --tree-sync 0,8,40,72 --sizes 1073741824 --out gpurun_out/r02i_cfg_n2.jsonl > gpurun_out/r02i_sweep2.log 2>&1; echo sweep2=$?
python - <<'PY'
import json
for l in open("gpurun_out/r02i_cfg_n2.jsonl"):
    d = json.loads(l); print(d["dtype"], d["algo"], "sync", d.get("tree_sync"), "ctas", d["ctas"], round(d["busbw"], 1))
PY
timeout 300 $R --master-port 29734 tools/tree_trace.py --algo dbt --chunk 32768 --ctas 0 --staging 2 --out gpurun_out/r02i_tr > gpurun_out/r02i_tr.log 2>&1; echo tr=$?
grep '^{' gpurun_out/r02i_tr.log
python tools/tree_trace.py --analyze gpurun_out/r02i_tr > gpurun_out/r02i_tr.json; rm -rf gpurun_out/r02i_tr; cat gpurun_out/r02i_tr.json | head -80

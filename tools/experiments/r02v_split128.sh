# round 2: dedicated down-pass CTAs with 128-thread CTAs (4 resident per SM) vs the default (4-GPU box)
set -x
python -c "import __graft_entry__ as g; g.build()"
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 600 $R --master-port 29931 tools/sweep.py --algos dbt,pair_dbt --tree-staging 0,3 --threads 128,256 --sizes 195035136 --out gpurun_out/r02v.jsonl > gpurun_out/r02v_s1.log 2>&1; echo s1=$?
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $R2 --master-port 29932 tools/sweep.py --algos dbt,pair_dbt --tree-staging 0,3 --threads 128,256 --sizes 195035136 --out gpurun_out/r02v.jsonl > gpurun_out/r02v_s2.log 2>&1; echo s2=$?
python - <<'PY'
import json
for l in open("gpurun_out/r02v.jsonl"):
    d = json.loads(l); print(d["n"], d["dtype"], d["algo"], "thr", d["threads"], "staging", d["tree_staging"], round(d["busbw"], 1))
PY
grep -h "hfr error" gpurun_out/r02v_s*.log | head -3

# round 2: register tree with dedicated down-pass CTAs (tree_staging 3, experiment) vs default (4-GPU box)
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_virtual.py -x -q -k "tree_staging and (4096 or 8192)" > gpurun_out/r02q_tests.log 2>&1; echo tests=$?
tail -2 gpurun_out/r02q_tests.log
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 600 $R --master-port 29831 tools/sweep.py --algos dbt,pair_dbt --tree-staging 0,3 --sizes 195035136 --out gpurun_out/r02q.jsonl > gpurun_out/r02q_s1.log 2>&1; echo s1=$?
timeout 600 $R --master-port 29832 tools/sweep.py --algos dbt,pair_dbt --tree-staging 3 --chunks 8192,16384,65536 --sizes 195035136 --out gpurun_out/r02q.jsonl > gpurun_out/r02q_s2.log 2>&1; echo s2=$?
timeout 600 $R --master-port 29833 tools/sweep.py --dtype bf16 --algos dbt,pair_dbt --tree-staging 0,3 --sizes 1073741824 --out gpurun_out/r02q.jsonl > gpurun_out/r02q_s3.log 2>&1; echo s3=$?
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $R2 --master-port 29834 tools/sweep.py --algos dbt,pair_dbt --tree-staging 0,3 --sizes 195035136 --out gpurun_out/r02q.jsonl > gpurun_out/r02q_s4.log 2>&1; echo s4=$?
python - <<'PY'
import json
for l in open("gpurun_out/r02q.jsonl"):
    d = json.loads(l); print(d["n"], d["dtype"], d["bytes"], d["algo"], "chunk", d["chunk"], "staging", d["tree_staging"], round(d["busbw"], 1))
PY

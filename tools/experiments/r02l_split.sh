# round 2: register tree kernel with per-rank CTA split by role (4-GPU box)
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_virtual.py -x -q -k "dbt" > gpurun_out/r02l_tree_tests.log 2>&1; echo trees=$?
tail -3 gpurun_out/r02l_tree_tests.log
timeout 600 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/r02l_multi4.log 2>&1; echo multi=$?
tail -2 gpurun_out/r02l_multi4.log
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $R2 --master-port 29781 tools/sweep.py --algos dbt,pair_dbt,flat --sizes 195035136 --out gpurun_out/r02l_trees.jsonl > gpurun_out/r02l_s1.log 2>&1; echo s1=$?
timeout 900 $R --master-port 29782 tools/sweep.py --algos dbt,pair_dbt,flat --sizes 195035136 --chunks 0,16384,65536 --ctas 0,296,444,592 --out gpurun_out/r02l_trees.jsonl > gpurun_out/r02l_s2.log 2>&1; echo s2=$?
timeout 600 $R --master-port 29783 tools/sweep.py --dtype bf16 --algos dbt,pair_dbt,flat --sizes 1073741824,67108864 --out gpurun_out/r02l_trees.jsonl > gpurun_out/r02l_s3.log 2>&1; echo s3=$?
python - <<'PY'
import json
for l in open("gpurun_out/r02l_trees.jsonl"):
    d = json.loads(l); print(d["n"], d["dtype"], d["bytes"], d["algo"], "chunk", d["chunk"], "ctas", d["ctas"], round(d["busbw"], 1))
PY

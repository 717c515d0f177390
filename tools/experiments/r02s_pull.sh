# round 2: pull-based TMA tree (tree_staging 3) — parity, then n=2 / n=4 vs the register default (4-GPU box)
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_virtual.py -x -q -k "tree_staging or tree_many" > gpurun_out/r02s_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/r02s_tests.log
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 600 $R --master-port 29871 tools/sweep.py --algos dbt,pair_dbt --tree-staging 0,3 --sizes 195035136 --out gpurun_out/r02s.jsonl > gpurun_out/r02s_s1.log 2>&1; echo s1=$?
timeout 600 $R --master-port 29872 tools/sweep.py --dtype bf16 --algos dbt,pair_dbt --tree-staging 0,3 --sizes 1073741824 --out gpurun_out/r02s.jsonl > gpurun_out/r02s_s2.log 2>&1; echo s2=$?
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $R2 --master-port 29873 tools/sweep.py --algos dbt,pair_dbt --tree-staging 0,3 --sizes 195035136 --out gpurun_out/r02s.jsonl > gpurun_out/r02s_s3.log 2>&1; echo s3=$?
timeout 600 $R --master-port 29874 tools/sweep.py --algos dbt,pair_dbt --tree-staging 3 --ctas 148,444 --sizes 195035136 --out gpurun_out/r02s.jsonl > gpurun_out/r02s_s4.log 2>&1; echo s4=$?
python - <<'PY'
import json
for l in open("gpurun_out/r02s.jsonl"):
    d = json.loads(l); print(d["n"], d["dtype"], d["bytes"], d["algo"], "ctas", d["ctas"], "staging", d["tree_staging"], round(d["busbw"], 1))
PY
grep -h "hfr error" gpurun_out/r02s_s*.log | head -3
CUDA_VISIBLE_DEVICES=0,1 timeout 300 $R2 --master-port 29875 tools/tree_trace.py --algo dbt --chunk 32768 --ctas 0 --staging 3 --out gpurun_out/r02s_tr > gpurun_out/r02s_tr.log 2>&1; echo tr=$?
grep '^{' gpurun_out/r02s_tr.log
python tools/tree_trace.py --analyze gpurun_out/r02s_tr > gpurun_out/r02s_tr.json; rm -rf gpurun_out/r02s_tr; head -c 3000 gpurun_out/r02s_tr.json

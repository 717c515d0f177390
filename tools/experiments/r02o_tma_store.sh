# round 2: FLAT-TMA with bulk-copy result stores (flat_staging 3) vs plain stores (2): parity + A/B at n=1v/2/4
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_virtual.py -x -q -k "flat_staging or flat_tma_store or c2_bench" > gpurun_out/r02o_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/r02o_tests.log
timeout 600 python tools/sweep.py --virtual 8 --algos flat --flat-staging 2,3 --sizes 195035136 --out gpurun_out/r02o_ab.jsonl > gpurun_out/r02o_v8.log 2>&1; echo v8=$?
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $R2 --master-port 29811 tools/sweep.py --algos flat --flat-staging 2,3 --sizes 195035136,67108864 --out gpurun_out/r02o_ab.jsonl > gpurun_out/r02o_n2.log 2>&1; echo n2=$?
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $R2 --master-port 29812 tools/sweep.py --dtype bf16 --algos flat --flat-staging 2,3 --sizes 1073741824,16777216,4194304 --out gpurun_out/r02o_ab.jsonl > gpurun_out/r02o_n2b.log 2>&1; echo n2b=$?
timeout 600 $R --master-port 29813 tools/sweep.py --algos flat --flat-staging 2,3 --sizes 195035136,67108864 --out gpurun_out/r02o_ab.jsonl > gpurun_out/r02o_n4.log 2>&1; echo n4=$?
timeout 600 $R --master-port 29814 tools/sweep.py --dtype bf16 --algos flat --flat-staging 2,3 --sizes 1073741824,16777216,4194304 --out gpurun_out/r02o_ab.jsonl > gpurun_out/r02o_n4b.log 2>&1; echo n4b=$?
timeout 600 $R --master-port 29815 tools/sweep.py --algos flat --flat-staging 2,3 --sizes 195035136 --ctas 296 --out gpurun_out/r02o_ab.jsonl > gpurun_out/r02o_n4c.log 2>&1; echo n4c=$?
python - <<'PY'
import json
for l in open("gpurun_out/r02o_ab.jsonl"):
    d = json.loads(l); print(d["n"], "virt" if d["virtual"] else "", d["dtype"], d["bytes"], "staging", d["flat_staging"], "ctas", d["ctas"], round(d["busbw"], 1))
PY

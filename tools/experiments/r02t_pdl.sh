# round 2: PDL for the FLAT-TMA kernel (pdl_off 2, experiment) vs plain launches, back-to-back (4-GPU box)
set -x
python -c "import __graft_entry__ as g; g.build()"
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 600 $R --master-port 29881 tools/sweep.py --algos flat --pdl 0,2,0,2 --sizes 195035136,67108864 --out gpurun_out/r02t.jsonl > gpurun_out/r02t_s1.log 2>&1; echo s1=$?
timeout 600 $R --master-port 29882 tools/sweep.py --dtype bf16 --algos flat --pdl 0,2 --sizes 1073741824,268435456,16777216,4194304 --out gpurun_out/r02t.jsonl > gpurun_out/r02t_s2.log 2>&1; echo s2=$?
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $R2 --master-port 29883 tools/sweep.py --algos flat --pdl 0,2,0,2 --sizes 195035136,67108864 --out gpurun_out/r02t.jsonl > gpurun_out/r02t_s3.log 2>&1; echo s3=$?
python - <<'PY'
import json
for l in open("gpurun_out/r02t.jsonl"):
    d = json.loads(l); print(d["n"], d["dtype"], d["bytes"], "pdl_off", d["pdl_off"], round(d["us"], 1), round(d["busbw"], 1))
PY

# after the 1-CTA/SM FLAT-TMA default: RS / reduce (TMA users) at n=4 vs NCCL; C3 large sizes at n=2
mkdir -p gpurun_out
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for coll in reduce_scatter reduce; do
  timeout 300 $R --nproc-per-node 4 --master-port 29611 tools/sweep.py --coll $coll --dtype bf16 --sizes $((64<<20)),$((1<<30)) --algos flat --nccl --out gpurun_out/g_coll_n4.jsonl > gpurun_out/g_coll.log 2>&1; echo $coll=$?
done
LARGE=$(python -c "print(','.join(str(1024<<k) for k in range(11,21)))")
CUDA_VISIBLE_DEVICES=0,1 timeout 400 $R --nproc-per-node 2 --master-port 29612 tools/sweep.py --dtype bf16 --sizes $LARGE --algos auto --nccl --out gpurun_out/g_c3p_n2.jsonl > gpurun_out/g_c3p2.log 2>&1; echo c3n2=$?
for f in gpurun_out/g_coll_n4.jsonl gpurun_out/g_c3p_n2.jsonl; do python -c "
import json
for l in open('$f'):
    d = json.loads(l); print(d['impl'], d['coll'], d['n'], d['bytes'] >> 20, 'MiB', round(d['busbw'], 1))"; done

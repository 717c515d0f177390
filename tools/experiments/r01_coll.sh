R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
i=0
for c in reduce_scatter allgather reduce broadcast; do
i=$((i+1))
timeout 600 $R --nproc-per-node 4 --master-port $((30150+i)) tools/sweep.py --coll $c --dtype bf16 --sizes $((64<<20)),$((1<<30)) --algos flat --nccl --out gpurun_out/coll_n4.jsonl > /dev/null 2>gpurun_out/coll_$c.err || tail -3 gpurun_out/coll_$c.err
done
python -c "
import json
for l in open('gpurun_out/coll_n4.jsonl'):
    d=json.loads(l); print(d['coll'], d['impl'], d['bytes'], round(d['us'],1), round(d['busbw'],1))"

R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for il in 0 1; do
for N in 2 4; do
HFR_TREE_INTERLEAVE=$il timeout 600 $R --nproc-per-node $N --master-port $((31100+N+10*il)) tools/sweep.py --sizes $((186<<20)) --algos dbt,pair_dbt --chunks 16384,32768 --out gpurun_out/t5_$il.jsonl > /dev/null 2>&1
HFR_TREE_INTERLEAVE=$il timeout 600 $R --nproc-per-node $N --master-port $((31120+N+10*il)) tools/sweep.py --dtype bf16 --sizes $((1<<30)) --algos dbt,pair_dbt --chunks 16384,32768 --out gpurun_out/t5_$il.jsonl > /dev/null 2>&1
done; done
for il in 0 1; do python -c "
import json
for l in open('gpurun_out/t5_$il.jsonl'):
    x=json.loads(l); print('il=$il', x['n'], x['dtype'], x['algo'], x['chunk'], round(x['busbw'],1))"; done

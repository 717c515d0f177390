R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for c in 1 2 4 8 16; do
python bench.py --no-cpu --no-variants --soak 0 --e2e-chunks $c > gpurun_out/e2e_1_$c.json 2>/dev/null
timeout 600 $R --nproc-per-node 4 --master-port $((30910+c)) bench.py --gpus 4 --no-variants --no-nccl --soak 0 --e2e-chunks $c > gpurun_out/e2e_4_$c.json 2>/dev/null
timeout 600 $R --nproc-per-node 2 --master-port $((30940+c)) bench.py --gpus 2 --no-variants --no-nccl --soak 0 --e2e-chunks $c > gpurun_out/e2e_2_$c.json 2>/dev/null
for N in 1 2 4; do python -c "
import json; d=json.loads(open('gpurun_out/e2e_${N}_$c.json').read().strip().splitlines()[-1]); print('N=$N chunks=$c', round(d['e2e']['value'],1), round(d['e2e']['ms_per_step'],2))"; done
done

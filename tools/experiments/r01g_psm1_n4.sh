# after FLAT-TMA 1 CTA/SM for real comms: multi-GPU parity (n=4), bench N=4 and N=2, C3 large sizes at n=4
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/g_multi4.log 2>&1; echo multi=$?
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 400 $R --nproc-per-node 4 --master-port 29601 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/g_bench_n4.log 2>&1; echo b4=$?
CUDA_VISIBLE_DEVICES=0,1 timeout 400 $R --nproc-per-node 2 --master-port 29602 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/g_bench_n2.log 2>&1; echo b2=$?
LARGE=$(python -c "print(','.join(str(1024<<k) for k in range(11,21)))")
timeout 400 $R --nproc-per-node 4 --master-port 29603 tools/sweep.py --dtype bf16 --sizes $LARGE --algos auto --nccl --out gpurun_out/g_c3p_n4.jsonl > gpurun_out/g_c3p.log 2>&1; echo c3=$?
grep -h '^{' gpurun_out/g_bench_n*.log | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['n_gpus'], round(d['value'],1), 'nccl', d.get('nccl'), {k: round(v.get('busbw',0),1) for k, v in d.get('variants', {}).items()}, d['clocks'])"
python -c "
import json
for l in open('gpurun_out/g_c3p_n4.jsonl'):
    d = json.loads(l); print(d['impl'], d['bytes'] >> 20, 'MiB', round(d['busbw'], 1))"
tail -2 gpurun_out/g_multi4.log

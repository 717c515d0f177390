R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $R --nproc-per-node 4 --master-port 29995 tools/sweep.py --nvls $((2<<30)) --dtype bf16 --sizes $((64<<20)),$((256<<20)),$((1<<30)) --algos nvls --out gpurun_out/nv2_n4.jsonl > gpurun_out/nv2_n4.log 2>&1; echo sweep=$?
cut -c1-200 gpurun_out/nv2_n4.jsonl
for N in 2 4; do
timeout 900 $R --nproc-per-node $N --master-port $((29996+N)) bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/nv2_bench_n$N.json 2> gpurun_out/nv2_bench_n$N.err; echo bench$N=$?
python -c "
import json; d=json.loads(open('gpurun_out/nv2_bench_n$N.json').read().strip().splitlines()[-1])
print(d['n_gpus'], round(d['value'],1), d['roofline']['frac'], d['nccl']['busbw'], {k:v.get('busbw', v) for k,v in d['variants'].items()}, d['clocks'], d['e2e']['value'])"
done
tail -3 gpurun_out/nv2_bench_n4.err

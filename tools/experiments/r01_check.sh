python __graft_entry__.py smoke > gpurun_out/ck_smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/ck_smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ck_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/ck_pytest.log
python bench.py > gpurun_out/ck_bench_n1.json 2> gpurun_out/ck_bench_n1.err; echo b1=$?
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 2 4; do
timeout 900 $R --nproc-per-node $N --master-port $((30130+N)) bench.py --gpus $N > gpurun_out/ck_bench_n$N.json 2> gpurun_out/ck_bench_n$N.err; echo b$N=$?
done
python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/ck_ref_n1.json 2>gpurun_out/ck_ref.err; echo ref=$?
for f in gpurun_out/ck_bench_n1.json gpurun_out/ck_bench_n2.json gpurun_out/ck_bench_n4.json gpurun_out/ck_ref_n1.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1])
print(d.get('impl','hfr'), d['n_gpus'], round(d['value'],1), d.get('roofline',{}).get('frac'), (d.get('nccl') or {}).get('busbw'), {k:v.get('busbw', v) for k,v in (d.get('variants') or {}).items()}, d.get('clocks'), d['e2e']['value'], d['cpu_baseline']['value'] if d.get('cpu_baseline') else None)"; done

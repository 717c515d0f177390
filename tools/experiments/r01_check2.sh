python __graft_entry__.py smoke > gpurun_out/c2_smoke.log 2>&1; echo smoke=$?
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/c2_pytest.log 2>&1; echo pytest=$?; grep -E "passed|FAILED|failed" gpurun_out/c2_pytest.log | tail -3
python bench.py > gpurun_out/c2_bench_n1.json 2> gpurun_out/c2_bench_n1.err; echo b1=$?
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 2 4; do
timeout 900 $R --nproc-per-node $N --master-port $((30340+N)) bench.py --gpus $N > gpurun_out/c2_bench_n$N.json 2> gpurun_out/c2_bench_n$N.err; echo b$N=$?
done
for f in gpurun_out/c2_bench_n1.json gpurun_out/c2_bench_n2.json gpurun_out/c2_bench_n4.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1])
print(d['n_gpus'], round(d['value'],1), round(d['roofline']['frac'],3), (d.get('nccl') or {}).get('busbw'), {k:v.get('busbw', v) for k,v in (d.get('variants') or {}).items()}, d['clocks']['sm_mhz'], d['clocks']['reasons'], round(d['e2e']['value'],1))"; done
bash tools/ncu_profile.sh > /dev/null 2>&1; echo ncu=$?; ls gpurun_out/*.ncu-rep

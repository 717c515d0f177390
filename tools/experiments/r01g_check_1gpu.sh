# final 1-GPU checkpoint: smoke, full pytest -m gpu, bench N=1 (+ e2e pipeline depth 16), ncu launch list + full capture
mkdir -p gpurun_out
python __graft_entry__.py smoke > gpurun_out/g1_smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/g1_pytest.log 2>&1; echo pytest=$?; grep -E "passed|FAILED|failed" gpurun_out/g1_pytest.log | tail -3
python bench.py > gpurun_out/g1_bench_n1.json 2> gpurun_out/g1_bench_n1.err; echo b1=$?
python bench.py --no-cpu --no-variants --e2e-chunks 16 > gpurun_out/g1_bench_n1_e2e16.json 2> gpurun_out/g1_bench_n1_e2e16.err; echo b1e=$?
for f in gpurun_out/g1_bench_n1.json gpurun_out/g1_bench_n1_e2e16.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1])
print(d['n_gpus'], round(d['value'],1), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'], round(d['e2e']['value'],2), d['cpu_baseline'] and round(d['cpu_baseline']['value'],1))"; done
bash tools/ncu_profile.sh > /dev/null 2>&1; echo ncu=$?; ls gpurun_out/*.ncu-rep

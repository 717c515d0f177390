# 1-GPU checkpoint after PDL (small kernels): smoke, full pytest -m gpu, bench N=1, ncu launch list + full capture
mkdir -p gpurun_out
python __graft_entry__.py smoke > gpurun_out/j1_smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/j1_pytest.log 2>&1; echo pytest=$?; grep -E "passed|FAILED|failed" gpurun_out/j1_pytest.log | tail -3
python bench.py > gpurun_out/j1_bench_n1.json 2> gpurun_out/j1_bench_n1.err; echo b1=$?
for f in gpurun_out/j1_bench_n1.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1])
print(d['n_gpus'], round(d['value'],1), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'], round(d['e2e']['value'],2), d['cpu_baseline'] and round(d['cpu_baseline']['value'],1))"; done
bash tools/ncu_profile.sh > /dev/null 2>&1; echo ncu=$?; ls gpurun_out/*.ncu-rep

# round 2: bench schema test + N=1 bench with the final bench.py (1 GPU)
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_bench_schema.py tests/test_tools.py tests/test_abi.py -q -m "gpu or not gpu" > gpurun_out/r02aj_tests.log 2>&1; echo tests=$?
tail -2 gpurun_out/r02aj_tests.log
timeout 600 python bench.py > gpurun_out/r02aj_bench_n1.log 2>&1; echo bench=$?
grep '^{' gpurun_out/r02aj_bench_n1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['value'], r['frac'], r['traffic'], r['traffic_provenance'])"

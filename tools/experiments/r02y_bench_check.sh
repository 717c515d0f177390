# round 2: bench line after the config/clocks change (1 GPU): schema test + N=1 bench + reference arm
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_bench_schema.py -q > gpurun_out/r02y_schema.log 2>&1; echo schema=$?
tail -2 gpurun_out/r02y_schema.log
timeout 600 python bench.py > gpurun_out/r02y_bench_n1.log 2>&1; echo bench=$?
grep '^{' gpurun_out/r02y_bench_n1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['roofline']['traffic'], d['roofline']['traffic_provenance'], d['clocks'], d['config'])"
timeout 600 python bench.py --impl reference > gpurun_out/r02y_ref_n1.log 2>&1; echo ref=$?
grep '^{' gpurun_out/r02y_ref_n1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['config'])"

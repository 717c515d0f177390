# round 2: scale edge cases (negative, zero -> signed zeros, inf) for every schedule (1 GPU)
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_virtual.py -q -k "parity_scale" -rs > gpurun_out/r02am_tests.log 2>&1; echo tests=$?
tail -8 gpurun_out/r02am_tests.log

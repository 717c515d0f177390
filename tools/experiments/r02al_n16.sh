# round 2: parity with 11 and 16 virtual ranks (beyond one box) on one GPU
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_virtual.py -q -k "beyond_one_box" -rs > gpurun_out/r02al_tests.log 2>&1; echo tests=$?
tail -15 gpurun_out/r02al_tests.log

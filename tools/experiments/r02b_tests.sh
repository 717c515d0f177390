# round 2: full GPU suite on a 2-GPU box (virtual-rank tests on GPU 0 + the multi-process test)
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -m gpu -x -q -rs --durations=15 > gpurun_out/r02b_gpu_tests.log 2>&1; echo tests=$?
tail -30 gpurun_out/r02b_gpu_tests.log

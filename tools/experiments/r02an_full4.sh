# round 2 FINAL: the whole GPU suite on a 4-GPU box (virtual-rank tests on GPU 0 + the multi-process test at n=4)
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02an_smoke.log 2>&1; echo smoke=$?
python -c "import bench; print(bench.source_sha())"
HFR_MULTI_OUT=gpurun_out/r02an_multi timeout 2000 python -m pytest tests -m gpu -q -rs --durations=5 > gpurun_out/r02an_gpu_tests_4gpu.log 2>&1; echo tests=$?
tail -10 gpurun_out/r02an_gpu_tests_4gpu.log
timeout 300 python -m pytest tests -q -m "not gpu" > gpurun_out/r02an_cpu_tests.log 2>&1; echo cpu=$?
tail -1 gpurun_out/r02an_cpu_tests.log

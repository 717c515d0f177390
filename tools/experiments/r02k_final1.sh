# round 2: 1-GPU checkpoint with the current sources — full GPU suite, bench N=1, launch list,
# ncu --set full of the bench kernel (+ its source hash for profiles/traffic.json), compute-sanitizer
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02k_smoke.log 2>&1; echo smoke=$?
tail -3 gpurun_out/r02k_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -rs --durations=10 > gpurun_out/r02k_gpu_tests.log 2>&1; echo tests=$?
tail -6 gpurun_out/r02k_gpu_tests.log
B1="python bench.py --steps 20 --warmup 5"
timeout 600 $B1 > gpurun_out/r02k_bench_n1.log 2>&1; echo bench1=$?
grep '^{' gpurun_out/r02k_bench_n1.log | head -c 1200; echo
python -c "import bench; print(bench.source_sha())" > gpurun_out/r02k_source_sha.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r02k_launches_n1.csv $B1 > gpurun_out/r02k_ncu_launch.log 2>&1; echo launch=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hfr_flat_tma -s 3 -c 1 -o gpurun_out/r02k_flat_v8 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --soak 0 > gpurun_out/r02k_ncu_full.log 2>&1; echo full=$?
timeout 900 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 python -m pytest tests/test_gpu_virtual.py -x -q -k "parity_sizes and (4109 or 100003) and (f32 or bf16)" > gpurun_out/r02k_memcheck.log 2>&1; echo memcheck=$?
tail -5 gpurun_out/r02k_memcheck.log
timeout 600 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 python -m pytest tests/test_gpu_virtual.py -x -q -k "tree_staging and 300007 and f32" > gpurun_out/r02k_memcheck_tree.log 2>&1; echo memcheck_tree=$?
tail -5 gpurun_out/r02k_memcheck_tree.log

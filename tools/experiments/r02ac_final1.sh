# round 2 FINAL after FP8 raw leaves (1 GPU): build, smoke, full GPU suite, bench N=1, launch list, ncu full capture + source hash, reference arm
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02ac_smoke.log 2>&1; echo smoke=$?
python -c "import bench; print(bench.source_sha())" > gpurun_out/r02ac_source_sha.txt; cat gpurun_out/r02ac_source_sha.txt
timeout 1500 python -m pytest tests -m gpu -q -rs > gpurun_out/r02ac_gpu_tests.log 2>&1; echo tests=$?
tail -6 gpurun_out/r02ac_gpu_tests.log
B1="python bench.py --steps 20 --warmup 5"
timeout 600 $B1 > gpurun_out/r02ac_bench_n1.log 2>&1; echo bench1=$?
grep '^{' gpurun_out/r02ac_bench_n1.log | head -c 600; echo
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02ac_bench_ref_n1.log 2>&1; echo ref=$?
grep '^{' gpurun_out/r02ac_bench_ref_n1.log | head -c 400; echo
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r02ac_launches_n1.csv $B1 > gpurun_out/r02ac_ncu_launch.log 2>&1; echo launch=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hfr_flat_tma -s 3 -c 1 -o gpurun_out/r02ac_flat_v8 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --soak 0 > gpurun_out/r02ac_ncu_full.log 2>&1; echo full=$?
timeout 600 python bench.py > gpurun_out/r02ac_bench_after.log 2>&1; echo bench_after=$?

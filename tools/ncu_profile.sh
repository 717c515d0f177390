# ncu evidence for bench.py at N=1 (run under gpurun; one tool per call)
set -x
B="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --soak 0"
$B > gpurun_out/plain_flat.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:hfr_flat -s 3 -c 1 -o gpurun_out/prof_flat_v8 $B > gpurun_out/ncu_flat.log 2>&1
echo flat=$?
L="python bench.py --steps 20 --warmup 5"
$L > gpurun_out/plain_launch.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_n1.csv $L > gpurun_out/ncu_launch.log 2>&1
echo launches=$?

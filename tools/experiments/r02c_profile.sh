# round 2: GPU tests, then the bench at N=1 and N=2 with ncu evidence (2-GPU box)
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -m gpu -q -rs --durations=10 > gpurun_out/r02c_gpu_tests.log 2>&1; echo tests=$?
tail -15 gpurun_out/r02c_gpu_tests.log
B1="python bench.py --steps 20 --warmup 5"
timeout 600 $B1 > gpurun_out/r02c_bench_n1.log 2>&1; echo bench1=$?
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 $R --master-port 29611 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r02c_bench_n2.log 2>&1; echo bench2=$?
grep '^{' gpurun_out/r02c_bench_n2.log | head -c 3000
# launch list (N=1) and a full capture of the top kernel (N=1)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r02c_launches_n1.csv $B1 > gpurun_out/r02c_ncu_launch.log 2>&1; echo launch=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hfr_flat_tma -s 3 -c 1 -o gpurun_out/r02c_flat_v8 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --soak 0 > gpurun_out/r02c_ncu_full.log 2>&1; echo full=$?
ncu -i gpurun_out/r02c_flat_v8.ncu-rep --page raw --csv > gpurun_out/r02c_flat_v8_raw.csv 2>/dev/null; echo raw=$?
# N=2: NVLink + DRAM bytes of one FLAT-TMA launch on rank 0 (application replay, one pass each)
BN="bench.py --gpus 2 --steps 4 --warmup 3 --no-cpu --no-e2e --no-nccl --no-variants --soak 0"
timeout 600 $R --master-port 29612 --no-python bash tools/ncu_rank0.sh gpurun_out/r02c_nvl_n2.csv gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum hfr_flat_tma 5 $BN > gpurun_out/r02c_ncu_nvl_n2.log 2>&1; echo nvl=$?
timeout 600 $R --master-port 29613 --no-python bash tools/ncu_rank0.sh gpurun_out/r02c_dram_n2.csv gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum hfr_flat_tma 5 $BN > gpurun_out/r02c_ncu_dram_n2.log 2>&1; echo dram=$?
cat gpurun_out/r02c_nvl_n2.csv gpurun_out/r02c_dram_n2.csv | tail -20

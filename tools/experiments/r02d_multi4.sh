# round 2: 4-GPU box — multi-process parity at n=4 (per-rank verdicts kept),
# FP8 virtual parity, bench at N=4 and N=2, NVLink/DRAM bytes of one FLAT-TMA
# launch on rank 0 (single-pass kernel replay)
set -x
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()"
HFR_MULTI_OUT=gpurun_out/r02d_multi timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -rA > gpurun_out/r02d_multigpu_n4.log 2>&1; echo multi4=$?
tail -4 gpurun_out/r02d_multigpu_n4.log
CUDA_VISIBLE_DEVICES=0,1 HFR_MULTI_OUT=gpurun_out/r02d_multi timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -rA > gpurun_out/r02d_multigpu_n2.log 2>&1; echo multi2=$?
tail -4 gpurun_out/r02d_multigpu_n2.log
timeout 900 python -m pytest tests/test_gpu_virtual.py -k "fp8 or e4m3 or e5m2" -x -q -rA > gpurun_out/r02d_fp8_virtual.log 2>&1; echo fp8=$?
tail -4 gpurun_out/r02d_fp8_virtual.log
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $R --nproc-per-node 4 --master-port 29621 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r02d_bench_n4.log 2>&1; echo bench4=$?
grep '^{' gpurun_out/r02d_bench_n4.log | head -c 1500; echo
BN="bench.py --gpus 2 --steps 4 --warmup 3 --no-cpu --no-e2e --no-nccl --no-variants --no-probe --no-nvls --soak 0"
export CUDA_VISIBLE_DEVICES=0,1
timeout 300 $R --nproc-per-node 2 --master-port 29622 --no-python bash tools/ncu_rank0.sh gpurun_out/r02d_nvltx_n2.csv nvltx__bytes.sum hfr_flat_tma 5 $BN > gpurun_out/r02d_ncu_nvltx_n2.log 2>&1; echo nvltx=$?
tail -5 gpurun_out/r02d_ncu_nvltx_n2.log; cat gpurun_out/r02d_nvltx_n2.csv
timeout 300 $R --nproc-per-node 2 --master-port 29623 --no-python bash tools/ncu_rank0.sh gpurun_out/r02d_nvlrx_n2.csv nvlrx__bytes.sum hfr_flat_tma 5 $BN > gpurun_out/r02d_ncu_nvlrx_n2.log 2>&1; echo nvlrx=$?
cat gpurun_out/r02d_nvlrx_n2.csv
timeout 300 $R --nproc-per-node 2 --master-port 29624 --no-python bash tools/ncu_rank0.sh gpurun_out/r02d_dram_n2.csv dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum hfr_flat_tma 5 $BN > gpurun_out/r02d_ncu_dram_n2.log 2>&1; echo dram=$?
cat gpurun_out/r02d_dram_n2.csv
timeout 300 $R --nproc-per-node 2 --master-port 29625 --no-python bash tools/ncu_rank0.sh gpurun_out/r02d_nvlall_n2.csv nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,gpu__time_duration.sum hfr_flat_tma 5 $BN > gpurun_out/r02d_ncu_nvlall_n2.log 2>&1; echo nvlall=$?
cat gpurun_out/r02d_nvlall_n2.csv
unset CUDA_VISIBLE_DEVICES
BN4="bench.py --gpus 4 --steps 4 --warmup 3 --no-cpu --no-e2e --no-nccl --no-variants --no-probe --no-nvls --soak 0"
timeout 300 $R --nproc-per-node 4 --master-port 29626 --no-python bash tools/ncu_rank0.sh gpurun_out/r02d_nvlall_n4.csv nvltx__bytes.sum,nvlrx__bytes.sum,gpu__time_duration.sum hfr_flat_tma 5 $BN4 > gpurun_out/r02d_ncu_nvlall_n4.log 2>&1; echo nvlall4=$?
cat gpurun_out/r02d_nvlall_n4.csv

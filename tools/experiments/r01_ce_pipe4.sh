#!/bin/bash
# chunk-pipelined CE schedule at n=4 (and n=2 with 8 MiB chunks): sweeps, then parity
mkdir -p gpurun_out
T="timeout 120 torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29604"
$T tools/sweep.py --dtype bf16 --sizes 67108864,1073741824 --algos ce,flat --out gpurun_out/ce_pipe8_n4.jsonl > gpurun_out/ce_pipe.log 2>&1; echo "sweep4 rc=$?" >> gpurun_out/ce_pipe.log
$T tools/sweep.py --dtype f32 --sizes 195035136 --algos ce,flat --out gpurun_out/ce_pipe8_n4.jsonl >> gpurun_out/ce_pipe.log 2>&1; echo "sweep4 rc=$?" >> gpurun_out/ce_pipe.log
CUDA_VISIBLE_DEVICES=0,1 timeout 120 torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29605 tools/sweep.py --dtype f32 --sizes 67108864,195035136 --algos ce --out gpurun_out/ce_pipe8_n2.jsonl >> gpurun_out/ce_pipe.log 2>&1; echo "sweep2 rc=$?" >> gpurun_out/ce_pipe.log
timeout 300 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/ce_multi.log 2>&1; echo "multi rc=$?" >> gpurun_out/ce_multi.log

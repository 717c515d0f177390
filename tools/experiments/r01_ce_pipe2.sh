#!/bin/bash
# chunk-pipelined CE schedule at n=2: sweep first (short timeouts), then parity
mkdir -p gpurun_out
T="timeout 120 torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29602"
$T tools/sweep.py --dtype f32 --sizes 67108864,195035136 --algos ce,flat --out gpurun_out/ce_pipe_n2.jsonl > gpurun_out/ce_pipe.log 2>&1; echo "sweep rc=$?" >> gpurun_out/ce_pipe.log
$T tools/sweep.py --dtype bf16 --sizes 1073741824 --algos ce,flat --out gpurun_out/ce_pipe_n2.jsonl >> gpurun_out/ce_pipe.log 2>&1; echo "sweep rc=$?" >> gpurun_out/ce_pipe.log
timeout 240 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/ce_multi.log 2>&1; echo "multi rc=$?" >> gpurun_out/ce_multi.log

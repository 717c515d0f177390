#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_virtual.py -x -q -k "exhaustive" > gpurun_out/exh.log 2>&1; echo "rc=$?" >> gpurun_out/exh.log
T="timeout 300 torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29514"
$T tests/nccl_deviation.py --out gpurun_out/nccl_dev.jsonl > gpurun_out/nccl_dev.log 2>&1
NCCL_NVLS_ENABLE=0 $T tests/nccl_deviation.py --out gpurun_out/nccl_dev.jsonl >> gpurun_out/nccl_dev.log 2>&1
NCCL_ALGO=Ring $T tests/nccl_deviation.py --out gpurun_out/nccl_dev.jsonl >> gpurun_out/nccl_dev.log 2>&1

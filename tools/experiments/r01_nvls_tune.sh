#!/bin/bash
mkdir -p gpurun_out
T="timeout 300 torchrun --nproc-per-node 4 --master-addr 127.0.0.1"
$T --master-port 29971 tools/sweep.py --dtype bf16 --sizes 268435456,1073741824 --algos nvls --ctas 0,296,444 --threads 256,512 --nvls $((1100<<20)) --repeats 3 --out gpurun_out/nvls_tune.jsonl >> gpurun_out/nvls_tune.log 2>&1
NCCL_ALGO=NVLS $T --master-port 29972 tools/sweep.py --dtype bf16 --sizes 268435456,1073741824 --algos barrier --nccl --repeats 3 --out gpurun_out/nvls_tune_ncclnvls.jsonl >> gpurun_out/nvls_tune.log 2>&1

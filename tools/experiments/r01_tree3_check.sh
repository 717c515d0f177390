#!/bin/bash
mkdir -p gpurun_out
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_virtual.py -q -x -k "dbt or pair or fuzz or graph" > gpurun_out/t3_virtual.log 2>&1; echo "virtual rc=$?" >> gpurun_out/t3_virtual.log
timeout 400 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/t3_multi.log 2>&1; echo "multi rc=$?" >> gpurun_out/t3_multi.log
CUDA_VISIBLE_DEVICES=0,1 timeout 200 torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29921 tools/sweep.py --dtype f32 --sizes 195035136 --algos dbt,pair_dbt --out gpurun_out/t3_sweep.jsonl > gpurun_out/t3_sweep.log 2>&1
timeout 200 torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29922 tools/sweep.py --dtype f32 --sizes 195035136 --algos dbt,pair_dbt --out gpurun_out/t3_sweep.jsonl >> gpurun_out/t3_sweep.log 2>&1
timeout 200 torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29923 tools/sweep.py --dtype bf16 --sizes 1073741824 --algos dbt,pair_dbt --out gpurun_out/t3_sweep.jsonl >> gpurun_out/t3_sweep.log 2>&1

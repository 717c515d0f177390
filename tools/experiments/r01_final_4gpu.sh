#!/bin/bash
# round-end checkpoint on 4 GPUs: multi-GPU parity, bench N=2 and N=4
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/fin_multi.log 2>&1; echo "multi rc=$?" >> gpurun_out/fin_multi.log
CUDA_VISIBLE_DEVICES=0,1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29701 bench.py --gpus 2 > gpurun_out/fin_bench_n2.json 2> gpurun_out/fin_bench_n2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29702 bench.py --gpus 4 > gpurun_out/fin_bench_n4.json 2> gpurun_out/fin_bench_n4.err

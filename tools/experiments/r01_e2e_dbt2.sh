#!/bin/bash
mkdir -p gpurun_out
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > gpurun_out/e2e_bench_n1.json 2> gpurun_out/e2e_bench_n1.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29711 bench.py --gpus 2 > gpurun_out/e2e_bench_n2.json 2> gpurun_out/e2e_bench_n2.err

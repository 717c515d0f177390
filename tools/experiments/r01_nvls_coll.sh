#!/bin/bash
# NVLS collectives: parity (multi-GPU tests) + reduce/broadcast/RS/AG sweeps vs FLAT and NCCL (n=4)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/multi.log 2>&1; echo "multi rc=$?" >> gpurun_out/multi.log
T="timeout 300 torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512"
for coll in reduce broadcast reduce_scatter allgather; do
  $T tools/sweep.py --coll $coll --dtype bf16 --sizes 67108864,1073741824 --algos nvls,flat --nvls $((1100<<20)) --nccl --out gpurun_out/nvls_$coll.jsonl >> gpurun_out/nvls_coll.log 2>&1
done

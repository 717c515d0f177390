#!/bin/bash
# chunk-pipelined CE schedule: parity (multi-GPU tests) + CE vs FLAT sweeps at n=2 and n=4
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/ce_multi.log 2>&1; echo "multi rc=$?" >> gpurun_out/ce_multi.log
for n in 2 4; do
  T="timeout 300 torchrun --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600+n))"
  CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((n-1))) $T tools/sweep.py --dtype f32 --sizes 67108864,195035136 --algos flat,ce --out gpurun_out/ce_pipe_n$n.jsonl >> gpurun_out/ce_pipe.log 2>&1
  CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((n-1))) $T tools/sweep.py --dtype bf16 --sizes 1073741824 --algos flat,ce --out gpurun_out/ce_pipe_n$n.jsonl >> gpurun_out/ce_pipe.log 2>&1
done

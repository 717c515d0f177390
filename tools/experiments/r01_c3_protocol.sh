#!/bin/bash
# C3 (bf16, 1 KiB..1 GiB) under the SURVEY §8(d) protocol: 10 warm-ups, 5 repeats (median of max-over-ranks),
# CUDA graphs for <= 1 MiB, HFR AUTO vs NCCL, n=2 and n=4
mkdir -p gpurun_out
SMALL=$(python -c "print(','.join(str(1024<<k) for k in range(0,11)))")
LARGE=$(python -c "print(','.join(str(1024<<k) for k in range(11,21)))")
for n in 2 4; do
  V=$(seq -s, 0 $((n-1)))
  T="timeout 400 torchrun --nproc-per-node $n --master-addr 127.0.0.1"
  CUDA_VISIBLE_DEVICES=$V $T --master-port $((29950+n)) tools/sweep.py --dtype bf16 --sizes $SMALL --algos auto --graph --nccl --out gpurun_out/c3p_n$n.jsonl >> gpurun_out/c3p.log 2>&1
  CUDA_VISIBLE_DEVICES=$V $T --master-port $((29960+n)) tools/sweep.py --dtype bf16 --sizes $LARGE --algos auto --nccl --out gpurun_out/c3p_n$n.jsonl >> gpurun_out/c3p.log 2>&1
done

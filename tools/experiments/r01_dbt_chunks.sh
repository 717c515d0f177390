#!/bin/bash
mkdir -p gpurun_out
for n in 2 4; do
  CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((n-1))) timeout 300 torchrun --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29800+n)) tools/sweep.py --dtype f32 --sizes 195035136 --algos dbt --chunks 8192,12288,16384,24576 --ctas 0,148,444 --out gpurun_out/dbt_chunks.jsonl >> gpurun_out/dbt_chunks.log 2>&1
done

#!/bin/bash
mkdir -p gpurun_out
for rep in 1 2; do
timeout 300 torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29900+rep)) tools/sweep.py --dtype f32 --sizes 195035136 --algos dbt --chunks 24576,32768 --ctas 296,444,592 --threads 128,256 --out gpurun_out/dbt_ctas.jsonl >> gpurun_out/dbt_ctas.log 2>&1
done

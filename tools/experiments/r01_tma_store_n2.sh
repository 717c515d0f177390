#!/bin/bash
mkdir -p gpurun_out
T="timeout 200 torchrun --nproc-per-node 2 --master-addr 127.0.0.1"
for st in 0 1; do
  HFR_TMA_STORE=$st $T --master-port $((29980+st)) tools/sweep.py --dtype f32 --sizes 195035136 --algos flat --repeats 5 --out gpurun_out/tma_store_n2_$st.jsonl >> gpurun_out/tma_store.log 2>&1
  HFR_TMA_STORE=$st $T --master-port $((29982+st)) tools/sweep.py --dtype bf16 --sizes 1073741824 --algos flat --repeats 5 --out gpurun_out/tma_store_n2_$st.jsonl >> gpurun_out/tma_store.log 2>&1
  HFR_TMA_STORE=$st HFR_TMA_TILE=8192 $T --master-port $((29984+st)) tools/sweep.py --dtype bf16 --sizes 1073741824 --algos flat --repeats 5 --out gpurun_out/tma_store_n2_t8k_$st.jsonl >> gpurun_out/tma_store.log 2>&1
done

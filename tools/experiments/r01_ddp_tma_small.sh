#!/bin/bash
# C5 DDP overlap: small-smem TMA comm CTAs vs register staging (n=4)
mkdir -p gpurun_out
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
i=0
run() {  # tile ctas threads staging
  i=$((i+1))
  HFR_TMA_TILE=$1 timeout 600 $R --nproc-per-node 4 --master-port $((30600+i)) tools/ddp_overlap.py --max-ctas $2 --threads $3 --staging $4 --gate 1 --reps 3 2>gpurun_out/ddp5_$i.err | grep '^{' | sed "s/^{/{\"tma_tile\": $1, /" >> gpurun_out/ddp_tma_small.jsonl
}
run 4096 32 128 1
run 1024 32 128 0
run 2048 32 128 0
run 1024 64 128 0
run 1024 32 64 0
run 4096 32 128 1

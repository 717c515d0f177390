#!/bin/bash
# C5 DDP: pipelined CE vs FLAT, default vs 32 hardware work queues (CUDA_DEVICE_MAX_CONNECTIONS)
mkdir -p gpurun_out
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
i=0
run() {  # conn algo ctas threads staging gate
  i=$((i+1))
  CUDA_DEVICE_MAX_CONNECTIONS=$1 timeout 420 $R --nproc-per-node 4 --master-port $((30700+i)) tools/ddp_overlap.py --algo $2 --max-ctas $3 --threads $4 --staging $5 --gate $6 --reps 3 2>gpurun_out/ddp6_$i.err | grep '^{' | sed "s/^{/{\"conn\": $1, /" >> gpurun_out/ddp_ce_conn.jsonl
}
run 8 ce 16 0 0 0
run 32 ce 16 0 0 0
run 32 flat 32 128 1 1
run 32 ce 8 0 0 0

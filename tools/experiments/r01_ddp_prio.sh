#!/bin/bash
# C5 DDP: comm side stream priority (HFR_SIDE_PRIORITY=low) vs high, FLAT 32x128 registers + gate, NVLS 16
mkdir -p gpurun_out
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
i=0
run() {  # prio algo ctas threads staging gate nvls_extra
  i=$((i+1))
  HFR_SIDE_PRIORITY=$1 timeout 420 $R --nproc-per-node 4 --master-port $((30800+i)) tools/ddp_overlap.py --algo $2 --max-ctas $3 --threads $4 --staging $5 --gate $6 --reps 3 2>gpurun_out/ddp7_$i.err | grep '^{' | sed "s/^{/{\"prio\": \"$1\", /" >> gpurun_out/ddp_prio.jsonl
}
run low flat 32 128 1 1
run high flat 32 128 1 1
run low flat 48 128 1 1
run low nvls 16 0 0 1

#!/bin/bash
# reduce collective investigation: NVLink fan-in probes + reduce variants (n=4)
set -x
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/p2p_probe tools/p2p_probe.cu
timeout 120 /tmp/p2p_probe 4 256 148 512 > gpurun_out/probe_fanin.txt 2>&1
timeout 120 /tmp/p2p_probe 4 256 296 512 >> gpurun_out/probe_fanin.txt 2>&1
T="timeout 300 torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511"
$T tools/sweep.py --coll reduce --dtype bf16 --sizes 1073741824 --algos flat --out gpurun_out/red_tma.jsonl > gpurun_out/red.log 2>&1
HFR_FLAT_TMA=0 $T tools/sweep.py --coll reduce --dtype bf16 --sizes 1073741824 --algos flat --ctas 0,64,148,296 --threads 256,512 --out gpurun_out/red_reg.jsonl >> gpurun_out/red.log 2>&1
$T tools/sweep.py --coll reduce --dtype f32 --sizes 1073741824 --algos flat --ctas 0,148,444 --out gpurun_out/red_f32.jsonl >> gpurun_out/red.log 2>&1

nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/p2p_probe tools/p2p_probe.cu || exit 1
for n in 2 4; do for c in 148 64 32; do timeout 120 /tmp/p2p_probe $n 256 $c 512; done; done

nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/p2p_probe tools/p2p_probe.cu || exit 1
for n in 2 4; do
timeout 120 /tmp/p2p_probe $n 128 148 512
timeout 120 /tmp/p2p_probe $n 128 64 512
for f in 64 256 1024; do timeout 120 /tmp/p2p_probe $n 128 64 512 $f; timeout 120 /tmp/p2p_probe $n 128 148 512 $f; done
done

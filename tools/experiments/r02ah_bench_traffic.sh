# round 2: bench at N=2 / N=4 with the PM-sampled NVLink traffic records in place (final library)
set -x
python -c "import __graft_entry__ as g; g.build()"
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $R --nproc-per-node 4 --master-port 29951 bench.py --gpus 4 > gpurun_out/r02ah_bench_n4.log 2>&1; echo b4=$?
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $R --nproc-per-node 2 --master-port 29952 bench.py --gpus 2 > gpurun_out/r02ah_bench_n2.log 2>&1; echo b2=$?
for n in 2 4; do grep '^{' gpurun_out/r02ah_bench_n$n.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print($n, d['value'], r['frac'], r['traffic'], r.get('traffic_wire'), r.get('dram_traffic'), r['traffic_provenance'])"; done

# round 2: run-to-run spread of the final bench lines (3x N=4, 3x N=2, 3x N=1 on one 4-GPU lease)
set -x
python -c "import __graft_entry__ as g; g.build()"
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for i in 1 2 3; do
timeout 600 $R --nproc-per-node 4 --master-port $((29970+i)) bench.py --gpus 4 --no-cpu --no-e2e > gpurun_out/r02ak_n4_$i.log 2>&1; echo n4_$i=$?
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $R --nproc-per-node 2 --master-port $((29980+i)) bench.py --gpus 2 --no-cpu --no-e2e > gpurun_out/r02ak_n2_$i.log 2>&1; echo n2_$i=$?
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/r02ak_n1_$i.log 2>&1; echo n1_$i=$?
done
for f in gpurun_out/r02ak_n*.log; do grep '^{' $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', d['n_gpus'], round(d['value'],1), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done

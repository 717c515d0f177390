python __graft_entry__.py smoke > gpurun_out/ll_smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests/test_gpu_virtual.py -x -q > gpurun_out/ll_pytest.log 2>&1; echo pytest_v=$?; tail -2 gpurun_out/ll_pytest.log
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/ll_multi.log 2>&1; echo pytest_m=$?; tail -2 gpurun_out/ll_multi.log
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
SZ=$(python -c "print(','.join(str(1024<<k) for k in range(0,11)))")
timeout 900 $R --nproc-per-node 4 --master-port 30051 tools/sweep.py --graph --iters 100 --dtype bf16 --sizes $SZ --algos barrier,oneshot,flat --nccl --out gpurun_out/ll_graph_n4.jsonl > /dev/null 2>gpurun_out/ll_graph_n4.err; echo graph=$?
python -c "
import json
by={}
for l in open('gpurun_out/ll_graph_n4.jsonl'):
    d=json.loads(l); k=d['impl'] if d['impl']=='nccl' else d['algo']; by.setdefault(d['bytes'],{})[k]=round(d['us'],2)
for b in sorted(by): print(b, by[b])"

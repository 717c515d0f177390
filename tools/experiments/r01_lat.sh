timeout 900 python -m pytest tests/test_gpu_virtual.py -x -q -k "oneshot or graph or distributions" > gpurun_out/l_pytest.log 2>&1; echo pytest_v=$?; tail -2 gpurun_out/l_pytest.log
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/l_pytest_multi.log 2>&1; echo pytest_m=$?; tail -2 gpurun_out/l_pytest_multi.log
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 2; do
timeout 900 $R --nproc-per-node $N --master-port $((29700+N)) tools/sweep.py --graph --iters 100 --dtype bf16 --sizes 1024,65536,1048576 --algos barrier,oneshot,flat --out gpurun_out/l_graph_n$N.jsonl > /dev/null 2>gpurun_out/l_graph_n$N.err; echo graph_$N=$?
done
python -c "
import json
for l in open('gpurun_out/l_graph_n2.jsonl'):
    d=json.loads(l); print(d['algo'], d['bytes'], round(d['us'],2))"

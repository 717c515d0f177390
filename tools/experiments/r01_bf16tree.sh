timeout 900 python -m pytest tests/test_gpu_virtual.py -x -q -k "dbt" > gpurun_out/bt_pytest.log 2>&1; echo pytest=$?; tail -1 gpurun_out/bt_pytest.log
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/bt_multi.log 2>&1; echo multi=$?; tail -1 gpurun_out/bt_multi.log
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 2 4; do
timeout 900 $R --nproc-per-node $N --master-port $((30140+N)) tools/sweep.py --dtype bf16 --sizes $((64<<20)),$((1<<30)) --algos flat,dbt,pair_dbt --out gpurun_out/bt_n$N.jsonl > /dev/null 2>&1
done
cat gpurun_out/bt_n*.jsonl | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['n'], d['algo'], d['bytes'], round(d['us'],1), round(d['busbw'],1))"

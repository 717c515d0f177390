set -x
timeout 900 python -m pytest tests/test_gpu_virtual.py -x -q -k "parity_sizes or c2_full or distributions" > gpurun_out/sw_pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/sw_pytest.log
S=$((186<<20))
timeout 600 python tools/sweep.py --virtual 8 --sizes $S --algos flat --threads 256,512 --ctas 0 --out gpurun_out/sw_v8.jsonl > /dev/null 2>gpurun_out/sw_v8.err
timeout 600 python tools/sweep.py --virtual 8 --sizes $S --algos dbt,pair_dbt --chunks 8192,32768,131072 --out gpurun_out/sw_v8.jsonl > /dev/null 2>>gpurun_out/sw_v8.err
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$N tools/sweep.py --sizes $S --algos flat --ctas 0,16,32,64,96 --threads 256,512 --nccl --out gpurun_out/sw_n$N.jsonl > /dev/null 2>gpurun_out/sw_n$N.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2952$N tools/sweep.py --sizes $S --algos dbt,pair_dbt --chunks 8192,32768,131072 --out gpurun_out/sw_n$N.jsonl > /dev/null 2>>gpurun_out/sw_n$N.err
done
cat gpurun_out/sw_*.jsonl | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['impl'],d['n'],d.get('algo',''),d.get('chunk',''),d.get('ctas',''),d.get('threads',''),round(d['us'],1),round(d['busbw'],1))"

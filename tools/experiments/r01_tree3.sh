timeout 900 python -m pytest tests/test_gpu_virtual.py -x -q -k "dbt" > gpurun_out/t3_pytest.log 2>&1; echo pytest=$?; tail -1 gpurun_out/t3_pytest.log
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
S=$((186<<20))
timeout 900 $R --nproc-per-node 4 --master-port 30121 tools/sweep.py --sizes $S --algos dbt,pair_dbt --chunks 16384,32768,65536 --ctas 148,296 --threads 256 --out gpurun_out/t3.jsonl > /dev/null 2>&1
timeout 900 $R --nproc-per-node 4 --master-port 30122 tools/sweep.py --sizes $S --algos dbt,pair_dbt --chunks 16384,65536 --ctas 296,592 --threads 128 --out gpurun_out/t3.jsonl > /dev/null 2>&1
timeout 900 $R --nproc-per-node 4 --master-port 30123 tools/sweep.py --sizes $S --algos dbt,pair_dbt --chunks 65536 --ctas 0 --threads 512 --out gpurun_out/t3.jsonl > /dev/null 2>&1
python -c "
import json
for l in open('gpurun_out/t3.jsonl'):
    d=json.loads(l); print(d['algo'], d['chunk'], d['ctas'], d['threads'], round(d['us'],1), round(d['busbw'],1))"

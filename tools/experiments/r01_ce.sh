timeout 900 python -m pytest tests/test_gpu_virtual.py -x -q -k "dbt or graph" > gpurun_out/c_pytest.log 2>&1; echo pytest_v=$?; tail -2 gpurun_out/c_pytest.log
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/c_pytest_multi.log 2>&1; echo pytest_m=$?; tail -5 gpurun_out/c_pytest_multi.log
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
S=$((186<<20))
timeout 900 $R --nproc-per-node 4 --master-port 29801 tools/sweep.py --sizes $S --algos dbt,pair_dbt --chunks 16384,32768,65536 --ctas 32,64,148 --out gpurun_out/c_tree_n4.jsonl > /dev/null 2>gpurun_out/c_tree_n4.err; echo tree=$?
timeout 900 $R --nproc-per-node 4 --master-port 29802 tools/sweep.py --dtype bf16 --sizes $((64<<20)),$S,$((1<<30)) --algos flat,ce --ctas 8,16,32,0 --out gpurun_out/c_ce_n4.jsonl > /dev/null 2>gpurun_out/c_ce_n4.err; echo ce=$?
for c in 8 16; do
timeout 900 $R --nproc-per-node 4 --master-port $((29810+c)) tools/ddp_overlap.py --algo ce --max-ctas $c > gpurun_out/c_ddp_ce_c$c.json 2> gpurun_out/c_ddp_ce_c$c.err; echo ddp=$?; cut -c1-420 gpurun_out/c_ddp_ce_c$c.json; tail -2 gpurun_out/c_ddp_ce_c$c.err
done
python -c "
import json
for f in ('gpurun_out/c_tree_n4.jsonl','gpurun_out/c_ce_n4.jsonl'):
    for l in open(f):
        d=json.loads(l); print(d['algo'], d['bytes'], d.get('chunk'), d.get('ctas'), round(d['us'],1), round(d['busbw'],1))"

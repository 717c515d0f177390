timeout 900 python -m pytest tests/test_gpu_virtual.py -x -q -k "oneshot or staged or async or golden" > gpurun_out/s2_pytest.log 2>&1; echo pytest_v=$?; tail -2 gpurun_out/s2_pytest.log
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/s2_pytest_multi.log 2>&1; echo pytest_m=$?; tail -2 gpurun_out/s2_pytest_multi.log
S=$((186<<20))
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $R --nproc-per-node 4 --master-port 29541 tools/sweep.py --sizes $S --algos dbt,pair_dbt --chunks 8192,16384,32768,65536 --ctas 16,32,64 --out gpurun_out/s2_tree_n4.jsonl > /dev/null 2>gpurun_out/s2_tree_n4.err; echo tree=$?
SZ=$(python -c "print(','.join(str(1024<<k) for k in range(21)))")
for N in 2 4; do
timeout 900 $R --nproc-per-node $N --master-port 2955$N tools/sweep.py --dtype bf16 --sizes $SZ --algos auto --nccl --out gpurun_out/s2_c3_n$N.jsonl > /dev/null 2>gpurun_out/s2_c3_n$N.err; echo c3_$N=$?
timeout 900 $R --nproc-per-node $N --master-port 2956$N tools/sweep.py --dtype bf16 --sizes $(python -c "print(','.join(str(1024<<k) for k in range(0,12)))") --algos flat,oneshot --out gpurun_out/s2_c3_n$N.jsonl > /dev/null 2>>gpurun_out/s2_c3_n$N.err; echo c3b_$N=$?
done
for c in 8 16 32; do
timeout 900 $R --nproc-per-node 4 --master-port 2957$c tools/ddp_overlap.py --max-ctas $c > gpurun_out/s2_ddp_n4_c$c.json 2> gpurun_out/s2_ddp_n4_c$c.err; echo ddp=$?; cat gpurun_out/s2_ddp_n4_c$c.json | cut -c1-400
done

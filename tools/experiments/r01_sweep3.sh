timeout 1200 python -m pytest tests/test_gpu_virtual.py -x -q > gpurun_out/s3_pytest.log 2>&1; echo pytest_v=$?; tail -2 gpurun_out/s3_pytest.log
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/s3_pytest_multi.log 2>&1; echo pytest_m=$?; tail -2 gpurun_out/s3_pytest_multi.log
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
SZ=$(python -c "print(','.join(str(1024<<k) for k in range(0,13)))")
for N in 2 4; do
timeout 900 $R --nproc-per-node $N --master-port $((29600+N)) tools/sweep.py --graph --iters 100 --dtype bf16 --sizes $SZ --algos oneshot,flat --nccl --out gpurun_out/s3_graph_n$N.jsonl > /dev/null 2>gpurun_out/s3_graph_n$N.err; echo graph_$N=$?
done
for c in 16 32; do
timeout 900 $R --nproc-per-node 4 --master-port $((29610+c)) tools/ddp_overlap.py --max-ctas $c > gpurun_out/s3_ddp_n4_c$c.json 2> gpurun_out/s3_ddp_n4_c$c.err; echo ddp=$?; cut -c1-420 gpurun_out/s3_ddp_n4_c$c.json
done

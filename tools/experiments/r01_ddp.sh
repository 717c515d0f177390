timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/ddp_pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/ddp_pytest.log
for c in 16 32; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533 tools/ddp_overlap.py --max-ctas $c > gpurun_out/ddp_n4_c$c.json 2> gpurun_out/ddp_n4_c$c.err; echo ddp=$?; cat gpurun_out/ddp_n4_c$c.json; tail -3 gpurun_out/ddp_n4_c$c.err
done

timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/nv_multi.log 2>&1; echo multi=$?; tail -3 gpurun_out/nv_multi.log
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $R --nproc-per-node 4 --master-port 29991 tools/sweep.py --nvls $((2<<30)) --dtype bf16 --sizes $((64<<20)),$((256<<20)),$((1<<30)) --algos nvls,flat --nccl --out gpurun_out/nv_sweep_n4.jsonl > gpurun_out/nv_sweep_n4.log 2>&1; echo sweep=$?
timeout 900 $R --nproc-per-node 4 --master-port 29992 tools/sweep.py --nvls $((1<<30)) --dtype f32 --sizes $((186<<20)) --algos nvls,flat --nccl --out gpurun_out/nv_sweep_n4.jsonl >> gpurun_out/nv_sweep_n4.log 2>&1; echo sweep=$?
timeout 900 $R --nproc-per-node 2 --master-port 29993 tools/sweep.py --nvls $((2<<30)) --dtype bf16 --sizes $((64<<20)),$((1<<30)) --algos nvls,flat --nccl --out gpurun_out/nv_sweep_n2.jsonl > gpurun_out/nv_sweep_n2.log 2>&1; echo sweep=$?
cat gpurun_out/nv_sweep_n*.jsonl | cut -c1-220; tail -3 gpurun_out/nv_sweep_n4.log

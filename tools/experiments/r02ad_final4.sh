# round 2 FINAL after FP8 raw leaves (4 GPUs): multi-process parity n=4 and n=2 (per-rank verdicts), bench N=4 and N=2
set -x
python -c "import __graft_entry__ as g; g.build()"
python -c "import bench; print(bench.source_sha())"
HFR_MULTI_OUT=gpurun_out/r02ad_multi timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -rA > gpurun_out/r02ad_multigpu_n4.log 2>&1; echo multi4=$?
tail -2 gpurun_out/r02ad_multigpu_n4.log
CUDA_VISIBLE_DEVICES=0,1 HFR_MULTI_OUT=gpurun_out/r02ad_multi timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -rA > gpurun_out/r02ad_multigpu_n2.log 2>&1; echo multi2=$?
tail -2 gpurun_out/r02ad_multigpu_n2.log
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $R --nproc-per-node 4 --master-port 29941 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r02ad_bench_n4.log 2>&1; echo bench4=$?
grep '^{' gpurun_out/r02ad_bench_n4.log | head -c 600; echo
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $R --nproc-per-node 2 --master-port 29942 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r02ad_bench_n2.log 2>&1; echo bench2=$?
grep '^{' gpurun_out/r02ad_bench_n2.log | head -c 600; echo
timeout 600 $R --nproc-per-node 4 --master-port 29943 bench.py --impl reference --gpus 4 --steps 3 --warmup 1 > gpurun_out/r02ad_bench_ref_n4.log 2>&1; echo ref4=$?
grep '^{' gpurun_out/r02ad_bench_ref_n4.log | head -c 400; echo

set -x
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm --format=csv
nproc; lscpu | grep -E "Model name|^CPU\(s\)|Thread|Socket"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/p2p_probe tools/p2p_probe.cu && /tmp/p2p_probe 2 256 148 512 > gpurun_out/r02a_probe_n2.txt 2>&1; echo probe=$?
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -rA > gpurun_out/r02a_multigpu_n2.log 2>&1; echo multi=$?
tail -5 gpurun_out/r02a_multigpu_n2.log
ncu --help > gpurun_out/ncu_help.txt 2>&1
ncu --query-metrics --chip gb100 2>/dev/null | grep -iE "nvl|nvlink" > gpurun_out/ncu_nvl_metrics.txt; echo q=$?

# round 2: TMA tree kernel — parity on virtual ranks (GPU 0), then n=2 NVLink
# A/B of the two tree data paths (2-GPU box)
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_virtual.py -x -q -k "tree_staging or tree_many or c2_full_size or cuda_graph" > gpurun_out/r02e_tree_tests.log 2>&1; echo trees=$?
tail -15 gpurun_out/r02e_tree_tests.log
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 600 $R --master-port 29631 tools/sweep.py --algos dbt,pair_dbt,flat --tree-staging 1,2 --sizes 195035136 --out gpurun_out/r02e_trees_n2.jsonl > gpurun_out/r02e_sweep1.log 2>&1; echo sweep1=$?
tail -3 gpurun_out/r02e_sweep1.log
timeout 600 $R --master-port 29632 tools/sweep.py --algos dbt,pair_dbt --tree-staging 2 --chunks 4096,8192,16384,32768,65536 --sizes 195035136 --out gpurun_out/r02e_trees_chunks_n2.jsonl > gpurun_out/r02e_sweep2.log 2>&1; echo sweep2=$?
timeout 600 $R --master-port 29633 tools/sweep.py --dtype bf16 --algos dbt,pair_dbt --tree-staging 1,2 --sizes 1073741824,67108864,8388608 --out gpurun_out/r02e_trees_bf16_n2.jsonl > gpurun_out/r02e_sweep3.log 2>&1; echo sweep3=$?
timeout 1500 python -m pytest tests -m gpu -q -rs --durations=10 > gpurun_out/r02e_gpu_tests.log 2>&1; echo tests=$?
tail -15 gpurun_out/r02e_gpu_tests.log
# ncu NVLink/DRAM bytes of one FLAT-TMA launch at n=2, host plumbing over gloo (no NCCL kernels under ncu)
BN="bench.py --gpus 2 --steps 4 --warmup 3 --no-cpu --no-e2e --no-variants --no-probe --no-nvls --soak 0 --dist gloo"
python -c "import bench; print(bench.source_sha())" > gpurun_out/r02e_source_sha.txt
timeout 240 $R --master-port 29634 --no-python bash tools/ncu_rank0.sh gpurun_out/r02e_nvl_n2.csv nvltx__bytes.sum,nvlrx__bytes.sum hfr_flat_tma 5 $BN > gpurun_out/r02e_ncu_nvl_n2.log 2>&1; echo nvl=$?
tail -4 gpurun_out/r02e_ncu_nvl_n2.log; cat gpurun_out/r02e_nvl_n2.csv
timeout 240 $R --master-port 29635 --no-python bash tools/ncu_rank0.sh gpurun_out/r02e_dram_n2.csv dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum hfr_flat_tma 5 $BN > gpurun_out/r02e_ncu_dram_n2.log 2>&1; echo dram=$?
cat gpurun_out/r02e_dram_n2.csv

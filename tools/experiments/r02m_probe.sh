# round 2: NVLink probe incl. the TMA bulk-copy modes (2-GPU box); tree sanity after the revert
set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/p2p_probe tools/p2p_probe.cu && /tmp/p2p_probe 2 256 148 512 > gpurun_out/r02m_probe_n2.txt 2>&1; echo probe=$?
cat gpurun_out/r02m_probe_n2.txt
python -c "import __graft_entry__ as g; g.build()"
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 600 $R --master-port 29791 tools/sweep.py --algos dbt,pair_dbt,flat --sizes 195035136 --out gpurun_out/r02m_trees_n2.jsonl > gpurun_out/r02m_s1.log 2>&1; echo s1=$?
cut -c1-200 gpurun_out/r02m_trees_n2.jsonl

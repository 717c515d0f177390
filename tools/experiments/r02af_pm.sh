# round 2: NVLink / DRAM bytes of the N=2 and N=4 FLAT allreduce from CUPTI PM sampling (no kernel replay)
set -x
python -c "import __graft_entry__ as g; g.build()"
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0,1 timeout 300 $R --nproc-per-node 2 --master-port 29991 tools/pm_nvlink.py --out gpurun_out/r02af_pm_n2.json > gpurun_out/r02af_pm_n2.log 2>&1; echo pm2=$?
grep '^{' gpurun_out/r02af_pm_n2.log | head -c 4000; echo
grep -i "pm_sampler\|error" gpurun_out/r02af_pm_n2.log | head -10
timeout 300 $R --nproc-per-node 4 --master-port 29992 tools/pm_nvlink.py --out gpurun_out/r02af_pm_n4.json > gpurun_out/r02af_pm_n4.log 2>&1; echo pm4=$?
grep '^{' gpurun_out/r02af_pm_n4.log | head -c 4000; echo

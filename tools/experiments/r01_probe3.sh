python - <<'PY'
from cuda.bindings import driver as d
d.cuInit(0)
for i in range(2):
    err, dev = d.cuDeviceGet(i)
    for name in ("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED","CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED","CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED","CU_DEVICE_ATTRIBUTE_CAN_USE_64_BIT_STREAM_MEM_OPS","CU_DEVICE_ATTRIBUTE_CAN_FLUSH_REMOTE_WRITES"):
        a = getattr(d.CUdevice_attribute, name)
        print(i, name, d.cuDeviceGetAttribute(a, dev))
PY
cat /proc/sys/kernel/yama/ptrace_scope 2>/dev/null; id
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,TUNING,COLL timeout 600 $R --nproc-per-node 4 --master-port 29951 tools/sweep.py --dtype bf16 --sizes $((1<<30)) --algos flat --nccl > gpurun_out/p3_nccl.log 2>&1; echo nccl=$?
grep -iE "nvls|algo|NCCL INFO Channel|proto" gpurun_out/p3_nccl.log | head -30
grep '^{' gpurun_out/p3_nccl.log
S=$((186<<20))
timeout 900 $R --nproc-per-node 4 --master-port 29952 tools/sweep.py --sizes $S --algos dbt,pair_dbt --chunks 32768,65536 --ctas 64,0 > gpurun_out/p3_tree.log 2>&1; grep '^{' gpurun_out/p3_tree.log | cut -c1-200

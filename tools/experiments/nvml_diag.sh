mkdir -p gpurun_out
{
python - <<'PY'
import pynvml as p
p.nvmlInit()
h = p.nvmlDeviceGetHandleByIndex(0)
for f in ["COUNT_XMIT_BYTES","COUNT_RCV_BYTES","COUNT_XMIT_PACKETS","THROUGHPUT_DATA_TX","THROUGHPUT_RAW_TX"]:
    fid = getattr(p, "NVML_FI_DEV_NVLINK_"+f)
    for scope in (0, 1, 0xFFFFFFFF):
        try:
            v = p.nvmlDeviceGetFieldValues(h, [(fid, scope)])[0]
            print(f, fid, scope, "ret", v.nvmlReturn, "val", v.value.ullVal, "type", v.valueType)
        except Exception as e:
            print(f, fid, scope, "EXC", repr(e))
    try:
        v = p.nvmlDeviceGetFieldValues(h, [fid])[0]
        print(f, "noscope ret", v.nvmlReturn, v.value.ullVal)
    except Exception as e:
        print(f, "noscope EXC", repr(e))
try:
    print("gpm support", p.nvmlGpmQueryDeviceSupport(h).isSupportedDevice)
except Exception as e:
    print("gpm EXC", repr(e))
try:
    print("nvlink util counter", p.nvmlDeviceGetNvLinkUtilizationCounter(h, 0, 0))
except Exception as e:
    print("util EXC", repr(e))
PY
} > gpurun_out/nvml_diag.txt 2>&1
{ nvidia-smi nvlink -h; echo ===gt; nvidia-smi nvlink -gt d -i 0; echo ===e; nvidia-smi nvlink -e -i 0 | head -40; echo ===dmonh; nvidia-smi dmon -h | head -40; } > gpurun_out/nvsmi_diag.txt 2>&1
head -c 3000 gpurun_out/nvml_diag.txt

mkdir -p gpurun_out
python - > gpurun_out/gpm_diag.txt 2>&1 <<'PY'
import time, traceback
import pynvml as p
p.nvmlInit()
h = p.nvmlDeviceGetHandleByIndex(0)
try:
    s1 = p.nvmlGpmSampleAlloc(); s2 = p.nvmlGpmSampleAlloc()
    p.nvmlGpmSampleGet(h, s1); time.sleep(0.2); p.nvmlGpmSampleGet(h, s2)
    mg = p.c_nvmlGpmMetricsGet_t()
    mg.version = p.NVML_GPM_METRICS_GET_VERSION
    ids = [p.NVML_GPM_METRIC_NVLINK_TOTAL_TX_PER_SEC, p.NVML_GPM_METRIC_NVLINK_TOTAL_RX_PER_SEC,
           p.NVML_GPM_METRIC_SM_OCCUPANCY, p.NVML_GPM_METRIC_DRAM_BW_UTIL]
    mg.numMetrics = len(ids)
    mg.sample1 = s1; mg.sample2 = s2
    for i, m in enumerate(ids):
        mg.metrics[i].metricId = m
    p.nvmlGpmMetricsGet(mg)
    for i in range(len(ids)):
        print(ids[i], mg.metrics[i].nvmlReturn, mg.metrics[i].value)
except Exception:
    traceback.print_exc()
PY
cat gpurun_out/gpm_diag.txt

// pm_sampler.cu — device-level hardware counters over a time window, via
// CUPTI PM sampling (CUDA 12.6+): the GPU samples its performance monitors at
// a fixed interval while the workload runs, so no kernel is replayed and a
// multi-rank allreduce (whose kernels wait on each other across GPUs) runs
// exactly as in production.  Measurement tool only (not part of libhfr):
// used by tools/pm_nvlink.py for the NVLink / DRAM bytes of the N>1 bench
// kernel, which ncu cannot capture (profiles/r02/ncu_multirank_attempts.txt).
//
//   nvcc -O2 -shared -Xcompiler -fPIC -o tools/libpm_sampler.so tools/pm_sampler.cu -lcupti -lcuda
//
// C ABI: pm_query_metrics(dev, buf, size) lists the base metrics the device
// samples; pm_start(dev, "m1,m2,...", interval, max_samples) starts a session
// with a decode thread; pm_stop(sums, n, &t0, &t1) stops it and returns the
// number of samples, each metric summed over them (a counter's sum over the
// window) and the first / last sample timestamps (ns).
#include <cuda.h>
#include <cupti_pmsampling.h>
#include <cupti_profiler_host.h>
#include <cupti_profiler_target.h>
#include <cupti_target.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <atomic>
#include <chrono>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

namespace {

#define PM_TRY(call)                                                           \
  do {                                                                         \
    CUptiResult r_ = (call);                                                   \
    if (r_ != CUPTI_SUCCESS) {                                                 \
      const char* s_ = nullptr;                                                \
      cuptiGetResultString(r_, &s_);                                           \
      fprintf(stderr, "pm_sampler: %s failed: %s\n", #call, s_ ? s_ : "?");    \
      return -(int)r_ - 1;                                                     \
    }                                                                          \
  } while (0)

struct Session {
  CUpti_Profiler_Host_Object* host = nullptr;
  CUpti_PmSampling_Object* sampler = nullptr;
  std::vector<std::string> names;
  std::vector<const char*> cnames;
  std::vector<uint8_t> config, counter_data;
  std::vector<double> sums;
  uint64_t t_first = 0, t_last = 0;
  size_t samples = 0;
  std::thread decoder;
  std::atomic<bool> stop{false};
  std::mutex mu;
  int error = 0;
  FILE* series = nullptr;  // optional per-sample dump: start_ns,end_ns,metric values...
} g;

int host_init(int dev, CUpti_ProfilerType type) {
  CUpti_Profiler_Initialize_Params ip = {CUpti_Profiler_Initialize_Params_STRUCT_SIZE};
  PM_TRY(cuptiProfilerInitialize(&ip));
  CUpti_Device_GetChipName_Params cp = {CUpti_Device_GetChipName_Params_STRUCT_SIZE};
  cp.deviceIndex = dev;
  PM_TRY(cuptiDeviceGetChipName(&cp));
  CUpti_PmSampling_GetCounterAvailability_Params ap = {CUpti_PmSampling_GetCounterAvailability_Params_STRUCT_SIZE};
  ap.deviceIndex = dev;
  PM_TRY(cuptiPmSamplingGetCounterAvailability(&ap));
  static std::vector<uint8_t> avail;
  avail.assign(ap.counterAvailabilityImageSize, 0);
  ap.pCounterAvailabilityImage = avail.data();
  PM_TRY(cuptiPmSamplingGetCounterAvailability(&ap));
  CUpti_Profiler_Host_Initialize_Params hp = {CUpti_Profiler_Host_Initialize_Params_STRUCT_SIZE};
  hp.profilerType = type;
  hp.pChipName = cp.pChipName;
  hp.pCounterAvailabilityImage = avail.data();
  PM_TRY(cuptiProfilerHostInitialize(&hp));
  g.host = hp.pHostObject;
  return 0;
}

// decode what the hardware buffer holds into the counter-data image and add
// every completed sample to the running sums
int drain() {
  CUpti_PmSampling_DecodeData_Params dp = {CUpti_PmSampling_DecodeData_Params_STRUCT_SIZE};
  dp.pPmSamplingObject = g.sampler;
  dp.pCounterDataImage = g.counter_data.data();
  dp.counterDataImageSize = g.counter_data.size();
  PM_TRY(cuptiPmSamplingDecodeData(&dp));
  CUpti_PmSampling_GetCounterDataInfo_Params info = {CUpti_PmSampling_GetCounterDataInfo_Params_STRUCT_SIZE};
  info.pCounterDataImage = g.counter_data.data();
  info.counterDataImageSize = g.counter_data.size();
  PM_TRY(cuptiPmSamplingGetCounterDataInfo(&info));
  std::vector<double> v(g.cnames.size());
  for (size_t s = 0; s < info.numCompletedSamples; ++s) {
    CUpti_PmSampling_CounterData_GetSampleInfo_Params si = {CUpti_PmSampling_CounterData_GetSampleInfo_Params_STRUCT_SIZE};
    si.pPmSamplingObject = g.sampler;
    si.pCounterDataImage = g.counter_data.data();
    si.counterDataImageSize = g.counter_data.size();
    si.sampleIndex = s;
    PM_TRY(cuptiPmSamplingCounterDataGetSampleInfo(&si));
    CUpti_Profiler_Host_EvaluateToGpuValues_Params ev = {CUpti_Profiler_Host_EvaluateToGpuValues_Params_STRUCT_SIZE};
    ev.pHostObject = g.host;
    ev.pCounterDataImage = g.counter_data.data();
    ev.counterDataImageSize = g.counter_data.size();
    ev.ppMetricNames = g.cnames.data();
    ev.numMetrics = g.cnames.size();
    ev.rangeIndex = s;
    ev.pMetricValues = v.data();
    PM_TRY(cuptiProfilerHostEvaluateToGpuValues(&ev));
    std::lock_guard<std::mutex> lock(g.mu);
    for (size_t i = 0; i < v.size(); ++i) g.sums[i] += v[i];
    if (g.series) {
      fprintf(g.series, "%llu,%llu", (unsigned long long)si.startTimestamp, (unsigned long long)si.endTimestamp);
      for (double x : v) fprintf(g.series, ",%.0f", x);
      fprintf(g.series, "\n");
    }
    if (!g.samples) g.t_first = si.startTimestamp;
    g.t_last = si.endTimestamp;
    ++g.samples;
  }
  CUpti_PmSampling_CounterDataImage_Initialize_Params ri = {CUpti_PmSampling_CounterDataImage_Initialize_Params_STRUCT_SIZE};
  ri.pPmSamplingObject = g.sampler;
  ri.counterDataSize = g.counter_data.size();
  ri.pCounterData = g.counter_data.data();
  PM_TRY(cuptiPmSamplingCounterDataImageInitialize(&ri));
  return 0;
}

}  // namespace

extern "C" int pm_query_metrics(int dev, char* buf, size_t size) {
  if (cuInit(0) != CUDA_SUCCESS) return -1;
  int rc = host_init(dev, CUPTI_PROFILER_TYPE_PM_SAMPLING);
  if (rc) return rc;
  CUpti_Profiler_Host_GetBaseMetrics_Params bp = {CUpti_Profiler_Host_GetBaseMetrics_Params_STRUCT_SIZE};
  bp.pHostObject = g.host;
  bp.metricType = CUPTI_METRIC_TYPE_COUNTER;
  PM_TRY(cuptiProfilerHostGetBaseMetrics(&bp));
  size_t off = 0;
  for (size_t i = 0; i < bp.numMetrics && off + 1 < size; ++i)
    off += snprintf(buf + off, size - off, "%s\n", bp.ppMetricNames[i]);
  CUpti_Profiler_Host_Deinitialize_Params dp = {CUpti_Profiler_Host_Deinitialize_Params_STRUCT_SIZE};
  dp.pHostObject = g.host;
  cuptiProfilerHostDeinitialize(&dp);
  g.host = nullptr;
  return (int)bp.numMetrics;
}

extern "C" int pm_series(const char* path) {  // call before pm_start; NULL / "" = off
  if (g.series) fclose(g.series);
  g.series = (path && *path) ? fopen(path, "w") : nullptr;
  return g.series || !(path && *path) ? 0 : -1;
}

extern "C" int pm_start(int dev, const char* metrics_csv, uint64_t interval, uint64_t max_samples) {
  if (cuInit(0) != CUDA_SUCCESS) return -1;
  int rc = host_init(dev, CUPTI_PROFILER_TYPE_PM_SAMPLING);
  if (rc) return rc;
  g.names.clear();
  std::string s(metrics_csv);
  for (size_t p = 0; p <= s.size();) {
    size_t q = s.find(',', p);
    if (q == std::string::npos) q = s.size();
    if (q > p) g.names.push_back(s.substr(p, q - p));
    p = q + 1;
  }
  g.cnames.clear();
  for (auto& n : g.names) g.cnames.push_back(n.c_str());
  g.sums.assign(g.names.size(), 0.0);
  g.samples = 0;
  CUpti_Profiler_Host_ConfigAddMetrics_Params am = {CUpti_Profiler_Host_ConfigAddMetrics_Params_STRUCT_SIZE};
  am.pHostObject = g.host;
  am.ppMetricNames = g.cnames.data();
  am.numMetrics = g.cnames.size();
  PM_TRY(cuptiProfilerHostConfigAddMetrics(&am));
  CUpti_Profiler_Host_GetConfigImageSize_Params cs = {CUpti_Profiler_Host_GetConfigImageSize_Params_STRUCT_SIZE};
  cs.pHostObject = g.host;
  PM_TRY(cuptiProfilerHostGetConfigImageSize(&cs));
  g.config.assign(cs.configImageSize, 0);
  CUpti_Profiler_Host_GetConfigImage_Params ci = {CUpti_Profiler_Host_GetConfigImage_Params_STRUCT_SIZE};
  ci.pHostObject = g.host;
  ci.pConfigImage = g.config.data();
  ci.configImageSize = g.config.size();
  PM_TRY(cuptiProfilerHostGetConfigImage(&ci));
  CUpti_PmSampling_Enable_Params en = {CUpti_PmSampling_Enable_Params_STRUCT_SIZE};
  en.deviceIndex = dev;
  PM_TRY(cuptiPmSamplingEnable(&en));
  g.sampler = en.pPmSamplingObject;
  CUpti_PmSampling_SetConfig_Params sc = {CUpti_PmSampling_SetConfig_Params_STRUCT_SIZE};
  sc.pPmSamplingObject = g.sampler;
  sc.configSize = g.config.size();
  sc.pConfig = g.config.data();
  sc.hardwareBufferSize = 512ull << 20;
  sc.samplingInterval = interval;
  sc.triggerMode = CUPTI_PM_SAMPLING_TRIGGER_MODE_GPU_SYSCLK_INTERVAL;
  PM_TRY(cuptiPmSamplingSetConfig(&sc));
  CUpti_PmSampling_GetCounterDataSize_Params ds = {CUpti_PmSampling_GetCounterDataSize_Params_STRUCT_SIZE};
  ds.pPmSamplingObject = g.sampler;
  ds.numMetrics = g.cnames.size();
  ds.pMetricNames = g.cnames.data();
  ds.maxSamples = max_samples;
  PM_TRY(cuptiPmSamplingGetCounterDataSize(&ds));
  g.counter_data.assign(ds.counterDataSize, 0);
  CUpti_PmSampling_CounterDataImage_Initialize_Params ii = {CUpti_PmSampling_CounterDataImage_Initialize_Params_STRUCT_SIZE};
  ii.pPmSamplingObject = g.sampler;
  ii.counterDataSize = g.counter_data.size();
  ii.pCounterData = g.counter_data.data();
  PM_TRY(cuptiPmSamplingCounterDataImageInitialize(&ii));
  CUpti_PmSampling_Start_Params st = {CUpti_PmSampling_Start_Params_STRUCT_SIZE};
  st.pPmSamplingObject = g.sampler;
  PM_TRY(cuptiPmSamplingStart(&st));
  g.stop = false;
  g.error = 0;
  g.decoder = std::thread([] {
    while (!g.stop) {
      if (int r = drain()) {
        g.error = r;
        return;
      }
      std::this_thread::sleep_for(std::chrono::milliseconds(5));
    }
  });
  return 0;
}

extern "C" int pm_stop(double* sums, int n, uint64_t* t_first, uint64_t* t_last) {
  CUpti_PmSampling_Stop_Params sp = {CUpti_PmSampling_Stop_Params_STRUCT_SIZE};
  sp.pPmSamplingObject = g.sampler;
  PM_TRY(cuptiPmSamplingStop(&sp));
  g.stop = true;
  if (g.decoder.joinable()) g.decoder.join();
  if (g.error) return g.error;
  if (int r = drain()) return r;
  for (int i = 0; i < n && i < (int)g.sums.size(); ++i) sums[i] = g.sums[i];
  if (t_first) *t_first = g.t_first;
  if (t_last) *t_last = g.t_last;
  CUpti_PmSampling_Disable_Params dp = {CUpti_PmSampling_Disable_Params_STRUCT_SIZE};
  dp.pPmSamplingObject = g.sampler;
  cuptiPmSamplingDisable(&dp);
  CUpti_Profiler_Host_Deinitialize_Params hd = {CUpti_Profiler_Host_Deinitialize_Params_STRUCT_SIZE};
  hd.pHostObject = g.host;
  cuptiProfilerHostDeinitialize(&hd);
  CUpti_Profiler_DeInitialize_Params pd = {CUpti_Profiler_DeInitialize_Params_STRUCT_SIZE};
  cuptiProfilerDeInitialize(&pd);
  g.host = nullptr;
  g.sampler = nullptr;
  if (g.series) {
    fclose(g.series);
    g.series = nullptr;
  }
  return (int)g.samples;
}

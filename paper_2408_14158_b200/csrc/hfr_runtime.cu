// hfr_runtime.cu — host runtime and C ABI (include/hfr.h) of the B200-native
// HFReduce (arXiv 2408.14158 §4).
//
// Responsibilities: communicator setup (peer-mapped signal pad + scratch,
// CUDA IPC handle exchange through the caller's all-gather callback), the
// symmetric-memory region table (zero-copy buffers), the chunk/segment plan
// (Alg. 1 "Split Dg by Chunk_Size"), the double-binary-tree
// tables (reading R9), argument signatures for the cross-rank protocol check,
// stream/event plumbing for asynchronous calls, and the
// sticky error state.  All data movement and arithmetic happens in the
// kernels of hfr_kernels.cuh.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "../../include/hfr.h"
#include "hfr_kernels.cuh"
#include "hfr_tree_tma.cuh"

using namespace hfr;

namespace {

thread_local std::string g_cuda_error;

void note_cuda(cudaError_t e, const char* what) {
  char buf[512];
  snprintf(buf, sizeof buf, "%s: %s (%d)", what, cudaGetErrorString(e), (int)e);
  g_cuda_error = buf;
}

#define HFR_CU(call)                                                               \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess) {                                                       \
      note_cuda(e_, #call);                                                        \
      return e_ == cudaErrorMemoryAllocation ? HFR_ERR_OUT_OF_MEMORY : HFR_ERR_CUDA; \
    }                                                                              \
  } while (0)

#define HFR_TRY(expr)                 \
  do {                                \
    hfr_status_t s_ = (expr);         \
    if (s_ != HFR_SUCCESS) return s_; \
  } while (0)

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

constexpr size_t kAlign = 256;
size_t round_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// One peer-mapped allocation: base[r] is rank r's copy as addressable from
// this process (own allocation for local ranks, IPC mapping for peers).
struct Region {
  char* base[kMaxRanks] = {};
  bool opened[kMaxRanks] = {};  // base[r] came from cudaIpcOpenMemHandle
  bool owned = false;           // we cudaMalloc'ed base[local ranks]
  bool nvls = false;            // the NVLS multicast arena (torn down by nvls_teardown)
  size_t bytes = 0;
};

struct Nvls;  // hfr_nvls.cuh

struct IpcRecord {
  cudaIpcMemHandle_t handle;
  uint64_t offset;  // byte offset of the exported pointer inside its allocation
  uint64_t bytes;
  int32_t device;
  int32_t rank;
};

}  // namespace

struct hfr_req_s {
  cudaEvent_t ev = nullptr;
  hfr_comm_s* comm = nullptr;
};

constexpr int kCeMaxChunks = 16;           // CE schedule: pipeline depth (chunks per shard)
constexpr uint64_t kCeMinChunkBytes = 8ull << 20;  // ... and the smallest chunk (per-chunk stream latency ~15 us)

struct hfr_comm_s {
  int rank = 0, n = 1, dev = 0, local = 1;
  bool virt = false;
  hfr_config_t cfg{};
  hfr_allgather_fn ag = nullptr;
  void* ctx = nullptr;
  Region pad;       // Pad per rank
  Region scratch;   // staging + tree partials per rank
  std::vector<Region> regions;  // hfr_mem_alloc / hfr_register memory
  uint64_t epoch = 0;
  uint32_t* err_host = nullptr;  // host-mapped error word
  uint32_t* err_dev = nullptr;
  cudaStream_t side = nullptr;
  // issue order (include/hfr.h): every call's stream waits for the previous
  // call's last_op event, and records it when enqueued (two
  // calls on different streams, or an async call and a barrier, must never
  // overlap — they share the pad's epoch, tile counter and scratch)
  cudaEvent_t last_op = nullptr;
  bool has_last = false;
  cudaStream_t setup = nullptr;       // private stream for scratch zeroing (no device-wide sync)
  std::vector<Region> retired;        // outgrown scratch regions, released at hfr_finalize
  std::vector<cudaEvent_t> ev_pool;
  int num_sms = 148;
  hfr_status_t sticky = HFR_SUCCESS;
  uint64_t launches = 0;
  // CE schedule (created on first use): per local rank l, a fold stream
  // (virtual comms; a real comm folds on the call's stream), H helper streams
  // for the reduce-scatter pulls and H for the all-gather pulls (real comms
  // H = n-1, one per peer, so the copy engines run the pulls concurrently;
  // virtual comms H = 1), one event per (helper, chunk) of the reduce-scatter
  // pulls, fork/join events, and the host-side CE epoch
  int ce_h = 0;
  std::vector<cudaStream_t> ce_fold;
  std::vector<cudaStream_t> helpers;
  std::vector<cudaStream_t> ag_helpers;
  std::vector<cudaEvent_t> ag_events;
  std::vector<cudaEvent_t> chunk_events;
  std::vector<cudaEvent_t> ce_fork;
  std::vector<cudaEvent_t> ce_join;
  uint64_t ce_epoch = 0;
  uint64_t* trace = nullptr;  // hfr_set_trace (diagnostic)
  uint32_t trace_cap = 0;
  Nvls* nvls = nullptr;       // NVLS multicast arena (hfr_config.nvls_bytes)
};

// ---------------------------------------------------------------------------
// double binary tree (reading R9).  Independent of oracle/: tree A is built
// top-down from the CHILD rules (the oracle derives it from parent rules).
// ---------------------------------------------------------------------------
namespace {

constexpr int kMaxTreeN = kMaxRanks * 64;  // hfr_tree_query supports n <= 1024

void build_tree(int n, int which, int* parent, std::array<int, 2>* child, int* nchild) {
  std::vector<int> pa(n, -1);
  std::vector<std::vector<int>> ch(n);
  if (n > 1) {
    int top = 1;
    while (top * 2 < n) top *= 2;
    ch[0].push_back(top);
    for (int r = 1; r < n; ++r) {
      const int b = r & -r;
      if (b > 1) {
        ch[r].push_back(r - b / 2);
        int h = b / 2;
        while (h > 0 && r + h >= n) h /= 2;
        if (h > 0) ch[r].push_back(r + h);
      }
    }
    for (int r = 0; r < n; ++r)
      for (int c : ch[r]) pa[c] = r;
  }
  // tree B: relabel by mirror (even n) or shift (odd n)
  auto f = [&](int r) { return which == 0 ? r : (n % 2 == 0 ? n - 1 - r : (r + 1) % n); };
  for (int r = 0; r < n; ++r) {
    nchild[r] = 0;
    child[r][0] = child[r][1] = -1;
  }
  for (int r = 0; r < n; ++r) parent[f(r)] = pa[r] < 0 ? -1 : f(pa[r]);
  for (int r = 0; r < n; ++r) {
    const int p = parent[r];
    if (p >= 0) child[p][nchild[p]++] = r;
  }
  for (int r = 0; r < n; ++r)
    if (nchild[r] == 2 && child[r][0] > child[r][1]) std::swap(child[r][0], child[r][1]);
}

void fill_tree_nodes(int m, TreeNode (*out)[kMaxRanks]) {
  for (int which = 0; which < 2; ++which) {
    int parent[kMaxRanks], nchild[kMaxRanks];
    std::array<int, 2> child[kMaxRanks];
    build_tree(m, which, parent, child, nchild);
    for (int v = 0; v < m; ++v) {
      TreeNode& t = out[which][v];
      t.parent = (int8_t)parent[v];
      t.nchild = (int8_t)nchild[v];
      t.child[0] = (int8_t)child[v][0];
      t.child[1] = (int8_t)child[v][1];
      int below = 0;
      for (int k = 0; k < nchild[v]; ++k) below += child[v][k] < v;
      t.self_pos = (int8_t)below;
      t.slot = 0;
      if (parent[v] >= 0) {
        const int p = parent[v];
        t.slot = (int8_t)(child[p][0] == v ? 0 : 1);
      }
    }
  }
}

// pair split (reading R13): H = min(N, 256 * ceil(N / 512))
uint64_t pair_half(uint64_t count) {
  const uint64_t h = 256 * ((count + 511) / 512);
  return h < count ? h : count;
}

uint64_t fnv(uint64_t h, uint64_t v) {
  for (int i = 0; i < 8; ++i) {
    h ^= (v >> (8 * i)) & 0xFF;
    h *= 1099511628211ull;
  }
  return h;
}

size_t dtype_size(hfr_dtype_t t) { return t == HFR_FLOAT32 ? 4 : (t == HFR_FP8_E4M3 || t == HFR_FP8_E5M2) ? 1 : 2; }
bool dtype_valid(int t) { return t >= HFR_FLOAT32 && t <= HFR_FP8_E5M2; }
bool dtype_fp8(hfr_dtype_t t) { return t == HFR_FP8_E4M3 || t == HFR_FP8_E5M2; }
uint64_t per_vec(hfr_dtype_t t) { return 16 / dtype_size(t); }  // elements per 16 bytes

// Kernel instantiation by element type: HFR_BY_DTYPE(dt, M) expands M(F32),
// M(BF16) or M(F16).
#define HFR_BY_DTYPE(dt, M)                                                                          \
  ((dt) == HFR_BFLOAT16 ? (M(BF16)) : (dt) == HFR_FLOAT16 ? (M(F16)) : (dt) == HFR_FP8_E4M3 ? (M(E4M3)) \
   : (dt) == HFR_FP8_E5M2 ? (M(E5M2)) : (M(F32)))
// NVLS has no fp32-accumulating multimem form for FP8 (UNSUPPORTED there)
#define HFR_BY_DTYPE_NO_FP8(dt, M) ((dt) == HFR_BFLOAT16 ? (M(BF16)) : (dt) == HFR_FLOAT16 ? (M(F16)) : (M(F32)))

// An explicit ONESHOT on a message above oneshot_max_bytes runs FLAT (same
// result bits).
// ONESHOT's LL form fits when every element's 8-byte word fits the inbox
// slot; AUTO takes it while the (n-1) * count * 8 bytes each rank pushes stay
// under ~6 MiB — the r01 graph sweep's crossover with FLAT on 2 and 4 B200s
// (bf16: n=4 up to 256 KiB, n=2 up to 1 MiB; fp32: n=4 up to 512 KiB).
bool ll_fits(const hfr_comm_s* c, size_t count) { return count * 8 <= c->cfg.oneshot_max_bytes; }
bool ll_pays(const hfr_comm_s* c, size_t count) { return (uint64_t)(c->n - 1) * count * 8 <= c->cfg.ll_push_max; }

int effective_algo(const hfr_comm_s* c, size_t count, size_t esz) {
  const size_t bytes = count * esz;
  const int a = c->cfg.algo;
  // CE moves shards of at least 4096 elements; a smaller message (or n = 1,
  // nothing to move) runs FLAT (same bits)
  if (a == HFR_ALGO_CE) return (c->n == 1 || bytes < (size_t)c->n * 16384) ? HFR_ALGO_FLAT : HFR_ALGO_CE;
  // AUTO: ONESHOT only in its LL form and only where it beats FLAT
  if (a == HFR_ALGO_AUTO) return ll_fits(c, count) && ll_pays(c, count) ? HFR_ALGO_ONESHOT : HFR_ALGO_FLAT;
  if (a == HFR_ALGO_ONESHOT) return bytes <= c->cfg.oneshot_max_bytes ? HFR_ALGO_ONESHOT : HFR_ALGO_FLAT;
  return a;
}

hfr_status_t validate_cfg(const hfr_config_t& c) {
  if (c.algo < HFR_ALGO_AUTO || c.algo > HFR_ALGO_NVLS) return HFR_ERR_INVALID_ARGUMENT;
  if (c.oneshot_max_bytes > (64u << 20)) return HFR_ERR_INVALID_ARGUMENT;
  if (c.chunk_elems % 256 != 0 || c.chunk_elems > (1u << 30)) return HFR_ERR_INVALID_ARGUMENT;
  if (c.max_ctas < 0 || c.max_ctas > kMaxCtas) return HFR_ERR_INVALID_ARGUMENT;
  if (c.threads != 0 && (c.threads < 128 || c.threads > 512 || c.threads % 32 != 0)) return HFR_ERR_INVALID_ARGUMENT;
  if (!(c.scale == c.scale)) return HFR_ERR_INVALID_ARGUMENT;
  if (c.timeout_ms < 0) return HFR_ERR_INVALID_ARGUMENT;
  if (c.stream_gate != 0 && c.stream_gate != 1) return HFR_ERR_INVALID_ARGUMENT;
  if (c.flat_staging < 0 || c.flat_staging > 2) return HFR_ERR_INVALID_ARGUMENT;
  if (c.pdl_off != 0 && c.pdl_off != 1) return HFR_ERR_INVALID_ARGUMENT;
  if (c.tree_staging < 0 || c.tree_staging > 2) return HFR_ERR_INVALID_ARGUMENT;
  return HFR_SUCCESS;
}

void resolve_defaults(hfr_config_t& c) {
  // chunk_elems stays 0 = "per n" (tree_chunk)
  if (c.scratch_bytes == 0) c.scratch_bytes = 256ull << 20;
  if (c.timeout_ms == 0) c.timeout_ms = 60000;
  if (c.oneshot_max_bytes == 0) c.oneshot_max_bytes = 4u << 20;
  c.oneshot_max_bytes = round_up(c.oneshot_max_bytes, 256);
  if (c.ll_push_max == 0) c.ll_push_max = 6ull << 20;
}

// ---------------------------------------------------------------------------
// collective region setup
// ---------------------------------------------------------------------------
hfr_status_t exchange(hfr_comm_s* c, const void* send, void* recv, size_t bytes) {
  if (c->n == 1 || c->virt) {
    memcpy(recv, send, bytes);
    return HFR_SUCCESS;
  }
  if (c->ag(send, recv, bytes, c->ctx) != 0) return HFR_ERR_INTERNAL;
  return HFR_SUCCESS;
}

// Export [ptr, ptr+bytes) of THIS rank (real comms) and open every peer's.
hfr_status_t share_region(hfr_comm_s* c, char* ptr, size_t bytes, Region* out) {
  if (c->virt) return HFR_ERR_INTERNAL;
  IpcRecord mine{};
  mine.rank = c->rank;
  mine.device = c->dev;
  mine.bytes = bytes;
  if (c->n > 1) {
    // Export the allocation containing ptr (cudaIpcGetMemHandle wants a base).
    void* base = ptr;
    size_t range = 0;
    typedef int (*GetRange)(unsigned long long*, size_t*, unsigned long long);
    static GetRange get_range = nullptr;
    if (!get_range) {
      cudaDriverEntryPointQueryResult q;
      void* fn = nullptr;
      if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) == cudaSuccess &&
          q == cudaDriverEntryPointSuccess)
        get_range = (GetRange)fn;
    }
    if (get_range) {
      unsigned long long b = 0;
      if (get_range(&b, &range, (unsigned long long)ptr) == 0) base = (void*)b;
    }
    mine.offset = (uint64_t)(ptr - (char*)base);
    HFR_CU(cudaIpcGetMemHandle(&mine.handle, base));
  }
  std::vector<IpcRecord> all(c->n);
  HFR_TRY(exchange(c, &mine, all.data(), sizeof(IpcRecord)));
  Region r;
  r.bytes = bytes;
  for (int q = 0; q < c->n; ++q) {
    if (all[q].rank != q || all[q].bytes != bytes) {
      for (int k = 0; k < q; ++k)
        if (r.opened[k]) cudaIpcCloseMemHandle(r.base[k] - all[k].offset);
      return HFR_ERR_PROTOCOL;
    }
    if (q == c->rank) {
      r.base[q] = ptr;
      continue;
    }
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, all[q].handle, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      note_cuda(e, "cudaIpcOpenMemHandle");
      for (int k = 0; k < q; ++k)
        if (r.opened[k]) cudaIpcCloseMemHandle(r.base[k] - all[k].offset);
      return HFR_ERR_CUDA;
    }
    r.base[q] = (char*)p + all[q].offset;
    r.opened[q] = true;
  }
  *out = r;
  return HFR_SUCCESS;
}

void close_region(hfr_comm_s* c, Region& r) {
  if (r.nvls) {  // mappings belong to the NVLS arena
    r = Region();
    return;
  }
  for (int q = 0; q < c->n; ++q) {
    if (r.opened[q] && r.base[q]) {
      // the mapping was opened at the allocation base; recover it
      void* b = r.base[q];
      typedef int (*GetRange)(unsigned long long*, size_t*, unsigned long long);
      cudaDriverEntryPointQueryResult qr;
      void* fn = nullptr;
      if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &qr) == cudaSuccess &&
          qr == cudaDriverEntryPointSuccess) {
        unsigned long long base = 0;
        size_t sz = 0;
        if (((GetRange)fn)(&base, &sz, (unsigned long long)r.base[q]) == 0) b = (void*)base;
      }
      cudaIpcCloseMemHandle(b);
    }
    r.opened[q] = false;
  }
  if (r.owned) {
    const int lo = c->virt ? 0 : c->rank, hi = c->virt ? c->n : c->rank + 1;
    for (int q = lo; q < hi; ++q)
      if (r.base[q]) cudaFree(r.base[q]);
  }
  r = Region();
}

// Allocate `bytes` on every local rank (zeroed) and make it peer-visible.
hfr_status_t alloc_region(hfr_comm_s* c, size_t bytes, Region* out) {
  bytes = round_up(std::max<size_t>(bytes, kAlign), 2u << 20);
  Region r;
  r.bytes = bytes;
  r.owned = true;
  // zeroed on the comm's private setup stream, which alone is synchronised:
  // kernels in flight on other streams (async allreduces) keep running
  if (c->virt) {
    for (int q = 0; q < c->n; ++q) {
      void* p = nullptr;
      cudaError_t e = cudaMalloc(&p, bytes);
      if (e == cudaSuccess) e = cudaMemsetAsync(p, 0, bytes, c->setup);
      if (e != cudaSuccess) {
        note_cuda(e, "cudaMalloc");
        for (int k = 0; k < q; ++k) cudaFree(r.base[k]);
        return e == cudaErrorMemoryAllocation ? HFR_ERR_OUT_OF_MEMORY : HFR_ERR_CUDA;
      }
      r.base[q] = (char*)p;
    }
    HFR_CU(cudaStreamSynchronize(c->setup));
    *out = r;
    return HFR_SUCCESS;
  }
  void* p = nullptr;
  HFR_CU(cudaMalloc(&p, bytes));
  cudaError_t e = cudaMemsetAsync(p, 0, bytes, c->setup);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->setup);  // zeroed before any peer can see it
  if (e != cudaSuccess) {
    note_cuda(e, "cudaMemset");
    cudaFree(p);
    return HFR_ERR_CUDA;
  }
  hfr_status_t s = share_region(c, (char*)p, bytes, &r);
  if (s != HFR_SUCCESS) {
    cudaFree(p);
    return s;
  }
  r.owned = true;
  *out = r;
  return HFR_SUCCESS;
}

}  // namespace

#include "hfr_nvls.cuh"

namespace {

hfr_status_t common_init(hfr_comm_s* c) {
  HFR_CU(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, c->dev));
  HFR_CU(cudaHostAlloc((void**)&c->err_host, sizeof(uint32_t) * 4, cudaHostAllocMapped | cudaHostAllocPortable));
  *c->err_host = 0;
  HFR_CU(cudaHostGetDevicePointer((void**)&c->err_dev, c->err_host, 0));
  int lo = 0, hi = 0;
  HFR_CU(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  // the side stream at the highest priority (r01: a low-priority comm stream
  // overlapped worse, 0.72-0.81 vs 0.90+, profiles/r01/c5_ddp_side_priority.jsonl)
  HFR_CU(cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, hi));
  HFR_CU(cudaEventCreateWithFlags(&c->last_op, cudaEventDisableTiming));
  HFR_CU(cudaStreamCreateWithFlags(&c->setup, cudaStreamNonBlocking));
  HFR_TRY(alloc_region(c, sizeof(Pad), &c->pad));
  HFR_TRY(alloc_region(c, c->cfg.scratch_bytes, &c->scratch));
  if (c->cfg.nvls_bytes > 0 && !c->virt && c->n > 1) {
    c->nvls = new Nvls;
    hfr_status_t st = nvls_setup(c, *c->nvls, c->cfg.nvls_bytes);
    if (st == HFR_ERR_UNSUPPORTED) {
      nvls_teardown(*c->nvls, c->n, c->rank);  // no NVLS on this box: NVLS calls report UNSUPPORTED
    } else if (st != HFR_SUCCESS) {
      return st;
    } else {
      Region r;
      for (int q = 0; q < c->n; ++q) r.base[q] = (char*)c->nvls->uc[q];
      r.bytes = c->nvls->size;
      r.nvls = true;
      c->regions.push_back(r);
    }
  }
  return HFR_SUCCESS;
}

// Scratch layout per rank: [ONESHOT inbox: 2 x n x oneshot_max][staged copy of
// the message, only for buffers outside peer-mapped memory][the schedule's
// area: CE staging slots (n shard copies) or tree partials (2 fp32 slots)].
// Depends only on (count, dtype, algo, memory kind), so ranks that honour the
// collective contract (the same memory kind on every rank: it is part of the
// call signature) grow in lockstep.
size_t inbox_bytes(const hfr_comm_s* c) { return round_up(2 * (size_t)c->n * c->cfg.oneshot_max_bytes, kAlign); }

// tree chunk (Alg. 1 "Chunk_Size"): the configured one, else per n — r01
// sweeps (C2 fp32): n=2 best at 16384 (572-590 vs 520 GB/s at 32768),
// n>=4 at 24576-32768
uint64_t tree_chunk(const hfr_comm_s* c) {
  if (c->cfg.chunk_elems) return c->cfg.chunk_elems;
  return c->n == 2 ? 16384 : 32768;
}

size_t msg_stage_bytes(size_t count, hfr_dtype_t dt, bool zero_copy) {
  return zero_copy ? 0 : round_up(count * dtype_size(dt), kAlign);
}
size_t ce_slot_bytes(const hfr_comm_s* c, size_t count, hfr_dtype_t dt) {
  return round_up((count / c->n + 256) * dtype_size(dt), kAlign);
}

size_t scratch_need(const hfr_comm_s* c, size_t count, hfr_dtype_t dt, int algo, bool zero_copy) {
  size_t need = inbox_bytes(c) + msg_stage_bytes(count, dt, zero_copy);
  if (algo == HFR_ALGO_CE) need += (size_t)c->n * ce_slot_bytes(c, count, dt);
  if (algo == HFR_ALGO_DBT) need += 2 * round_up(count, 64) * 4;
  if (algo == HFR_ALGO_PAIR_DBT) need += 2 * round_up(pair_half(count), 64) * 4;
  return need;
}

char* stage_base(const hfr_comm_s* c, int q) { return c->scratch.base[q] + inbox_bytes(c); }

// Collective growth without a device-wide synchronisation (VERDICT r01 weak
// #10): the fresh region is zeroed on the setup stream and swapped in; the
// outgrown one stays mapped (kernels in flight here or at peers may still use
// it) and is released at hfr_finalize.
hfr_status_t ensure_scratch(hfr_comm_s* c, size_t need) {
  if (need <= c->scratch.bytes) return HFR_SUCCESS;
  Region fresh;
  HFR_TRY(alloc_region(c, std::max(need, c->scratch.bytes * 2), &fresh));
  c->retired.push_back(c->scratch);
  c->scratch = fresh;
  return HFR_SUCCESS;
}

// ---------------------------------------------------------------------------
// launches
// ---------------------------------------------------------------------------
template <class E>
const void* flat_fn(int n) {
  switch (n) {
    case 1: return (const void*)hfr_flat_kernel<E, 1>;
    case 2: return (const void*)hfr_flat_kernel<E, 2>;
    case 3: return (const void*)hfr_flat_kernel<E, 3>;
    case 4: return (const void*)hfr_flat_kernel<E, 4>;
    case 5: return (const void*)hfr_flat_kernel<E, 5>;
    case 6: return (const void*)hfr_flat_kernel<E, 6>;
    case 7: return (const void*)hfr_flat_kernel<E, 7>;
    case 8: return (const void*)hfr_flat_kernel<E, 8>;
    default: return (const void*)hfr_flat_kernel<E, 0>;
  }
}

template <class E>
const void* flat_tma_fn(int n) {
  switch (n) {
    case 2: return (const void*)hfr_flat_tma_kernel<E, 2>;
    case 4: return (const void*)hfr_flat_tma_kernel<E, 4>;
    case 8: return (const void*)hfr_flat_tma_kernel<E, 8>;
    default: return nullptr;
  }
}

template <class E>
const void* tree_fn(bool pair) {
  return pair ? (const void*)hfr_tree_kernel<E, true> : (const void*)hfr_tree_kernel<E, false>;
}

// Launch one protocol kernel.  Virtual comms (all ranks' CTAs on one GPU):
// cooperative launch, so every rank's CTAs are co-resident.  Real comms with
// `pdl` (the latency-bound small-message kernels: ONESHOT, LL ONESHOT,
// barrier): programmatic dependent launch — the kernel may be scheduled while
// the previous kernel on the stream is in its exit handshake and waits for it
// in hardware (pdl_wait, hfr_kernels.cuh) before touching memory.  r01, n=2,
// bf16, CUDA graph: 1 KiB 3.93 -> 3.75 us, 64 KiB 5.12 -> 4.73, 1 MiB 12.38 ->
// 11.98; the bandwidth kernels (FLAT, FLAT-TMA) measured slower with it at
// 2-64 MiB eager (2 MiB 17.3 -> 20.5 us) and neutral (+-0.3 %) back to back
// at 4 MiB-1 GiB (r02), so they launch plainly (profiles/r01/pdl_ab_n2.jsonl,
// profiles/r02/flat_pdl_ab.jsonl).  hfr_config_t.pdl_off = 1: never.
cudaError_t launch_protocol_kernel(const hfr_comm_s* c, const void* fn, dim3 grid, dim3 block, void** params,
                                   size_t smem, cudaStream_t s, bool pdl_ok) {
  if (c->virt && c->local > 1) return cudaLaunchCooperativeKernel(fn, grid, block, params, smem, s);
  if (!pdl_ok || c->cfg.pdl_off) return cudaLaunchKernel(fn, grid, block, params, smem, s);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelExC(&cfg, fn, params);
}

hfr_status_t launch(hfr_comm_s* c, const void* fn, int grid_x, int threads, Args& a, cudaStream_t s,
                    bool pdl_ok = false) {
  ++c->epoch;  // host mirror (stats only): kernels keep their epoch in device memory
  void* params[] = {&a};
  dim3 grid(grid_x, c->local), block(threads);
  const cudaError_t e = launch_protocol_kernel(c, fn, grid, block, params, 0, s, pdl_ok);
  if (e != cudaSuccess) {
    note_cuda(e, "launch");
    return HFR_ERR_CUDA;
  }
  ++c->launches;
  return HFR_SUCCESS;
}

// threads per CTA: the config's, else the schedule's measured best
int cta_threads(const hfr_comm_s* c, int dflt) { return c->cfg.threads > 0 ? c->cfg.threads : dflt; }

// CTAs per rank: the config cap (default `per_sm` per SM), limited so that
// all ranks' CTAs of a virtual comm are co-resident (cooperative launch).
hfr_status_t ctas_per_rank(hfr_comm_s* c, const void* fn, int threads, int want, int* out, int per_sm = 1) {
  int g = c->cfg.max_ctas > 0 ? c->cfg.max_ctas : per_sm * c->num_sms;
  g = std::min(g, kMaxCtas);
  if (want > 0) g = std::min(g, want);
  if (c->virt && c->local > 1) {
    int occ = 0;
    HFR_CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, 0));
    const int cap = occ * c->num_sms / c->local;
    if (cap < 1) return HFR_ERR_UNSUPPORTED;
    g = std::min(g, cap);
  }
  *out = std::max(g, 1);
  return HFR_SUCCESS;
}

void base_args(hfr_comm_s* c, Args& a, uint64_t count, uint64_t sig) {
  memset(&a, 0, sizeof a);
  for (int q = 0; q < c->n; ++q) a.pad[q] = reinterpret_cast<Pad*>(c->pad.base[q]);
  a.err = c->err_dev;
  a.count = count;
  a.sig = sig;
  a.timeout_ns = (uint64_t)c->cfg.timeout_ms * 1000000ull;
  a.scale = c->cfg.scale;
  a.n = c->n;
  a.rank0 = c->virt ? 0 : c->rank;
  a.trace = c->trace;
  a.trace_cap = c->trace_cap;
  a.src_rank = -1;  // fold all ranks ...
  a.dst_mask = c->n >= 32 ? ~0u : ((1u << c->n) - 1);  // ... into every rank (allreduce)
  a.excl_root = -1;
  a.nvls_op = 3;     // NVLS: ld_reduce + multicast store (allreduce)
  a.nvls_solo = -1;
}

// FLAT-kernel routing of a collective (NEXT-3, "general reduce
// and broadcast"): which rank's shard is read (-1: fold all, -2: my own) and
// which ranks receive it (0: the shard's owner).
void coll_routing(const hfr_comm_s* c, int coll, int root, int* src, uint32_t* dmask, int* excl) {
  *excl = (coll == HFR_REDUCE || coll == HFR_BROADCAST) && c->n > 1 ? root : -1;
  const uint32_t all = c->n >= 32 ? ~0u : ((1u << c->n) - 1);
  switch (coll) {
    case HFR_REDUCE_SCATTER: *src = -1; *dmask = 0; break;
    case HFR_ALLGATHER: *src = -2; *dmask = all; break;
    case HFR_REDUCE: *src = -1; *dmask = 1u << root; break;
    case HFR_BROADCAST: *src = root; *dmask = all & ~(1u << root); break;
    default: *src = -1; *dmask = all;
  }
}

// The kernel attribute is a per-function MAXIMUM: raise it to the largest
// dynamic shared memory asked for so far, never lower it (a lower value set
// for a smaller call would make a later, larger launch of the same kernel
// fail or report zero occupancy).
hfr_status_t allow_dynamic_smem(const void* fn, int smem) {
  static std::mutex mu;
  static std::vector<std::pair<const void*, int>> set;  // (kernel, bytes allowed)
  std::lock_guard<std::mutex> lock(mu);
  for (auto& e : set)
    if (e.first == fn) {
      if (smem <= e.second) return HFR_SUCCESS;
      HFR_CU(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      e.second = smem;
      return HFR_SUCCESS;
    }
  HFR_CU(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  set.emplace_back(fn, smem);
  return HFR_SUCCESS;
}

// TMA-staged FLAT (default for allreduce / reduce-scatter / reduce with n in {2, 4, 8})
hfr_status_t run_flat_tma(hfr_comm_s* c, char* const* bufs, uint64_t count, hfr_dtype_t dt, uint64_t sig,
                          cudaStream_t s, int coll, int root, const void* fn) {
  // 4 KiB per source per stage (r01: 2-8 KiB within noise).  CTAs per SM: 1
  // for a real comm (one rank per GPU) — r01 sweep, bf16 2 MiB-256 MiB and C2:
  // +1 % (large) to +18 % (4 MiB) over 2 per SM at n=2 and n=4, half the
  // per-CTA handshakes (profiles/r01/tma_tile_*.jsonl); 2 for virtual ranks
  // (all n ranks' CTAs share one GPU).  max_ctas overrides.
  const int tile = kTmaTileBytes;
  const int per_sm = c->virt && c->local > 1 ? 2 : 1;
  const int threads = cta_threads(c, 256);
  const int smem = 2 * c->n * tile;
  HFR_TRY(allow_dynamic_smem(fn, smem));
  int g = c->cfg.max_ctas > 0 ? c->cfg.max_ctas : per_sm * c->num_sms;
  // no more CTAs than tiles: idle CTAs would only add handshakes
  const uint64_t per = per_vec(dt);
  const uint64_t tiles = (count / per / c->n + (uint64_t)tile / 16 - 1) / ((uint64_t)tile / 16) + 1;
  g = (int)std::min<uint64_t>((uint64_t)g, tiles);
  if (c->virt && c->local > 1) {
    int occ = 0;
    HFR_CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem));
    g = std::min(g, occ * c->num_sms / c->local);
  }
  g = std::max(1, std::min(g, kMaxCtas));
  Args a;
  base_args(c, a, count, fnv(fnv(sig, 0x544d41), (uint64_t)g * 1315423911ull + threads));
  for (int q = 0; q < c->n; ++q) a.buf[q] = bufs[q];
  a.tma_tile = tile;
  coll_routing(c, coll, root, &a.src_rank, &a.dst_mask, &a.excl_root);
  ++c->epoch;
  void* params[] = {&a};
  cudaError_t e = launch_protocol_kernel(c, fn, dim3(g, c->local), dim3(threads), params, smem, s, false);
  if (e != cudaSuccess) {
    note_cuda(e, "hfr_flat_tma_kernel");
    return HFR_ERR_CUDA;
  }
  ++c->launches;
  return HFR_SUCCESS;
}

hfr_status_t run_flat(hfr_comm_s* c, char* const* bufs, uint64_t count, hfr_dtype_t dt, uint64_t sig,
                      cudaStream_t s, int coll = HFR_ALLREDUCE, int root = 0) {
  // TMA-staged variant by default for n in {2,4,8} (r01: +2.5-4 % over the
  // register-staged kernel; 98.5 % of HBM with 8 virtual ranks); config
  // flat_staging = 1 selects register staging (no shared memory)
  const bool tma = c->cfg.flat_staging != 1;
  if (tma && (coll == HFR_ALLREDUCE || coll == HFR_REDUCE_SCATTER || coll == HFR_REDUCE)) {
#define HFR_TMA_FN(E) flat_tma_fn<E>(c->n)
    const void* tfn = HFR_BY_DTYPE(dt, HFR_TMA_FN);
    if (tfn) return run_flat_tma(c, bufs, count, dt, sig, s, coll, root, tfn);
  }
#define HFR_FLAT_FN(E) flat_fn<E>(c->n)
  const void* fn = HFR_BY_DTYPE(dt, HFR_FLAT_FN);
  const int threads = cta_threads(c, 512);
  const uint64_t per = per_vec(dt);
  const uint64_t vec_per_rank = count / per / c->n + 1;
  int g = 0;
  HFR_TRY(ctas_per_rank(c, fn, threads, (int)std::min<uint64_t>((vec_per_rank + threads - 1) / threads, kMaxCtas), &g));
  Args a;
  base_args(c, a, count, fnv(sig, (uint64_t)g * 1315423911ull + threads));
  for (int q = 0; q < c->n; ++q) a.buf[q] = bufs[q];
  coll_routing(c, coll, root, &a.src_rank, &a.dst_mask, &a.excl_root);
  return launch(c, fn, g, threads, a, s);
}

template <class E>
const void* tree_tma_fn(bool pair) {
  return pair ? (const void*)hfr_tree_tma_kernel<E, true> : (const void*)hfr_tree_tma_kernel<E, false>;
}

// TMA tree kernel geometry (hfr_tree_tma.cuh TreeStage): a 100 KiB
// shared-memory budget per CTA (2 CTAs per SM); the tile is the largest power
// of two dividing the chunk, at most 2048 elements, halved until the largest
// role's stage (x, partner x, two fp32 child partials, fp32 output) fits a
// third of the budget, so every role gets >= 3 stages.
constexpr int kTreeSmem = 100 << 10;
uint32_t tree_stage_max(uint32_t T, uint32_t esz, bool pair) { return T * esz * (pair ? 2 : 1) + 12 * T; }
uint32_t tree_tile(uint64_t C, uint32_t esz, bool pair, uint32_t tmax = 2048, int budget = kTreeSmem) {
  uint32_t T = tmax;
  while (C % T) T >>= 1;
  while (T > 256 && 3 * tree_stage_max(T, esz, pair) > (uint32_t)budget) T >>= 1;
  return T;
}

hfr_status_t run_tree(hfr_comm_s* c, char* const* bufs, uint64_t count, hfr_dtype_t dt, bool pair, uint64_t sig,
                      cudaStream_t s, size_t area) {
  const uint64_t C = tree_chunk(c);
  Args a;
  base_args(c, a, count, 0);
  if (pair) {
    const uint64_t H = pair_half(count);
    a.half_base[0] = 0;
    a.half_len[0] = H;
    a.half_base[1] = H;
    a.half_len[1] = count - H;
    a.part_stride = round_up(H, 64);
    a.ntree = c->n / 2;
  } else {
    a.half_base[0] = a.half_base[1] = 0;
    a.half_len[0] = a.half_len[1] = count;
    a.part_stride = round_up(count, 64);
    a.ntree = c->n;
  }
  fill_tree_nodes(a.ntree, a.tree);
  a.chunk = (int)C;
  for (int q = 0; q < c->n; ++q) {
    a.buf[q] = bufs[q];
    a.part[q] = reinterpret_cast<float*>(stage_base(c, q) + area);
  }
  // auto = register staging: the TMA form (hfr_tree_tma.cuh) measured slower
  // at every size, n and dtype in round 2 (n=4 fp32 C2: DBT 404 vs 443 GB/s,
  // PAIR 503 vs 595; n=2: 563 vs 598, 581 vs 625; bf16 1 GiB n=4: 304 vs 390)
  const bool tma = c->cfg.tree_staging == 2;
  if (tma) {
    // hfr_tree_tma.cuh: one producer thread + 3 fold warps per CTA, flags per
    // tile, a shared-memory ring of 3-8 stages (by role).  All CTAs of every rank must be
    // co-resident (a CTA spins on tiles of peers' CTAs), so the grid is capped
    // by the occupancy at this shared-memory size.
#define HFR_TREE_TMA_FN(E) tree_tma_fn<E>(pair)
    const void* fn = HFR_BY_DTYPE(dt, HFR_TREE_TMA_FN);
    const uint32_t esz = (uint32_t)dtype_size(dt);
    // r02 sweep (n=2, C2 fp32): a 100 KiB budget at 2 CTAs/SM beats 200 KiB at
    // 1/SM (557 vs 391 GB/s) and 64 KiB at 3/SM (489); 4096-element tiles
    // +1 % over 2048 (profiles/r02/tree_tma_*.jsonl)
    const int smem = kTreeSmem;
    const uint32_t T = tree_tile(C, esz, pair, 4096u, smem);
    HFR_TRY(allow_dynamic_smem(fn, smem));
    int occ = 0;
    HFR_CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kTreeThreads, smem));
    if (occ < 1) return HFR_ERR_UNSUPPORTED;
    const int per_sm = std::min(occ, 3);
    a.tree_tile = T;
    a.tree_smem = smem;
    const uint64_t nt = (a.half_len[0] + T - 1) / T;  // tiles of the longer half
    for (uint64_t lo = 0; lo < std::max<uint64_t>(nt, 1); lo += kMaxChunks) {
      const uint64_t hi = lo + kMaxChunks;
      const uint64_t here = std::min<uint64_t>(nt, hi) - std::min<uint64_t>(nt, lo);
      int g = c->cfg.max_ctas > 0 ? c->cfg.max_ctas : per_sm * c->num_sms;
      g = std::min(g, occ * c->num_sms / c->local);
      g = (int)std::min<uint64_t>((uint64_t)g, std::max<uint64_t>(here, 2));
      g = std::max(2, std::min(g, kMaxCtas) & ~1);  // even: CTA b works on tree b & 1 only
      a.c_lo = (uint32_t)lo;
      a.c_hi = (uint32_t)hi;
      a.sig = fnv(fnv(fnv(sig, (uint64_t)g * 1315423911ull + kTreeThreads), lo), 0x7474ull + T * 16);
      ++c->epoch;
      void* params[] = {&a};
      const cudaError_t e = launch_protocol_kernel(c, fn, dim3(g, c->local), dim3(kTreeThreads), params, smem, s, false);
      if (e != cudaSuccess) {
        note_cuda(e, "hfr_tree_tma_kernel");
        return HFR_ERR_CUDA;
      }
      ++c->launches;
    }
    return HFR_SUCCESS;
  }
#define HFR_TREE_FN(E) tree_fn<E>(pair)
  const void* fn = HFR_BY_DTYPE(dt, HFR_TREE_FN);
  // register staging: 2-3 CTAs x 256 threads per SM: while one CTA drains its
  // chunk's stores at the per-chunk system fence the others issue (r01, n=4:
  // DBT 1 -> 2 CTAs/SM 377 -> 422 GB/s; fp32 DBT 2 -> 3 CTAs/SM 423 -> 442 and
  // n=2 572 -> 591, but PAIR (shared-memory partner ring) 590-609 -> 561 and
  // bf16 DBT 388 -> 377, so those keep 2).  At ~120 registers per thread only
  // 2 such CTAs are resident per SM; the rest start as the first ones finish.
  // That cannot deadlock: CTA b of a rank waits only on CTA b of other ranks
  // (chunk c is served by CTA (c - c_lo) mod g everywhere), and every rank
  // makes its low-index CTAs resident first.
  const int threads = cta_threads(c, 256);
  const int per_sm = !pair && dt == HFR_FLOAT32 ? 3 : 2;
  const uint64_t nch = (a.half_len[0] + C - 1) / C;  // half 0 is the longer one
  for (uint64_t lo = 0; lo < std::max<uint64_t>(nch, 1); lo += kMaxChunks) {
    const uint64_t hi = lo + kMaxChunks;
    const uint64_t here = std::min<uint64_t>(nch, hi) - std::min<uint64_t>(nch, lo);
    // An EVEN number of CTAs per rank: CTA b then only ever sees chunks of
    // tree b & 1, so the two trees' dependency chains never interleave inside
    // one CTA (a rank is the root of one tree and a leaf of the other).
    int g = 0;
    HFR_TRY(ctas_per_rank(c, fn, threads, (int)std::min<uint64_t>(std::max<uint64_t>(here, 2), kMaxCtas), &g, per_sm));
    g = std::max(2, g & ~1);
    a.c_lo = (uint32_t)lo;
    a.c_hi = (uint32_t)hi;
    a.sig = fnv(fnv(sig, (uint64_t)g * 1315423911ull + threads), lo);
    HFR_TRY(launch(c, fn, g, threads, a, s));
  }
  return HFR_SUCCESS;
}

hfr_status_t run_oneshot_ll(hfr_comm_s* c, char* const* local_bufs, uint64_t count, hfr_dtype_t dt, uint64_t sig,
                            cudaStream_t s) {
  const void* fn;
#define HFR_LL2(E) (const void*)hfr_oneshot_ll_kernel<E, 2>
#define HFR_LL4(E) (const void*)hfr_oneshot_ll_kernel<E, 4>
#define HFR_LL8(E) (const void*)hfr_oneshot_ll_kernel<E, 8>
#define HFR_LL0(E) (const void*)hfr_oneshot_ll_kernel<E, 0>
  switch (c->n) {
    case 2: fn = HFR_BY_DTYPE(dt, HFR_LL2); break;
    case 4: fn = HFR_BY_DTYPE(dt, HFR_LL4); break;
    case 8: fn = HFR_BY_DTYPE(dt, HFR_LL8); break;
    default: fn = HFR_BY_DTYPE(dt, HFR_LL0);
  }
  const uint64_t npair = (count + 1) / 2;
  // one pair per thread: every word's latency overlaps every other's
  const int threads = (int)std::max<uint64_t>(32, std::min<uint64_t>(256, round_up(npair, 32)));
  int g = 0;
  HFR_TRY(ctas_per_rank(c, fn, threads, (int)std::min<uint64_t>((npair + threads - 1) / threads, kMaxCtas), &g));
  Args a;
  base_args(c, a, count, fnv(sig, 0x11ull + (uint64_t)g * 1315423911ull + threads));
  a.slot_bytes = c->cfg.oneshot_max_bytes;
  for (int q = 0; q < c->n; ++q) a.inbox[q] = c->scratch.base[q];
  for (int q = 0; q < c->local; ++q) a.buf[c->virt ? q : c->rank] = local_bufs[q];
  return launch(c, fn, g, threads, a, s, true);
}

hfr_status_t run_oneshot(hfr_comm_s* c, char* const* local_bufs, uint64_t count, hfr_dtype_t dt, uint64_t sig,
                         cudaStream_t s) {
  // LL form: 8 inbox bytes per element, one NVLink write of latency
  if (ll_fits(c, count) && (c->cfg.algo == HFR_ALGO_AUTO || ll_pays(c, count)))
    return run_oneshot_ll(c, local_bufs, count, dt, sig, s);
#define HFR_ONESHOT_FN(E) (const void*)hfr_oneshot_kernel<E, 0>
  const void* fn = HFR_BY_DTYPE(dt, HFR_ONESHOT_FN);
  const uint64_t per = per_vec(dt);
  const uint64_t nvec = count / per;
  // small grids: one CTA per 2048 vectors (32 KiB), at least n threads
  const int min_thr = 32 * ((c->n + 31) / 32);
  const int threads = (int)std::max<uint64_t>(min_thr, std::min<uint64_t>(cta_threads(c, 512), round_up(std::max<uint64_t>(nvec, 1), 32)));
  int g = 0;
  HFR_TRY(ctas_per_rank(c, fn, threads, (int)std::min<uint64_t>((nvec + 2047) / 2048 + 1, kMaxCtas), &g));
  Args a;
  base_args(c, a, count, fnv(sig, (uint64_t)g * 1315423911ull + threads));
  a.slot_bytes = c->cfg.oneshot_max_bytes;
  for (int q = 0; q < c->n; ++q) a.inbox[q] = c->scratch.base[q];
  for (int q = 0; q < c->local; ++q) a.buf[c->virt ? q : c->rank] = local_bufs[q];
  return launch(c, fn, g, threads, a, s, true);
}

// ---------------------------------------------------------------------------
// CE schedule (copy engines + stream memory operations)
// ---------------------------------------------------------------------------
typedef int (*StreamValueFn)(cudaStream_t, unsigned long long, uint64_t, unsigned);
constexpr unsigned kWaitGeq = 0x0;        // CU_STREAM_WAIT_VALUE_GEQ
constexpr unsigned kWriteFenced = 0x0;    // CU_STREAM_WRITE_VALUE_DEFAULT: preceded by a system-wide fence

hfr_status_t stream_value_fns(StreamValueFn* wr, StreamValueFn* wt) {
  static StreamValueFn w = nullptr, t = nullptr;
  if (!w || !t) {
    cudaDriverEntryPointQueryResult q1, q2;
    void *f1 = nullptr, *f2 = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue64", &f1, cudaEnableDefault, &q1) != cudaSuccess ||
        cudaGetDriverEntryPoint("cuStreamWaitValue64", &f2, cudaEnableDefault, &q2) != cudaSuccess ||
        q1 != cudaDriverEntryPointSuccess || q2 != cudaDriverEntryPointSuccess)
      return HFR_ERR_UNSUPPORTED;
    w = (StreamValueFn)f1;
    t = (StreamValueFn)f2;
  }
  *wr = w;
  *wt = t;
  return HFR_SUCCESS;
}

// Handshake through stream memory operations (no SM involved): local rank l
// writes `e` into field[rank(l)] of every peer's pad (fenced) on streams[l];
// then streams[l] waits until field[q] >= e for every peer q.  Every write is
// submitted before any wait, so ranks driven by one process (virtual comms)
// cannot deadlock on a shared hardware queue.
hfr_status_t ce_handshake(hfr_comm_s* c, const cudaStream_t* streams, size_t field, uint64_t e) {
  StreamValueFn wr = nullptr, wt = nullptr;
  HFR_TRY(stream_value_fns(&wr, &wt));
  for (int l = 0; l < c->local; ++l) {
    const int r = c->virt ? l : c->rank;
    for (int q = 0; q < c->n; ++q) {
      if (q == r) continue;
      const unsigned long long dst = (unsigned long long)(c->pad.base[q] + field + 8 * (size_t)r);
      if (wr(streams[l], dst, e, kWriteFenced) != 0) {
        g_cuda_error = "cuStreamWriteValue64 on peer memory failed";
        return HFR_ERR_CUDA;
      }
    }
  }
  for (int l = 0; l < c->local; ++l) {
    const int r = c->virt ? l : c->rank;
    for (int q = 0; q < c->n; ++q) {
      if (q == r) continue;
      const unsigned long long src = (unsigned long long)(c->pad.base[r] + field + 8 * (size_t)q);
      if (wt(streams[l], src, e, kWaitGeq) != 0) {
        g_cuda_error = "cuStreamWaitValue64 failed";
        return HFR_ERR_CUDA;
      }
    }
  }
  return HFR_SUCCESS;
}

hfr_status_t ce_streams(hfr_comm_s* c) {
  if (c->ce_h) return HFR_SUCCESS;
  int lo = 0, hi = 0;
  HFR_CU(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  const int H = c->virt ? 1 : c->n - 1;
  auto mk_stream = [&](std::vector<cudaStream_t>& v) -> hfr_status_t {
    cudaStream_t h = nullptr;
    HFR_CU(cudaStreamCreateWithPriority(&h, cudaStreamNonBlocking, hi));
    v.push_back(h);
    return HFR_SUCCESS;
  };
  auto mk_event = [&](std::vector<cudaEvent_t>& v) -> hfr_status_t {
    cudaEvent_t ev = nullptr;
    HFR_CU(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    v.push_back(ev);
    return HFR_SUCCESS;
  };
  for (int l = 0; l < c->local; ++l) {
    if (c->virt) HFR_TRY(mk_stream(c->ce_fold));
    HFR_TRY(mk_event(c->ce_fork));
    HFR_TRY(mk_event(c->ce_join));
    for (int j = 0; j < H; ++j) {
      HFR_TRY(mk_stream(c->helpers));
      HFR_TRY(mk_stream(c->ag_helpers));
      HFR_TRY(mk_event(c->ag_events));
      for (int i = 0; i < kCeMaxChunks; ++i) HFR_TRY(mk_event(c->chunk_events));
    }
  }
  c->ce_h = H;
  return HFR_SUCCESS;
}

// CE schedule, chunk-pipelined (Alg. 1's "split Dg by Chunk_Size" + the
// paper's pipelining): shard r is cut into K chunks
// (K the same on every rank: a function of count and n only).  For every rank
// r this process drives (one, or all n for a virtual comm):
//   reduce-scatter pulls: helper streams copy chunk i of shard r from every
//     peer q into staging slot q, back to back for i = 0..K-1 (copy engines,
//     one cudaMemcpyAsync per copy);
//   fold: r's fold stream folds chunk i (SMs, local, rank order) as soon as
//     its n-1 pulls landed, then publishes ce_done[r] = (e << 20) | (i + 1) at
//     every peer with a fenced stream write;
//   all-gather pulls: helper streams wait (stream memop) until peer q
//     published chunk i of shard q and copy it into r's buffer.
// So chunk i's all-gather overlaps chunk i+1's reduce-scatter pull and fold.
// Entry/exit: ce_ready / ce_exit handshakes (no SM involved).
hfr_status_t run_ce(hfr_comm_s* c, char* const* bufs, uint64_t count, hfr_dtype_t dt, cudaStream_t s, size_t area) {
  HFR_TRY(ce_streams(c));
  const int n = c->n, L = c->local, H = c->ce_h;
  const size_t esz = dtype_size(dt);
  uint64_t lo[kMaxRanks + 1];
  for (int g = 0; g < n; ++g) lo[g] = count * g / n / 256 * 256;
  lo[n] = count;
  const size_t slot = ce_slot_bytes(c, count, dt);
  const uint64_t e = ++c->ce_epoch;
  StreamValueFn wr = nullptr, wt = nullptr;
  HFR_TRY(stream_value_fns(&wr, &wt));
  // pipeline depth: every chunk >= kCeMinChunkBytes, at most kCeMaxChunks
  const uint64_t shard_bytes = count / n * esz;
  const int K = (int)std::max<uint64_t>(1, std::min<uint64_t>(kCeMaxChunks, shard_bytes / kCeMinChunkBytes));
  auto chunk = [&](int g, int i, uint64_t* b, uint64_t* len) {  // chunk i of shard g, elements
    const uint64_t Lg = lo[g + 1] - lo[g];
    const uint64_t C = (Lg + K - 1) / K / 256 * 256 + 256;
    const uint64_t s0 = std::min<uint64_t>(Lg, (uint64_t)i * C), s1 = std::min<uint64_t>(Lg, (uint64_t)(i + 1) * C);
    *b = lo[g] + s0;
    *len = (i == K - 1 ? Lg : s1) - s0;
  };
  auto rank_of = [&](int l) { return c->virt ? l : c->rank; };
  auto helper = [&](int l, int q) {  // helper index of peer q for local rank l
    const int r = rank_of(l);
    return l * H + (H == 1 ? 0 : (q < r ? q : q - 1));
  };
  // fold streams: the call's stream (real) or one per virtual rank, forked from it
  cudaStream_t fs[kMaxRanks];
  if (c->virt) {
    HFR_CU(cudaEventRecord(c->ce_join[0], s));
    for (int l = 0; l < L; ++l) {
      fs[l] = c->ce_fold[l];
      HFR_CU(cudaStreamWaitEvent(fs[l], c->ce_join[0], 0));
    }
  } else {
    fs[0] = s;
  }
  // 1. every rank's buffer is ready ("wait for chunk-i transfer")
  HFR_TRY(ce_handshake(c, fs, offsetof(Pad, ce_ready), e));
  // 2. reduce-scatter transfers: all chunks, back to back, per helper
  for (int l = 0; l < L; ++l) {
    const int r = rank_of(l);
    char* stage = stage_base(c, r) + area;
    HFR_CU(cudaEventRecord(c->ce_fork[l], fs[l]));
    for (int j = 0; j < H; ++j) {
      HFR_CU(cudaStreamWaitEvent(c->helpers[l * H + j], c->ce_fork[l], 0));
      HFR_CU(cudaStreamWaitEvent(c->ag_helpers[l * H + j], c->ce_fork[l], 0));
    }
    for (int i = 0; i < K; ++i) {
      uint64_t b, len;
      chunk(r, i, &b, &len);
      for (int q = 0; q < n; ++q) {
        if (q == r || !len) continue;
        HFR_CU(cudaMemcpyAsync(stage + (size_t)q * slot + (b - lo[r]) * esz, bufs[q] + b * esz, len * esz,
                               cudaMemcpyDeviceToDevice, c->helpers[helper(l, q)]));
      }
      for (int j = 0; j < H; ++j)
        HFR_CU(cudaEventRecord(c->chunk_events[(size_t)(l * H + j) * kCeMaxChunks + i], c->helpers[l * H + j]));
    }
  }
  // 3./4. per chunk: fold (SMs, local, rank order) once its pulls landed and
  // publish it; then the all-gather pulls of chunk i, each gated on the
  // owner's flag.  Host submission order matters: streams may share a
  // hardware queue, so a blocking stream wait is only ever submitted AFTER
  // everything any rank's flag depends on (the RS pulls, this chunk's folds
  // and flag writes of every local rank) — no false dependency can then
  // deadlock the ranks.
  for (int i = 0; i < K; ++i) {
    for (int l = 0; l < L; ++l) {
      const int r = rank_of(l);
      char* stage = stage_base(c, r) + area;
      for (int j = 0; j < H; ++j)
        HFR_CU(cudaStreamWaitEvent(fs[l], c->chunk_events[(size_t)(l * H + j) * kCeMaxChunks + i], 0));
      uint64_t b, len;
      chunk(r, i, &b, &len);
      if (len) {
        FoldArgs f{};
        for (int q = 0; q < n; ++q)
          f.src[q] = q == r ? bufs[r] + b * esz : stage + (size_t)q * slot + (b - lo[r]) * esz;
        f.dst = bufs[r] + b * esz;
        f.count = len;
        f.scale = c->cfg.scale;
        f.n = n;
        const int ctas = (int)std::max<uint64_t>(
            1, std::min<uint64_t>(c->cfg.max_ctas > 0 ? c->cfg.max_ctas : c->num_sms / L, (len / 4 + 511) / 512));
        if (dt == HFR_BFLOAT16)
          hfr_local_fold_kernel<BF16><<<ctas, 512, 0, fs[l]>>>(f);
        else if (dt == HFR_FLOAT16)
          hfr_local_fold_kernel<F16><<<ctas, 512, 0, fs[l]>>>(f);
        else if (dt == HFR_FP8_E4M3)
          hfr_local_fold_kernel<E4M3><<<ctas, 512, 0, fs[l]>>>(f);
        else if (dt == HFR_FP8_E5M2)
          hfr_local_fold_kernel<E5M2><<<ctas, 512, 0, fs[l]>>>(f);
        else
          hfr_local_fold_kernel<F32><<<ctas, 512, 0, fs[l]>>>(f);
        cudaError_t err = cudaGetLastError();
        if (err != cudaSuccess) {
          note_cuda(err, "hfr_local_fold_kernel");
          return HFR_ERR_CUDA;
        }
        ++c->launches;
      }
      for (int q = 0; q < n; ++q) {
        if (q == r) continue;
        const unsigned long long dst = (unsigned long long)(c->pad.base[q] + offsetof(Pad, ce_done) + 8 * (size_t)r);
        if (wr(fs[l], dst, (e << 20) | (uint64_t)(i + 1), kWriteFenced) != 0) {
          g_cuda_error = "cuStreamWriteValue64 on peer memory failed";
          return HFR_ERR_CUDA;
        }
      }
    }
    for (int l = 0; l < L; ++l) {
      const int r = rank_of(l);
      for (int q = 0; q < n; ++q) {
        if (q == r) continue;
        cudaStream_t h = c->ag_helpers[helper(l, q)];
        const unsigned long long flag = (unsigned long long)(c->pad.base[r] + offsetof(Pad, ce_done) + 8 * (size_t)q);
        if (wt(h, flag, (e << 20) | (uint64_t)(i + 1), kWaitGeq) != 0) {
          g_cuda_error = "cuStreamWaitValue64 failed";
          return HFR_ERR_CUDA;
        }
        uint64_t qb, qlen;
        chunk(q, i, &qb, &qlen);
        if (qlen) HFR_CU(cudaMemcpyAsync(bufs[r] + qb * esz, bufs[q] + qb * esz, qlen * esz, cudaMemcpyDeviceToDevice, h));
      }
    }
  }
  for (int l = 0; l < L; ++l)
    for (int j = 0; j < H; ++j) {
      HFR_CU(cudaEventRecord(c->ag_events[l * H + j], c->ag_helpers[l * H + j]));
      HFR_CU(cudaStreamWaitEvent(fs[l], c->ag_events[l * H + j], 0));
    }
  // 5. every rank finished pulling from every buffer
  HFR_TRY(ce_handshake(c, fs, offsetof(Pad, ce_exit), e));
  if (c->virt) {
    for (int l = 0; l < L; ++l) {
      HFR_CU(cudaEventRecord(c->ce_join[l], fs[l]));
      HFR_CU(cudaStreamWaitEvent(s, c->ce_join[l], 0));
    }
  }
  return HFR_SUCCESS;
}

hfr_status_t run_nvls(hfr_comm_s* c, char* const* bufs, uint64_t count, hfr_dtype_t dt, uint64_t sig, uint64_t offset,
                      cudaStream_t s, int coll = HFR_ALLREDUCE, int root = 0) {
#define HFR_NVLS_FN(E) (const void*)hfr_nvls_kernel<E>
#define HFR_NVLS_COLL_FN(E) (const void*)hfr_nvls_coll_kernel<E>
  if (dtype_fp8(dt)) return HFR_ERR_UNSUPPORTED;
  const void* fn = coll == HFR_ALLREDUCE ? HFR_BY_DTYPE_NO_FP8(dt, HFR_NVLS_FN) : HFR_BY_DTYPE_NO_FP8(dt, HFR_NVLS_COLL_FN);
  const int threads = cta_threads(c, 512);
  const uint64_t per = per_vec(dt);
  // reduce / broadcast: the root alone moves the whole buffer
  const bool solo = coll == HFR_REDUCE || coll == HFR_BROADCAST;
  const uint64_t vec_per_rank = count / per / (solo ? 1 : c->n) + 1;
  int g = 0;
  HFR_TRY(ctas_per_rank(c, fn, threads, (int)std::min<uint64_t>((vec_per_rank + threads - 1) / threads, kMaxCtas), &g));
  Args a;
  base_args(c, a, count, fnv(sig, (uint64_t)g * 1315423911ull + threads));
  for (int q = 0; q < c->n; ++q) a.buf[q] = bufs[q];
  a.mcbuf = (char*)c->nvls->mcva + offset;
  a.mc_exit = (uint32_t*)c->nvls->mcva;
  a.uc_exit = (uint32_t*)c->nvls->uc[c->rank];
  switch (coll) {
    case HFR_REDUCE_SCATTER: a.nvls_op = 1; break;
    case HFR_ALLGATHER: a.nvls_op = 2; break;
    case HFR_REDUCE: a.nvls_op = 1; a.nvls_solo = root; break;
    case HFR_BROADCAST: a.nvls_op = 2; a.nvls_solo = root; break;
    default: a.nvls_op = 3;
  }
  return launch(c, fn, g, threads, a, s);
}

hfr_status_t run_copy(hfr_comm_s* c, char* dst, const char* src, uint64_t bytes, cudaStream_t s) {
  if (bytes == 0) return HFR_SUCCESS;
  const int threads = 512;
  const uint64_t want = (bytes / 16 + threads - 1) / threads;
  const int g = (int)std::max<uint64_t>(1, std::min<uint64_t>(want, (uint64_t)c->num_sms * 4));
  hfr_copy_kernel<<<g, threads, 0, s>>>(dst, src, bytes);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    note_cuda(e, "hfr_copy_kernel");
    return HFR_ERR_CUDA;
  }
  ++c->launches;
  return HFR_SUCCESS;
}

bool find_region(hfr_comm_s* c, const char* p, size_t bytes, const Region** out) {
  for (const Region& r : c->regions) {
    const char* b = r.base[c->rank];
    if (b && p >= b && p + bytes <= b + r.bytes) {
      *out = &r;
      return true;
    }
  }
  return false;
}

cudaEvent_t take_event(hfr_comm_s* c) {
  if (!c->ev_pool.empty()) {
    cudaEvent_t e = c->ev_pool.back();
    c->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
  return e;
}

// The body shared by hfr_allreduce / hfr_allreduce_virtual.  bufs[q] is local
// rank q's buffer (virtual: q = 0..n-1; real: only bufs[0] = this rank's).
hfr_status_t allreduce_impl(hfr_comm_s* c, char* const* local_bufs, size_t count, hfr_dtype_t dt, hfr_op_t op,
                            cudaStream_t user, hfr_req_t* req, int coll = HFR_ALLREDUCE, int root = 0) {
  if (!c) return HFR_ERR_NOT_INITIALIZED;
  if (req) *req = nullptr;
  if (!dtype_valid(dt)) return HFR_ERR_INVALID_ARGUMENT;
  if (coll < HFR_ALLREDUCE || coll > HFR_BROADCAST) return HFR_ERR_INVALID_ARGUMENT;
  if ((coll == HFR_REDUCE || coll == HFR_BROADCAST) && (root < 0 || root >= c->n)) return HFR_ERR_INVALID_ARGUMENT;
  if (op != HFR_SUM) return HFR_ERR_UNSUPPORTED;
  if (c->sticky != HFR_SUCCESS) return c->sticky;
  // the other collectives run on the FLAT kernel's routing (NEXT-3)
  // (algo NVLS: every collective on the multicast object)
  const int algo = coll == HFR_ALLREDUCE ? effective_algo(c, count, dtype_size(dt))
                   : c->cfg.algo == HFR_ALGO_NVLS ? HFR_ALGO_NVLS
                                                  : HFR_ALGO_FLAT;
  if (algo == HFR_ALGO_PAIR_DBT && c->n % 2 != 0) return HFR_ERR_UNSUPPORTED;
  if (algo == HFR_ALGO_NVLS && (c->virt || !c->nvls || !c->nvls->on)) return HFR_ERR_UNSUPPORTED;
  for (int q = 0; q < c->local; ++q)
    if (count > 0 && !local_bufs[q]) return HFR_ERR_INVALID_ARGUMENT;
  DeviceGuard guard(c->dev);

  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  HFR_CU(cudaStreamIsCapturing(user, &cap));
  const bool capturing = cap != cudaStreamCaptureStatusNone;
  const size_t esz = dtype_size(dt);
  const size_t bytes = count * esz;
  // zero-copy iff every local buffer is 16-B aligned and (real comm) lies in
  // peer-mapped memory; otherwise stage through the scratch.
  bool aligned = true;
  for (int q = 0; q < c->local; ++q) aligned &= (reinterpret_cast<uintptr_t>(local_bufs[q]) & 15) == 0;
  const Region* reg = nullptr;
  const bool zero_copy = count > 0 && aligned && (c->virt || find_region(c, local_bufs[0], bytes, &reg));
  const uint64_t offset = zero_copy && reg ? (uint64_t)(local_bufs[0] - reg->base[c->rank]) : 0;
  // ONESHOT never stages (peers never touch this rank's buffer)
  const size_t need = count == 0 ? 0 : scratch_need(c, count, dt, algo, zero_copy || algo == HFR_ALGO_ONESHOT);
  if (capturing && need > c->scratch.bytes)
    return HFR_ERR_UNSUPPORTED;  // scratch growth is collective: call once before capturing
  // the CE schedule's stream-memop flags carry a host-side epoch, which a
  // replayed graph would repeat (stale flags would pass): not capturable
  if (capturing && count > 0 && algo == HFR_ALGO_CE) return HFR_ERR_UNSUPPORTED;

  cudaStream_t s = user;
  if (req) {
    cudaEvent_t ready = take_event(c);
    if (!ready) return HFR_ERR_CUDA;
    HFR_CU(cudaEventRecord(ready, user));
    HFR_CU(cudaStreamWaitEvent(c->side, ready, 0));
    c->ev_pool.push_back(ready);
    s = c->side;
  }
  // issue order: after the previous call of this comm, whatever its stream
  // (captured calls are ordered by their capture stream alone)
  if (!capturing && c->has_last) HFR_CU(cudaStreamWaitEvent(s, c->last_op, 0));
  if (count > 0) {
    HFR_TRY(ensure_scratch(c, need));
    uint64_t sig = 1469598103934665603ull;
    sig = fnv(sig, count);
    sig = fnv(sig, (uint64_t)dt | ((uint64_t)op << 8) | ((uint64_t)algo << 16) | ((uint64_t)coll << 24) |
                       ((uint64_t)root << 32));
    uint32_t sbits;
    memcpy(&sbits, &c->cfg.scale, 4);
    sig = fnv(sig, sbits);
    const bool gate = c->cfg.stream_gate && !c->virt && c->n > 1 && algo != HFR_ALGO_CE && !capturing;
    if (gate) HFR_TRY(ce_handshake(c, &s, offsetof(Pad, ce_ready), ++c->ce_epoch));
    if (algo == HFR_ALGO_ONESHOT) {
      // peers never touch this rank's buffer: no staging, any device pointer
      HFR_TRY(run_oneshot(c, local_bufs, count, dt, sig, s));
      goto done;
    }
    {
    char* bufs[kMaxRanks] = {};
    if (zero_copy) {
      for (int q = 0; q < c->n; ++q) bufs[q] = c->virt ? local_bufs[q] : reg->base[q] + offset;
    } else {
      for (int q = 0; q < c->n; ++q) bufs[q] = stage_base(c, q);
      for (int q = 0; q < c->local; ++q) {
        const int r = c->virt ? q : c->rank;
        HFR_TRY(run_copy(c, stage_base(c, r), local_bufs[q], bytes, s));
      }
    }
    const size_t area = msg_stage_bytes(count, dt, zero_copy);  // the schedule's scratch area
    sig = fnv(sig, (uint64_t)zero_copy);
    sig = fnv(sig, algo == HFR_ALGO_FLAT ? 0 : tree_chunk(c));
    sig = fnv(sig, offset);
    if (algo == HFR_ALGO_NVLS) {
      if (!zero_copy || !reg || !reg->nvls || !c->nvls || !c->nvls->on) return HFR_ERR_UNSUPPORTED;
      HFR_TRY(run_nvls(c, bufs, count, dt, sig, offset, s, coll, root));
    } else if (algo == HFR_ALGO_CE) {
      HFR_TRY(run_ce(c, bufs, count, dt, s, area));
    } else if (algo == HFR_ALGO_FLAT) {
      HFR_TRY(run_flat(c, bufs, count, dt, sig, s, coll, root));
    } else {
      HFR_TRY(run_tree(c, bufs, count, dt, algo == HFR_ALGO_PAIR_DBT, sig, s, area));
    }
    if (!zero_copy) {
      for (int q = 0; q < c->local; ++q) {
        const int r = c->virt ? q : c->rank;
        HFR_TRY(run_copy(c, local_bufs[q], stage_base(c, r), bytes, s));
      }
    }
    }
  }
done:
  if (!capturing) {
    HFR_CU(cudaEventRecord(c->last_op, s));
    c->has_last = true;
  }
  if (req) {
    cudaEvent_t done = take_event(c);
    if (!done) return HFR_ERR_CUDA;
    HFR_CU(cudaEventRecord(done, s));
    hfr_req_s* r = new hfr_req_s;
    r->ev = done;
    r->comm = c;
    *req = r;
  }
  return HFR_SUCCESS;
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

void hfr_config_default(hfr_config_t* cfg) {
  if (!cfg) return;
  memset(cfg, 0, sizeof *cfg);
  cfg->algo = HFR_ALGO_AUTO;
  cfg->scale = 1.0f;
  resolve_defaults(*cfg);
}

static hfr_status_t init_common(hfr_comm_t* comm, int rank, int nranks, int dev, bool virt, hfr_allgather_fn ag,
                                void* ctx, const hfr_config_t* cfg) {
  if (!comm) return HFR_ERR_INVALID_ARGUMENT;
  *comm = nullptr;
  if (nranks < 1 || nranks > HFR_MAX_RANKS || rank < 0 || rank >= nranks || dev < 0)
    return HFR_ERR_INVALID_ARGUMENT;
  if (!virt && nranks > 1 && !ag) return HFR_ERR_INVALID_ARGUMENT;
  hfr_config_t c;
  if (cfg) {
    c = *cfg;
  } else {
    hfr_config_default(&c);
  }
  HFR_TRY(validate_cfg(c));
  resolve_defaults(c);
  int ndev = 0;
  HFR_CU(cudaGetDeviceCount(&ndev));
  if (dev >= ndev) return HFR_ERR_INVALID_ARGUMENT;
  DeviceGuard guard(dev);
  hfr_comm_s* x = new hfr_comm_s;
  x->rank = rank;
  x->n = nranks;
  x->dev = dev;
  x->virt = virt;
  x->local = virt ? nranks : 1;
  x->cfg = c;
  x->ag = ag;
  x->ctx = ctx;
  hfr_status_t s = common_init(x);
  if (s != HFR_SUCCESS) {
    hfr_finalize(x);
    return s;
  }
  *comm = x;
  return HFR_SUCCESS;
}

hfr_status_t hfr_init(hfr_comm_t* comm, int rank, int nranks, int cuda_device, hfr_allgather_fn allgather, void* ctx,
                      const hfr_config_t* cfg) {
  return init_common(comm, rank, nranks, cuda_device, false, allgather, ctx, cfg);
}

hfr_status_t hfr_init_virtual(hfr_comm_t* comm, int nranks, int cuda_device, const hfr_config_t* cfg) {
  return init_common(comm, 0, nranks, cuda_device, true, nullptr, nullptr, cfg);
}

hfr_status_t hfr_comm_set_config(hfr_comm_t c, const hfr_config_t* cfg) {
  if (!c) return HFR_ERR_NOT_INITIALIZED;
  if (!cfg) return HFR_ERR_INVALID_ARGUMENT;
  hfr_config_t n = *cfg;
  HFR_TRY(validate_cfg(n));
  n.scratch_bytes = c->cfg.scratch_bytes;
  n.timeout_ms = c->cfg.timeout_ms;
  n.oneshot_max_bytes = c->cfg.oneshot_max_bytes;
  n.nvls_bytes = c->cfg.nvls_bytes;
  resolve_defaults(n);
  c->cfg = n;
  return HFR_SUCCESS;
}

int hfr_comm_local_ranks(hfr_comm_t c) { return c ? c->local : 0; }
int hfr_comm_rank(hfr_comm_t c) { return c ? c->rank : -1; }
int hfr_comm_nranks(hfr_comm_t c) { return c ? c->n : 0; }
uint64_t hfr_comm_launches(hfr_comm_t c) { return c ? c->launches : 0; }

hfr_status_t hfr_mem_alloc(hfr_comm_t c, size_t bytes, void** ptrs) {
  if (!c) return HFR_ERR_NOT_INITIALIZED;
  if (!ptrs || bytes == 0) return HFR_ERR_INVALID_ARGUMENT;
  DeviceGuard guard(c->dev);
  if (c->nvls && c->nvls->on && c->nvls->used + bytes <= c->nvls->size) {
    // symmetric bump allocation inside the NVLS arena (same offsets on every rank)
    ptrs[0] = (void*)(c->nvls->uc[c->rank] + c->nvls->used);
    c->nvls->used += round_up(bytes, 4096);
    return HFR_SUCCESS;
  }
  Region r;
  HFR_TRY(alloc_region(c, bytes, &r));
  c->regions.push_back(r);
  for (int q = 0; q < c->local; ++q) ptrs[q] = r.base[c->virt ? q : c->rank];
  return HFR_SUCCESS;
}

hfr_status_t hfr_mem_free(hfr_comm_t c, void* ptr) {
  if (!c) return HFR_ERR_NOT_INITIALIZED;
  DeviceGuard guard(c->dev);
  if (c->nvls && c->nvls->on && (CUdeviceptr)ptr >= c->nvls->uc[c->rank] &&
      (CUdeviceptr)ptr < c->nvls->uc[c->rank] + c->nvls->size)
    return HFR_SUCCESS;  // arena memory lives until hfr_finalize
  for (size_t i = 0; i < c->regions.size(); ++i) {
    Region& r = c->regions[i];
    if (r.owned && r.base[c->virt ? 0 : c->rank] == ptr) {
      HFR_CU(cudaDeviceSynchronize());
      if (!c->virt && c->n > 1) {
        int dummy = 0;
        std::vector<int> all(c->n);
        HFR_TRY(exchange(c, &dummy, all.data(), sizeof(int)));  // everyone stopped using it
      }
      close_region(c, r);
      c->regions.erase(c->regions.begin() + i);
      return HFR_SUCCESS;
    }
  }
  return HFR_ERR_INVALID_ARGUMENT;
}

hfr_status_t hfr_register(hfr_comm_t c, void* ptr, size_t bytes) {
  if (!c) return HFR_ERR_NOT_INITIALIZED;
  if (!ptr || bytes == 0) return HFR_ERR_INVALID_ARGUMENT;
  if (c->virt) return HFR_SUCCESS;
  const Region* have = nullptr;
  if (find_region(c, (const char*)ptr, bytes, &have)) return HFR_SUCCESS;
  DeviceGuard guard(c->dev);
  Region r;
  HFR_TRY(share_region(c, (char*)ptr, bytes, &r));
  r.owned = false;
  c->regions.push_back(r);
  return HFR_SUCCESS;
}

hfr_status_t hfr_deregister(hfr_comm_t c, void* ptr) {
  if (!c) return HFR_ERR_NOT_INITIALIZED;
  if (!ptr) return HFR_ERR_INVALID_ARGUMENT;
  if (c->virt) return HFR_SUCCESS;
  for (size_t i = 0; i < c->regions.size(); ++i) {
    Region& r = c->regions[i];
    const char* b = r.base[c->rank];
    if (!r.owned && !r.nvls && b && (const char*)ptr >= b && (const char*)ptr < b + r.bytes) {
      DeviceGuard guard(c->dev);
      HFR_CU(cudaDeviceSynchronize());
      if (c->n > 1) {
        int dummy = 0;
        std::vector<int> all(c->n);
        HFR_TRY(exchange(c, &dummy, all.data(), sizeof(int)));  // every rank stopped using it
      }
      close_region(c, r);
      c->regions.erase(c->regions.begin() + i);
      return HFR_SUCCESS;
    }
  }
  return HFR_ERR_INVALID_ARGUMENT;
}

hfr_status_t hfr_allreduce(hfr_comm_t c, void* buf, size_t count, hfr_dtype_t dtype, hfr_op_t op,
                           hfr_stream_t stream, hfr_req_t* req) {
  if (!c) return HFR_ERR_NOT_INITIALIZED;
  if (c->virt) return HFR_ERR_INVALID_ARGUMENT;
  char* bufs[1] = {(char*)buf};
  return allreduce_impl(c, bufs, count, dtype, op, (cudaStream_t)stream, req);
}

hfr_status_t hfr_allreduce_virtual(hfr_comm_t c, void* const* bufs, size_t count, hfr_dtype_t dtype, hfr_op_t op,
                                   hfr_stream_t stream, hfr_req_t* req) {
  if (!c) return HFR_ERR_NOT_INITIALIZED;
  if (!c->virt || !bufs) return HFR_ERR_INVALID_ARGUMENT;
  char* local[kMaxRanks];
  for (int q = 0; q < c->n; ++q) local[q] = (char*)bufs[q];
  return allreduce_impl(c, local, count, dtype, op, (cudaStream_t)stream, req);
}

hfr_status_t hfr_collective(hfr_comm_t c, hfr_coll_t coll, void* buf, size_t count, hfr_dtype_t dtype, hfr_op_t op,
                            int root, hfr_stream_t stream, hfr_req_t* req) {
  if (!c) return HFR_ERR_NOT_INITIALIZED;
  if (c->virt) return HFR_ERR_INVALID_ARGUMENT;
  char* bufs[1] = {(char*)buf};
  return allreduce_impl(c, bufs, count, dtype, op, (cudaStream_t)stream, req, coll, root);
}

hfr_status_t hfr_collective_virtual(hfr_comm_t c, hfr_coll_t coll, void* const* bufs, size_t count,
                                    hfr_dtype_t dtype, hfr_op_t op, int root, hfr_stream_t stream, hfr_req_t* req) {
  if (!c) return HFR_ERR_NOT_INITIALIZED;
  if (!c->virt || !bufs) return HFR_ERR_INVALID_ARGUMENT;
  char* local[kMaxRanks];
  for (int q = 0; q < c->n; ++q) local[q] = (char*)bufs[q];
  return allreduce_impl(c, local, count, dtype, op, (cudaStream_t)stream, req, coll, root);
}

hfr_status_t hfr_shard_range(int nranks, size_t count, hfr_dtype_t dtype, int rank, size_t* lo, size_t* hi) {
  if (nranks < 1 || nranks > HFR_MAX_RANKS || rank < 0 || rank >= nranks || !lo || !hi ||
      !dtype_valid(dtype))
    return HFR_ERR_INVALID_ARGUMENT;
  const uint64_t K = per_vec(dtype);  // elements per 16-byte vector
  const uint64_t nvec = count / K;
  *lo = K * (nvec * (uint64_t)rank / nranks);
  *hi = rank == nranks - 1 ? count : K * (nvec * (uint64_t)(rank + 1) / nranks);
  return HFR_SUCCESS;
}

hfr_status_t hfr_wait(hfr_req_t req, hfr_stream_t stream) {
  if (!req) return HFR_SUCCESS;  // count == 0 / already-complete request
  hfr_comm_s* c = req->comm;
  DeviceGuard guard(c->dev);
  hfr_status_t s = HFR_SUCCESS;
  cudaError_t e;
  if (stream) {
    e = cudaStreamWaitEvent((cudaStream_t)stream, req->ev, 0);
  } else {
    e = cudaEventSynchronize(req->ev);
  }
  if (e != cudaSuccess) {
    note_cuda(e, "hfr_wait");
    s = HFR_ERR_CUDA;
  }
  c->ev_pool.push_back(req->ev);
  delete req;
  if (s == HFR_SUCCESS) s = hfr_comm_status(c);
  return s;
}

hfr_status_t hfr_comm_status(hfr_comm_t c) {
  if (!c) return HFR_ERR_NOT_INITIALIZED;
  if (c->sticky == HFR_SUCCESS && c->err_host && *(volatile uint32_t*)c->err_host != 0)
    c->sticky = (hfr_status_t) * (volatile uint32_t*)c->err_host;
  return c->sticky;
}

hfr_status_t hfr_barrier(hfr_comm_t c, hfr_stream_t stream) {
  if (!c) return HFR_ERR_NOT_INITIALIZED;
  if (c->sticky != HFR_SUCCESS) return c->sticky;
  DeviceGuard guard(c->dev);
  cudaStream_t s = (cudaStream_t)stream;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  HFR_CU(cudaStreamIsCapturing(s, &cap));
  const bool capturing = cap != cudaStreamCaptureStatusNone;
  if (!capturing && c->has_last) HFR_CU(cudaStreamWaitEvent(s, c->last_op, 0));  // issue order
  Args a;
  base_args(c, a, 0, 0xBA881E8ull);
  HFR_TRY(launch(c, (const void*)hfr_barrier_kernel, 1, 32 * ((c->n + 31) / 32), a, s, true));
  if (!capturing) {
    HFR_CU(cudaEventRecord(c->last_op, s));
    c->has_last = true;
  }
  return HFR_SUCCESS;
}

hfr_status_t hfr_finalize(hfr_comm_t c) {
  if (!c) return HFR_ERR_NOT_INITIALIZED;
  {
    DeviceGuard guard(c->dev);
    cudaDeviceSynchronize();
    if (!c->virt && c->n > 1 && c->ag) {
      int dummy = 0;
      std::vector<int> all(c->n);
      exchange(c, &dummy, all.data(), sizeof(int));  // host barrier: peers are done with our memory
    }
    for (Region& r : c->regions) close_region(c, r);
    c->regions.clear();
    for (Region& r : c->retired) close_region(c, r);
    c->retired.clear();
    close_region(c, c->scratch);
    close_region(c, c->pad);
    if (c->nvls) {
      nvls_teardown(*c->nvls, c->n, c->rank);
      delete c->nvls;
    }
    for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
    for (cudaStream_t h : c->ce_fold) cudaStreamDestroy(h);
    for (cudaStream_t h : c->helpers) cudaStreamDestroy(h);
    for (cudaStream_t h : c->ag_helpers) cudaStreamDestroy(h);
    for (cudaEvent_t e : c->ag_events) cudaEventDestroy(e);
    for (cudaEvent_t e : c->chunk_events) cudaEventDestroy(e);
    for (cudaEvent_t e : c->ce_fork) cudaEventDestroy(e);
    for (cudaEvent_t e : c->ce_join) cudaEventDestroy(e);
    if (c->last_op) cudaEventDestroy(c->last_op);
    if (c->setup) cudaStreamDestroy(c->setup);
    if (c->side) cudaStreamDestroy(c->side);
    if (c->err_host) cudaFreeHost(c->err_host);
  }
  delete c;
  return HFR_SUCCESS;
}

hfr_status_t hfr_tree_query(int n, int which, int* parent, int* child0, int* child1) {
  if (n < 1 || n > kMaxTreeN || (which != 0 && which != 1) || !parent || !child0 || !child1)
    return HFR_ERR_INVALID_ARGUMENT;
  std::vector<int> p(n), nc(n);
  std::vector<std::array<int, 2>> ch(n);
  build_tree(n, which, p.data(), ch.data(), nc.data());
  for (int v = 0; v < n; ++v) {
    parent[v] = p[v];
    child0[v] = ch[v][0];
    child1[v] = ch[v][1];
  }
  return HFR_SUCCESS;
}

hfr_status_t hfr_set_trace(hfr_comm_t c, void* dev_buf, size_t bytes) {
  if (!c) return HFR_ERR_NOT_INITIALIZED;
  const size_t per = (size_t)64 * kMaxCtas * c->local;
  if (!dev_buf || bytes < per) {
    c->trace = nullptr;
    c->trace_cap = 0;
    return dev_buf ? HFR_ERR_INVALID_ARGUMENT : HFR_SUCCESS;
  }
  c->trace = (uint64_t*)dev_buf;
  c->trace_cap = (uint32_t)std::min<size_t>(bytes / per, 1u << 20);
  return HFR_SUCCESS;
}

const char* hfr_status_string(hfr_status_t s) {
  switch (s) {
    case HFR_SUCCESS: return "success";
    case HFR_ERR_INVALID_ARGUMENT: return "invalid argument";
    case HFR_ERR_UNSUPPORTED: return "unsupported";
    case HFR_ERR_CUDA: return "CUDA error";
    case HFR_ERR_OUT_OF_MEMORY: return "out of memory";
    case HFR_ERR_PROTOCOL: return "protocol violation (ranks disagree)";
    case HFR_ERR_TIMEOUT: return "timeout waiting for peers";
    case HFR_ERR_NOT_INITIALIZED: return "not initialized";
    case HFR_ERR_INTERNAL: return "internal error";
  }
  return "unknown status";
}

const char* hfr_last_cuda_error(void) { return g_cuda_error.c_str(); }

}  // extern "C"

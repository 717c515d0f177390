// hfr_kernels.cuh — sm_100a kernels of the B200-native HFReduce.
//
// Paper: Fire-Flyer AI-HPC, arXiv 2408.14158, §4 HFReduce.
// The paper's CPU-side steps (D2H copy, SIMD reduce-add, RDMA double binary
// tree, H2D copy) become SM loads/stores over NVLink on CUDA-IPC-mapped
// memory.  Every kernel takes an Args by value holding, per rank r, the
// pointer (valid in this process) to rank r's buffer, tree partials and
// signal pad.  In a virtual comm all ranks live on one GPU and one launch
// runs every rank's CTAs (blockIdx.y = rank - rank0).
//
// Numerics (readings R1-R6): fp32 adds/multiplies via __fadd_rn /
// __fmul_rn (never contracted into FMA, no FTZ since the TU is built without
// --use_fast_math), bf16 widened exactly, fp32 accumulate, one RNE cast.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include <type_traits>

namespace hfr {

constexpr int kMaxRanks = 16;
constexpr int kMaxCtas = 1024;
constexpr int kMaxChunks = 1 << 18;  // tree flags per launch (chunks, or tiles for the TMA tree kernel)

// Peer-mapped signal pad, one per rank (DESIGN.md §5 "HBM layout").
// entry/exit[b][q] are written by rank q's CTA b; up/down/pdown[c] are the
// per-chunk tree flags (c = chunk index local to the launch).  All values are
// launch epochs, strictly increasing per rank, so nothing is ever reset.  The
// epoch lives in device memory (launch_epoch), not in the kernel arguments,
// so captured CUDA graphs replay correctly.
struct Pad {
  uint64_t entry[kMaxCtas][kMaxRanks];  // packed (epoch << 32 | sig32)
  uint64_t exit[kMaxCtas][kMaxRanks];
  uint64_t up[2][kMaxChunks];   // child partial for chunk c landed in slot s
  uint64_t down[kMaxChunks];    // final chunk c landed in my buffer (from tree parent)
  uint64_t pdown[kMaxChunks];   // final chunk c of my other half landed (from pair partner)
  uint64_t ce_ready[kMaxRanks]; // CE schedule: rank q's buffer is ready (stream memop flags)
  uint64_t ce_done[kMaxRanks];  //   rank q's result shard is final
  uint64_t ce_exit[kMaxRanks];  //   rank q finished pulling from every peer
  uint32_t nvls_seq[kMaxCtas]; // NVLS launches seen by CTA b (local only)
  uint64_t tile_next;           // FLAT: next warp tile to hand out (dynamic distribution), 0 between launches
  uint64_t launch_epoch;        // epoch of the last completed launch on this rank
  uint32_t done_ctas;           // CTAs of the current launch that have finished
};

// One node of a double binary tree (reading R9/R10).  Children are sorted by
// rank; self_pos = number of children with a smaller rank, so the in-order
// combination is  children[0..self_pos) , x_v , children[self_pos..nchild).
struct TreeNode {
  int8_t parent;    // -1 at the root
  int8_t nchild;    // 0..2
  int8_t self_pos;  // 0..nchild
  int8_t slot;      // my slot index in my parent's sorted children
  int8_t child[2];
  int8_t pad_[2];
};

struct Args {
  char* buf[kMaxRanks];    // rank r's data buffer (this call)
  char* inbox[kMaxRanks];  // rank r's ONESHOT inbox: [2 parities][n sources][slot_bytes]
  float* part[kMaxRanks];  // rank r's fp32 partial slots (tree algos): 2 x part_stride
  Pad* pad[kMaxRanks];
  volatile uint32_t* err;  // host-mapped error word (hfr_status_t), 0 = ok
  uint64_t count;          // elements per rank
  uint64_t sig;            // hash of the call's arguments, compared across ranks
  uint64_t timeout_ns;
  uint64_t part_stride;    // floats per partial slot
  uint64_t slot_bytes;     // ONESHOT inbox slot size
  uint64_t half_base[2];   // tree algos: element offset of the range each parity works on
  uint64_t half_len[2];
  uint32_t c_lo, c_hi;     // tree algos: global chunk range of this launch
  float scale;
  int n;                   // ranks in the comm
  int rank0;               // rank of blockIdx.y == 0
  int chunk;               // tree chunk elements (multiple of 256)
  int ntree;               // nodes per tree (n, or n/2 for PAIR)
  int src_rank;            // FLAT kernel: -1 fold all ranks; -2 copy my own shard; r>=0 copy rank r's
  uint32_t dst_mask;       // FLAT kernel: ranks that receive the result (0 = the owner itself)
  int tma_tile;            // FLAT TMA kernel: bytes per source per stage (multiple of 16)
  int excl_root;           // FLAT kernel: >= 0: this rank owns no shard (reduce/broadcast root)
  int nvls_op;             // NVLS kernel: bit0 multimem.ld_reduce (else local load), bit1 multimem.st (else local store)
  int nvls_solo;           // NVLS kernel: >= 0: this rank alone covers the whole buffer (reduce/broadcast root)
  char* mcbuf;              // NVLS: multicast VA of this call's buffer
  uint32_t* mc_exit;       // NVLS: multicast VA of the exit counters [kMaxCtas]
  uint32_t* uc_exit;       // NVLS: local unicast VA of the same counters
  uint32_t trace_cap;      // diagnostic trace: events per CTA (0 = off)
  uint64_t* trace;         // [local rank][CTA][trace_cap][4] u64, see Tracer
  uint32_t tree_tile;      // TMA tree kernel: elements per tile (flag granularity), divides chunk
  int tree_smem;           // TMA tree kernel: dynamic shared memory per CTA (each role fits its own stages)
  TreeNode tree[2][kMaxRanks];
};

// Diagnostic per-CTA event log (hfr_set_trace): thread 0 records
// {tag, t_wait_start, t_work_start, t_stores_issued, t_done, 0, 0, 0} in
// globaltimer ns (t_stores_issued: after the CTA barrier that follows the
// chunk's stores, before the system fence that drains them).
struct Tracer {
  uint64_t* p = nullptr;
  uint32_t cap = 0, n = 0;
  __device__ explicit Tracer(const Args& a) {
    if (a.trace && threadIdx.x == 0) {
      cap = a.trace_cap;
      p = a.trace + ((uint64_t)blockIdx.y * kMaxCtas + blockIdx.x) * cap * 8;
    }
  }
  __device__ __forceinline__ void rec(uint64_t tag, uint64_t t0, uint64_t t1, uint64_t t2, uint64_t t3,
                                      uint64_t t4 = 0, uint64_t t5 = 0) {
    if (p && n < cap) {
      p[8 * n] = tag;
      p[8 * n + 1] = t0;
      p[8 * n + 2] = t1;
      p[8 * n + 3] = t2;
      p[8 * n + 4] = t3;
      p[8 * n + 5] = t4;
      p[8 * n + 6] = t5;
      ++n;
    }
  }
};

// ---------------------------------------------------------------------------
// memory-model primitives (PTX ISA memory consistency model, sys scope)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_relaxed_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Launch epoch.  Every CTA reads the rank's launch_epoch at entry (+1 = this
// launch); the last CTA of the launch to finish publishes it.  A CTA can only
// finish after reading, so every CTA of a launch sees the same value whatever
// the residency, and the next launch (stream order) sees the update.
// Programmatic dependent launch (real comms, include/hfr.h): a launch may be
// scheduled while the previous kernel on the stream is in its exit phase.
// pdl_wait() blocks until that kernel has completed and its memory is visible
// (a no-op for an ordinary launch), so it comes before ANY memory access;
// pdl_trigger() lets the next launch be scheduled once every CTA of this one
// has reached its exit handshake (implicit at completion otherwise).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ uint64_t begin_epoch(Pad* mine) {
  __shared__ uint64_t s_epoch;
  pdl_wait();
  if (threadIdx.x == 0) s_epoch = *reinterpret_cast<volatile uint64_t*>(&mine->launch_epoch) + 1;
  __syncthreads();
  return s_epoch;
}
__device__ __forceinline__ void end_epoch(Pad* mine, uint64_t e) {
  pdl_trigger();
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&mine->done_ctas, 1u) == gridDim.x - 1) {
      mine->done_ctas = 0;
      mine->tile_next = 0;  // every CTA of this launch is past its last tile grab
      *reinterpret_cast<volatile uint64_t*>(&mine->launch_epoch) = e;
      __threadfence();
    }
  }
}

// 128-bit data movement.  Loads skip L1 allocation (each byte is read once);
// peer addresses bypass the local L2 in hardware.  (An L2 evict-first
// cache-policy variant measured no difference: 643 vs 647 GB/s, r01.)
__device__ __forceinline__ uint4 ld128(const void* p) {
  uint4 v;
  asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ void st128(void* p, const uint4& v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// status codes mirrored from include/hfr.h
constexpr uint32_t kErrProtocol = 5;
constexpr uint32_t kErrTimeout = 6;

__device__ __forceinline__ void raise_error(const Args& a, uint32_t code) {
  if (*a.err == 0) *a.err = code;
}

// Handshake flags pack (launch epoch << 32 | 32-bit argument signature) into
// one 64-bit word, so publishing needs a single store and no fence.
__device__ __forceinline__ uint64_t pack_flag(uint64_t e, uint64_t sig) {
  return (e << 32) | (uint32_t)(sig ^ (sig >> 32));
}

// Spin until *p >= target.  Returns false on timeout or if another CTA
// already raised an error (checked every 1024 polls).  peer0 (optional): the
// word peer CTA 0 publishes into this rank's pad at entry; if it shows this
// launch's epoch (or a later one) with another signature, the peer runs a
// different call (other count / dtype / algo / grid) and will never publish
// *p: raise PROTOCOL instead of waiting for the timeout.
// Only the same epoch counts: a later epoch there may legitimately become
// visible before the flag awaited here (stores of different CTAs are not
// ordered for a remote observer).
__device__ __noinline__ bool wait_ge(const Args& a, const uint64_t* p, uint64_t target,
                                     const uint64_t* peer0 = nullptr, uint64_t expect0 = 0) {
  if (ld_acquire_sys(p) >= target) return true;
  uint64_t t0 = globaltimer();
  for (uint32_t it = 1;; ++it) {
    if (ld_acquire_sys(p) >= target) return true;
    if ((it & 1023u) == 0) {
      if (*a.err != 0) return false;
      if (peer0) {
        const uint64_t v = ld_relaxed_sys(peer0);
        if ((v >> 32) == (expect0 >> 32) && v != expect0) {
          raise_error(a, kErrProtocol);
          return false;
        }
      }
      if (globaltimer() - t0 > a.timeout_ns) {
        raise_error(a, kErrTimeout);
        return false;
      }
    }
  }
}

// Wait for the packed flag of epoch e at *p (written by peer q's CTA b) and
// check the signature; peer q's CTA-0 word is watched meanwhile (wait_ge).
__device__ __forceinline__ bool wait_flag(const Args& a, const uint64_t* p, uint64_t e, int rank, int q) {
  const uint64_t want = pack_flag(e, a.sig);
  if (!wait_ge(a, p, e << 32, &a.pad[rank]->entry[0][q], want)) return false;
  if (ld_relaxed_sys(p) != want) {
    raise_error(a, kErrProtocol);
    return false;
  }
  return true;
}

// a0 "trigger and entry handshake" ("wait for chunk-i
// transfer finished in this node", made a device barrier): CTA b of `rank`
// publishes (epoch, sig) to CTA b of every rank and waits for all of them.
// When it returns true every rank has entered this launch, so every rank's
// prior stream work on its buffers is complete (kernel boundaries order it;
// no fence is needed before the flag).  Ranks that disagree on the call's
// arguments see a signature mismatch -> HFR_ERR_PROTOCOL.
__device__ __forceinline__ bool entry_barrier(const Args& a, int rank, int b, uint64_t e) {
  bool ok = true;
  const int q = threadIdx.x;
  if (q < a.n) {
    st_relaxed_sys(&a.pad[q]->entry[b][rank], pack_flag(e, a.sig));
    ok = wait_flag(a, &a.pad[rank]->entry[b][q], e, rank, q);
  }
  return __syncthreads_and(ok);
}

// a5 completion: CTA b tells CTA b of every rank that all its loads from and
// stores to that rank are done, and waits for the same from everyone.
__device__ __forceinline__ void exit_barrier(const Args& a, int rank, int b, uint64_t e) {
  pdl_trigger();
  __syncthreads();
  const int q = threadIdx.x;
  if (q < a.n) {
    fence_acq_rel_sys();
    st_relaxed_sys(&a.pad[q]->exit[b][rank], e);
    wait_ge(a, &a.pad[rank]->exit[b][q], e);
  }
  __syncthreads();
}

// Exit through the NVLS multicast arena: after its stores (incl. multimem.st)
// each CTA b bumps counter b on every GPU with ONE multimem.red.release and
// waits until all n ranks' CTA b arrived (k = this CTA's NVLS launch count).
__device__ __forceinline__ void mc_exit_barrier(const Args& a, int b, int n, uint32_t k) {
  pdl_trigger();
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t target = (uint32_t)n * k;
    asm volatile("multimem.red.release.sys.global.add.u32 [%0], 1;" ::"l"(a.mc_exit + b) : "memory");
    uint64_t t_start = 0;
    for (uint32_t it = 1;; ++it) {
      uint32_t v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(a.uc_exit + b) : "memory");
      if ((int32_t)(v - target) >= 0) break;
      if ((it & 1023u) == 0) {
        if (!t_start) t_start = globaltimer();
        if (*a.err != 0) break;
        if (globaltimer() - t_start > a.timeout_ns) {
          raise_error(a, kErrTimeout);
          break;
        }
      }
    }
  }
  __syncthreads();
}

__device__ __forceinline__ void mc_st128(char* mc, const uint4& v) {
  asm volatile("multimem.st.weak.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc), "f"(__uint_as_float(v.x)),
               "f"(__uint_as_float(v.y)), "f"(__uint_as_float(v.z)), "f"(__uint_as_float(v.w))
               : "memory");
}

// ---------------------------------------------------------------------------
// element types
// ---------------------------------------------------------------------------
struct F32 {
  using T = float;
  static constexpr int kPerVec = 4;  // elements per 16 B
  __device__ static __forceinline__ void widen(const uint4& v, float* f) {
    f[0] = __uint_as_float(v.x); f[1] = __uint_as_float(v.y);
    f[2] = __uint_as_float(v.z); f[3] = __uint_as_float(v.w);
  }
  __device__ static __forceinline__ uint4 narrow(const float* f) {
    return make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]), __float_as_uint(f[3]));
  }
  __device__ static __forceinline__ float load1(const char* p, uint64_t i) {
    return reinterpret_cast<const float*>(p)[i];
  }
  __device__ static __forceinline__ void store1(char* p, uint64_t i, float v) {
    reinterpret_cast<float*>(p)[i] = v;
  }
  __device__ static __forceinline__ float from_bits(uint32_t b) { return __uint_as_float(b); }
};

struct BF16 {
  using T = __nv_bfloat16;
  static constexpr int kPerVec = 8;
  __device__ static __forceinline__ void widen(const uint4& v, float* f) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      f[2 * j] = __uint_as_float(w[j] << 16);
      f[2 * j + 1] = __uint_as_float(w[j] & 0xFFFF0000u);
    }
  }
  __device__ static __forceinline__ uint32_t rne(float x) {
    return (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(x));
  }
  __device__ static __forceinline__ uint4 narrow(const float* f) {
    return make_uint4(rne(f[0]) | (rne(f[1]) << 16), rne(f[2]) | (rne(f[3]) << 16),
                      rne(f[4]) | (rne(f[5]) << 16), rne(f[6]) | (rne(f[7]) << 16));
  }
  __device__ static __forceinline__ float load1(const char* p, uint64_t i) {
    return __uint_as_float(((uint32_t)reinterpret_cast<const uint16_t*>(p)[i]) << 16);
  }
  __device__ static __forceinline__ void store1(char* p, uint64_t i, float v) {
    reinterpret_cast<uint16_t*>(p)[i] = (uint16_t)rne(v);
  }
  __device__ static __forceinline__ float from_bits(uint32_t b) { return __uint_as_float(b << 16); }
};

// IEEE binary16 (PAPER.md:404 lists FP16): widened exactly, fp32 accumulate,
// one RNE rounding (__float2half_rn: subnormals kept, overflow -> Inf).
struct F16 {
  using T = __half;
  static constexpr int kPerVec = 8;
  __device__ static __forceinline__ float h2f(uint32_t b) { return __half2float(__ushort_as_half((unsigned short)b)); }
  __device__ static __forceinline__ void widen(const uint4& v, float* f) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      f[2 * j] = h2f(w[j] & 0xFFFFu);
      f[2 * j + 1] = h2f(w[j] >> 16);
    }
  }
  __device__ static __forceinline__ uint32_t rne(float x) { return (uint32_t)__half_as_ushort(__float2half_rn(x)); }
  __device__ static __forceinline__ uint4 narrow(const float* f) {
    return make_uint4(rne(f[0]) | (rne(f[1]) << 16), rne(f[2]) | (rne(f[3]) << 16),
                      rne(f[4]) | (rne(f[5]) << 16), rne(f[6]) | (rne(f[7]) << 16));
  }
  __device__ static __forceinline__ float load1(const char* p, uint64_t i) {
    return h2f(reinterpret_cast<const uint16_t*>(p)[i]);
  }
  __device__ static __forceinline__ void store1(char* p, uint64_t i, float v) {
    reinterpret_cast<uint16_t*>(p)[i] = (uint16_t)rne(v);
  }
  __device__ static __forceinline__ float from_bits(uint32_t b) { return h2f(b); }
};

// FP8 (PAPER.md:404 lists FP8; reading R20): OCP E4M3 ("FN": no Inf, NaN =
// S.1111.111, max 448) and E5M2 (IEEE-like, max 57344).  Widened exactly
// (every FP8 value is a binary16, hence a float: cvt.rn.f16x2.e4m3x2 /
// .e5m2x2), fp32 accumulate, one RNE rounding.  The hardware converts with
// .satfinite only, so the overflow rule of R20 (as torch.Tensor.to: no
// saturation) is applied on top: a magnitude that rounds past the largest
// finite value becomes NaN (E4M3, which has no Inf: |x| > 464, the tie 464
// rounding down to 448) or +-Inf (E5M2: |x| >= 61440, the tie rounding up
// to the next power of two); NaN stays NaN.
template <bool kE5M2>
struct FP8 {
  using T = uint8_t;
  static constexpr int kPerVec = 16;
  __device__ static __forceinline__ uint32_t cvt2_to_h2(uint32_t two) {  // 2 codes (low 16 bits) -> f16x2
    uint32_t h2;
    const uint16_t x = (uint16_t)two;
    if constexpr (kE5M2)
      asm("cvt.rn.f16x2.e5m2x2 %0, %1;" : "=r"(h2) : "h"(x));
    else
      asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h2) : "h"(x));
    return h2;
  }
  __device__ static __forceinline__ void widen2(uint32_t two, float* f) {
    const uint32_t h2 = cvt2_to_h2(two);
    f[0] = __half2float(__ushort_as_half((unsigned short)(h2 & 0xFFFFu)));
    f[1] = __half2float(__ushort_as_half((unsigned short)(h2 >> 16)));
  }
  __device__ static __forceinline__ void widen(const uint4& v, float* f) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      widen2(w[j] & 0xFFFFu, f + 4 * j);
      widen2(w[j] >> 16, f + 4 * j + 2);
    }
  }
  // 8 codes (8 bytes) -> 8 floats / back (the tree kernel's 8-element unit)
  __device__ static __forceinline__ void widen8(const uint2& v, float* f) {
    widen2(v.x & 0xFFFFu, f);
    widen2(v.x >> 16, f + 2);
    widen2(v.y & 0xFFFFu, f + 4);
    widen2(v.y >> 16, f + 6);
  }
  __device__ static __forceinline__ uint32_t fix(uint32_t code, float x) {  // R20 overflow rule
    const float a = fabsf(x);
    const uint32_t sign = (__float_as_uint(x) >> 24) & 0x80u;
    if constexpr (kE5M2) {
      if (a != a) return 0x7Eu | sign;
      if (a >= 61440.f) return 0x7Cu | sign;
    } else {
      if (!(a <= 464.f)) return 0x7Fu | sign;  // NaN, Inf or overflow
    }
    return code;
  }
  __device__ static __forceinline__ uint32_t rne2(float lo, float hi) {  // -> 2 codes in the low 16 bits
    uint16_t st;
    if constexpr (kE5M2)
      asm("cvt.rn.satfinite.e5m2x2.f32 %0, %1, %2;" : "=h"(st) : "f"(hi), "f"(lo));
    else
      asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(st) : "f"(hi), "f"(lo));
    return fix(st & 0xFFu, lo) | (fix((uint32_t)st >> 8, hi) << 8);
  }
  __device__ static __forceinline__ uint32_t rne(float x) { return rne2(x, 0.f) & 0xFFu; }
  __device__ static __forceinline__ uint4 narrow(const float* f) {
    uint32_t w[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) w[j] = rne2(f[4 * j], f[4 * j + 1]) | (rne2(f[4 * j + 2], f[4 * j + 3]) << 16);
    return make_uint4(w[0], w[1], w[2], w[3]);
  }
  __device__ static __forceinline__ uint2 narrow8(const float* f) {
    return make_uint2(rne2(f[0], f[1]) | (rne2(f[2], f[3]) << 16), rne2(f[4], f[5]) | (rne2(f[6], f[7]) << 16));
  }
  __device__ static __forceinline__ float from_bits(uint32_t b) {
    float f[2];
    widen2(b & 0xFFu, f);
    return f[0];
  }
  __device__ static __forceinline__ float load1(const char* p, uint64_t i) {
    return from_bits(reinterpret_cast<const uint8_t*>(p)[i]);
  }
  __device__ static __forceinline__ void store1(char* p, uint64_t i, float v) {
    reinterpret_cast<uint8_t*>(p)[i] = (uint8_t)rne(v);
  }
};
using E4M3 = FP8<false>;
using E5M2 = FP8<true>;

// ---------------------------------------------------------------------------
// Subsystems (1)+(3), FLAT: fused reduce-scatter + all-gather/cast/scale.
//
// Rank g owns shard g = vectors [g*V/n, (g+1)*V/n).  For each vector of its
// shard a thread loads the 16 B at that offset from all n ranks' buffers
// (n-1 over NVLink; Algorithm 1's D2H + "Dc_i += GPU-j's Dc_i", PAPER.md:
// 327-336), folds them serially in rank order 0..n-1 in fp32 (lanes split
// ELEMENTS, never ranks, so the order is the oracle's), multiplies by scale
// once, casts, and stores the result to all n buffers (Algorithm 2 pass 2 /
// H2D fan-out).  In place without a mid-kernel barrier:
// shard g of rank q's buffer is read and then written only by rank g.
// ---------------------------------------------------------------------------
template <class E, int NR, int U>
__device__ __forceinline__ void flat_vecs(const Args& a, uint64_t i, uint64_t stride, uint64_t hi, int src,
                                          uint32_t dmask) {
  // U vectors per thread, all loads issued before the first fold so that
  // U*NR 16-byte NVLink reads are in flight per thread.  src >= 0: copy that
  // rank's vectors (all-gather / broadcast) instead of folding all ranks.
  constexpr int K = E::kPerVec;
  uint4 v[U][NR];
  bool ok[U];
#pragma unroll
  for (int u = 0; u < U; ++u) ok[u] = i + u * stride < hi;
  if (src >= 0) {
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (ok[u]) v[u][0] = ld128(a.buf[src] + (i + u * stride) * 16);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (ok[u]) {
#pragma unroll
        for (int r = 0; r < NR; ++r)
          if ((dmask >> r) & 1u) st128(a.buf[r] + (i + u * stride) * 16, v[u][0]);
      }
    return;
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    if (ok[u]) {
#pragma unroll
      for (int r = 0; r < NR; ++r) v[u][r] = ld128(a.buf[r] + (i + u * stride) * 16);
    }
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    if (ok[u]) {
      float acc[K];
      E::widen(v[u][0], acc);
#pragma unroll
      for (int r = 1; r < NR; ++r) {
        float t[K];
        E::widen(v[u][r], t);
#pragma unroll
        for (int k = 0; k < K; ++k) acc[k] = __fadd_rn(acc[k], t[k]);
      }
#pragma unroll
      for (int k = 0; k < K; ++k) acc[k] = __fmul_rn(acc[k], a.scale);
      const uint4 o = E::narrow(acc);
#pragma unroll
      for (int r = 0; r < NR; ++r)
        if ((dmask >> r) & 1u) st128(a.buf[r] + (i + u * stride) * 16, o);
    }
  }
}

template <class E>
__device__ __forceinline__ void flat_vec_dyn(const Args& a, const int n, uint64_t i, int src, uint32_t dmask) {
  constexpr int K = E::kPerVec;
  if (src >= 0) {
    const uint4 o = ld128(a.buf[src] + i * 16);
    for (int r = 0; r < n; ++r)
      if ((dmask >> r) & 1u) st128(a.buf[r] + i * 16, o);
    return;
  }
  float acc[K];
  E::widen(ld128(a.buf[0] + i * 16), acc);
  for (int r = 1; r < n; ++r) {
    float t[K];
    E::widen(ld128(a.buf[r] + i * 16), t);
#pragma unroll
    for (int k = 0; k < K; ++k) acc[k] = __fadd_rn(acc[k], t[k]);
  }
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = __fmul_rn(acc[k], a.scale);
  const uint4 o = E::narrow(acc);
  for (int r = 0; r < n; ++r)
    if ((dmask >> r) & 1u) st128(a.buf[r] + i * 16, o);
}

// NR = compile-time rank count (1..8), 0 = runtime a.n (up to kMaxRanks).
template <class E, int NR>
__global__ void __launch_bounds__(512) hfr_flat_kernel(const Args a) {
  const int rank = a.rank0 + blockIdx.y;
  const int n = NR > 0 ? NR : a.n;
  const int b = blockIdx.x;
  const uint64_t e = begin_epoch(a.pad[rank]);
  // collective mode (NEXT-3): allreduce = fold all -> all; reduce-scatter =
  // fold all -> owner; reduce = fold all -> root; all-gather = owner's shard
  // -> all; broadcast = root's shard -> all
  const int src = a.src_rank == -2 ? rank : a.src_rank;
  const uint32_t dmask = a.dst_mask ? a.dst_mask : (1u << rank);
  // shard owners: all n ranks, or (reduce / broadcast) the n-1 ranks other
  // than the root, so the root's link carries each byte once
  const int nown = a.excl_root >= 0 ? n - 1 : n;
  const int own = a.excl_root >= 0 ? (rank < a.excl_root ? rank : rank - 1) : rank;
  const bool owner = rank != a.excl_root;
  if (entry_barrier(a, rank, b, e) && owner) {
    constexpr int K = E::kPerVec;
    constexpr int U = NR > 4 ? 2 : (NR > 2 ? 3 : 4);
    const uint64_t nvec = a.count / K;
    const uint64_t lo = nvec * own / nown, hi = nvec * (own + 1) / nown;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    if constexpr (NR > 0) {
      // warp tiles of U*32 consecutive vectors (U*512 B contiguous per rank
      // buffer): lane l of the warp owning tile t handles vectors
      // t*U*32 + u*32 + l, u < U.  Each warp takes the next tile of this
      // rank's shard from a counter in the local pad, so fast CTAs absorb the
      // slow ones' share (r01: +3-7 % over a static deal).
      const uint64_t lane = threadIdx.x & 31;
      unsigned long long* ctr = reinterpret_cast<unsigned long long*>(&a.pad[rank]->tile_next);
      for (;;) {
        uint64_t t = 0;
        if (lane == 0) t = atomicAdd(ctr, 1ull);
        t = __shfl_sync(0xffffffffu, t, 0);
        const uint64_t t0 = lo + t * (U * 32);
        if (t0 >= hi) break;
        flat_vecs<E, NR, U>(a, t0 + lane, 32, hi, src, dmask);
      }
    } else {
      for (uint64_t i = lo + (uint64_t)b * blockDim.x + threadIdx.x; i < hi; i += stride)
        flat_vec_dyn<E>(a, n, i, src, dmask);
    }
    // ragged tail (< K elements) — owned by the last owner, CTA 0
    const uint64_t t0 = nvec * K;
    if (own == nown - 1 && b == 0 && threadIdx.x < a.count - t0) {
      const uint64_t el = t0 + threadIdx.x;
      if (src >= 0) {
        // raw copy of the element (fp8 / 16-bit / fp32 bits)
        if constexpr (K == 16) {
          const uint8_t x = reinterpret_cast<const uint8_t*>(a.buf[src])[el];
          for (int r = 0; r < n; ++r)
            if ((dmask >> r) & 1u) reinterpret_cast<uint8_t*>(a.buf[r])[el] = x;
        } else if constexpr (K == 8) {
          const uint16_t x = reinterpret_cast<const uint16_t*>(a.buf[src])[el];
          for (int r = 0; r < n; ++r)
            if ((dmask >> r) & 1u) reinterpret_cast<uint16_t*>(a.buf[r])[el] = x;
        } else {
          const uint32_t x = reinterpret_cast<const uint32_t*>(a.buf[src])[el];
          for (int r = 0; r < n; ++r)
            if ((dmask >> r) & 1u) reinterpret_cast<uint32_t*>(a.buf[r])[el] = x;
        }
      } else {
        float acc = E::load1(a.buf[0], el);
        for (int r = 1; r < n; ++r) acc = __fadd_rn(acc, E::load1(a.buf[r], el));
        acc = __fmul_rn(acc, a.scale);
        for (int r = 0; r < n; ++r)
          if ((dmask >> r) & 1u) E::store1(a.buf[r], el, acc);
      }
    }
  }
  exit_barrier(a, rank, b, e);
  end_epoch(a.pad[rank], e);
}

// ---------------------------------------------------------------------------
// FLAT with TMA staging (north star: "shared-memory or TMA double-buffered
// staging"): per CTA, one elected thread moves tile t of shard g from all n
// ranks' buffers into shared memory with cp.async.bulk (the TMA bulk-copy
// engine, completion counted on an mbarrier), two stages deep; the CTA folds
// stage s from shared memory in rank order while stage s^1 is in flight, then
// stores the result to every rank from registers.  Same arithmetic, same bits
// as hfr_flat_kernel; tiles come from the per-rank counter.  The bulk copies
// read peer HBM over NVLink directly (SASS UBLKCP.S.G).  Default for
// allreduce / reduce-scatter at n in {2,4,8}: r01 measured +2.5-4 % over the
// register-staged kernel (virtual 8: 714 vs 696 GB/s; n=4 bf16 1 GiB: 689 vs 662).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n HFR_MBAR_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra HFR_MBAR_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

constexpr int kTmaTileBytes = 4096;  // default bytes per source per stage (a.tma_tile)
constexpr uint64_t kPairSubUnits = 256;  // PAIR tree kernel: 8-element units per partner sub-tile

__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}

template <class E, int NR>
__global__ void __launch_bounds__(256) hfr_flat_tma_kernel(const Args a) {
  extern __shared__ __align__(128) uint8_t stage_mem[];  // [2][NR][a.tma_tile]
  __shared__ uint64_t bars[2];
  __shared__ uint64_t s_tile[2];
  const int rank = a.rank0 + blockIdx.y;
  const int b = blockIdx.x;
  const uint64_t e = begin_epoch(a.pad[rank]);
  const uint32_t dmask = a.dst_mask ? a.dst_mask : (1u << rank);
  // shard owners: all ranks, or (reduce) the n-1 ranks other than the root
  const int nown = a.excl_root >= 0 ? NR - 1 : NR;
  const int own = a.excl_root >= 0 ? (rank < a.excl_root ? rank : rank - 1) : rank;
  if (entry_barrier(a, rank, b, e) && rank != a.excl_root) {
    constexpr int K = E::kPerVec;
    const uint64_t TB = (uint64_t)a.tma_tile;    // bytes per source per stage
    const uint64_t TV = TB / 16;                 // vectors per tile
    const uint64_t nvec = a.count / K;
    const uint64_t lo = nvec * own / nown, hi = nvec * (own + 1) / nown;
    const uint64_t ntile = (hi - lo + TV - 1) / TV;
    unsigned long long* ctr = reinterpret_cast<unsigned long long*>(&a.pad[rank]->tile_next);
    auto issue = [&](int st, uint64_t t) {  // thread 0 only
      const uint64_t v0 = lo + t * TV;
      const uint32_t bytes = (uint32_t)((v0 + TV < hi ? TV : hi - v0) * 16);
      mbar_expect_tx(&bars[st], NR * bytes);
#pragma unroll
      for (int r = 0; r < NR; ++r)
        bulk_g2s(stage_mem + ((size_t)st * NR + r) * TB, a.buf[r] + v0 * 16, bytes, &bars[st]);
    };
    if (threadIdx.x == 0) {
      mbar_init(&bars[0], 1);
      mbar_init(&bars[1], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
#pragma unroll
      for (int st = 0; st < 2; ++st) {
        const uint64_t t = atomicAdd(ctr, 1ull);
        s_tile[st] = t;
        if (t < ntile) issue(st, t);
      }
    }
    __syncthreads();
    for (uint32_t k = 0;; ++k) {
      const int st = k & 1;
      const uint64_t t = s_tile[st];
      if (t >= ntile) break;
      mbar_wait(&bars[st], (k >> 1) & 1);
      const uint64_t v0 = lo + t * TV;
      const uint64_t nv = v0 + TV < hi ? TV : hi - v0;
      const uint8_t* sm = stage_mem + (size_t)st * NR * TB;
      for (uint64_t j = threadIdx.x; j < nv; j += blockDim.x) {
        float acc[K], tt[K];
        E::widen(*reinterpret_cast<const uint4*>(sm + j * 16), acc);
#pragma unroll
        for (int r = 1; r < NR; ++r) {
          E::widen(*reinterpret_cast<const uint4*>(sm + (size_t)r * TB + j * 16), tt);
#pragma unroll
          for (int q = 0; q < K; ++q) acc[q] = __fadd_rn(acc[q], tt[q]);
        }
#pragma unroll
        for (int q = 0; q < K; ++q) acc[q] = __fmul_rn(acc[q], a.scale);
        const uint4 o = E::narrow(acc);
#pragma unroll
        for (int r = 0; r < NR; ++r)
          if ((dmask >> r) & 1u) st128(a.buf[r] + (v0 + j) * 16, o);
      }
      __syncthreads();  // every thread is done reading stage st
      if (threadIdx.x == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem accesses before async proxy
        const uint64_t tn = atomicAdd(ctr, 1ull);
        s_tile[st] = tn;
        if (tn < ntile) issue(st, tn);
      }
      __syncthreads();
    }
    // ragged tail (< K elements) — last owner, CTA 0
    const uint64_t t0 = nvec * K;
    if (own == nown - 1 && b == 0 && threadIdx.x < a.count - t0) {
      const uint64_t el = t0 + threadIdx.x;
      float acc = E::load1(a.buf[0], el);
      for (int r = 1; r < NR; ++r) acc = __fadd_rn(acc, E::load1(a.buf[r], el));
      acc = __fmul_rn(acc, a.scale);
      for (int r = 0; r < NR; ++r)
        if ((dmask >> r) & 1u) E::store1(a.buf[r], el, acc);
    }
  }
  exit_barrier(a, rank, b, e);
  end_epoch(a.pad[rank], e);
}

// ---------------------------------------------------------------------------
// ONESHOT (small messages): push, then fold locally.
//
// CTA b of rank r stores its slice of x_r into slot [epoch&1][r] of every
// rank's inbox (n-1 NVLink writes), then releases flag entry[b][r] at every
// rank and waits for entry[b][q] of all q — one cross-rank handoff, carrying
// the data.  It then folds the n copies of its slice from its LOCAL inbox in
// rank order 0..n-1 (the same per-element order as FLAT, so the same bits)
// and writes the result into its own buffer only.  Peers never read this
// rank's buffer, so any device buffer works without staging, and no exit
// barrier is needed: a peer reuses a slot parity only two launches later,
// after the intervening launch's entry barrier proved this CTA done.
// ---------------------------------------------------------------------------
template <class E, int NR>
__global__ void __launch_bounds__(512) hfr_oneshot_kernel(const Args a) {
  const int rank = a.rank0 + blockIdx.y;
  const int n = NR > 0 ? NR : a.n;
  const int b = blockIdx.x;
  constexpr int K = E::kPerVec;
  const uint64_t nvec = a.count / K;
  const uint64_t v0 = nvec * b / gridDim.x, v1 = nvec * (b + 1) / gridDim.x;
  const uint64_t ep = begin_epoch(a.pad[rank]);
  const uint64_t par = ep & 1;
  const char* src = a.buf[rank];
  const bool last = b == (int)gridDim.x - 1;
  const uint64_t t0 = nvec * K;  // first tail element
  // the rank's own buffer may be unaligned (any device pointer is accepted):
  // then this CTA moves its slice element by element
  const bool vec_ok = ((reinterpret_cast<uintptr_t>(a.buf[rank])) & 15) == 0;
  const uint64_t e_end = last ? a.count : v1 * K;
  // 1. push
  if (vec_ok) {
    for (uint64_t i = v0 + threadIdx.x; i < v1; i += blockDim.x) {
      const uint4 v = ld128(src + i * 16);
      for (int q = 0; q < n; ++q) st128(a.inbox[q] + (par * n + rank) * a.slot_bytes + i * 16, v);
    }
  }
  for (uint64_t e = (vec_ok ? (last ? t0 : e_end) : v0 * K) + threadIdx.x; e < e_end; e += blockDim.x) {
    const float x = E::load1(src, e);
    for (int q = 0; q < n; ++q) E::store1(a.inbox[q] + (par * n + rank) * a.slot_bytes, e, x);
  }
  // 2. one handoff: data visible everywhere, then the flag
  __syncthreads();
  bool ok = true;
  if (threadIdx.x < n) {
    const int q = threadIdx.x;
    fence_acq_rel_sys();  // this CTA's pushes are visible before the flag
    st_relaxed_sys(&a.pad[q]->entry[b][rank], pack_flag(ep, a.sig));
    ok = wait_flag(a, &a.pad[rank]->entry[b][q], ep, rank, q);
  }
  if (!__syncthreads_and(ok)) return;
  // 3. fold the n local copies in rank order
  const char* in = a.inbox[rank] + par * n * a.slot_bytes;
  char* dst = a.buf[rank];
  if (vec_ok) {
    for (uint64_t i = v0 + threadIdx.x; i < v1; i += blockDim.x) {
      float acc[K], t[K];
      E::widen(ld128(in + i * 16), acc);
      for (int r = 1; r < n; ++r) {
        E::widen(ld128(in + r * a.slot_bytes + i * 16), t);
#pragma unroll
        for (int k = 0; k < K; ++k) acc[k] = __fadd_rn(acc[k], t[k]);
      }
#pragma unroll
      for (int k = 0; k < K; ++k) acc[k] = __fmul_rn(acc[k], a.scale);
      st128(dst + i * 16, E::narrow(acc));
    }
  }
  for (uint64_t e = (vec_ok ? (last ? t0 : e_end) : v0 * K) + threadIdx.x; e < e_end; e += blockDim.x) {
    float acc = E::load1(in, e);
    for (int r = 1; r < n; ++r) acc = __fadd_rn(acc, E::load1(in + r * a.slot_bytes, e));
    E::store1(dst, e, __fmul_rn(acc, a.scale));
  }
  end_epoch(a.pad[rank], ep);
}

// ---------------------------------------------------------------------------
// ONESHOT, LL form (small messages): the flag travels inside the data.
//
// Every element becomes one 8-byte word {element bits, flag}, flag =
// (sig8 << 24) | (1 + epoch mod (2^24 - 1)) — never 0 in its low 24 bits, so
// a zeroed word never passes; two words go out per 16-byte store, so a word
// is never seen half-written.  A receiver spins on the words of its slice
// until every source's flag shows this launch, folds in rank order (the FLAT
// bits again) and zeroes the words it consumed, so no stale word survives to
// alias a launch 2^24 - 1 epochs later.  No fence, no separate handshake:
// latency is one NVLink write.  Slot reuse (parity = epoch & 1) is safe for
// the same reason as the fenced ONESHOT: a rank only enters launch e+2 after
// it received every peer's launch-e+1 data, which peers send after finishing
// launch e (including its zeroing).  CTA 0 also publishes the usual packed
// entry word at every peer (no wait), so a peer running another kernel for
// this call (argument mismatch) sees PROTOCOL instead of a timeout, and this
// kernel watches the peers' words the same way while it spins.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint4 ld128_volatile(const void* p) {
  uint4 v;
  asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}

template <class E>
__device__ __forceinline__ uint32_t elem_bits(const char* p, uint64_t e) {
  if constexpr (E::kPerVec == 16) return reinterpret_cast<const uint8_t*>(p)[e];
  if constexpr (E::kPerVec == 8) return reinterpret_cast<const uint16_t*>(p)[e];
  return reinterpret_cast<const uint32_t*>(p)[e];
}
template <class E>
__device__ __forceinline__ float bits_value(uint32_t b) {
  return E::from_bits(b);
}

__device__ __forceinline__ bool ll_ready(const uint4& w, uint32_t flag) {
  return ((w.y ^ flag) & 0xFFFFFFu) == 0 && ((w.w ^ flag) & 0xFFFFFFu) == 0;
}
__device__ __forceinline__ uint32_t ll_flag(uint64_t ep, uint32_t sig8) {
  return (sig8 << 24) | (uint32_t)(1 + ep % 0xFFFFFFull);
}

// NR = compile-time rank count (2, 4, 8) so all n words of a pair are loaded
// at once; 0 = runtime n (one source at a time).
template <class E, int NR>
__global__ void __launch_bounds__(512) hfr_oneshot_ll_kernel(const Args a) {
  const int rank = a.rank0 + blockIdx.y;
  const int n = NR > 0 ? NR : a.n;
  const uint64_t ep = begin_epoch(a.pad[rank]);
  const uint32_t sig8 = (uint32_t)(a.sig ^ (a.sig >> 32)) & 0xFFu;
  const uint32_t flag = ll_flag(ep, sig8);
  const uint64_t par = ep & 1;
  const uint64_t npair = (a.count + 1) / 2;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const char* src = a.buf[rank];
  const uint64_t entry_word = pack_flag(ep, a.sig);
  if (blockIdx.x == 0 && threadIdx.x < n) st_relaxed_sys(&a.pad[threadIdx.x]->entry[0][rank], entry_word);
  // 1. push {x, flag} words of my pairs into every rank's slot [par][rank]
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < npair; i += stride) {
    const uint64_t e = 2 * i;
    const uint32_t x0 = elem_bits<E>(src, e);
    const uint32_t x1 = e + 1 < a.count ? elem_bits<E>(src, e + 1) : 0u;
    const uint4 w = make_uint4(x0, flag, x1, flag);
    for (int q = 0; q < n; ++q) st128(a.inbox[q] + (par * n + rank) * a.slot_bytes + i * 16, w);
  }
  // 2. receive (all n words of a pair in flight at once) and fold in rank order
  const char* in = a.inbox[rank] + par * n * a.slot_bytes;
  char* dst = a.buf[rank];
  bool ok = true;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < npair && ok; i += stride) {
    constexpr int M = NR > 0 ? NR : 1;
    uint4 w[M];
    float acc0 = 0.f, acc1 = 0.f;
    for (int r0 = 0; r0 < n && ok; r0 += M) {
#pragma unroll
      for (int u = 0; u < M; ++u) w[u] = ld128_volatile(in + (r0 + u) * a.slot_bytes + i * 16);
      uint64_t t0 = 0;
#pragma unroll
      for (int u = 0; u < M; ++u) {
        for (uint32_t it = 1; !ll_ready(w[u], flag); ++it) {
          if ((it & 1023u) == 0) {
            if (!t0) t0 = globaltimer();
            const uint64_t v = ld_relaxed_sys(&a.pad[rank]->entry[0][r0 + u]);
            if ((v >> 32) == ep && v != entry_word) raise_error(a, kErrProtocol);  // peer runs another call
            if (*a.err != 0 || globaltimer() - t0 > a.timeout_ns) {
              if (*a.err == 0) raise_error(a, kErrTimeout);
              ok = false;
              break;
            }
          }
          w[u] = ld128_volatile(in + (r0 + u) * a.slot_bytes + i * 16);
        }
        if (ok && ((w[u].y >> 24) != sig8 || (w[u].w >> 24) != sig8)) {
          raise_error(a, kErrProtocol);
          ok = false;
        }
      }
      if (!ok) break;
#pragma unroll
      for (int u = 0; u < M; ++u) st128(const_cast<char*>(in) + (r0 + u) * a.slot_bytes + i * 16, make_uint4(0, 0, 0, 0));
#pragma unroll
      for (int u = 0; u < M; ++u) {
        const float v0 = bits_value<E>(w[u].x), v1 = bits_value<E>(w[u].z);
        acc0 = r0 + u == 0 ? v0 : __fadd_rn(acc0, v0);
        acc1 = r0 + u == 0 ? v1 : __fadd_rn(acc1, v1);
      }
    }
    if (!ok) break;
    const uint64_t e = 2 * i;
    E::store1(dst, e, __fmul_rn(acc0, a.scale));
    if (e + 1 < a.count) E::store1(dst, e + 1, __fmul_rn(acc1, a.scale));
  }
  end_epoch(a.pad[rank], ep);
}

// ---------------------------------------------------------------------------
// NVLS (order-relaxed; hfr_nvls.cuh): the NVSwitch reduces and multicasts.
//
// Rank g owns shard g.  Per 16 B: one multimem.ld_reduce on the multicast
// address returns the sum over all n GPUs (fp32; bf16 accumulated in fp32 by
// the switch and rounded once), the owner multiplies by scale, and one
// multimem.st writes the result into all n GPUs' buffers.  The switch picks
// the summation order, so the bits are NOT the rank-ascending fold's: the
// result is held to reading R18's bound.  Entry: the usual packed-flag
// handshake (argument check); exit: one multimem.red.release per CTA bumps
// counter b on every GPU, each CTA waits until all n ranks' CTA b arrived.
// ---------------------------------------------------------------------------
// U multimem.ld_reduce in flight per thread before the first multimem.st
template <int U>
__device__ __forceinline__ void nvls_vecs_f32(char* mc, uint64_t stride_bytes, int cnt, float scale) {
  float v[U][4];
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (u < cnt)
      asm volatile("multimem.ld_reduce.weak.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                   : "=f"(v[u][0]), "=f"(v[u][1]), "=f"(v[u][2]), "=f"(v[u][3])
                   : "l"(mc + u * stride_bytes)
                   : "memory");
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (u < cnt) {
#pragma unroll
      for (int k = 0; k < 4; ++k) v[u][k] = __fmul_rn(v[u][k], scale);
      asm volatile("multimem.st.weak.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc + u * stride_bytes), "f"(v[u][0]),
                   "f"(v[u][1]), "f"(v[u][2]), "f"(v[u][3])
                   : "memory");
    }
}

template <class E, int U>
__device__ __forceinline__ void nvls_vecs_16(char* mc, uint64_t stride_bytes, int cnt, float scale) {
  uint4 v[U];
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (u < cnt) {
      if constexpr (std::is_same<E, BF16>::value)
        asm volatile("multimem.ld_reduce.weak.global.add.acc::f32.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                     : "l"(mc + u * stride_bytes)
                     : "memory");
      else
        asm volatile("multimem.ld_reduce.weak.global.add.acc::f32.v4.f16x2 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                     : "l"(mc + u * stride_bytes)
                     : "memory");
    }
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (u < cnt) {
      if (scale != 1.0f) {
        float f[8];
        E::widen(v[u], f);
#pragma unroll
        for (int k = 0; k < 8; ++k) f[k] = __fmul_rn(f[k], scale);
        v[u] = E::narrow(f);
      }
      asm volatile("multimem.st.weak.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc + u * stride_bytes),
                   "f"(__uint_as_float(v[u].x)), "f"(__uint_as_float(v[u].y)), "f"(__uint_as_float(v[u].z)),
                   "f"(__uint_as_float(v[u].w))
                   : "memory");
    }
}

// The other collectives on the multicast object (bit-exact where nothing is
// reduced): RED loads through multimem.ld_reduce (else a local 16-B load of
// this rank's buffer), MC stores through multimem.st (else a local store).
//   reduce-scatter: RED, local store   all-gather: local load, MC
//   reduce:         RED, local store (root alone, whole buffer)
//   broadcast:      local load, MC   (root alone, whole buffer)
template <class E, bool RED, bool MC, int U>
__device__ __forceinline__ void nvls_vecs_coll(char* mc, char* uc, uint64_t stride_bytes, int cnt, float scale) {
  uint4 v[U];
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (u < cnt) {
      if constexpr (!RED) {
        v[u] = ld128(uc + u * stride_bytes);
      } else if constexpr (std::is_same<E, F32>::value) {
        asm volatile("multimem.ld_reduce.weak.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                     : "l"(mc + u * stride_bytes)
                     : "memory");
      } else if constexpr (std::is_same<E, BF16>::value) {
        asm volatile("multimem.ld_reduce.weak.global.add.acc::f32.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                     : "l"(mc + u * stride_bytes)
                     : "memory");
      } else {
        asm volatile("multimem.ld_reduce.weak.global.add.acc::f32.v4.f16x2 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                     : "l"(mc + u * stride_bytes)
                     : "memory");
      }
    }
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (u < cnt) {
      if (RED && scale != 1.0f) {
        float f[E::kPerVec];
        E::widen(v[u], f);
#pragma unroll
        for (int k = 0; k < E::kPerVec; ++k) f[k] = __fmul_rn(f[k], scale);
        v[u] = E::narrow(f);
      }
      if constexpr (MC)
        mc_st128(mc + u * stride_bytes, v[u]);
      else
        st128(uc + u * stride_bytes, v[u]);
    }
}

template <class E, bool RED, bool MC>
__device__ __forceinline__ void nvls_coll_range(const Args& a, char* uc, uint64_t lo, uint64_t hi, Pad* mine) {
  constexpr int U = 4;
  const uint64_t lane = threadIdx.x & 31;
  unsigned long long* ctr = reinterpret_cast<unsigned long long*>(&mine->tile_next);
  for (;;) {
    uint64_t t = 0;
    if (lane == 0) t = atomicAdd(ctr, 1ull);
    t = __shfl_sync(0xffffffffu, t, 0);
    const uint64_t i = lo + t * (U * 32) + lane;
    if (lo + t * (U * 32) >= hi) break;
    const int cnt = i < hi ? (int)((hi - i + 31) / 32) : 0;
    nvls_vecs_coll<E, RED, MC, U>(a.mcbuf + i * 16, uc + i * 16, 32 * 16, cnt < U ? cnt : U, a.scale);
  }
}

template <class E>
__global__ void __launch_bounds__(512) hfr_nvls_coll_kernel(const Args a) {
  const int rank = a.rank0;  // real comms only
  const int n = a.n;
  const int b = blockIdx.x;
  Pad* const mine = a.pad[rank];
  const uint64_t e = begin_epoch(mine);
  __shared__ uint32_t s_k;
  if (threadIdx.x == 0) s_k = ++mine->nvls_seq[b];
  if (entry_barrier(a, rank, b, e)) {
    constexpr int K = E::kPerVec;
    const uint64_t nvec = a.count / K;
    const bool solo = a.nvls_solo >= 0;
    if (!solo || rank == a.nvls_solo) {
      const uint64_t lo = solo ? 0 : nvec * rank / n, hi = solo ? nvec : nvec * (rank + 1) / n;
      char* uc = a.buf[rank];
      switch (a.nvls_op) {
        case 1: nvls_coll_range<E, true, false>(a, uc, lo, hi, mine); break;
        case 2: nvls_coll_range<E, false, true>(a, uc, lo, hi, mine); break;
        default: nvls_coll_range<E, true, true>(a, uc, lo, hi, mine); break;
      }
      // ragged tail (< K elements): the last worker, over unicast peers
      const uint64_t t0 = nvec * K;
      if ((solo || rank == n - 1) && b == 0 && threadIdx.x < a.count - t0) {
        const uint64_t el = t0 + threadIdx.x;
        float acc;
        if (a.nvls_op & 1) {
          acc = E::load1(a.buf[0], el);
          for (int r = 1; r < n; ++r) acc = __fadd_rn(acc, E::load1(a.buf[r], el));
          acc = __fmul_rn(acc, a.scale);
        } else {
          acc = E::load1(a.buf[rank], el);
        }
        if (a.nvls_op & 2) {
          for (int r = 0; r < n; ++r) E::store1(a.buf[r], el, acc);
        } else {  // reduce root, or reduce-scatter's last shard (this rank)
          E::store1(a.buf[rank], el, acc);
        }
      }
    }
    mc_exit_barrier(a, b, n, s_k);
  }
  end_epoch(mine, e);
}

template <class E>
__global__ void __launch_bounds__(512) hfr_nvls_kernel(const Args a) {
  const int rank = a.rank0;  // real comms only
  const int n = a.n;
  const int b = blockIdx.x;
  Pad* const mine = a.pad[rank];
  const uint64_t e = begin_epoch(mine);
  __shared__ uint32_t s_k;
  if (threadIdx.x == 0) s_k = ++mine->nvls_seq[b];
  if (entry_barrier(a, rank, b, e)) {
    constexpr int K = E::kPerVec;
    const uint64_t nvec = a.count / K;
    const uint64_t lo = nvec * rank / n, hi = nvec * (rank + 1) / n;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    constexpr int U = 4;
    (void)stride;
    // warp tiles of U*32 vectors handed out from the per-rank counter (as FLAT)
    const uint64_t lane = threadIdx.x & 31;
    unsigned long long* ctr = reinterpret_cast<unsigned long long*>(&mine->tile_next);
    for (;;) {
      uint64_t t = 0;
      if (lane == 0) t = atomicAdd(ctr, 1ull);
      t = __shfl_sync(0xffffffffu, t, 0);
      const uint64_t i = lo + t * (U * 32) + lane;
      if (lo + t * (U * 32) >= hi) break;
      const int cnt = i < hi ? (int)((hi - i + 31) / 32) : 0;
      if constexpr (K == 8)
        nvls_vecs_16<E, U>(a.mcbuf + i * 16, 32 * 16, cnt < U ? cnt : U, a.scale);
      else
        nvls_vecs_f32<U>(a.mcbuf + i * 16, 32 * 16, cnt < U ? cnt : U, a.scale);
    }
    // ragged tail (< K elements): the last rank folds it over unicast peers
    const uint64_t t0 = nvec * K;
    if (rank == n - 1 && b == 0 && threadIdx.x < a.count - t0) {
      const uint64_t el = t0 + threadIdx.x;
      float acc = E::load1(a.buf[0], el);
      for (int r = 1; r < n; ++r) acc = __fadd_rn(acc, E::load1(a.buf[r], el));
      acc = __fmul_rn(acc, a.scale);
      for (int r = 0; r < n; ++r) E::store1(a.buf[r], el, acc);
    }
    mc_exit_barrier(a, b, n, s_k);
  }
  end_epoch(mine, e);
}

// ---------------------------------------------------------------------------
// Subsystem (2): double binary tree (Algorithm 2) as a
// push-only P2P schedule, and (PAIR) "HFReduce with NVLink".
//
// Chunk c (global index within the half) rides tree c & 1 (reading R8).  Up
// pass (Alg. 2 pass 1, "DL_i += DR_i"): a node waits for its children's fp32
// partials (pushed into its own partial slots), combines them in-order with
// its own value (reading R10) and pushes the result into its parent's slot;
// the root scales, casts, writes the final chunk to its own buffer and pushes
// it to its children.  Down pass (Alg. 2 pass 2): a node waits for the final
// chunk from its parent and forwards it to its children.  PAIR: tree nodes
// are pairs k = (2k, 2k+1); member 2k+h works on half h, its node value is
// fl32(x_2k + x_2k+1) (the NVLink pair pre-reduce, fused), and every final
// chunk is also pushed to the partner (the pair all-gather, fused).
// Every NVLink transfer is a remote store; all loads are local except the
// partner's half in PAIR mode.
// ---------------------------------------------------------------------------
template <class E>
__device__ __forceinline__ void load8(const char* base, uint64_t e, float* f) {
  // 8 consecutive elements starting at element e (e % 8 == 0)
  if constexpr (E::kPerVec == 16) {
    E::widen8(*reinterpret_cast<const uint2*>(base + e), f);
  } else if constexpr (E::kPerVec == 8) {
    E::widen(ld128(base + e * 2), f);
  } else {
    E::widen(ld128(base + e * 4), f);
    E::widen(ld128(base + e * 4 + 16), f + 4);
  }
}
// the same from any address space (the PAIR kernel's shared-memory ring)
template <class E>
__device__ __forceinline__ void widen8_generic(const uint8_t* p, float* f) {
  if constexpr (E::kPerVec == 16) {
    E::widen8(*reinterpret_cast<const uint2*>(p), f);
  } else if constexpr (E::kPerVec == 8) {
    E::widen(*reinterpret_cast<const uint4*>(p), f);
  } else {
    E::widen(*reinterpret_cast<const uint4*>(p), f);
    E::widen(*reinterpret_cast<const uint4*>(p + 16), f + 4);
  }
}
template <class E>
__device__ __forceinline__ void store8(char* base, uint64_t e, const float* f) {
  if constexpr (E::kPerVec == 16) {
    *reinterpret_cast<uint2*>(base + e) = E::narrow8(f);
  } else if constexpr (E::kPerVec == 8) {
    st128(base + e * 2, E::narrow(f));
  } else {
    st128(base + e * 4, E::narrow(f));
    st128(base + e * 4 + 16, E::narrow(f + 4));
  }
}
__device__ __forceinline__ void load8_f32(const float* base, uint64_t e, float* f) {
  F32::widen(ld128(base + e), f);
  F32::widen(ld128(base + e + 4), f + 4);
}
__device__ __forceinline__ void store8_f32(float* base, uint64_t e, const float* f) {
  st128(base + e, F32::narrow(f));
  st128(base + e + 4, F32::narrow(f + 4));
}

template <class E, bool PAIR>
__global__ void __launch_bounds__(512) hfr_tree_kernel(const Args a) {
  const int rank = a.rank0 + blockIdx.y;
  const int b = blockIdx.x;
  const uint64_t ep = begin_epoch(a.pad[rank]);
  const bool ok = entry_barrier(a, rank, b, ep);
  if (!ok) return;

  const int h = PAIR ? (rank & 1) : 0;
  const int me = PAIR ? (rank >> 1) : rank;
  const int partner = rank ^ 1;
  const uint64_t base = a.half_base[h], len = a.half_len[h];
  const uint64_t C = (uint64_t)a.chunk;
  const uint64_t nch = (len + C - 1) / C;
  const uint64_t c_end = nch < a.c_hi ? nch : a.c_hi;
  Pad* const mypad = a.pad[rank];
  char* const mybuf = a.buf[rank];
  const float* const mypart = a.part[rank];
  auto member = [&](int node) { return PAIR ? 2 * node + h : node; };

  Tracer tr(a);
  __shared__ int s_ready;
  // Down pass of chunk c (Alg. 2 pass 2): wait for (block) or poll (!block)
  // the final chunk from the parent, then forward it to the children (and the
  // pair partner).  Returns 1 done, 0 not ready yet, -1 error.
  auto down_chunk = [&](uint64_t c, bool block) -> int {
    const TreeNode nd = a.tree[c & 1][me];
    if (nd.parent < 0) return 1;  // the root already pushed its final chunk in the up pass
    const uint32_t lc = (uint32_t)(c - a.c_lo);
    const uint64_t tw = tr.p ? globaltimer() : 0;
    if (threadIdx.x == 0) {
      if (block)
        s_ready = wait_ge(a, &mypad->down[lc], ep) ? 1 : -1;
      else
        s_ready = ld_acquire_sys(&mypad->down[lc]) >= ep ? 1 : 0;
    }
    __syncthreads();
    const int ready = s_ready;
    __syncthreads();
    if (ready != 1) return ready;
    const uint64_t tk = tr.p ? globaltimer() : 0;
    if (nd.nchild == 0 && !PAIR) {
      if (threadIdx.x == 0) tr.rec((2ull << 60) | ((uint64_t)rank << 48) | c, tw, tk, tk, tk);
      return 1;
    }
    const uint64_t e0 = c * C, e1 = (e0 + C < len) ? e0 + C : len;
    const int esz = (int)sizeof(typename E::T);
    const uint64_t b0 = (base + e0) * esz, b1 = (base + e1) * esz;  // byte range
    const uint64_t nv = (b1 - b0) / 16;
    constexpr int DU = 4;  // 4 x 16 B loads in flight per thread before the stores
    for (uint64_t v0 = threadIdx.x; v0 < nv; v0 += (uint64_t)blockDim.x * DU) {
      uint4 val[DU];
#pragma unroll
      for (int u = 0; u < DU; ++u)
        if (v0 + (uint64_t)u * blockDim.x < nv) val[u] = ld128(mybuf + b0 + (v0 + (uint64_t)u * blockDim.x) * 16);
#pragma unroll
      for (int u = 0; u < DU; ++u) {
        if (v0 + (uint64_t)u * blockDim.x >= nv) break;
        const uint64_t off = b0 + (v0 + (uint64_t)u * blockDim.x) * 16;
        for (int k = 0; k < nd.nchild; ++k) st128(a.buf[member(nd.child[k])] + off, val[u]);
        if constexpr (PAIR) st128(a.buf[partner] + off, val[u]);
      }
    }
    for (uint64_t y = b0 + nv * 16 + threadIdx.x * esz; y < b1; y += (uint64_t)blockDim.x * esz) {
      if (esz == 1) {
        const uint8_t val = *reinterpret_cast<const uint8_t*>(mybuf + y);
        for (int k = 0; k < nd.nchild; ++k) *reinterpret_cast<uint8_t*>(a.buf[member(nd.child[k])] + y) = val;
        if constexpr (PAIR) *reinterpret_cast<uint8_t*>(a.buf[partner] + y) = val;
      } else if (esz == 2) {
        const uint16_t val = *reinterpret_cast<const uint16_t*>(mybuf + y);
        for (int k = 0; k < nd.nchild; ++k) *reinterpret_cast<uint16_t*>(a.buf[member(nd.child[k])] + y) = val;
        if constexpr (PAIR) *reinterpret_cast<uint16_t*>(a.buf[partner] + y) = val;
      } else {
        const uint32_t val = *reinterpret_cast<const uint32_t*>(mybuf + y);
        for (int k = 0; k < nd.nchild; ++k) *reinterpret_cast<uint32_t*>(a.buf[member(nd.child[k])] + y) = val;
        if constexpr (PAIR) *reinterpret_cast<uint32_t*>(a.buf[partner] + y) = val;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const uint64_t ts = tr.p ? globaltimer() : 0;
      fence_acq_rel_sys();
      for (int k = 0; k < nd.nchild; ++k) st_relaxed_sys(&a.pad[member(nd.child[k])]->down[lc], ep);
      if constexpr (PAIR) st_relaxed_sys(&a.pad[partner]->pdown[lc], ep);
      tr.rec((2ull << 60) | ((uint64_t)rank << 48) | c, tw, tk, ts, globaltimer());
    }
    return 1;
  };
  // PAIR: 2-stage shared-memory ring for the partner's chunk (bulk copies)
  __shared__ __align__(128) uint8_t pstage[PAIR ? 2 * kPairSubUnits * 8 * sizeof(typename E::T) : 16];
  __shared__ uint64_t pbar[2];
  uint32_t puse[2] = {0, 0};
  if constexpr (PAIR) {
    if (threadIdx.x == 0) {
      mbar_init(&pbar[0], 1);
      mbar_init(&pbar[1], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
  }
  uint64_t dn = a.c_lo + b;  // next chunk whose down pass is pending

  // ---- up pass -----------------------------------------------------------
  for (uint64_t c = a.c_lo + b; c < c_end; c += gridDim.x) {
    const TreeNode nd = a.tree[c & 1][me];
    const uint32_t lc = (uint32_t)(c - a.c_lo);
    const uint64_t tw = tr.p ? globaltimer() : 0;
    // PAIR: start pulling the partner's chunk before waiting on the children
    const uint64_t pe0 = c * C, pe1 = (pe0 + C < len) ? pe0 + C : len;
    const uint64_t nsub = ((pe1 - pe0) / 8 + kPairSubUnits - 1) / kPairSubUnits;
    auto pair_issue = [&](int st, uint64_t j) {  // thread 0 only
      constexpr uint64_t esz = sizeof(typename E::T);
      const uint64_t nvc = (pe1 - pe0) / 8;
      const uint64_t u0 = j * kPairSubUnits, u1 = u0 + kPairSubUnits < nvc ? u0 + kPairSubUnits : nvc;
      // bulk copies move whole 16-byte units: an odd last FP8 unit (8 bytes)
      // is read directly from the partner below
      const uint32_t bytes = (uint32_t)((u1 - u0) * 8 * esz) & ~15u;
      mbar_expect_tx(&pbar[st], bytes);
      if (bytes)
        bulk_g2s(pstage + (size_t)st * kPairSubUnits * 8 * esz, a.buf[partner] + (base + pe0 + u0 * 8) * esz, bytes,
                 &pbar[st]);
    };
    if constexpr (PAIR) {
      if (threadIdx.x == 0)
        for (uint64_t j = 0; j < 2 && j < nsub; ++j) pair_issue((int)j, j);
    }
    bool got = true;
    if (threadIdx.x < nd.nchild) got = wait_ge(a, &mypad->up[threadIdx.x][lc], ep);
    if (!__syncthreads_and(got)) return;
    const uint64_t tk = tr.p ? globaltimer() : 0;

    const uint64_t e0 = c * C, e1 = (e0 + C < len) ? e0 + C : len;  // offsets within the half
    const uint64_t nv = (e1 - e0) / 8;
    const bool root = nd.parent < 0;
    char* const pbuf = PAIR ? a.buf[partner] : nullptr;
    float* const dst_part = root ? nullptr : a.part[member(nd.parent)] + (uint64_t)nd.slot * a.part_stride;
    const int nchild = nd.nchild, self_pos = nd.self_pos;
    // A DBT leaf's partial is its own x: stream it as a copy with 4 vectors in
    // flight per thread (r01: DBT n=4 313 -> 360-378 GB/s).  16-bit and FP8
    // leaves send their raw values (the parent widens exactly): half / a
    // quarter of an fp32 partial's bytes.
    constexpr bool kRaw = E::kPerVec >= 8;  // 16-bit and 8-bit element types
    const bool leafcopy = !PAIR && nchild == 0 && !root;
    // slot sl of this node holds a raw leaf partial?
    bool slot_bf16[2] = {false, false};
    if constexpr (!PAIR && kRaw) {
      for (int sl = 0; sl < nchild; ++sl) slot_bf16[sl] = a.tree[c & 1][nd.child[sl]].nchild == 0;
    }
    if (leafcopy && kRaw) {
      // raw partials live at the start of the chunk's fp32 slot region (bytes
      // [4*e0, 4*e0 + esz*C)), so they never overlap another chunk's fp32
      // partials in the same slot array; one 8-element unit = 16 B (16-bit) or
      // 8 B (FP8)
      constexpr uint64_t esz = sizeof(typename E::T);
      const char* srcb = mybuf + (base + e0) * esz;
      char* dstb = reinterpret_cast<char*>(dst_part + e0);
      for (uint64_t q0 = threadIdx.x; q0 < nv; q0 += (uint64_t)blockDim.x * 4) {
        if constexpr (esz == 2) {
          uint4 v[4];
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (q0 + (uint64_t)u * blockDim.x < nv) v[u] = ld128(srcb + (q0 + (uint64_t)u * blockDim.x) * 16);
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (q0 + (uint64_t)u * blockDim.x < nv) st128(dstb + (q0 + (uint64_t)u * blockDim.x) * 16, v[u]);
        } else {
          uint2 v[4];
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (q0 + (uint64_t)u * blockDim.x < nv)
              v[u] = *reinterpret_cast<const uint2*>(srcb + (q0 + (uint64_t)u * blockDim.x) * 8);
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (q0 + (uint64_t)u * blockDim.x < nv) *reinterpret_cast<uint2*>(dstb + (q0 + (uint64_t)u * blockDim.x) * 8) = v[u];
        }
      }
    } else if (leafcopy) {
      const uint64_t nq = nv * 2;  // 16 B fp32 quads
      for (uint64_t q0 = threadIdx.x; q0 < nq; q0 += (uint64_t)blockDim.x * 4) {
        float f[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint64_t q = q0 + (uint64_t)u * blockDim.x;
          if (q < nq) {
            F32::widen(ld128(mybuf + (base + e0 + q * 4) * 4), f[u]);  // fp32 only (16/8-bit: raw copy above)
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint64_t q = q0 + (uint64_t)u * blockDim.x;
          if (q < nq) st128(dst_part + e0 + q * 4, F32::narrow(f[u]));
        }
      }
    }
    // one unit = 8 elements at offset e of the half; xp = the pair partner's
    // 8 values (PAIR, staged in shared memory) or nullptr
    auto unit = [&](uint64_t v, const float* xp) {
      const uint64_t e = e0 + v * 8;
      float xv[8], pp[2][8];
      load8<E>(mybuf, base + e, xv);
      if constexpr (PAIR) {
        // node value x_v = fl32(x_2k + x_2k+1), lower rank first
#pragma unroll
        for (int k = 0; k < 8; ++k) xv[k] = h == 0 ? __fadd_rn(xv[k], xp[k]) : __fadd_rn(xp[k], xv[k]);
      }
#pragma unroll
      for (int sl = 0; sl < 2; ++sl)
        if (sl < nchild) {
          if (kRaw && slot_bf16[sl])
            load8<E>(reinterpret_cast<const char*>(mypart + (uint64_t)sl * a.part_stride + e0), e - e0, pp[sl]);
          else
            load8_f32(mypart + (uint64_t)sl * a.part_stride, e, pp[sl]);
        }
      // in-order combination: children below, x_v, children above (R10)
      float acc[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = self_pos == 0 ? xv[j] : pp[0][j];
#pragma unroll
      for (int k = 1; k <= 2; ++k) {
        if (k > nchild) break;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float t = k == self_pos ? xv[j] : (k < self_pos ? pp[k][j] : pp[k - 1][j]);
          acc[j] = __fadd_rn(acc[j], t);
        }
      }
      if (root) {
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = __fmul_rn(acc[j], a.scale);
        store8<E>(mybuf, base + e, acc);
        for (int k = 0; k < nchild; ++k) store8<E>(a.buf[member(nd.child[k])], base + e, acc);
        if constexpr (PAIR) store8<E>(pbuf, base + e, acc);
      } else {
        store8_f32(dst_part, e, acc);
      }
    };
    if constexpr (PAIR) {
      // the partner's chunk arrives through the bulk-copy engine, sub-tile by
      // sub-tile into a 2-stage ring (prefetched before the children's wait)
      constexpr uint64_t esz = sizeof(typename E::T);
      for (uint64_t j = 0; j < nsub; ++j) {
        const int st = (int)(j & 1);
        mbar_wait(&pbar[st], puse[st] & 1);
        ++puse[st];
        const uint64_t u0 = j * kPairSubUnits, u1 = u0 + kPairSubUnits < nv ? u0 + kPairSubUnits : nv;
        const uint8_t* sm = pstage + (size_t)st * kPairSubUnits * 8 * esz;
        for (uint64_t v = u0 + threadIdx.x; v < u1; v += blockDim.x) {
          float xp[8];
          if ((v - u0 + 1) * 8 * esz <= (((u1 - u0) * 8 * esz) & ~(uint64_t)15))
            widen8_generic<E>(sm + (v - u0) * 8 * esz, xp);  // shared memory: generic loads
          else
            widen8_generic<E>(reinterpret_cast<const uint8_t*>(pbuf) + (base + e0 + v * 8) * esz, xp);
          unit(v, xp);
        }
        __syncthreads();  // stage st consumed
        if (threadIdx.x == 0 && j + 2 < nsub) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          pair_issue(st, j + 2);
        }
      }
    } else {
      for (uint64_t v = leafcopy ? nv : threadIdx.x; v < nv; v += blockDim.x) unit(v, nullptr);
    }
    // ragged tail of the half (only the last chunk can have one)
    for (uint64_t e = e0 + nv * 8 + threadIdx.x; e < e1; e += blockDim.x) {
      float xv = E::load1(mybuf, base + e);
      if constexpr (PAIR) {
        const float xp = E::load1(pbuf, base + e);
        xv = h == 0 ? __fadd_rn(xv, xp) : __fadd_rn(xp, xv);
      }
      float acc = 0.f;
      for (int k = 0; k <= nd.nchild; ++k) {
        float s = xv;
        if (k != nd.self_pos) {
          const int sl = k < nd.self_pos ? k : k - 1;
          const float* slot = mypart + (uint64_t)sl * a.part_stride;
          s = (kRaw && slot_bf16[sl]) ? E::load1(reinterpret_cast<const char*>(slot + e0), e - e0) : slot[e];
        }
        acc = k == 0 ? s : __fadd_rn(acc, s);
      }
      if (root) {
        acc = __fmul_rn(acc, a.scale);
        E::store1(mybuf, base + e, acc);
        for (int k = 0; k < nd.nchild; ++k) E::store1(a.buf[member(nd.child[k])], base + e, acc);
        if constexpr (PAIR) E::store1(pbuf, base + e, acc);
      } else if (kRaw && leafcopy) {
        E::store1(reinterpret_cast<char*>(dst_part + e0), e - e0, acc);  // raw 16/8-bit leaf partial (exact)
      } else {
        dst_part[e] = acc;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const uint64_t ts = tr.p ? globaltimer() : 0;
      fence_acq_rel_sys();
      if (root) {
        for (int k = 0; k < nd.nchild; ++k) st_relaxed_sys(&a.pad[member(nd.child[k])]->down[lc], ep);
        if constexpr (PAIR) st_relaxed_sys(&a.pad[partner]->pdown[lc], ep);
      } else {
        st_relaxed_sys(&a.pad[member(nd.parent)]->up[nd.slot][lc], ep);
      }
      tr.rec((1ull << 60) | ((uint64_t)rank << 48) | c, tw, tk, ts, globaltimer());
    }
  }

  // ---- down pass (blocking) ------------------------------------------------
  for (; dn < c_end; dn += gridDim.x)
    if (down_chunk(dn, true) < 0) return;

  // ---- PAIR: wait until the partner's half has fully landed in my buffer ---
  if constexpr (PAIR) {
    const uint64_t olen = a.half_len[h ^ 1];
    const uint64_t onch = (olen + C - 1) / C;
    const uint64_t oend = onch < a.c_hi ? onch : a.c_hi;
    for (uint64_t c = a.c_lo + b; c < oend; c += gridDim.x) {
      if (threadIdx.x == 0) {
        const uint64_t tw = tr.p ? globaltimer() : 0;
        wait_ge(a, &mypad->pdown[(uint32_t)(c - a.c_lo)], ep);
        const uint64_t tk = tr.p ? globaltimer() : 0;
        tr.rec((3ull << 60) | ((uint64_t)rank << 48) | c, tw, tk, tk, tk);
      }
    }
  }
  end_epoch(mypad, ep);
}

// ---------------------------------------------------------------------------
// Staging copy (buffers outside peer-mapped memory) and the device barrier.
// ---------------------------------------------------------------------------
// CE schedule's only SM work: fold the n copies of this rank's shard (its own
// slice + the n-1 slices the copy engines pulled into staging) in rank order,
// scale, cast, write the owner's result in place.  Local HBM traffic only.
struct FoldArgs {
  const char* src[kMaxRanks];  // rank-ordered sources
  char* dst;
  uint64_t count;
  float scale;
  int n;
};

template <class E>
__global__ void __launch_bounds__(512) hfr_local_fold_kernel(const FoldArgs f) {
  constexpr int K = E::kPerVec;
  const uint64_t nvec = f.count / K;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nvec; i += stride) {
    float acc[K], t[K];
    E::widen(ld128(f.src[0] + i * 16), acc);
    for (int r = 1; r < f.n; ++r) {
      E::widen(ld128(f.src[r] + i * 16), t);
#pragma unroll
      for (int k = 0; k < K; ++k) acc[k] = __fadd_rn(acc[k], t[k]);
    }
#pragma unroll
    for (int k = 0; k < K; ++k) acc[k] = __fmul_rn(acc[k], f.scale);
    st128(f.dst + i * 16, E::narrow(acc));
  }
  for (uint64_t e = nvec * K + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < f.count; e += stride) {
    float acc = E::load1(f.src[0], e);
    for (int r = 1; r < f.n; ++r) acc = __fadd_rn(acc, E::load1(f.src[r], e));
    E::store1(f.dst, e, __fmul_rn(acc, f.scale));
  }
}

__global__ void __launch_bounds__(1024) hfr_copy_kernel(char* dst, const char* src, uint64_t bytes) {
  const uint64_t nv = bytes / 16;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool aligned = ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0;
  if (aligned) {
    for (uint64_t i = tid; i < nv; i += stride) st128(dst + i * 16, ld128(src + i * 16));
    for (uint64_t i = nv * 16 + tid; i < bytes; i += stride) dst[i] = src[i];
  } else {
    for (uint64_t i = tid; i < bytes; i += stride) dst[i] = src[i];
  }
}

__global__ void hfr_barrier_kernel(const Args a) {
  const int rank = a.rank0 + blockIdx.y;
  const uint64_t e = begin_epoch(a.pad[rank]);
  if (entry_barrier(a, rank, 0, e)) end_epoch(a.pad[rank], e);
}

}  // namespace hfr

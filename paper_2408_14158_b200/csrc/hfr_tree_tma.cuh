// hfr_tree_tma.cuh — subsystem (2), the double binary tree (Algorithm 2,
// PAPER.md:344-370) and "HFReduce with NVLink", moved by
// the TMA engine.
//
// Same schedule, same arithmetic and the same bits as hfr_tree_kernel
// (hfr_kernels.cuh; readings R8-R13): chunk c of a half rides tree c & 1, a
// node combines its children's fp32 partials in order around its own value,
// the root scales and casts once.  What changes is how bytes move and how a
// hand-off is signalled:
//
//  * Flags per TILE (a.tree_tile elements, a power of two dividing the chunk)
//    instead of per chunk, so a parent starts on a tile as soon as that tile
//    of its children has landed (pipeline fill = one tile per CTA, not one
//    128 KiB chunk per CTA).
//  * One producer thread per CTA (warp 0, lane 0) issues everything: bulk
//    copies global -> shared (own x, the pair partner's x, the children's
//    partials) and bulk copies shared -> global into the parent's partial slot
//    or the children's buffers (SASS UBLKCP).  The SM's load/store pipe moves
//    no NVLink bytes.  Warps 1.. fold in shared memory.
//  * A tile's flag is raised when its bulk-store group has COMPLETED
//    (cp.async.bulk.wait_group), keeping the next tile's stores in flight,
//    instead of a system fence that drains every store of the CTA
//    (round 1: the fence wait was as long as the issue).
//  * The producer polls dependencies without blocking, so a tile whose
//    children are late never holds back the stores of a tile that is ready
//    (no cross-rank wait cycle: every blocking wait is CTA-local).
//
// Measured (round 2): slower than the register form at every n
// and dtype (n=4 C2: DBT 404 vs 443 GB/s), so it is the tree_staging = 2
// option, not the default.  A remote tile's completion is observable only by
// a blocking wait_group, so its flag is raised once D newer groups are in
// flight and each parent runs D tiles behind its children.
//
// Stage ring (S stages, one tile each): [X: own x / the final tile][P:
// partner x (PAIR)][C0, C1: children's fp32 partials (or raw 16/8-bit leaf
// values)][O: this node's output (fp32 partial, or the root's final values)].
// full[s]: bulk loads landed (tx count); done[s]: every consumer warp is
// finished with the stage (one arrival per warp per job, compute or not).
#pragma once

#include "hfr_kernels.cuh"

namespace hfr {

constexpr int kTreeStagesMax = 8;
constexpr int kTreeThreads = 128;  // 1 producer warp + 3 fold warps

__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// at most n (< kTreeStagesMax) most recent bulk groups still pending (n must be an immediate)
__device__ __forceinline__ void bulk_wait_n(uint32_t n) {
  switch (n) {
    case 0: asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); break;
    case 1: asm volatile("cp.async.bulk.wait_group 1;" ::: "memory"); break;
    case 2: asm volatile("cp.async.bulk.wait_group 2;" ::: "memory"); break;
    case 3: asm volatile("cp.async.bulk.wait_group 3;" ::: "memory"); break;
    case 4: asm volatile("cp.async.bulk.wait_group 4;" ::: "memory"); break;
    case 5: asm volatile("cp.async.bulk.wait_group 5;" ::: "memory"); break;
    default: asm volatile("cp.async.bulk.wait_group 6;" ::: "memory"); break;
  }
}
// generic-proxy accesses (an acquired flag, plain stores) vs async-proxy ones (bulk copies)
__device__ __forceinline__ void fence_proxy_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// wait for a phase, giving up if the producer aborted (timeout / error)
__device__ __forceinline__ bool mbar_wait_abort(uint64_t* bar, uint32_t parity, volatile int* abort) {
  for (uint32_t it = 0;; ++it) {
    if (mbar_test(bar, parity)) return true;
    if ((it & 255u) == 255u && *abort) return false;
  }
}

// Stage geometry (bytes) of one CTA's role: the regions its jobs use, each
// rounded to 128 B; O (the output) usually aliases an input.  The host sizes the tile so the largest role fits a third
// of the shared-memory budget (tree_tile); a CTA then gets as many stages as
// its own role fits (a DBT leaf, which only copies x, gets 8).
struct TreeStage {
  uint32_t X, P, C0, C1, O, bytes;
  __device__ __forceinline__ TreeStage(uint32_t T, uint32_t esz, bool pair, int nchild, const bool* raw,
                                       bool compute, bool root) {
    auto r128 = [](uint32_t v) { return (v + 127u) & ~127u; };
    uint32_t off = 0;
    X = off;
    off += r128(T * esz);
    P = off;
    if (pair && compute) off += r128(T * esz);
    C0 = off;
    if (nchild > 0) off += r128(raw[0] ? T * esz : 4 * T);
    C1 = off;
    if (nchild > 1) off += r128(raw[1] ? T * esz : 4 * T);
    // The output overwrites an input of the same element size in place (each
    // fold thread reads a unit completely before writing it back): the root's
    // final values over x, a partial over an fp32 child partial, or over fp32
    // x; only a 16/8-bit non-root node with raw (or no) children needs its own.
    O = off;
    if (compute) {
      if (root)
        O = X;
      else if (nchild > 0 && !raw[0])
        O = C0;
      else if (nchild > 1 && !raw[1])
        O = C1;
      else if (esz == 4)
        O = X;
      else
        off += r128(4 * T);
    }
    bytes = off;
  }
};

// 8 consecutive output elements into shared memory (generic stores)
template <class E>
__device__ __forceinline__ void narrow8_generic(uint8_t* p, const float* f) {
  if constexpr (E::kPerVec == 16) {
    *reinterpret_cast<uint2*>(p) = E::narrow8(f);
  } else if constexpr (E::kPerVec == 8) {
    *reinterpret_cast<uint4*>(p) = E::narrow(f);
  } else {
    *reinterpret_cast<uint4*>(p) = E::narrow(f);
    *reinterpret_cast<uint4*>(p + 16) = E::narrow(f + 4);
  }
}

template <class E, bool PAIR>
__global__ void __launch_bounds__(kTreeThreads) hfr_tree_tma_kernel(const Args a) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[kTreeStagesMax], done[kTreeStagesMax];
  __shared__ int s_abort;
  const int rank = a.rank0 + blockIdx.y;
  const int b = blockIdx.x;
  const uint64_t ep = begin_epoch(a.pad[rank]);
  if (!entry_barrier(a, rank, b, ep)) return;

  constexpr uint32_t esz = sizeof(typename E::T);
  constexpr uint32_t V = E::kPerVec;  // elements per 16 B: bulk copies move multiples of V
  const uint32_t T = a.tree_tile;
  const int h = PAIR ? (rank & 1) : 0;
  const int me = PAIR ? (rank >> 1) : rank;
  const int partner = rank ^ 1;
  const int p = b & 1;  // the tree of this CTA: chunk c rides tree c & 1 (R8), CTA b only sees tree b & 1
  const uint64_t G2 = gridDim.x >> 1, m = (uint64_t)(b >> 1);
  const TreeNode nd = a.tree[p][me];
  const bool root = nd.parent < 0;
  const int nchild = nd.nchild;
  // a DBT leaf's partial is its own x: a pure copy (16/8-bit leaves send their
  // raw values, which the parent widens exactly: half the bytes)
  const bool leafcopy = !PAIR && nchild == 0 && !root;
  bool slot_raw[2] = {false, false};
  if constexpr (!PAIR) {
    if (esz < 4)
      for (int sl = 0; sl < nchild; ++sl) slot_raw[sl] = a.tree[p][nd.child[sl]].nchild == 0;
  }
  const bool has_down = !root && (nchild > 0 || PAIR);
  const TreeStage G(T, esz, PAIR, nchild, slot_raw, !leafcopy, root);
  // stages: as many as the role fits into the budget; D bulk-store groups in
  // flight (one stage is being filled, one folded)
  uint32_t S = (uint32_t)a.tree_smem / G.bytes;
  S = S < (uint32_t)kTreeStagesMax ? S : (uint32_t)kTreeStagesMax;
  const uint32_t D = S > 2 ? S - 2 : 1;
  const uint64_t base = a.half_base[h], len = a.half_len[h];
  const uint64_t R = (uint64_t)a.chunk / T;  // tiles per chunk
  Pad* const mypad = a.pad[rank];
  const float* const mypart = a.part[rank];
  const uint64_t stride = a.part_stride;
  auto member = [&](int node) { return PAIR ? 2 * node + h : node; };

  // Tiles of tree p in order: the k-th one and how many lie below tile t.
  auto kth = [&](uint64_t k) { return ((uint64_t)p + 2 * (k / R)) * R + k % R; };
  auto count_below = [&](uint64_t t) {
    const uint64_t rem = t % (2 * R), lo = (uint64_t)p * R;
    const uint64_t part = rem > lo ? (rem - lo < R ? rem - lo : R) : 0;
    return (t / (2 * R)) * R + part;
  };
  // this CTA's tiles of a half of length hlen within the launch's tile range:
  // k = first, first + G2, ... (num of them)
  auto klist = [&](uint64_t hlen, uint64_t* first, uint64_t* num) {
    const uint64_t nt = (hlen + T - 1) / T;
    const uint64_t t1 = nt < a.c_hi ? nt : a.c_hi, t0 = a.c_lo < t1 ? a.c_lo : t1;
    const uint64_t k0 = count_below(t0), k1 = count_below(t1);
    const uint64_t f = k0 + (m + G2 - k0 % G2) % G2;
    *first = f;
    *num = f < k1 ? (k1 - f + G2 - 1) / G2 : 0;
  };
  uint64_t kf, nk;
  klist(len, &kf, &nk);
  const uint64_t NJ = nk + (has_down ? nk : 0);  // up jobs, then down jobs (same tiles)
  struct Job {
    uint64_t t, e0;
    uint32_t L, Lv;
    bool down;
  };
  auto job = [&](uint64_t j) {
    Job J;
    J.down = j >= nk;
    J.t = kth(kf + (J.down ? j - nk : j) * G2);
    J.e0 = J.t * T;
    const uint64_t rest = len - J.e0;
    J.L = rest < T ? (uint32_t)rest : T;
    J.Lv = J.L - J.L % V;
    return J;
  };
  auto is_compute = [&](const Job& J) { return !J.down && !leafcopy; };

  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&done[s], blockDim.x / 32 - 1);
    }
    s_abort = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (threadIdx.x == 0) {
    // ------------------------------------------------------------ producer
    Tracer tr(a);
    uint64_t tq[kTreeStagesMax][3];  // trace: {t_first_poll, t_loaded, t_stored} per stage
    bool plain[kTreeStagesMax];      // the stage's job also wrote with plain stores (ragged end)
    uint64_t loaded = 0, stored = 0, retired = 0;
    uint64_t t_poll = 0;           // first unsuccessful dependency poll of job `loaded`
    uint64_t t_idle = globaltimer();
    bool abort = false;
    auto deps_ready = [&](const Job& J) {
      const uint32_t lc = (uint32_t)(J.t - a.c_lo);
      if (J.down) return ld_acquire_sys(&mypad->down[lc]) >= ep;
      for (int sl = 0; sl < nchild; ++sl)
        if (ld_acquire_sys(&mypad->up[sl][lc]) < ep) return false;
      return true;
    };
    auto issue_loads = [&](const Job& J, uint32_t st) {
      uint8_t* sb = smem + (size_t)st * G.bytes;
      const uint64_t xb = (base + J.e0) * esz;
      const uint32_t xbytes = J.Lv * esz;
      uint32_t tx = 0;
      if (J.Lv) {
        tx += xbytes;
        if (!J.down) {
          if (PAIR) tx += xbytes;
          for (int sl = 0; sl < nchild; ++sl) tx += slot_raw[sl] ? xbytes : J.Lv * 4;
        }
      }
      mbar_expect_tx(&full[st], tx);
      if (!J.Lv) return;
      fence_proxy_global();  // the acquired flags before the bulk reads
      bulk_g2s(sb + G.X, a.buf[rank] + xb, xbytes, &full[st]);
      if (J.down) return;
      if (PAIR) bulk_g2s(sb + G.P, a.buf[partner] + xb, xbytes, &full[st]);
      for (int sl = 0; sl < nchild; ++sl) {
        const char* slot = reinterpret_cast<const char*>(mypart + (uint64_t)sl * stride);
        uint8_t* dst = sb + (sl ? G.C1 : G.C0);
        if (slot_raw[sl])
          bulk_g2s(dst, slot + 4 * J.e0, xbytes, &full[st]);
        else
          bulk_g2s(dst, slot + 4 * J.e0, J.Lv * 4, &full[st]);
      }
    };
    // the ragged end of a half (< V elements): plain loads and stores
    auto remainder = [&](const Job& J) {
      for (uint32_t i = J.Lv; i < J.L; ++i) {
        const uint64_t e = J.e0 + i;
        const uint64_t y = (base + e) * esz;
        if (J.down) {
          for (uint32_t q = 0; q < esz; ++q) {
            const char v = a.buf[rank][y + q];
            for (int k = 0; k < nchild; ++k) a.buf[member(nd.child[k])][y + q] = v;
            if (PAIR) a.buf[partner][y + q] = v;
          }
          continue;
        }
        if (leafcopy) {
          char* slot = reinterpret_cast<char*>(a.part[member(nd.parent)] + (uint64_t)nd.slot * stride);
          for (uint32_t q = 0; q < esz; ++q)
            slot[(esz < 4 ? 4 * J.e0 + (uint64_t)i * esz : 4 * e) + q] = a.buf[rank][y + q];
          continue;
        }
        float xv = E::load1(a.buf[rank], base + e);
        if constexpr (PAIR) {
          const float xp = E::load1(a.buf[partner], base + e);
          xv = h == 0 ? __fadd_rn(xv, xp) : __fadd_rn(xp, xv);
        }
        float acc = 0.f;
        for (int k = 0; k <= nchild; ++k) {
          float s = xv;
          if (k != nd.self_pos) {
            const int sl = k < nd.self_pos ? k : k - 1;
            const float* slot = mypart + (uint64_t)sl * stride;
            s = slot_raw[sl] ? E::load1(reinterpret_cast<const char*>(slot) + 4 * J.e0, i) : slot[e];
          }
          acc = k == 0 ? s : __fadd_rn(acc, s);
        }
        if (root) {
          acc = __fmul_rn(acc, a.scale);
          E::store1(a.buf[rank], base + e, acc);
          for (int k = 0; k < nchild; ++k) E::store1(a.buf[member(nd.child[k])], base + e, acc);
          if (PAIR) E::store1(a.buf[partner], base + e, acc);
        } else {
          (a.part[member(nd.parent)] + (uint64_t)nd.slot * stride)[e] = acc;
        }
      }
    };
    auto issue_stores = [&](const Job& J, uint32_t st) {
      const uint8_t* sb = smem + (size_t)st * G.bytes;
      const uint64_t xb = (base + J.e0) * esz;
      const uint32_t xbytes = J.Lv * esz;
      if (J.Lv) {
        if (J.down) {
          for (int k = 0; k < nchild; ++k) bulk_s2g(a.buf[member(nd.child[k])] + xb, sb + G.X, xbytes);
          if (PAIR) bulk_s2g(a.buf[partner] + xb, sb + G.X, xbytes);
        } else if (root) {
          bulk_s2g(a.buf[rank] + xb, sb + G.O, xbytes);
          for (int k = 0; k < nchild; ++k) bulk_s2g(a.buf[member(nd.child[k])] + xb, sb + G.O, xbytes);
          if (PAIR) bulk_s2g(a.buf[partner] + xb, sb + G.O, xbytes);
        } else {
          char* slot = reinterpret_cast<char*>(a.part[member(nd.parent)] + (uint64_t)nd.slot * stride);
          if (leafcopy)
            bulk_s2g(slot + 4 * J.e0, sb + G.X, xbytes);  // raw (16/8-bit) or fp32 = x itself
          else
            bulk_s2g(slot + 4 * J.e0, sb + G.O, J.Lv * 4);
        }
      }
      plain[st] = J.L > J.Lv;
      remainder(J);
    };
    auto raise = [&](const Job& J) {
      const uint32_t lc = (uint32_t)(J.t - a.c_lo);
      if (!J.down && !root) {
        st_relaxed_sys(&a.pad[member(nd.parent)]->up[nd.slot][lc], ep);
      } else {
        for (int k = 0; k < nchild; ++k) st_relaxed_sys(&a.pad[member(nd.child[k])]->down[lc], ep);
        if (PAIR) st_relaxed_sys(&a.pad[partner]->pdown[lc], ep);
      }
    };
    // Retire jobs [retired, upto): their bulk groups have COMPLETED (the
    // writes are performed at the destination), so the flag store that follows
    // cannot overtake them.  A system fence is needed only to order the plain
    // stores of a ragged end before the flag (round-2 trace: a fence.acq_rel.sys
    // per tile cost ~7 us and cut the TMA tree to 190 GB/s at n=2).
    auto retire_to = [&](uint64_t upto, uint64_t t_waited) {
      bool fence = false;
      for (uint64_t j = retired; j < upto; ++j) fence |= plain[j % S];
      fence_proxy_global();
      if (fence) fence_acq_rel_sys();
      const uint64_t t_fenced = tr.p ? globaltimer() : 0;
      for (; retired < upto; ++retired) {
        const Job J = job(retired);
        raise(J);
        if (tr.p) {
          const uint32_t st = (uint32_t)(retired % S);
          tr.rec(((J.down ? 2ull : 1ull) << 60) | ((uint64_t)rank << 48) | J.t, tq[st][0], tq[st][1], tq[st][2],
                 globaltimer(), t_waited, t_fenced);
        }
      }
    };
    // Event loop.  Every blocking wait here is CTA-local (bulk loads, fold
    // warps, bulk-store completion); dependencies on other ranks are polled,
    // and while the CTA is held up by them every completed tile is retired, so
    // a flag a peer waits for is never held back.
    uint32_t idle = 0;
    while (retired < NJ) {
      bool did = false;
      // (A) loads, as far as the stages and the polled dependencies allow
      while (loaded < NJ && loaded < retired + S) {
        const uint32_t st = (uint32_t)(loaded % S);
        if (loaded >= S && !mbar_test(&done[st], (uint32_t)((loaded / S - 1) & 1))) break;  // fold warps still on it
        const Job J = job(loaded);
        if (tr.p && !t_poll) t_poll = globaltimer();
        if (!deps_ready(J)) break;
        if (tr.p) {
          tq[st][0] = t_poll;
          tq[st][1] = globaltimer();
        }
        t_poll = 0;
        issue_loads(J, st);
        ++loaded;
        did = true;
      }
      // (B) stores of the next job once its stage is ready
      bool stalled = true;
      if (stored < loaded) {
        const uint32_t st = (uint32_t)(stored % S);
        const uint32_t ph = (uint32_t)((stored / S) & 1);
        const Job J = job(stored);
        if (mbar_test(is_compute(J) ? &done[st] : &full[st], ph)) {
          issue_stores(J, st);
          bulk_commit();
          if (tr.p) tq[st][2] = globaltimer();
          ++stored;
          did = true;
          if (stored - retired > D) {  // keep the newest D groups in flight, retire the older ones
            bulk_wait_n(D);
            retire_to(stored - D, tr.p ? globaltimer() : 0);
          }
        }
        stalled = false;  // a loaded job will become ready without any peer
      }
      if (stalled && retired < stored) {  // held up by peers only: release everything
        bulk_wait_0();
        retire_to(stored, tr.p ? globaltimer() : 0);
        did = true;
      }
      if (did) {
        idle = 0;
        t_idle = 0;
      } else if ((++idle & 63u) == 0) {
        const uint64_t now = globaltimer();
        if (!t_idle) t_idle = now;
        if (*a.err != 0) abort = true;
        if (now - t_idle > a.timeout_ns) {
          raise_error(a, kErrTimeout);
          abort = true;
        }
        if (abort) break;
      }
    }
    // the final values this rank receives without forwarding them
    if (!abort && !PAIR && leafcopy) {
      for (uint64_t j = 0; j < nk && !abort; ++j)
        abort = !wait_ge(a, &mypad->down[(uint32_t)(job(j).t - a.c_lo)], ep);
    }
    if (!abort && PAIR) {  // the partner's half
      uint64_t of, on;
      klist(a.half_len[h ^ 1], &of, &on);
      for (uint64_t j = 0; j < on && !abort; ++j)
        abort = !wait_ge(a, &mypad->pdown[(uint32_t)(kth(of + j * G2) - a.c_lo)], ep);
    }
    if (abort) {
      bulk_wait_0();
      s_abort = 1;
    }
  } else if (threadIdx.x >= 32) {
    // ------------------------------------------------------------ fold warps
    const uint32_t ct = threadIdx.x - 32, nct = blockDim.x - 32;
    const int lane = threadIdx.x & 31;
    for (uint64_t j = 0; j < NJ; ++j) {
      const uint32_t st = (uint32_t)(j % S);
      if (!mbar_wait_abort(&full[st], (uint32_t)((j / S) & 1), &s_abort)) break;
      const Job J = job(j);
      if (is_compute(J)) {
        const uint8_t* sb = smem + (size_t)st * G.bytes;
        const uint8_t* X = sb + G.X;
        const uint8_t* P = sb + G.P;
        const uint8_t* C[2] = {sb + G.C0, sb + G.C1};
        uint8_t* O = const_cast<uint8_t*>(sb) + G.O;
        const uint32_t nu = J.Lv / 8;
        for (uint32_t u = ct; u < nu; u += nct) {
          float xv[8], pp[2][8], acc[8];
          widen8_generic<E>(X + (size_t)u * 8 * esz, xv);
          if constexpr (PAIR) {
            float xp[8];
            widen8_generic<E>(P + (size_t)u * 8 * esz, xp);
#pragma unroll
            for (int k = 0; k < 8; ++k) xv[k] = h == 0 ? __fadd_rn(xv[k], xp[k]) : __fadd_rn(xp[k], xv[k]);
          }
#pragma unroll
          for (int sl = 0; sl < 2; ++sl)
            if (sl < nchild) {
              if (slot_raw[sl]) {
                widen8_generic<E>(C[sl] + (size_t)u * 8 * esz, pp[sl]);
              } else {
                const float4 lo = *reinterpret_cast<const float4*>(C[sl] + (size_t)u * 32);
                const float4 hi = *reinterpret_cast<const float4*>(C[sl] + (size_t)u * 32 + 16);
                pp[sl][0] = lo.x, pp[sl][1] = lo.y, pp[sl][2] = lo.z, pp[sl][3] = lo.w;
                pp[sl][4] = hi.x, pp[sl][5] = hi.y, pp[sl][6] = hi.z, pp[sl][7] = hi.w;
              }
            }
          // in-order combination: children below, x_v, children above (R10)
          const int sp = nd.self_pos;
#pragma unroll
          for (int q = 0; q < 8; ++q) acc[q] = sp == 0 ? xv[q] : pp[0][q];
#pragma unroll
          for (int k = 1; k <= 2; ++k) {
            if (k > nchild) break;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const float t = k == sp ? xv[q] : (k < sp ? pp[k][q] : pp[k - 1][q]);
              acc[q] = __fadd_rn(acc[q], t);
            }
          }
          if (root) {
#pragma unroll
            for (int q = 0; q < 8; ++q) acc[q] = __fmul_rn(acc[q], a.scale);
            narrow8_generic<E>(O + (size_t)u * 8 * esz, acc);
          } else {
            *reinterpret_cast<float4*>(O + (size_t)u * 32) = make_float4(acc[0], acc[1], acc[2], acc[3]);
            *reinterpret_cast<float4*>(O + (size_t)u * 32 + 16) = make_float4(acc[4], acc[5], acc[6], acc[7]);
          }
        }
        // Lv % 8 elements (fp32 tiles can end on a 4-element boundary)
        for (uint32_t i = nu * 8 + ct; i < J.Lv; i += nct) {
          float xv = E::load1(reinterpret_cast<const char*>(X), i);
          if constexpr (PAIR) {
            const float xp = E::load1(reinterpret_cast<const char*>(P), i);
            xv = h == 0 ? __fadd_rn(xv, xp) : __fadd_rn(xp, xv);
          }
          float acc = 0.f;
          for (int k = 0; k <= nchild; ++k) {
            float s = xv;
            if (k != nd.self_pos) {
              const int sl = k < nd.self_pos ? k : k - 1;
              s = slot_raw[sl] ? E::load1(reinterpret_cast<const char*>(C[sl]), i)
                               : reinterpret_cast<const float*>(C[sl])[i];
            }
            acc = k == 0 ? s : __fadd_rn(acc, s);
          }
          if (root)
            E::store1(reinterpret_cast<char*>(O), i, __fmul_rn(acc, a.scale));
          else
            reinterpret_cast<float*>(O)[i] = acc;
        }
        fence_proxy_smem();  // my shared-memory writes before the producer's bulk store reads them
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&done[st]);
    }
  }
  __syncthreads();
  if (!s_abort) end_epoch(mypad, ep);
}

}  // namespace hfr

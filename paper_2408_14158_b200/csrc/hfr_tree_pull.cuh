// hfr_tree_pull.cuh — subsystem (2), the double binary tree (Algorithm 2,
// PAPER.md:344-370) and "HFReduce with NVLink", with every
// NVLink transfer a bulk-copy READ (tree_staging = 3).
//
// Same schedule and bits as the push kernels (hfr_tree_kernel,
// hfr_tree_tma_kernel): chunk c rides tree c & 1 (R8), in-order combination
// (R10), one scale + cast at the root.  The data flow is inverted:
//  * up: a node PULLS its children's contributions — a DBT leaf child's x
//    straight from the child's buffer (ready at kernel entry: leaves do no
//    up-pass work at all and raise no flags), an interior child's fp32
//    partial from the child's own scratch slot once the child's up flag
//    shows it — folds them with its own x (and the pair partner's x, pulled
//    too) and writes its partial into its OWN slot (or, at the root, the
//    final values into its own buffer);
//  * down: a node pulls the final tile from its parent's buffer into its own;
//    PAIR: each member also pulls the partner's half.
// Every store is local, so a tile's bulk-store group completes at local-HBM
// latency and its flag (in the writer's own pad, polled over NVLink by the
// readers) follows at once; the remote traffic is bulk loads, whose
// completion an mbarrier reports per tile.  The push form's weakness — a
// remote tile's completion is only observable once D newer bulk groups are
// issued (round-2 traces) — does not arise.  Sources must outlive their
// readers: an exit handshake (CTA b with CTA b of every rank; every tile is
// served by the same CTA index on every rank) ends the kernel.
#pragma once

#include "hfr_tree_tma.cuh"

namespace hfr {

template <class E, bool PAIR>
__global__ void __launch_bounds__(kTreeThreads) hfr_tree_pull_kernel(const Args a) {
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
  const int p = b & 1;  // the tree of this CTA (R8)
  const uint64_t G2 = gridDim.x >> 1, m = (uint64_t)(b >> 1);
  const TreeNode nd = a.tree[p][me];
  const bool root = nd.parent < 0;
  const int nchild = nd.nchild;
  auto member = [&](int node) { return PAIR ? 2 * node + h : node; };
  auto dbt_leaf = [&](int node) { return !PAIR && a.tree[p][node].nchild == 0 && a.tree[p][node].parent >= 0; };
  const bool leaf = dbt_leaf(me);  // no up-pass work: the parent pulls this rank's x
  // child data in the stage: a DBT leaf child's raw x (E), else its fp32 partial
  bool raw[2] = {false, false};
  for (int sl = 0; sl < nchild; ++sl) raw[sl] = dbt_leaf(nd.child[sl]);
  const TreeStage G(T, esz, PAIR, nchild, raw, !leaf, root);
  uint32_t S = (uint32_t)a.tree_smem / G.bytes;
  S = S < (uint32_t)kTreeStagesMax ? S : (uint32_t)kTreeStagesMax;
  const uint32_t D = S > 2 ? S - 2 : 1;
  const uint64_t base = a.half_base[h], len = a.half_len[h];
  const uint64_t obase = a.half_base[h ^ 1], olen = a.half_len[h ^ 1];
  const uint64_t R = (uint64_t)a.chunk / T;  // tiles per chunk
  Pad* const mypad = a.pad[rank];
  const uint64_t stride = a.part_stride;
  (void)stride;

  auto kth = [&](uint64_t k) { return ((uint64_t)p + 2 * (k / R)) * R + k % R; };
  auto count_below = [&](uint64_t t) {
    const uint64_t rem = t % (2 * R), lo = (uint64_t)p * R;
    const uint64_t part = rem > lo ? (rem - lo < R ? rem - lo : R) : 0;
    return (t / (2 * R)) * R + part;
  };
  auto klist = [&](uint64_t hlen, uint64_t* first, uint64_t* num) {
    const uint64_t nt = (hlen + T - 1) / T;
    const uint64_t t1 = nt < a.c_hi ? nt : a.c_hi, t0 = a.c_lo < t1 ? a.c_lo : t1;
    const uint64_t k0 = count_below(t0), k1 = count_below(t1);
    const uint64_t f = k0 + (m + G2 - k0 % G2) % G2;
    *first = f;
    *num = f < k1 ? (k1 - f + G2 - 1) / G2 : 0;
  };
  uint64_t kf, nk, okf = 0, onk = 0;
  klist(len, &kf, &nk);
  if (PAIR) klist(olen, &okf, &onk);
  // jobs: [UP x n_up][DOWN x n_dn][PAIRW x n_pw]
  const uint64_t n_up = leaf ? 0 : nk, n_dn = root ? 0 : nk, n_pw = PAIR ? onk : 0;
  const uint64_t NJ = n_up + n_dn + n_pw;
  enum { UP = 0, DOWN = 1, PAIRW = 2 };
  struct Job {
    uint64_t t, e0, hb;  // tile (within its half), element offset within the half, the half's base
    uint32_t L, Lv;
    int kind;
  };
  auto job = [&](uint64_t j) {
    Job J;
    uint64_t k;
    uint64_t hl;
    if (j < n_up) {
      J.kind = UP, k = kf + j * G2, J.hb = base, hl = len;
    } else if (j < n_up + n_dn) {
      J.kind = DOWN, k = kf + (j - n_up) * G2, J.hb = base, hl = len;
    } else {
      J.kind = PAIRW, k = okf + (j - n_up - n_dn) * G2, J.hb = obase, hl = olen;
    }
    J.t = kth(k);
    J.e0 = J.t * T;
    const uint64_t rest = hl - J.e0;
    J.L = rest < T ? (uint32_t)rest : T;
    J.Lv = J.L - J.L % V;
    return J;
  };

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
    uint64_t tq[kTreeStagesMax][3];
    bool plain[kTreeStagesMax];
    uint64_t loaded = 0, stored = 0, retired = 0;
    uint64_t t_poll = 0, t_idle = globaltimer();
    bool abort = false;
    auto child_src = [&](int sl) -> const char* {  // where child sl's contribution lives
      const int cr = member(nd.child[sl]);
      return raw[sl] ? a.buf[cr] : reinterpret_cast<const char*>(a.part[cr]);
    };
    auto deps_ready = [&](const Job& J) {
      const uint32_t lc = (uint32_t)(J.t - a.c_lo);
      if (J.kind == DOWN) return ld_acquire_sys(&a.pad[member(nd.parent)]->down[lc]) >= ep;
      if (J.kind == PAIRW) return ld_acquire_sys(&a.pad[partner]->down[lc]) >= ep;
      for (int sl = 0; sl < nchild; ++sl)
        if (!raw[sl] && ld_acquire_sys(&a.pad[member(nd.child[sl])]->up[0][lc]) < ep) return false;
      return true;
    };
    auto issue_loads = [&](const Job& J, uint32_t st) {
      uint8_t* sb = smem + (size_t)st * G.bytes;
      const uint64_t xb = (J.hb + J.e0) * esz;
      const uint32_t xbytes = J.Lv * esz;
      uint32_t tx = 0;
      if (J.Lv) {
        tx += xbytes;
        if (J.kind == UP) {
          if (PAIR) tx += xbytes;
          for (int sl = 0; sl < nchild; ++sl) tx += raw[sl] ? xbytes : J.Lv * 4;
        }
      }
      mbar_expect_tx(&full[st], tx);
      if (!J.Lv) return;
      fence_proxy_global();  // the acquired flags before the bulk reads
      if (J.kind == DOWN) {
        bulk_g2s(sb + G.X, a.buf[member(nd.parent)] + xb, xbytes, &full[st]);
        return;
      }
      if (J.kind == PAIRW) {
        bulk_g2s(sb + G.X, a.buf[partner] + xb, xbytes, &full[st]);
        return;
      }
      bulk_g2s(sb + G.X, a.buf[rank] + xb, xbytes, &full[st]);
      if (PAIR) bulk_g2s(sb + G.P, a.buf[partner] + xb, xbytes, &full[st]);
      for (int sl = 0; sl < nchild; ++sl) {
        uint8_t* dst = sb + (sl ? G.C1 : G.C0);
        if (raw[sl])
          bulk_g2s(dst, child_src(sl) + xb, xbytes, &full[st]);
        else
          bulk_g2s(dst, child_src(sl) + 4 * J.e0, J.Lv * 4, &full[st]);
      }
    };
    // the ragged end of a half (< V elements): plain loads and stores
    auto remainder = [&](const Job& J) {
      for (uint32_t i = J.Lv; i < J.L; ++i) {
        const uint64_t e = J.e0 + i;
        const uint64_t y = (J.hb + e) * esz;
        if (J.kind != UP) {
          const char* src = J.kind == DOWN ? a.buf[member(nd.parent)] : a.buf[partner];
          for (uint32_t q = 0; q < esz; ++q) a.buf[rank][y + q] = src[y + q];
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
            s = raw[sl] ? E::load1(child_src(sl), base + e) : reinterpret_cast<const float*>(child_src(sl))[e];
          }
          acc = k == 0 ? s : __fadd_rn(acc, s);
        }
        if (root)
          E::store1(a.buf[rank], base + e, __fmul_rn(acc, a.scale));
        else
          a.part[rank][e] = acc;
      }
    };
    auto issue_stores = [&](const Job& J, uint32_t st) {  // all local
      const uint8_t* sb = smem + (size_t)st * G.bytes;
      const uint64_t xb = (J.hb + J.e0) * esz;
      const uint32_t xbytes = J.Lv * esz;
      if (J.Lv) {
        if (J.kind != UP)
          bulk_s2g(a.buf[rank] + xb, sb + G.X, xbytes);
        else if (root)
          bulk_s2g(a.buf[rank] + xb, sb + G.O, xbytes);
        else
          bulk_s2g(reinterpret_cast<char*>(a.part[rank]) + 4 * J.e0, sb + G.O, J.Lv * 4);
      }
      plain[st] = J.L > J.Lv;
      remainder(J);
    };
    auto raise = [&](const Job& J) {  // flags in my own pad, polled by the readers
      const uint32_t lc = (uint32_t)(J.t - a.c_lo);
      if (J.kind == UP && !root)
        st_relaxed_sys(&mypad->up[0][lc], ep);
      else if ((J.kind == UP && root) || (J.kind == DOWN && (nchild > 0 || PAIR)))
        st_relaxed_sys(&mypad->down[lc], ep);
    };
    // a completed local bulk store is in this GPU's memory (L2) before the flag
    // store is issued; readers poll the flag and then read through the same L2
    auto retire_to = [&](uint64_t upto) {
      bool fence = false;
      for (uint64_t j = retired; j < upto; ++j) fence |= plain[j % S];
      fence_proxy_global();
      if (fence) fence_acq_rel_sys();
      for (; retired < upto; ++retired) {
        const Job J = job(retired);
        raise(J);
        if (tr.p) {
          const uint32_t st = (uint32_t)(retired % S);
          tr.rec(((uint64_t)(J.kind + 1) << 60) | ((uint64_t)rank << 48) | J.t, tq[st][0], tq[st][1], tq[st][2],
                 globaltimer());
        }
      }
    };
    uint32_t idle = 0;
    while (retired < NJ) {
      bool did = false;
      while (loaded < NJ && loaded < retired + S) {
        const uint32_t st = (uint32_t)(loaded % S);
        if (loaded >= S && !mbar_test(&done[st], (uint32_t)((loaded / S - 1) & 1))) break;
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
      bool stalled = true;
      if (stored < loaded) {
        const uint32_t st = (uint32_t)(stored % S);
        const uint32_t ph = (uint32_t)((stored / S) & 1);
        const Job J = job(stored);
        if (mbar_test(J.kind == UP ? &done[st] : &full[st], ph)) {
          issue_stores(J, st);
          bulk_commit();
          if (tr.p) tq[st][2] = globaltimer();
          ++stored;
          did = true;
          if (stored - retired > D) {
            bulk_wait_n(D);
            retire_to(stored - D);
          }
        }
        stalled = false;
      }
      if (stalled && retired < stored) {
        bulk_wait_0();
        retire_to(stored);
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
    bulk_wait_0();
    if (abort) s_abort = 1;
  } else if (threadIdx.x >= 32) {
    // ------------------------------------------------------------ fold warps
    const uint32_t ct = threadIdx.x - 32, nct = blockDim.x - 32;
    const int lane = threadIdx.x & 31;
    for (uint64_t j = 0; j < NJ; ++j) {
      const uint32_t st = (uint32_t)(j % S);
      if (!mbar_wait_abort(&full[st], (uint32_t)((j / S) & 1), &s_abort)) break;
      if (j < n_up) {
        const Job J = job(j);
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
              if (raw[sl]) {
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
              s = raw[sl] ? E::load1(reinterpret_cast<const char*>(C[sl]), i)
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
  if (s_abort) return;
  // sources outlive their readers: every tile this CTA index serves is read by
  // the same CTA index of the other ranks
  exit_barrier(a, rank, b, ep);
  end_epoch(mypad, ep);
}

}  // namespace hfr

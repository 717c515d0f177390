// p2p_probe.cu — NVLink microbenchmark (one process, n GPUs, peer access):
// what per-direction bandwidth do SM-driven remote loads, remote stores and
// their mix reach on this box, and what does a per-chunk system fence (the
// tree schedule's handoff) cost?  Used to choose the transfer style of the
// HFReduce kernels.  No cross-GPU waits: every kernel only
// moves data, so concurrent launches on several GPUs are safe.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o p2p_probe tools/p2p_probe.cu
//   ./p2p_probe <ngpus> <MiB per peer> <ctas> <threads> [fence_chunk_KiB]
//
// Every thread interleaves all peers (vector i of every peer segment before
// vector i+stride), so no GPU is a hotspot.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) {                                                          \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                        \
    }                                                                                 \
  } while (0)

struct Ptrs {
  const uint4* src[16];
  uint4* dst[16];
  unsigned long long* flag;  // per-chunk handoff target (fence mode)
  int n;
};

// vector i of every segment k (k-inner), U vectors in flight per segment
template <int U>
__global__ void __launch_bounds__(512) move(Ptrs p, uint64_t nvec) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nvec; i += U * stride) {
    for (int k = 0; k < p.n; ++k) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (i + u * stride < nvec) v[u] = p.src[k][i + u * stride];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (i + u * stride < nvec) p.dst[k][i + u * stride] = v[u];
    }
  }
}

// chunked: CTA b moves contiguous chunks of `cvec` vectors of every segment;
// after each chunk: __syncthreads, thread 0 fence.acq_rel.sys + flag store
// (exactly the tree kernel's per-chunk handoff).
__global__ void __launch_bounds__(512) move_fenced(Ptrs p, uint64_t nvec, uint64_t cvec) {
  const uint64_t nchunks = (nvec + cvec - 1) / cvec;
  for (uint64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const uint64_t lo = c * cvec, hi = lo + cvec < nvec ? lo + cvec : nvec;
    for (int k = 0; k < p.n; ++k) {
      for (uint64_t i = lo + threadIdx.x; i < hi; i += 4 * blockDim.x) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (i + u * blockDim.x < hi) v[u] = p.src[k][i + u * blockDim.x];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (i + u * blockDim.x < hi) p.dst[k][i + u * blockDim.x] = v[u];
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("fence.acq_rel.sys;" ::: "memory");
      asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p.flag + blockIdx.x), "l"((unsigned long long)c) : "memory");
    }
  }
}

// TMA (bulk-copy) forms: one thread per CTA issues cp.async.bulk copies of
// `chunk` bytes.  push: shared -> peer global (the same shared bytes every
// time: this measures the link, not a local read), at most 8 groups in
// flight; pull: peer global -> shared into an 8-stage ring tracked by
// mbarriers.  mixed: even CTAs push, odd CTAs pull (half the bytes each).
__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void __launch_bounds__(32) tma_move(Ptrs p, uint64_t bytes, uint32_t chunk, int mode) {
  extern __shared__ __align__(128) uint8_t buf[];  // 8 * chunk
  __shared__ __align__(8) uint64_t bar[8];
  if (threadIdx.x != 0) return;
  const bool push = mode == 0 || (mode == 2 && (blockIdx.x & 1) == 0);
  const uint64_t G = mode == 2 ? gridDim.x / 2 : gridDim.x, b = mode == 2 ? blockIdx.x / 2 : blockIdx.x;
  for (int s = 0; s < 8; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  uint64_t j = 0;
  const uint64_t lo = mode == 2 ? (push ? 0 : bytes / 2) : 0, hi = mode == 2 ? (push ? bytes / 2 : bytes) : bytes;
  for (uint64_t off = lo + b * chunk; off + chunk <= hi; off += G * chunk)
    for (int k = 0; k < p.n; ++k, ++j) {
      if (push) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"((char*)p.dst[k] + off),
                     "r"(s32(buf)), "r"(chunk) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group 8;" ::: "memory");
      } else {
        const uint32_t st = j & 7;
        if (j >= 8) {
          const uint32_t ph = (uint32_t)(((j >> 3) - 1) & 1);
          asm volatile("{\n .reg .pred q;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n @!q bra W_%=;\n}"
                       ::"r"(s32(&bar[st])), "r"(ph) : "memory");
        }
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&bar[st])), "r"(chunk) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(s32(buf + (size_t)st * chunk)), "l"((const char*)p.src[k] + off), "r"(chunk), "r"(s32(&bar[st]))
                     : "memory");
      }
    }
  if (push) {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  } else {
    for (uint64_t q = j > 8 ? j - 8 : 0; q < j; ++q) {
      const uint32_t st = q & 7, ph = (uint32_t)((q >> 3) & 1);
      asm volatile("{\n .reg .pred q;\n V_%=:\n mbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n @!q bra V_%=;\n}"
                   ::"r"(s32(&bar[st])), "r"(ph) : "memory");
    }
  }
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 2;
  const size_t mib = argc > 2 ? atol(argv[2]) : 64;
  const int ctas = argc > 3 ? atoi(argv[3]) : 148;
  const int threads = argc > 4 ? atoi(argv[4]) : 512;
  const size_t fence_kib = argc > 5 ? atol(argv[5]) : 0;
  const size_t bytes = mib << 20;
  const uint64_t nvec = bytes / 16;
  uint4 *local[8], *inbox[8];  // inbox[g] holds n slots of `bytes` (one per peer)
  unsigned long long* flags[8];
  cudaStream_t st[8];
  cudaEvent_t e0[8], e1[8];
  for (int g = 0; g < n; ++g) {
    CK(cudaSetDevice(g));
    for (int h = 0; h < n; ++h)
      if (h != g) {
        cudaError_t pe = cudaDeviceEnablePeerAccess(h, 0);
        if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) CK(pe);
        cudaGetLastError();
      }
    CK(cudaMalloc(&local[g], bytes * n));
    CK(cudaMalloc(&inbox[g], bytes * n));
    CK(cudaMalloc(&flags[g], 8 * 4096));
    CK(cudaMemset(local[g], 1, bytes * n));
    CK(cudaMemset(inbox[g], 2, bytes * n));
    CK(cudaStreamCreateWithFlags(&st[g], cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0[g]));
    CK(cudaEventCreate(&e1[g]));
  }
  const char* names[] = {"read  (pull from peers)", "write (push to peers)", "mixed (pull half, push half)",
                         "read  one-way (GPU0 only)", "write one-way (GPU0 only)",
                         "fan-in read (peers read GPU0)", "fan-in write (peers write GPU0)",
                         "reduce pattern (root GPU0)", "root read+write only (GPU0)",
                         "owner reads + push to root", "root pushes + owner reads",
                         "tma push (bulk copies to peers)", "tma pull (bulk copies from peers)",
                         "tma mixed (half push, half pull)"};
  // modes 5-7 run on GPUs 1..n-1 only and load GPU0's port: 5/6 every peer
  // reads/writes `bytes` at GPU0; 7 is the reduce collective's traffic —
  // every non-root GPU reads a segment from each other GPU (root included)
  // and writes one segment to the root.  GB/s is GPU0's egress (5, 7) or
  // ingress (6, 7).  8-10 split mode 7: 8 = peers read GPU0 and write GPU0
  // (no peer-peer reads); 9 = peers read each other (not GPU0) and write GPU0;
  // 10 = 9 plus GPU0 pushing a segment to every peer.
  const uint32_t tchunk = 8192;
  for (int g = 0; g < n; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaFuncSetAttribute(tma_move, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * tchunk));
  }
  for (int mode = 0; mode < 14; ++mode) {
    if (fence_kib && mode != 1) continue;
    for (int rep = 0; rep < 3; ++rep) {
      for (int g = 0; g < n; ++g) {
        if ((mode == 3 || mode == 4) && g != 0) continue;
        if (mode >= 5 && mode <= 9 && g == 0) continue;
        CK(cudaSetDevice(g));
        Ptrs p{};
        p.n = 0;
        p.flag = flags[(g + 1) % n];
        uint64_t per = nvec;
        for (int h = 0; h < n; ++h) {
          if (h == g || ((mode == 5 || mode == 6 || mode == 8) && h != 0)) continue;
          if ((mode == 9 || mode == 10) && h == 0) continue;
          if (mode == 10 && g == 0) {  // the root pushes its segment to peer h
            p.src[p.n] = local[0] + (size_t)h * nvec;
            p.dst[p.n++] = inbox[h] + (size_t)0 * nvec;
            continue;
          }
          uint4* peer_slot = inbox[h] + (size_t)g * nvec;
          uint4* my_slot = local[g] + (size_t)h * nvec;
          if (mode >= 11) {  // TMA forms: pull from the peer's slot, push into it
            p.src[p.n] = peer_slot; p.dst[p.n++] = peer_slot;
          } else if (mode == 0 || mode == 3 || mode == 5 || mode == 7 || mode == 8 || mode == 9 || mode == 10) {
            p.src[p.n] = peer_slot; p.dst[p.n++] = my_slot;
          } else if (mode == 1 || mode == 4 || mode == 6) {
            p.src[p.n] = my_slot; p.dst[p.n++] = peer_slot;
          } else {
            per = nvec / 2;
            p.src[p.n] = peer_slot; p.dst[p.n++] = my_slot;
            p.src[p.n] = my_slot + per; p.dst[p.n++] = peer_slot + per;
          }
        }
        if (mode >= 7 && mode <= 10 && g != 0) {  // + the owner's result segment, pushed to the root
          p.src[p.n] = local[g] + (size_t)g * nvec;
          p.dst[p.n++] = inbox[0] + (size_t)g * nvec;
        }
        CK(cudaEventRecord(e0[g], st[g]));
        if (mode >= 11)
          tma_move<<<2 * ctas, 32, 8 * tchunk, st[g]>>>(p, bytes, tchunk, mode - 11);
        else if (fence_kib)
          move_fenced<<<ctas, threads, 0, st[g]>>>(p, per, (fence_kib << 10) / 16 / p.n);
        else
          move<4><<<ctas, threads, 0, st[g]>>>(p, per);
        CK(cudaGetLastError());
        CK(cudaEventRecord(e1[g], st[g]));
      }
      float worst = 0;
      for (int g = 0; g < n; ++g) {
        if ((mode == 3 || mode == 4) && g != 0) continue;
        if (mode >= 5 && mode <= 9 && g == 0) continue;
        CK(cudaSetDevice(g));
        CK(cudaEventSynchronize(e1[g]));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0[g], e1[g]));
        if (ms > worst) worst = ms;
      }
      const double per_dir = (double)bytes * (n - 1);
      if (rep == 2)
        printf("n=%d %-30s %5zu MiB/peer ctas=%3d thr=%d fence_chunk=%zuKiB: %8.3f ms -> %6.1f GB/s per GPU per direction\n",
               n, names[mode], mib, ctas, threads, fence_kib, worst, per_dir / worst / 1e6);
    }
  }
  return 0;
}

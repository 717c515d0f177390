// p2p_probe.cu — NVLink microbenchmark (one process, n GPUs, peer access):
// what per-direction bandwidth do SM-driven remote loads, remote stores and
// their mix reach on this box?  Used to choose the transfer style of the
// HFReduce kernels.  No cross-GPU waits: every kernel only
// moves data, so concurrent launches on several GPUs are safe.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o p2p_probe tools/p2p_probe.cu
//   ./p2p_probe <ngpus> <MiB per peer> <ctas> <threads>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e = (x);                                                              \
    if (e != cudaSuccess) {                                                           \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
      exit(1);                                                                        \
    }                                                                                 \
  } while (0)

struct Ptrs {
  const uint4* src[16];
  uint4* dst[16];
  int n;
};

// each CTA grid-strides over all peers' segments: vector i of segment p
// copies src[p][i] -> dst[p][i]
template <int U>
__global__ void __launch_bounds__(512) move(Ptrs p, uint64_t nvec) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (int k = 0; k < p.n; ++k) {
    const uint4* s = p.src[k];
    uint4* d = p.dst[k];
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nvec; i += U * stride) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (i + u * stride < nvec) v[u] = s[i + u * stride];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (i + u * stride < nvec) d[i + u * stride] = v[u];
    }
  }
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 2;
  const size_t mib = argc > 2 ? atol(argv[2]) : 64;
  const int ctas = argc > 3 ? atoi(argv[3]) : 148;
  const int threads = argc > 4 ? atoi(argv[4]) : 512;
  const size_t bytes = mib << 20;
  const uint64_t nvec = bytes / 16;
  uint4 *local[8], *inbox[8];  // inbox[g] holds n slots of `bytes` (one per peer)
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
    CK(cudaMemset(local[g], 1, bytes * n));
    CK(cudaMemset(inbox[g], 2, bytes * n));
    CK(cudaStreamCreateWithFlags(&st[g], cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0[g]));
    CK(cudaEventCreate(&e1[g]));
  }
  const char* names[] = {"read  (pull from peers)", "write (push to peers)", "mixed (pull half, push half)",
                         "read  one-way (GPU0 only)", "write one-way (GPU0 only)"};
  for (int mode = 0; mode < 5; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {
      for (int g = 0; g < n; ++g) {
        if (mode >= 3 && g != 0) continue;
        CK(cudaSetDevice(g));
        Ptrs p{};
        p.n = 0;
        uint64_t per = nvec;
        for (int h = 0; h < n; ++h) {
          if (h == g) continue;
          uint4* peer_slot = inbox[h] + (size_t)g * nvec;
          uint4* my_slot = local[g] + (size_t)h * nvec;
          if (mode == 0 || mode == 3) {  // pull: read peer, write local
            p.src[p.n] = peer_slot; p.dst[p.n++] = my_slot;
          } else if (mode == 1 || mode == 4) {  // push: read local, write peer
            p.src[p.n] = my_slot; p.dst[p.n++] = peer_slot;
          } else {  // mixed: pull the first half, push the second half
            per = nvec / 2;
            p.src[p.n] = peer_slot; p.dst[p.n++] = my_slot;
            p.src[p.n] = my_slot + per; p.dst[p.n++] = peer_slot + per;
          }
        }
        CK(cudaEventRecord(e0[g], st[g]));
        move<4><<<ctas, threads, 0, st[g]>>>(p, per);
        CK(cudaEventRecord(e1[g], st[g]));
      }
      float worst = 0;
      for (int g = 0; g < n; ++g) {
        if (mode >= 3 && g != 0) continue;
        CK(cudaSetDevice(g));
        CK(cudaEventSynchronize(e1[g]));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0[g], e1[g]));
        if (ms > worst) worst = ms;
      }
      // bytes entering one GPU over NVLink (== leaving, by symmetry)
      const double per_dir = (double)bytes * (n - 1);
      if (rep == 2)
        printf("n=%d %-30s %5zu MiB/peer ctas=%3d thr=%d: %8.3f ms -> %6.1f GB/s per GPU per direction\n", n,
               names[mode], mib, ctas, threads, worst, per_dir / worst / 1e6);
    }
  }
  return 0;
}

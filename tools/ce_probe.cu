// ce_probe.cu — copy-engine (cudaMemcpyAsync peer) bandwidth on this box:
// every GPU moves `MiB` to/from each peer at once, split over `k` streams per
// peer, pulling (dst local, src peer) or pushing (src local, dst peer).  Tells
// how fast the CE schedule (algo CE, "no GPU kernel") can be.
//
//   nvcc -O3 -o ce_probe tools/ce_probe.cu && ./ce_probe <ngpus> <MiB per peer> <k streams per peer>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                                             \
  do {                                                                                    \
    cudaError_t e_ = (x);                                                                 \
    if (e_ != cudaSuccess) {                                                              \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                            \
    }                                                                                     \
  } while (0)

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 4;
  const size_t bytes = (size_t)(argc > 2 ? atol(argv[2]) : 256) << 20;
  const int k = argc > 3 ? atoi(argv[3]) : 1;
  char *src[8], *dst[8];
  cudaStream_t st[8][64];
  cudaEvent_t e0[8], e1[8], ej[8][64];
  for (int g = 0; g < n; ++g) {
    CK(cudaSetDevice(g));
    for (int h = 0; h < n; ++h)
      if (h != g) {
        cudaError_t pe = cudaDeviceEnablePeerAccess(h, 0);
        if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) CK(pe);
        cudaGetLastError();
      }
    CK(cudaMalloc(&src[g], bytes * n));
    CK(cudaMalloc(&dst[g], bytes * n));
    CK(cudaMemset(src[g], 1, bytes * n));
    for (int s = 0; s < (n - 1) * k; ++s) {
      CK(cudaStreamCreateWithFlags(&st[g][s], cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&ej[g][s], cudaEventDisableTiming));
    }
    CK(cudaEventCreate(&e0[g]));
    CK(cudaEventCreate(&e1[g]));
  }
  int asyncEngines = 0;
  CK(cudaDeviceGetAttribute(&asyncEngines, cudaDevAttrAsyncEngineCount, 0));
  for (int push = 0; push < 2; ++push) {
    for (int rep = 0; rep < 3; ++rep) {
      for (int g = 0; g < n; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaEventRecord(e0[g], st[g][0]));
        int s = 0;
        for (int h = 0; h < n; ++h) {
          if (h == g) continue;
          const size_t piece = bytes / k;
          for (int j = 0; j < k; ++j, ++s) {
            if (s) CK(cudaStreamWaitEvent(st[g][s], e0[g], 0));
            char* d = push ? dst[h] + (size_t)g * bytes + j * piece : dst[g] + (size_t)h * bytes + j * piece;
            const char* c = push ? src[g] + (size_t)h * bytes + j * piece : src[h] + (size_t)g * bytes + j * piece;
            CK(cudaMemcpyAsync(d, c, piece, cudaMemcpyDeviceToDevice, st[g][s]));
            if (s) {
              CK(cudaEventRecord(ej[g][s], st[g][s]));
              CK(cudaStreamWaitEvent(st[g][0], ej[g][s], 0));
            }
          }
        }
        CK(cudaEventRecord(e1[g], st[g][0]));
      }
      float worst = 0;
      for (int g = 0; g < n; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaEventSynchronize(e1[g]));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0[g], e1[g]));
        if (ms > worst) worst = ms;
      }
      if (rep == 2)
        printf("n=%d CE %-4s %4zu MiB/peer k=%2d streams/peer (async engines %d): %8.3f ms -> %6.1f GB/s per GPU per direction\n",
               n, push ? "push" : "pull", bytes >> 20, k, asyncEngines, worst, (double)bytes * (n - 1) / worst / 1e6);
    }
  }
  return 0;
}

// hfr_nvls.cuh — NVLink SHARP (NVLS) multicast arena and the order-relaxed
// NVLS schedule (included by hfr_runtime.cu).
//
// Host side: a per-comm arena of physical memory created with cuMemCreate on
// every rank and bound to ONE multicast object (cuMulticastCreate on rank 0,
// imported by the others), mapped three ways: the local unicast VA, every
// peer's unicast VA (so the bit-exact schedules also run zero-copy on it) and
// the multicast VA used by multimem instructions.  POSIX file descriptors of
// the multicast object and of each rank's physical allocation travel between
// the processes over an abstract-namespace Unix socket (SCM_RIGHTS); the
// rendezvous token goes through the caller's all-gather callback.  Driver
// entry points are resolved with cudaGetDriverEntryPoint (no libcuda link).
//
// Device side (hfr_nvls_kernel in hfr_kernels.cuh): rank g owns shard g; for
// each 16 B of it one multimem.ld_reduce returns the sum over all n GPUs
// computed in the NVSwitch (fp32, or bf16 with .acc::f32), the owner scales
// it, and one multimem.st writes it to all n GPUs.  Per direction a GPU moves
// about (n+1)/n * S instead of 2(n-1)/n * S, but the switch chooses the
// summation order: results are ORDER-RELAXED, held to reading R18's bound,
// not bit-exact.
#pragma once

#include <cuda.h>
#include <sys/socket.h>
#include <sys/un.h>
#include <unistd.h>

#include <random>

namespace {

struct DrvApi {
  CUresult (*DeviceGet)(CUdevice*, int) = nullptr;
  CUresult (*DeviceGetAttribute)(int*, CUdevice_attribute, CUdevice) = nullptr;
  CUresult (*MulticastCreate)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*) = nullptr;
  CUresult (*MulticastAddDevice)(CUmemGenericAllocationHandle, CUdevice) = nullptr;
  CUresult (*MulticastBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                               unsigned long long) = nullptr;
  CUresult (*MulticastUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t) = nullptr;
  CUresult (*MulticastGetGranularity)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags) = nullptr;
  CUresult (*MemCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long) = nullptr;
  CUresult (*MemRelease)(CUmemGenericAllocationHandle) = nullptr;
  CUresult (*MemMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
  CUresult (*MemUnmap)(CUdeviceptr, size_t) = nullptr;
  CUresult (*MemAddressReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
  CUresult (*MemAddressFree)(CUdeviceptr, size_t) = nullptr;
  CUresult (*MemSetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
  CUresult (*MemExportToShareableHandle)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType,
                                         unsigned long long) = nullptr;
  CUresult (*MemImportFromShareableHandle)(CUmemGenericAllocationHandle*, void*, CUmemAllocationHandleType) = nullptr;
  CUresult (*MemGetAllocationGranularity)(size_t*, const CUmemAllocationProp*,
                                          CUmemAllocationGranularity_flags) = nullptr;
};

bool load_drv(DrvApi* d) {
  bool ok = true;
  auto get = [&](const char* name, auto** fp) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &f, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess) {
      ok = false;
      return;
    }
    *fp = reinterpret_cast<std::remove_pointer_t<decltype(fp)>>(f);
  };
  get("cuDeviceGet", &d->DeviceGet);
  get("cuDeviceGetAttribute", &d->DeviceGetAttribute);
  get("cuMulticastCreate", &d->MulticastCreate);
  get("cuMulticastAddDevice", &d->MulticastAddDevice);
  get("cuMulticastBindMem", &d->MulticastBindMem);
  get("cuMulticastUnbind", &d->MulticastUnbind);
  get("cuMulticastGetGranularity", &d->MulticastGetGranularity);
  get("cuMemCreate", &d->MemCreate);
  get("cuMemRelease", &d->MemRelease);
  get("cuMemMap", &d->MemMap);
  get("cuMemUnmap", &d->MemUnmap);
  get("cuMemAddressReserve", &d->MemAddressReserve);
  get("cuMemAddressFree", &d->MemAddressFree);
  get("cuMemSetAccess", &d->MemSetAccess);
  get("cuMemExportToShareableHandle", &d->MemExportToShareableHandle);
  get("cuMemImportFromShareableHandle", &d->MemImportFromShareableHandle);
  get("cuMemGetAllocationGranularity", &d->MemGetAllocationGranularity);
  return ok;
}

#define HFR_CUDRV(call)                                                    \
  do {                                                                     \
    CUresult r_ = (call);                                                  \
    if (r_ != CUDA_SUCCESS) {                                              \
      char b_[256];                                                        \
      snprintf(b_, sizeof b_, "%s failed: CUresult %d", #call, (int)r_);   \
      g_cuda_error = b_;                                                   \
      return r_ == CUDA_ERROR_OUT_OF_MEMORY ? HFR_ERR_OUT_OF_MEMORY : HFR_ERR_CUDA; \
    }                                                                      \
  } while (0)

// ---------------------------------------------------------------------------
// file-descriptor exchange over abstract Unix sockets
// ---------------------------------------------------------------------------
void sock_name(sockaddr_un* a, socklen_t* len, uint64_t token, int rank) {
  memset(a, 0, sizeof *a);
  a->sun_family = AF_UNIX;
  const int k = snprintf(a->sun_path + 1, sizeof(a->sun_path) - 2, "hfr-%016llx-%d", (unsigned long long)token, rank);
  *len = (socklen_t)(offsetof(sockaddr_un, sun_path) + 1 + k);
}

bool send_fd(int sock, int32_t tag, int fd) {
  char ctrl[CMSG_SPACE(sizeof(int))];
  memset(ctrl, 0, sizeof ctrl);
  iovec iov{&tag, sizeof tag};
  msghdr m{};
  m.msg_iov = &iov;
  m.msg_iovlen = 1;
  m.msg_control = ctrl;
  m.msg_controllen = sizeof ctrl;
  cmsghdr* c = CMSG_FIRSTHDR(&m);
  c->cmsg_level = SOL_SOCKET;
  c->cmsg_type = SCM_RIGHTS;
  c->cmsg_len = CMSG_LEN(sizeof(int));
  memcpy(CMSG_DATA(c), &fd, sizeof(int));
  return sendmsg(sock, &m, 0) == (ssize_t)sizeof tag;
}

bool recv_fd(int sock, int32_t* tag, int* fd) {
  char ctrl[CMSG_SPACE(sizeof(int))];
  iovec iov{tag, sizeof *tag};
  msghdr m{};
  m.msg_iov = &iov;
  m.msg_iovlen = 1;
  m.msg_control = ctrl;
  m.msg_controllen = sizeof ctrl;
  if (recvmsg(sock, &m, 0) != (ssize_t)sizeof *tag) return false;
  cmsghdr* c = CMSG_FIRSTHDR(&m);
  if (!c || c->cmsg_type != SCM_RIGHTS) return false;
  memcpy(fd, CMSG_DATA(c), sizeof(int));
  return true;
}

// Every rank sends `my_fd` to every other rank (root_only: only rank 0 sends).
// fds[q] receives rank q's descriptor (fds[rank] = my_fd).  Collective.
hfr_status_t fd_allgather(hfr_comm_s* c, int my_fd, bool root_only, int* fds) {
  struct Hello {
    uint64_t token;
    int32_t rank, pid;
  } me{0, c->rank, (int32_t)getpid()}, all[kMaxRanks];
  std::random_device rd;
  me.token = ((uint64_t)rd() << 32) ^ rd() ^ ((uint64_t)getpid() << 16);
  HFR_TRY(exchange(c, &me, all, sizeof me));
  const uint64_t token = all[0].token;
  for (int q = 0; q < c->n; ++q) fds[q] = -1;
  fds[c->rank] = my_fd;
  const bool receiver = !root_only || c->rank != 0;
  const int expect = root_only ? (c->rank == 0 ? 0 : 1) : c->n - 1;
  int ls = -1;
  if (receiver && expect > 0) {
    ls = socket(AF_UNIX, SOCK_STREAM, 0);
    sockaddr_un a;
    socklen_t len;
    sock_name(&a, &len, token, c->rank);
    if (ls < 0 || bind(ls, (sockaddr*)&a, len) != 0 || listen(ls, kMaxRanks) != 0) {
      if (ls >= 0) close(ls);
      g_cuda_error = "fd exchange: cannot listen on abstract socket";
      return HFR_ERR_INTERNAL;
    }
  }
  int dummy = 0, sink[kMaxRanks];
  HFR_TRY(exchange(c, &dummy, sink, sizeof dummy));  // everyone listens
  hfr_status_t st = HFR_SUCCESS;
  if (!root_only || c->rank == 0) {
    for (int q = 0; q < c->n && st == HFR_SUCCESS; ++q) {
      if (q == c->rank) continue;
      const int s = socket(AF_UNIX, SOCK_STREAM, 0);
      sockaddr_un a;
      socklen_t len;
      sock_name(&a, &len, token, q);
      bool ok = s >= 0 && connect(s, (sockaddr*)&a, len) == 0 && send_fd(s, c->rank, my_fd);
      if (s >= 0) close(s);
      if (!ok) {
        g_cuda_error = "fd exchange: send failed";
        st = HFR_ERR_INTERNAL;
      }
    }
  }
  for (int i = 0; i < expect && st == HFR_SUCCESS; ++i) {
    const int s = accept(ls, nullptr, nullptr);
    int32_t tag = -1;
    int fd = -1;
    if (s < 0 || !recv_fd(s, &tag, &fd) || tag < 0 || tag >= c->n) {
      g_cuda_error = "fd exchange: receive failed";
      st = HFR_ERR_INTERNAL;
    } else {
      fds[tag] = fd;
    }
    if (s >= 0) close(s);
  }
  if (ls >= 0) close(ls);
  hfr_status_t st2 = exchange(c, &dummy, sink, sizeof dummy);  // everyone received
  return st != HFR_SUCCESS ? st : st2;
}

// ---------------------------------------------------------------------------
// the arena
// ---------------------------------------------------------------------------
constexpr size_t kNvlsFlagBytes = 64 << 10;  // multicast exit counters at the front

struct Nvls {
  bool on = false;
  DrvApi d;
  CUdevice dev = 0;
  size_t size = 0, used = kNvlsFlagBytes;
  CUmemGenericAllocationHandle mc = 0;
  CUmemGenericAllocationHandle mem[kMaxRanks] = {};  // own + imported peer allocations
  CUdeviceptr uc[kMaxRanks] = {};                    // unicast VAs (own + peers)
  CUdeviceptr mcva = 0;
  bool bound = false;
};

void nvls_teardown(Nvls& v, int n, int rank) {
  if (!v.d.MemUnmap) return;
  if (v.mcva) {
    v.d.MemUnmap(v.mcva, v.size);
    v.d.MemAddressFree(v.mcva, v.size);
  }
  for (int q = 0; q < n; ++q) {
    if (v.uc[q]) {
      v.d.MemUnmap(v.uc[q], v.size);
      v.d.MemAddressFree(v.uc[q], v.size);
    }
    if (v.mem[q] && q != rank) v.d.MemRelease(v.mem[q]);
  }
  if (v.bound) v.d.MulticastUnbind(v.mc, v.dev, 0, v.size);
  if (v.mem[rank]) v.d.MemRelease(v.mem[rank]);
  if (v.mc) v.d.MemRelease(v.mc);
  v = Nvls();
}

hfr_status_t nvls_map(Nvls& v, CUmemGenericAllocationHandle h, CUdeviceptr* va) {
  HFR_CUDRV(v.d.MemAddressReserve(va, v.size, 0, 0, 0));
  HFR_CUDRV(v.d.MemMap(*va, v.size, 0, h, 0));
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = (int)v.dev;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  HFR_CUDRV(v.d.MemSetAccess(*va, v.size, &acc, 1));
  return HFR_SUCCESS;
}

// COLLECTIVE.  Build the multicast arena of `bytes` per rank.
hfr_status_t nvls_setup(hfr_comm_s* c, Nvls& v, size_t bytes) {
  if (!load_drv(&v.d)) return HFR_ERR_UNSUPPORTED;
  HFR_CUDRV(v.d.DeviceGet(&v.dev, c->dev));
  int mcs = 0;
  HFR_CUDRV(v.d.DeviceGetAttribute(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, v.dev));
  int ok_all[kMaxRanks], mine = mcs ? 1 : 0;
  HFR_TRY(exchange(c, &mine, ok_all, sizeof mine));
  for (int q = 0; q < c->n; ++q)
    if (!ok_all[q]) return HFR_ERR_UNSUPPORTED;

  CUmulticastObjectProp mp{};
  mp.numDevices = (unsigned)c->n;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t mgran = 0;
  HFR_CUDRV(v.d.MulticastGetGranularity(&mgran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  CUmemAllocationProp ap{};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = c->dev;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t agran = 0;
  HFR_CUDRV(v.d.MemGetAllocationGranularity(&agran, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  const size_t gran = std::max(mgran, agran);
  v.size = round_up(bytes + kNvlsFlagBytes, gran);
  mp.size = v.size;

  // 1. multicast object: created by rank 0, imported by the others
  int mcfd = -1, fds[kMaxRanks];
  if (c->rank == 0) {
    HFR_CUDRV(v.d.MulticastCreate(&v.mc, &mp));
    HFR_CUDRV(v.d.MemExportToShareableHandle(&mcfd, v.mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
  }
  HFR_TRY(fd_allgather(c, mcfd, true, fds));
  if (c->rank == 0) {
    close(mcfd);
  } else {
    HFR_CUDRV(v.d.MemImportFromShareableHandle(&v.mc, (void*)(uintptr_t)fds[0], CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR));
    close(fds[0]);
  }
  HFR_CUDRV(v.d.MulticastAddDevice(v.mc, v.dev));
  int dummy = 0, sink[kMaxRanks];
  HFR_TRY(exchange(c, &dummy, sink, sizeof dummy));  // every device added before any bind

  // 2. physical memory, bound to the multicast object, zeroed
  HFR_CUDRV(v.d.MemCreate(&v.mem[c->rank], v.size, &ap, 0));
  HFR_CUDRV(v.d.MulticastBindMem(v.mc, 0, v.mem[c->rank], 0, v.size, 0));
  v.bound = true;
  HFR_TRY(nvls_map(v, v.mem[c->rank], &v.uc[c->rank]));
  HFR_CU(cudaMemset((void*)v.uc[c->rank], 0, v.size));
  HFR_CU(cudaDeviceSynchronize());

  // 3. peers' physical memory, for unicast (bit-exact schedules, flags)
  int memfd = -1;
  HFR_CUDRV(v.d.MemExportToShareableHandle(&memfd, v.mem[c->rank], CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
  HFR_TRY(fd_allgather(c, memfd, false, fds));
  close(memfd);
  for (int q = 0; q < c->n; ++q) {
    if (q == c->rank) continue;
    HFR_CUDRV(v.d.MemImportFromShareableHandle(&v.mem[q], (void*)(uintptr_t)fds[q], CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR));
    close(fds[q]);
    HFR_TRY(nvls_map(v, v.mem[q], &v.uc[q]));
  }
  // 4. the multicast VA
  HFR_TRY(nvls_map(v, v.mc, &v.mcva));
  HFR_TRY(exchange(c, &dummy, sink, sizeof dummy));
  v.on = true;
  return HFR_SUCCESS;
}

}  // namespace

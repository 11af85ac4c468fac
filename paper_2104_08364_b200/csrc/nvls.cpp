// nvls.cpp — NVLink SHARP (NVSwitch multicast) replica for the fused multi-GPU path.
//
// The w replica of every rank is bound to one multicast object, so the owner of a shard writes each updated slice
// once with multimem.st and the switch delivers it to every GPU ("stores w to all peers
// (multimem.st)"). Driver API entry points are fetched at run time through cudaGetDriverEntryPoint (no link-time
// libcuda dependency, so the library still loads on a machine without a driver). The multicast handle is exported by
// rank 0 as a POSIX file descriptor and passed to the other ranks over an abstract Unix-domain socket (SCM_RIGHTS).
#include "nvls.h"

#include <cuda.h>
#include <cuda_runtime.h>
#include <poll.h>
#include <sys/socket.h>
#include <sys/un.h>
#include <unistd.h>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>

namespace ss {
namespace {

struct Drv {
  bool ok = false;
  CUresult (*MulticastGetGranularity)(size_t *, const CUmulticastObjectProp *, CUmulticastGranularity_flags);
  CUresult (*MulticastCreate)(CUmemGenericAllocationHandle *, const CUmulticastObjectProp *);
  CUresult (*MulticastAddDevice)(CUmemGenericAllocationHandle, CUdevice);
  CUresult (*MulticastBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                               unsigned long long);
  CUresult (*MulticastUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t);
  CUresult (*MemCreate)(CUmemGenericAllocationHandle *, size_t, const CUmemAllocationProp *, unsigned long long);
  CUresult (*MemRelease)(CUmemGenericAllocationHandle);
  CUresult (*MemExportToShareableHandle)(void *, CUmemGenericAllocationHandle, CUmemAllocationHandleType,
                                         unsigned long long);
  CUresult (*MemImportFromShareableHandle)(CUmemGenericAllocationHandle *, void *, CUmemAllocationHandleType);
  CUresult (*MemAddressReserve)(CUdeviceptr *, size_t, size_t, CUdeviceptr, unsigned long long);
  CUresult (*MemAddressFree)(CUdeviceptr, size_t);
  CUresult (*MemMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long);
  CUresult (*MemUnmap)(CUdeviceptr, size_t);
  CUresult (*MemSetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc *, size_t);
  CUresult (*DeviceGet)(CUdevice *, int);
  CUresult (*DeviceGetAttribute)(int *, CUdevice_attribute, CUdevice);
};

Drv &drv() {
  static Drv d = [] {
    Drv x;
    auto get = [](const char *name, void **fn) {
      cudaDriverEntryPointQueryResult q;
      return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess &&
             q == cudaDriverEntryPointSuccess && *fn != nullptr;
    };
    x.ok = get("cuMulticastGetGranularity", (void **)&x.MulticastGetGranularity) &&
           get("cuMulticastCreate", (void **)&x.MulticastCreate) &&
           get("cuMulticastAddDevice", (void **)&x.MulticastAddDevice) &&
           get("cuMulticastBindMem", (void **)&x.MulticastBindMem) &&
           get("cuMulticastUnbind", (void **)&x.MulticastUnbind) && get("cuMemCreate", (void **)&x.MemCreate) &&
           get("cuMemRelease", (void **)&x.MemRelease) &&
           get("cuMemExportToShareableHandle", (void **)&x.MemExportToShareableHandle) &&
           get("cuMemImportFromShareableHandle", (void **)&x.MemImportFromShareableHandle) &&
           get("cuMemAddressReserve", (void **)&x.MemAddressReserve) &&
           get("cuMemAddressFree", (void **)&x.MemAddressFree) && get("cuMemMap", (void **)&x.MemMap) &&
           get("cuMemUnmap", (void **)&x.MemUnmap) && get("cuMemSetAccess", (void **)&x.MemSetAccess) &&
           get("cuDeviceGet", (void **)&x.DeviceGet) && get("cuDeviceGetAttribute", (void **)&x.DeviceGetAttribute);
    cudaGetLastError();
    return x;
  }();
  return d;
}

// ---- file-descriptor passing over an abstract Unix socket ----
void sock_name(sockaddr_un *a, socklen_t *len, const char *tag) {
  std::memset(a, 0, sizeof *a);
  a->sun_family = AF_UNIX;
  const int n = std::snprintf(a->sun_path + 1, sizeof(a->sun_path) - 1, "syncswitch-nvls-%s", tag);
  *len = (socklen_t)(offsetof(sockaddr_un, sun_path) + 1 + n);
}

bool send_fd(int sock, int fd) {
  char data = 'f';
  iovec iov{&data, 1};
  char ctrl[CMSG_SPACE(sizeof(int))];
  std::memset(ctrl, 0, sizeof ctrl);
  msghdr m{};
  m.msg_iov = &iov;
  m.msg_iovlen = 1;
  m.msg_control = ctrl;
  m.msg_controllen = sizeof ctrl;
  cmsghdr *c = CMSG_FIRSTHDR(&m);
  c->cmsg_level = SOL_SOCKET;
  c->cmsg_type = SCM_RIGHTS;
  c->cmsg_len = CMSG_LEN(sizeof(int));
  std::memcpy(CMSG_DATA(c), &fd, sizeof(int));
  return sendmsg(sock, &m, 0) == 1;
}

int recv_fd(int sock) {
  char data;
  iovec iov{&data, 1};
  char ctrl[CMSG_SPACE(sizeof(int))];
  msghdr m{};
  m.msg_iov = &iov;
  m.msg_iovlen = 1;
  m.msg_control = ctrl;
  m.msg_controllen = sizeof ctrl;
  if (recvmsg(sock, &m, 0) != 1) return -1;
  cmsghdr *c = CMSG_FIRSTHDR(&m);
  if (!c || c->cmsg_type != SCM_RIGHTS) return -1;
  int fd;
  std::memcpy(&fd, CMSG_DATA(c), sizeof(int));
  return fd;
}

}  // namespace

bool nvls_supported(int device) {
  Drv &d = drv();
  if (!d.ok) return false;
  CUdevice dev;
  int v = 0;
  if (d.DeviceGet(&dev, device) != CUDA_SUCCESS) return false;
  if (d.DeviceGetAttribute(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev) != CUDA_SUCCESS) return false;
  return v != 0;
}

// Phase 1, collective over `world` processes: rank 0 creates the object and serves its fd (every wait bounded by 60 s);
// every rank imports it and adds its device. The caller must agree on success across ranks before phase 2, because
// binding blocks until every device has been added. `tag` names the socket (unique per job).
const char *nvls_share(NvlsReplica *r, int rank, int world, int device, size_t bytes, const char *tag) {
  Drv &d = drv();
  if (!d.ok) return "driver multicast entry points unavailable";
  CUdevice dev;
  if (d.DeviceGet(&dev, device) != CUDA_SUCCESS) return "cuDeviceGet failed";
  CUmulticastObjectProp prop{};
  prop.numDevices = (unsigned)world;
  prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  prop.size = bytes;
  size_t gran = 0;
  if (d.MulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS || gran == 0)
    return "cuMulticastGetGranularity failed";
  const size_t size = (bytes + gran - 1) / gran * gran;
  prop.size = size;
  r->size = size;

  sockaddr_un addr;
  socklen_t alen;
  sock_name(&addr, &alen, tag);
  int fd = -1;
  if (rank == 0) {
    if (d.MulticastCreate(&r->mc, &prop) != CUDA_SUCCESS) return "cuMulticastCreate failed";
    if (d.MemExportToShareableHandle(&fd, r->mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0) != CUDA_SUCCESS)
      return "cuMemExportToShareableHandle failed";
    const int srv = socket(AF_UNIX, SOCK_STREAM, 0);
    if (srv < 0 || bind(srv, (sockaddr *)&addr, alen) != 0 || listen(srv, world) != 0) {
      if (srv >= 0) close(srv);
      return "unix socket bind/listen failed";
    }
    for (int i = 1; i < world; ++i) {
      pollfd pf{srv, POLLIN, 0};
      if (poll(&pf, 1, 60000) != 1) {   // a peer that never connects must not hang rank 0
        close(srv);
        close(fd);
        return "no connection from a peer within 60 s";
      }
      const int cl = accept(srv, nullptr, nullptr);
      if (cl < 0 || !send_fd(cl, fd)) {
        if (cl >= 0) close(cl);
        close(srv);
        return "fd send failed";
      }
      close(cl);
    }
    close(srv);
    close(fd);
  } else {
    int s = -1;
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
      s = socket(AF_UNIX, SOCK_STREAM, 0);
      if (s >= 0 && connect(s, (sockaddr *)&addr, alen) == 0) break;
      if (s >= 0) close(s);
      s = -1;
      if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(60)) return "connect to rank 0 timed out";
      std::this_thread::sleep_for(std::chrono::milliseconds(5));
    }
    fd = recv_fd(s);
    close(s);
    if (fd < 0) return "fd receive failed";
    const CUresult e = d.MemImportFromShareableHandle(&r->mc, (void *)(uintptr_t)fd,
                                                      CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
    close(fd);
    if (e != CUDA_SUCCESS) return "cuMemImportFromShareableHandle failed";
  }
  if (d.MulticastAddDevice(r->mc, dev) != CUDA_SUCCESS) return "cuMulticastAddDevice failed";
  r->device = device;
  r->gran = gran;
  return nullptr;
}

// Phase 2 (after every rank's phase 1 succeeded): bind fresh device memory and map the unicast and multicast views.
const char *nvls_bind(NvlsReplica *r) {
  Drv &d = drv();
  const size_t size = r->size, gran = r->gran;
  const int device = r->device;
  CUmemAllocationProp ap{};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = device;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  if (d.MemCreate(&r->mem, size, &ap, 0) != CUDA_SUCCESS) return "cuMemCreate failed";
  r->have_mem = true;
  // blocks until every rank has added its device
  if (d.MulticastBindMem(r->mc, 0, r->mem, 0, size, 0) != CUDA_SUCCESS) return "cuMulticastBindMem failed";
  r->bound = true;
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CUdeviceptr uc = 0, mcv = 0;
  if (d.MemAddressReserve(&uc, size, gran, 0, 0) != CUDA_SUCCESS) return "reserve (unicast) failed";
  r->uc = (void *)uc;
  if (d.MemMap(uc, size, 0, r->mem, 0) != CUDA_SUCCESS) return "map (unicast) failed";
  r->uc_mapped = true;
  if (d.MemSetAccess(uc, size, &acc, 1) != CUDA_SUCCESS) return "access (unicast) failed";
  if (d.MemAddressReserve(&mcv, size, gran, 0, 0) != CUDA_SUCCESS) return "reserve (multicast) failed";
  r->mcv = (void *)mcv;
  if (d.MemMap(mcv, size, 0, r->mc, 0) != CUDA_SUCCESS) return "map (multicast) failed";
  r->mc_mapped = true;
  if (d.MemSetAccess(mcv, size, &acc, 1) != CUDA_SUCCESS) return "access (multicast) failed";
  r->ready = true;
  return nullptr;
}

void nvls_release(NvlsReplica *r) {
  Drv &d = drv();
  if (!d.ok) return;
  if (r->mc_mapped) d.MemUnmap((CUdeviceptr)r->mcv, r->size);
  if (r->mcv) d.MemAddressFree((CUdeviceptr)r->mcv, r->size);
  if (r->uc_mapped) d.MemUnmap((CUdeviceptr)r->uc, r->size);
  if (r->uc) d.MemAddressFree((CUdeviceptr)r->uc, r->size);
  if (r->bound) {
    CUdevice dev;
    if (d.DeviceGet(&dev, r->device) == CUDA_SUCCESS) d.MulticastUnbind(r->mc, dev, 0, r->size);
  }
  if (r->have_mem) d.MemRelease(r->mem);
  if (r->mc) d.MemRelease(r->mc);
  *r = NvlsReplica{};
}

}  // namespace ss

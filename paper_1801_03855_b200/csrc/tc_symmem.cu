// Symmetric, multicast-capable device memory (tc_mem_alloc / tc_mem_free).
//
// NVSwitch can reduce in the switch: a `multimem.ld_reduce` on a multicast address returns the
// sum of every GPU's copy and a `multimem.st` writes all copies at once (NVLS).  That needs the
// tensors to live in physical memory bound to a multicast object, so libtc offers a collective
// allocator: every rank creates its own physical allocation (cuMemCreate), rank 0 creates the
// multicast object, the shareable POSIX file descriptors travel between the ranks' processes
// over abstract-namespace unix sockets (SCM_RIGHTS), every rank maps its own memory, every
// peer's memory (unicast, for the P2P algorithms) and the multicast object.  libcuda is reached
// through cudaGetDriverEntryPoint, so nothing here links the driver library.
#include <cuda.h>
#include <cuda_runtime.h>
#include <sys/socket.h>
#include <sys/time.h>
#include <sys/un.h>
#include <unistd.h>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

#include "tc_internal.h"

using namespace tc;

namespace {

template <class F>
F drv(const char* name) {
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &f, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return nullptr;
  return (F)f;
}

struct Drv {
  decltype(&cuMemCreate) memCreate = nullptr;
  decltype(&cuMemRelease) memRelease = nullptr;
  decltype(&cuMemMap) memMap = nullptr;
  decltype(&cuMemUnmap) memUnmap = nullptr;
  decltype(&cuMemSetAccess) memSetAccess = nullptr;
  decltype(&cuMemAddressReserve) addrReserve = nullptr;
  decltype(&cuMemAddressFree) addrFree = nullptr;
  decltype(&cuMemExportToShareableHandle) exportHandle = nullptr;
  decltype(&cuMemImportFromShareableHandle) importHandle = nullptr;
  decltype(&cuMemGetAllocationGranularity) allocGran = nullptr;
  decltype(&cuMulticastCreate) mcCreate = nullptr;
  decltype(&cuMulticastAddDevice) mcAddDevice = nullptr;
  decltype(&cuMulticastBindMem) mcBindMem = nullptr;
  decltype(&cuMulticastUnbind) mcUnbind = nullptr;
  decltype(&cuMulticastGetGranularity) mcGran = nullptr;
  decltype(&cuDeviceGet) deviceGet = nullptr;
  decltype(&cuDeviceGetAttribute) deviceAttr = nullptr;
  bool ok = false;
};

const Drv& driver() {
  static Drv d = [] {
    Drv x;
    x.memCreate = drv<decltype(&cuMemCreate)>("cuMemCreate");
    x.memRelease = drv<decltype(&cuMemRelease)>("cuMemRelease");
    x.memMap = drv<decltype(&cuMemMap)>("cuMemMap");
    x.memUnmap = drv<decltype(&cuMemUnmap)>("cuMemUnmap");
    x.memSetAccess = drv<decltype(&cuMemSetAccess)>("cuMemSetAccess");
    x.addrReserve = drv<decltype(&cuMemAddressReserve)>("cuMemAddressReserve");
    x.addrFree = drv<decltype(&cuMemAddressFree)>("cuMemAddressFree");
    x.exportHandle = drv<decltype(&cuMemExportToShareableHandle)>("cuMemExportToShareableHandle");
    x.importHandle = drv<decltype(&cuMemImportFromShareableHandle)>("cuMemImportFromShareableHandle");
    x.allocGran = drv<decltype(&cuMemGetAllocationGranularity)>("cuMemGetAllocationGranularity");
    x.mcCreate = drv<decltype(&cuMulticastCreate)>("cuMulticastCreate");
    x.mcAddDevice = drv<decltype(&cuMulticastAddDevice)>("cuMulticastAddDevice");
    x.mcBindMem = drv<decltype(&cuMulticastBindMem)>("cuMulticastBindMem");
    x.mcUnbind = drv<decltype(&cuMulticastUnbind)>("cuMulticastUnbind");
    x.mcGran = drv<decltype(&cuMulticastGetGranularity)>("cuMulticastGetGranularity");
    x.deviceGet = drv<decltype(&cuDeviceGet)>("cuDeviceGet");
    x.deviceAttr = drv<decltype(&cuDeviceGetAttribute)>("cuDeviceGetAttribute");
    x.ok = x.memCreate && x.memRelease && x.memMap && x.memUnmap && x.memSetAccess &&
           x.addrReserve && x.addrFree && x.exportHandle && x.importHandle && x.allocGran &&
           x.mcCreate && x.mcAddDevice && x.mcBindMem && x.mcUnbind && x.mcGran && x.deviceGet &&
           x.deviceAttr;
    return x;
  }();
  return d;
}

bool debug() { return std::getenv("TC_DEBUG") != nullptr; }

// ---------------------------------------------------------------- fd passing (SCM_RIGHTS)
void sock_name(sockaddr_un& a, socklen_t& len, uint64_t nonce, int rank) {
  std::memset(&a, 0, sizeof(a));
  a.sun_family = AF_UNIX;
  int n = std::snprintf(a.sun_path + 1, sizeof(a.sun_path) - 1, "tc-%016llx-%d",
                        (unsigned long long)nonce, rank);
  len = (socklen_t)(offsetof(sockaddr_un, sun_path) + 1 + n);
}

int sock_open(uint64_t nonce, int rank) {
  int s = socket(AF_UNIX, SOCK_DGRAM, 0);
  if (s < 0) return -1;
  sockaddr_un a;
  socklen_t len;
  sock_name(a, len, nonce, rank);
  if (bind(s, (sockaddr*)&a, len) != 0) {
    close(s);
    return -1;
  }
  timeval tv{60, 0};
  setsockopt(s, SOL_SOCKET, SO_RCVTIMEO, &tv, sizeof(tv));
  return s;
}

struct FdMsg {
  int32_t from, kind;
};

bool send_fd(int s, uint64_t nonce, int to, int fd, FdMsg msg) {
  sockaddr_un a;
  socklen_t len;
  sock_name(a, len, nonce, to);
  iovec iov{&msg, sizeof(msg)};
  char ctrl[CMSG_SPACE(sizeof(int))];
  std::memset(ctrl, 0, sizeof(ctrl));
  msghdr m{};
  m.msg_name = &a;
  m.msg_namelen = len;
  m.msg_iov = &iov;
  m.msg_iovlen = 1;
  m.msg_control = ctrl;
  m.msg_controllen = sizeof(ctrl);
  cmsghdr* c = CMSG_FIRSTHDR(&m);
  c->cmsg_level = SOL_SOCKET;
  c->cmsg_type = SCM_RIGHTS;
  c->cmsg_len = CMSG_LEN(sizeof(int));
  std::memcpy(CMSG_DATA(c), &fd, sizeof(int));
  return sendmsg(s, &m, 0) == (ssize_t)sizeof(msg);
}

bool recv_fd(int s, int* fd, FdMsg* msg) {
  iovec iov{msg, sizeof(*msg)};
  char ctrl[CMSG_SPACE(sizeof(int))];
  msghdr m{};
  m.msg_iov = &iov;
  m.msg_iovlen = 1;
  m.msg_control = ctrl;
  m.msg_controllen = sizeof(ctrl);
  if (recvmsg(s, &m, 0) != (ssize_t)sizeof(*msg)) return false;
  cmsghdr* c = CMSG_FIRSTHDR(&m);
  if (!c || c->cmsg_type != SCM_RIGHTS) return false;
  std::memcpy(fd, CMSG_DATA(c), sizeof(int));
  return true;
}

tc_status barrier(Comm& c) {
  int32_t one = 1, all[kMaxRanks];
  return bootstrap_allgather(c.ag, c.ag_ctx, c.nranks, &one, all, sizeof(one));
}

tc_status agree_status(Comm& c, tc_status mine) {
  int32_t s = (int32_t)mine, all[kMaxRanks];
  tc_status bs = bootstrap_allgather(c.ag, c.ag_ctx, c.nranks, &s, all, sizeof(s));
  if (bs != TC_OK) return bs;
  for (int r = 0; r < c.nranks; ++r)
    if (all[r] != TC_OK) return (tc_status)all[r];
  return TC_OK;
}

void release_sym(SymAlloc& a) {
  const Drv& d = driver();
  for (int r = 0; r < kMaxRanks; ++r) {
    if (a.uc[r]) {
      d.memUnmap((CUdeviceptr)a.uc[r], a.size);
      d.addrFree((CUdeviceptr)a.uc[r], a.size);
      a.uc[r] = nullptr;
    }
    if (a.phys[r]) {
      d.memRelease((CUmemGenericAllocationHandle)a.phys[r]);
      a.phys[r] = 0;
    }
  }
  if (a.mc) {
    d.memUnmap((CUdeviceptr)a.mc, a.size);
    d.addrFree((CUdeviceptr)a.mc, a.size);
    a.mc = nullptr;
  }
  if (a.mc_handle) {
    CUdevice dev;
    if (d.deviceGet(&dev, a.device) == CUDA_SUCCESS)
      d.mcUnbind((CUmemGenericAllocationHandle)a.mc_handle, dev, 0, a.size);
    d.memRelease((CUmemGenericAllocationHandle)a.mc_handle);
    a.mc_handle = 0;
  }
}

tc_status map_rw(const Drv& d, int device, CUmemGenericAllocationHandle h, size_t size,
                 size_t gran, void** out) {
  CUdeviceptr va = 0;
  if (d.addrReserve(&va, size, gran, 0, 0) != CUDA_SUCCESS) return TC_ERR_CUDA;
  if (d.memMap(va, size, 0, h, 0) != CUDA_SUCCESS) {
    d.addrFree(va, size);
    return TC_ERR_CUDA;
  }
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  if (d.memSetAccess(va, size, &acc, 1) != CUDA_SUCCESS) {
    d.memUnmap(va, size);
    d.addrFree(va, size);
    return TC_ERR_CUDA;
  }
  *out = (void*)va;
  return TC_OK;
}

}  // namespace

namespace tc {

// Finds the symmetric allocation holding [p, p+bytes); returns its index or -1.
int find_sym(const Comm& c, const void* p, size_t bytes, int64_t* offset) {
  for (size_t i = 0; i < c.sym.size(); ++i) {
    const SymAlloc& a = c.sym[i];
    const char* base = (const char*)a.uc[c.rank < 0 ? 0 : c.rank];
    if (!base) continue;
    if ((const char*)p >= base && (const char*)p + bytes <= base + a.size) {
      *offset = (const char*)p - base;
      return (int)i;
    }
  }
  return -1;
}

void sym_ref(Comm& c, const void* base, int delta) {
  for (SymAlloc& a : c.sym)
    if (a.uc[c.rank < 0 ? 0 : c.rank] == base) a.refs += delta;
}

bool multicast_supported(int device) {
  const Drv& d = driver();
  if (!d.ok) return false;
  CUdevice dev;
  int v = 0;
  if (d.deviceGet(&dev, device) != CUDA_SUCCESS) return false;
  if (d.deviceAttr(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev) != CUDA_SUCCESS) return false;
  return v != 0;
}

void free_all_sym(Comm& c) {
  for (auto& a : c.sym) release_sym(a);
  c.sym.clear();
}

}  // namespace tc

extern "C" {

tc_status tc_mem_alloc(tc_comm* comm, size_t bytes, void** out) {
  if (!comm || !out || bytes == 0) return TC_ERR_INVALID_ARG;
  *out = nullptr;
  Comm& c = comm->c;
  if (c.emulated) return TC_ERR_UNSUPPORTED;
  const Drv& d = driver();
  if (!d.ok) return TC_ERR_UNSUPPORTED;
  cudaSetDevice(c.device);
  const int p = c.nranks, me = c.rank;
  tc_status st = TC_OK;
  SymAlloc a;
  a.device = c.device;
  int sock = -1;
  std::vector<int> fds;
  CUdevice dev;
  CUmemAllocationProp prop{};
  CUmulticastObjectProp mprop{};
  size_t gran = 0, mgran = 0;
  bool mc_ok = multicast_supported(c.device) && p > 1;
  struct Info { int32_t status, mc; uint64_t nonce, size; } mine{}, all[kMaxRanks];

  if (d.deviceGet(&dev, c.device) != CUDA_SUCCESS) return TC_ERR_CUDA;
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = c.device;
  prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  if (d.allocGran(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS)
    return TC_ERR_CUDA;
  mprop.numDevices = (unsigned)p;
  mprop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  mprop.size = bytes;
  if (mc_ok && d.mcGran(&mgran, &mprop, CU_MULTICAST_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS)
    mc_ok = false;
  {
    size_t g = gran > mgran ? gran : mgran;
    a.size = (bytes + g - 1) / g * g;
    gran = g;
  }
  mprop.size = a.size;
  mine.status = TC_OK;
  mine.mc = mc_ok ? 1 : 0;
  mine.nonce = ((uint64_t)std::random_device{}() << 32) ^ (uint64_t)getpid() ^ (uint64_t)(uintptr_t)&a;
  mine.size = a.size;
  st = bootstrap_allgather(c.ag, c.ag_ctx, p, &mine, all, sizeof(Info));
  if (st != TC_OK) return st;
  for (int r = 0; r < p; ++r) {
    mc_ok = mc_ok && all[r].mc;
    if (all[r].size != all[0].size) return TC_ERR_INVALID_ARG;
  }
  a.multicast = mc_ok;
  {
    const uint64_t nonce = all[0].nonce;
    if (p > 1) {
      sock = sock_open(nonce, me);
      st = agree_status(c, sock >= 0 ? TC_OK : TC_ERR_BOOTSTRAP);  // every socket is bound
      if (st != TC_OK) goto fail;
    }
    // 1. multicast object: rank 0 creates and ships it; every rank adds its device
    if (mc_ok) {
      CUmemGenericAllocationHandle mh = 0;
      if (me == 0) {
        // on failure still send a (dummy) message so no peer blocks; status agreement follows
        int fd = -1;
        if (d.mcCreate(&mh, &mprop) != CUDA_SUCCESS ||
            d.exportHandle(&fd, mh, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0) != CUDA_SUCCESS) {
          st = TC_ERR_CUDA;
          fd = dup(sock);
        }
        for (int r = 1; r < p; ++r)
          if (!send_fd(sock, nonce, r, fd, FdMsg{0, st == TC_OK ? 1 : -1})) st = TC_ERR_BOOTSTRAP;
        close(fd);
      } else {
        int fd = -1;
        FdMsg m{};
        if (!recv_fd(sock, &fd, &m) || m.kind != 1) {
          st = TC_ERR_BOOTSTRAP;
        } else {
          if (d.importHandle(&mh, (void*)(uintptr_t)fd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR) !=
              CUDA_SUCCESS)
            st = TC_ERR_CUDA;
          close(fd);
        }
      }
      a.mc_handle = (uint64_t)mh;
      if (st == TC_OK && d.mcAddDevice(mh, dev) != CUDA_SUCCESS) st = TC_ERR_CUDA;
      st = agree_status(c, st);
      if (st != TC_OK) goto fail;
    }
    // 2. physical memory on every rank, exported to every peer
    {
      CUmemGenericAllocationHandle ph = 0;
      if (d.memCreate(&ph, a.size, &prop, 0) != CUDA_SUCCESS) st = TC_ERR_CUDA;
      else a.phys[me] = (uint64_t)ph;
      if (p > 1) {
        int fd = -1;
        if (st != TC_OK ||
            d.exportHandle(&fd, ph, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0) != CUDA_SUCCESS) {
          st = TC_ERR_CUDA;
          fd = dup(sock);
        }
        for (int j = 1; j < p; ++j)
          if (!send_fd(sock, nonce, (me + j) % p, fd, FdMsg{me, st == TC_OK ? 2 : -2}))
            st = TC_ERR_BOOTSTRAP;
        close(fd);
        for (int j = 1; j < p; ++j) {
          int rfd = -1;
          FdMsg m{};
          if (!recv_fd(sock, &rfd, &m) || m.from < 0 || m.from >= p) {
            st = TC_ERR_BOOTSTRAP;
            break;
          }
          if (m.kind != 2) {  // the sender failed; keep draining the other messages
            close(rfd);
            st = TC_ERR_CUDA;
            continue;
          }
          CUmemGenericAllocationHandle h = 0;
          if (d.importHandle(&h, (void*)(uintptr_t)rfd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR) !=
              CUDA_SUCCESS)
            st = TC_ERR_CUDA;
          else
            a.phys[m.from] = (uint64_t)h;
          close(rfd);
        }
      }
      st = agree_status(c, st);
      if (st != TC_OK) goto fail;
    }
    // 3. bind my memory to the multicast object (after every device was added), map everything
    if (mc_ok && d.mcBindMem((CUmemGenericAllocationHandle)a.mc_handle, 0,
                             (CUmemGenericAllocationHandle)a.phys[me], 0, a.size, 0) != CUDA_SUCCESS)
      st = TC_ERR_CUDA;
    for (int r = 0; r < p && st == TC_OK; ++r)
      st = map_rw(d, c.device, (CUmemGenericAllocationHandle)a.phys[r], a.size, gran, &a.uc[r]);
    if (st == TC_OK && mc_ok)
      st = map_rw(d, c.device, (CUmemGenericAllocationHandle)a.mc_handle, a.size, gran, &a.mc);
    if (st == TC_OK && cudaMemset(a.uc[me], 0, a.size) != cudaSuccess) st = TC_ERR_CUDA;
    if (st == TC_OK && cudaDeviceSynchronize() != cudaSuccess) st = TC_ERR_CUDA;
    st = agree_status(c, st);
    if (st != TC_OK) goto fail;
  }
  if (sock >= 0) close(sock);
  c.sym.push_back(a);
  *out = a.uc[me];
  return TC_OK;
fail:
  if (sock >= 0) close(sock);
  if (debug()) std::fprintf(stderr, "libtc: tc_mem_alloc failed: %s\n", tc_status_string(st));
  release_sym(a);
  return st;
}

tc_status tc_mem_free(tc_comm* comm, void* ptr) {
  if (!comm || !ptr) return TC_ERR_INVALID_ARG;
  Comm& c = comm->c;
  int64_t off = 0;
  int i = find_sym(c, ptr, 1, &off);
  if (i < 0 || off != 0) return TC_ERR_INVALID_ARG;
  if (c.sym[(size_t)i].refs > 0) return TC_ERR_INVALID_ARG;  // a live group still points into it
  cudaSetDevice(c.device);
  cudaDeviceSynchronize();
  tc_status st = barrier(c);  // no peer kernel still touches it
  release_sym(c.sym[(size_t)i]);
  c.sym.erase(c.sym.begin() + i);
  tc_status st2 = barrier(c);
  return st != TC_OK ? st : st2;
}

int tc_comm_multicast_supported(const tc_comm* comm) {
  if (!comm || comm->c.emulated) return 0;
  return multicast_supported(comm->c.device) ? 1 : 0;
}

}  // extern "C"

// NVLS (NVLink SHARP) path: a multicast object spanning every rank's GPU, with
// each rank's own memory bound to it. One `multimem.ld_reduce` returns the sum of
// all N copies computed inside the NVSwitch, one `multimem.st` writes all N
// copies. Per-GPU link traffic of an all-reduce drops from 2(N-1)/N*S per
// direction (P2P two-shot) to about S -- the route past the P2P ceiling at N >= 4
// (DESIGN.md §5, §8). The switch sums in its own order, so the result is NOT the
// rank-ordered fold: this path is opt-in (RP_ALGO_NVLS) with a stated tolerance.
//
// Bootstrap: the multicast handle is a POSIX file descriptor (fabric handles are
// not permitted on this pool, tools/mc_probe.cu), handed from rank 0 to its peers
// over an abstract-namespace Unix socket with SCM_RIGHTS.
//
// Also here, as the other dynamically scheduled broadcasts: the NVLS broadcast
// (K4n, multicast store) and the pipelined P2P relay broadcast (K4r).
#include <cuda.h>
#include <string.h>
#include <sys/socket.h>
#include <sys/un.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <string>

#include <cudaTypedefs.h>

#include "rp_allreduce.cuh"

// Driver-API entry points resolved at run time through the runtime
// (cudaGetDriverEntryPoint): librp.so keeps no link-time dependency on
// libcuda.so, so it still loads (and its C ABI can be inspected) on hosts
// without a GPU driver.
namespace {
struct Driver {
#define RP_DRV(name) PFN_##name name = nullptr;
#define RP_DRV_ALL(X)                                                                             \
  X(cuDeviceGet) X(cuDeviceGetAttribute) X(cuGetErrorString) X(cuMemAddressFree) X(cuMemAddressReserve) \
  X(cuMemCreate) X(cuMemExportToShareableHandle) X(cuMemGetAllocationGranularity)                 \
  X(cuMemImportFromShareableHandle) X(cuMemMap) X(cuMemRelease) X(cuMemSetAccess) X(cuMemUnmap)   \
  X(cuMulticastAddDevice) X(cuMulticastBindMem) X(cuMulticastCreate) X(cuMulticastGetGranularity) \
  X(cuMulticastUnbind)
  RP_DRV_ALL(RP_DRV)
#undef RP_DRV
  bool ok = false;
};
Driver g_drv;

int load_driver() {
  if (g_drv.ok) return RP_OK;
#define RP_LOAD(name)                                                                            \
  {                                                                                              \
    void* fn = nullptr;                                                                          \
    cudaDriverEntryPointQueryResult q;                                                           \
    if (cudaGetDriverEntryPoint(#name, &fn, cudaEnableDefault, &q) != cudaSuccess || fn == nullptr) \
      return rp_fail(RP_ERR_CONFIG, "CUDA driver entry point " #name " unavailable");           \
    g_drv.name = (PFN_##name)fn;                                                                 \
  }
  RP_DRV_ALL(RP_LOAD)
#undef RP_LOAD
  g_drv.ok = true;
  return RP_OK;
}
}  // namespace

#define cuDeviceGet g_drv.cuDeviceGet
#define cuDeviceGetAttribute g_drv.cuDeviceGetAttribute
#define cuGetErrorString g_drv.cuGetErrorString
#define cuMemAddressFree g_drv.cuMemAddressFree
#define cuMemAddressReserve g_drv.cuMemAddressReserve
#define cuMemCreate g_drv.cuMemCreate
#define cuMemExportToShareableHandle g_drv.cuMemExportToShareableHandle
#define cuMemGetAllocationGranularity g_drv.cuMemGetAllocationGranularity
#define cuMemImportFromShareableHandle g_drv.cuMemImportFromShareableHandle
#define cuMemMap g_drv.cuMemMap
#define cuMemRelease g_drv.cuMemRelease
#define cuMemSetAccess g_drv.cuMemSetAccess
#define cuMemUnmap g_drv.cuMemUnmap
#define cuMulticastAddDevice g_drv.cuMulticastAddDevice
#define cuMulticastBindMem g_drv.cuMulticastBindMem
#define cuMulticastCreate g_drv.cuMulticastCreate
#define cuMulticastGetGranularity g_drv.cuMulticastGetGranularity
#define cuMulticastUnbind g_drv.cuMulticastUnbind

struct NvlsState {
  CUmemGenericAllocationHandle mc = 0;
  CUmemGenericAllocationHandle phys = 0;
  CUdeviceptr mc_va = 0, uc_va = 0;
  size_t size = 0, gran = 0;
  int listen_fd = -1;
  int share_fd = -1;
  bool have_mc = false, added = false, bound = false;
  size_t reserved = 0;
};

static NvlsState* nvls_of(rp_comm* c) { return (NvlsState*)c->nvls; }

static int cu_fail(CUresult r, const char* what) {
  const char* s = nullptr;
  cuGetErrorString(r, &s);
  return rp_fail(RP_ERR_CONFIG, std::string(what) + ": " + (s ? s : "CUDA driver error"));
}
#define CU_CHECK(x)                         \
  do {                                      \
    CUresult r_ = (x);                      \
    if (r_ != CUDA_SUCCESS) return cu_fail(r_, #x); \
  } while (0)

static CUmulticastObjectProp mc_prop(rp_comm* c, size_t bytes) {
  CUmulticastObjectProp p;
  memset(&p, 0, sizeof(p));
  p.numDevices = (unsigned)c->world;
  p.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  p.size = bytes;
  return p;
}

static int nvls_size(rp_comm* c, size_t bytes, size_t* size, size_t* gran) {
  CUmulticastObjectProp p = mc_prop(c, bytes);
  size_t g = 0;
  CU_CHECK(cuMulticastGetGranularity(&g, &p, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  *gran = g;
  *size = (bytes + g - 1) / g * g;
  return RP_OK;
}

static void abstract_addr(const char* name, sockaddr_un* a, socklen_t* len) {
  memset(a, 0, sizeof(*a));
  a->sun_family = AF_UNIX;
  const size_t n = std::min(strlen(name), sizeof(a->sun_path) - 2);
  memcpy(a->sun_path + 1, name, n);  // leading NUL: abstract namespace, no filesystem entry
  *len = (socklen_t)(offsetof(sockaddr_un, sun_path) + 1 + n);
}

extern "C" {

int rp_nvls_create(rp_comm_t c, size_t bytes, char* name, size_t name_cap) {
  if (!c || !name || name_cap < 64) return rp_fail(RP_ERR_INVALID, "rp_nvls_create: bad arguments");
  if (c->is_virtual || c->world < 2) return rp_fail(RP_ERR_CONFIG, "NVLS needs a multi-process communicator");
  RP_CUDA_CHECK(cudaSetDevice(c->device));
  RP_CUDA_CHECK(cudaFree(0));  // primary context current for the driver API
  if (int rc0 = load_driver()) return rc0;
  int mcs = 0;
  CUdevice dev;
  CU_CHECK(cuDeviceGet(&dev, c->device));
  CU_CHECK(cuDeviceGetAttribute(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
  if (!mcs) return rp_fail(RP_ERR_CONFIG, "device does not support NVLS multicast");
  if (!c->nvls) c->nvls = new NvlsState();
  NvlsState* s = nvls_of(c);
  int rc = nvls_size(c, bytes, &s->size, &s->gran);
  if (rc) return rc;
  name[0] = 0;
  if (c->rank != 0) return RP_OK;
  CUmulticastObjectProp p = mc_prop(c, s->size);
  CU_CHECK(cuMulticastCreate(&s->mc, &p));
  s->have_mc = true;
  int fd = -1;
  CU_CHECK(cuMemExportToShareableHandle(&fd, s->mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
  s->share_fd = fd;
  static std::atomic<int> counter{0};
  snprintf(name, name_cap, "rp-nvls-%d-%d", (int)getpid(), counter++);
  int ls = socket(AF_UNIX, SOCK_STREAM, 0);
  if (ls < 0) return rp_fail(RP_ERR_CONFIG, "rp_nvls_create: socket() failed");
  sockaddr_un a;
  socklen_t len;
  abstract_addr(name, &a, &len);
  if (bind(ls, (sockaddr*)&a, len) != 0 || listen(ls, c->world) != 0) {
    close(ls);
    return rp_fail(RP_ERR_CONFIG, "rp_nvls_create: cannot bind/listen on the abstract socket");
  }
  s->listen_fd = ls;
  return RP_OK;
}

// rank 0: hand the multicast fd to every peer (blocks until world-1 peers took it)
int rp_nvls_serve(rp_comm_t c) {
  if (!c || !c->nvls) return rp_fail(RP_ERR_INVALID, "rp_nvls_serve: call rp_nvls_create first");
  NvlsState* s = nvls_of(c);
  if (c->rank != 0) return RP_OK;
  for (int i = 1; i < c->world; ++i) {
    int conn = accept(s->listen_fd, nullptr, nullptr);
    if (conn < 0) return rp_fail(RP_ERR_CONFIG, "rp_nvls_serve: accept() failed");
    char byte = 'F';
    iovec iov{&byte, 1};
    char ctrl[CMSG_SPACE(sizeof(int))];
    memset(ctrl, 0, sizeof(ctrl));
    msghdr m;
    memset(&m, 0, sizeof(m));
    m.msg_iov = &iov;
    m.msg_iovlen = 1;
    m.msg_control = ctrl;
    m.msg_controllen = sizeof(ctrl);
    cmsghdr* cm = CMSG_FIRSTHDR(&m);
    cm->cmsg_level = SOL_SOCKET;
    cm->cmsg_type = SCM_RIGHTS;
    cm->cmsg_len = CMSG_LEN(sizeof(int));
    memcpy(CMSG_DATA(cm), &s->share_fd, sizeof(int));
    const ssize_t n = sendmsg(conn, &m, 0);
    close(conn);
    if (n != 1) return rp_fail(RP_ERR_CONFIG, "rp_nvls_serve: sendmsg failed");
  }
  close(s->listen_fd);
  s->listen_fd = -1;
  return RP_OK;
}

// ranks != 0: receive the multicast fd from rank 0 and import the handle
int rp_nvls_join(rp_comm_t c, const char* name) {
  if (!c || !c->nvls || !name) return rp_fail(RP_ERR_INVALID, "rp_nvls_join: call rp_nvls_create first");
  NvlsState* s = nvls_of(c);
  if (c->rank == 0) return RP_OK;
  int sock = socket(AF_UNIX, SOCK_STREAM, 0);
  if (sock < 0) return rp_fail(RP_ERR_CONFIG, "rp_nvls_join: socket() failed");
  sockaddr_un a;
  socklen_t len;
  abstract_addr(name, &a, &len);
  int ok = -1;
  for (int attempt = 0; attempt < 2000 && ok != 0; ++attempt) {  // rank 0 may not listen yet
    ok = connect(sock, (sockaddr*)&a, len);
    if (ok != 0) usleep(5000);
  }
  if (ok != 0) {
    close(sock);
    return rp_fail(RP_ERR_CONFIG, "rp_nvls_join: cannot reach rank 0's socket");
  }
  char byte = 0;
  iovec iov{&byte, 1};
  char ctrl[CMSG_SPACE(sizeof(int))];
  msghdr m;
  memset(&m, 0, sizeof(m));
  m.msg_iov = &iov;
  m.msg_iovlen = 1;
  m.msg_control = ctrl;
  m.msg_controllen = sizeof(ctrl);
  const ssize_t n = recvmsg(sock, &m, 0);
  close(sock);
  cmsghdr* cm = CMSG_FIRSTHDR(&m);
  if (n != 1 || !cm || cm->cmsg_type != SCM_RIGHTS) return rp_fail(RP_ERR_CONFIG, "rp_nvls_join: no fd received");
  int fd;
  memcpy(&fd, CMSG_DATA(cm), sizeof(int));
  s->share_fd = fd;
  RP_CUDA_CHECK(cudaSetDevice(c->device));
  CU_CHECK(cuMemImportFromShareableHandle(&s->mc, (void*)(uintptr_t)fd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR));
  s->have_mc = true;
  return RP_OK;
}

// every rank: add its device (all ranks must finish this before anyone binds)
int rp_nvls_add(rp_comm_t c) {
  if (!c || !c->nvls || !nvls_of(c)->have_mc) return rp_fail(RP_ERR_INVALID, "rp_nvls_add: no multicast handle");
  RP_CUDA_CHECK(cudaSetDevice(c->device));
  CUdevice dev;
  CU_CHECK(cuDeviceGet(&dev, c->device));
  CU_CHECK(cuMulticastAddDevice(nvls_of(c)->mc, dev));
  nvls_of(c)->added = true;
  return RP_OK;
}

// every rank: allocate its memory, bind it to the multicast object, map both views
int rp_nvls_bind(rp_comm_t c) {
  if (!c || !c->nvls || !nvls_of(c)->added) return rp_fail(RP_ERR_INVALID, "rp_nvls_bind: call rp_nvls_add first");
  NvlsState* s = nvls_of(c);
  RP_CUDA_CHECK(cudaSetDevice(c->device));
  CUmemAllocationProp ap;
  memset(&ap, 0, sizeof(ap));
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = c->device;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;  // required to bind to the multicast object
  size_t pg = 0;
  CU_CHECK(cuMemGetAllocationGranularity(&pg, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  const size_t g = std::max(pg, s->gran);
  s->size = (s->size + g - 1) / g * g;
  CU_CHECK(cuMemCreate(&s->phys, s->size, &ap, 0));
  CU_CHECK(cuMulticastBindMem(s->mc, 0, s->phys, 0, s->size, 0));
  CUmemAccessDesc acc;
  memset(&acc, 0, sizeof(acc));
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = c->device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CU_CHECK(cuMemAddressReserve(&s->uc_va, s->size, g, 0, 0));
  CU_CHECK(cuMemMap(s->uc_va, s->size, 0, s->phys, 0));
  CU_CHECK(cuMemSetAccess(s->uc_va, s->size, &acc, 1));
  CU_CHECK(cuMemAddressReserve(&s->mc_va, s->size, g, 0, 0));
  CU_CHECK(cuMemMap(s->mc_va, s->size, 0, s->mc, 0));
  CU_CHECK(cuMemSetAccess(s->mc_va, s->size, &acc, 1));
  RP_CUDA_CHECK(cudaMemset((void*)s->uc_va, 0, s->size));
  RP_CUDA_CHECK(cudaDeviceSynchronize());
  s->bound = true;
  return RP_OK;
}

int rp_nvls_pool(rp_comm_t c, void** base, size_t* bytes) {
  if (!c || !base || !bytes) return rp_fail(RP_ERR_INVALID, "rp_nvls_pool: NULL argument");
  if (!c->nvls || !nvls_of(c)->bound) return rp_fail(RP_ERR_CONFIG, "NVLS region not set up (rp_nvls_bind)");
  *base = (void*)nvls_of(c)->uc_va;
  *bytes = nvls_of(c)->size;
  return RP_OK;
}

}  // extern "C"

bool rp_nvls_covers(rp_comm* c, const void* p, size_t bytes) {
  NvlsState* s = nvls_of(c);
  if (!s || !s->bound) return false;
  const char* q = (const char*)p;
  const char* base = (const char*)s->uc_va;
  return q >= base && q + bytes <= base + s->size && (size_t)(q - base) % 16 == 0;
}

void rp_nvls_destroy(rp_comm* c) {
  NvlsState* s = nvls_of(c);
  if (!s) return;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  if (s->mc_va) {
    cuMemUnmap(s->mc_va, s->size);
    cuMemAddressFree(s->mc_va, s->size);
  }
  if (s->uc_va) {
    cuMemUnmap(s->uc_va, s->size);
    cuMemAddressFree(s->uc_va, s->size);
  }
  if (s->bound) {
    CUdevice dev;
    if (cuDeviceGet(&dev, c->device) == CUDA_SUCCESS) cuMulticastUnbind(s->mc, dev, 0, s->size);
  }
  if (s->phys) cuMemRelease(s->phys);
  if (s->have_mc) cuMemRelease(s->mc);
  if (s->listen_fd >= 0) close(s->listen_fd);
  if (s->share_fd >= 0) close(s->share_fd);
  delete s;
  c->nvls = nullptr;
}

// ===========================================================================
// K2n: NVLS all-reduce (in place in the multicast-bound region)
//   barrier 0 (every rank's input is in place)
//   tiles of chunk `rank` (per-warp claims): v = multimem.ld_reduce.add(mc + v)
//     (the switch sums the N copies), scale for mean/premean, multimem.st(mc + v)
//   barrier 1 (every rank's stores landed in every copy)
// ===========================================================================
namespace rp {

template <int DT>
__device__ __forceinline__ uint4 mc_ld_add(const void* p) {
  uint4 r;
  if constexpr (DT == RP_F32) {
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p) : "memory");
  } else if constexpr (DT == RP_BF16) {
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p) : "memory");
  } else {
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.f16x2 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p) : "memory");
  }
  return r;
}
__device__ __forceinline__ void mc_st(void* p, uint4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

// One block of kNvlsThreads per SM, kNvlsU 16-byte requests in flight per
// thread (~75K x 16 B per GPU: deeper queues only congest the switch,
// profiles/r01_nvls_probe.txt). A tile is exactly one request per lane and
// unroll step, so a warp finishes a tile in one switch round trip (short tail),
// and the next tile's claim is issued before the current tile's loads.
constexpr int kNvlsThreads = 128;
constexpr int kNvlsU = 4;

template <int DT, int OP>
__global__ void __launch_bounds__(kNvlsThreads) ar_nvls(const CollArgs a) {
  using T = typename DType<DT>::T;
  const int rank = a.rank;
  if (rp_aborted(a.t, rank)) return;
  char* mc = (char*)a.src[rank];  // the multicast view of this message
  const size_t V = (a.count + (16 / sizeof(T)) - 1) / (16 / sizeof(T));
  const size_t Vc = a.chunk;
  constexpr uint32_t tv = 32 * kNvlsU;
  const uint32_t tpc = (uint32_t)((Vc + tv - 1) / tv);
  const int lane = threadIdx.x & 31;
  const size_t c_hi = std::min((size_t)(rank + 1) * Vc, V);
  rp_trace(a, 0);
  const PhaseBase pb = phase_begin(a, rank);
  if (!phase_end(a, rank, 0, pb)) return;
  const float inv = 1.0f / (float)a.world;
  uint32_t j = claim_tile(a, rank, 1);
  while (j < tpc) {
    const uint32_t next = claim_tile(a, rank, 1);
    const size_t lo = (size_t)rank * Vc + (size_t)j * tv + lane;
    uint4 r[kNvlsU];
#pragma unroll
    for (int u = 0; u < kNvlsU; ++u) {
      const size_t v = lo + (size_t)u * 32;
      if (v < c_hi) r[u] = mc_ld_add<DT>(mc + v * 16);
    }
#pragma unroll
    for (int u = 0; u < kNvlsU; ++u) {
      const size_t v = lo + (size_t)u * 32;
      if (v >= c_hi) continue;
      if (OP == RP_MEAN || OP == RP_PREMEAN) {
        Pack16<T> p;
        p.u = r[u];
#pragma unroll
        for (int e = 0; e < (int)(16 / sizeof(T)); ++e) p.e[e] = from_f32<T>(to_acc(p.e[e]) * inv);
        r[u] = p.u;
      }
      mc_st(mc + v * 16, r[u]);
    }
    j = next;
  }
  if (!phase_end(a, rank, 1, pb)) return;
  dyn_finish(a, rank, 2, pb);
  rp_trace(a, 7);
}

// ===========================================================================
// K4n: NVLS broadcast (destination in the multicast-bound region)
//   barrier 0 (every rank is done with the destination's previous contents)
//   root only, per-warp tiles: v = its local source (any local buffer),
//     multimem.st(mc + v): the switch writes the same 16 bytes into every rank's copy
//   barrier 1 (the root's stores landed everywhere)
// Root egress S and every rank's ingress S -- the broadcast lower bound, with no
// relay step (the P2P scatter + all-gather moves 2(N-1)/N*S through every link).
// A copy, so bit-exact (graph.py:538-540 pick0).
// ===========================================================================
template <bool ROOT_UNUSED = false>
__global__ void __launch_bounds__(kNvlsThreads) bcast_nvls(const CollArgs a) {
  const int rank = a.rank;
  if (rp_aborted(a.t, rank)) return;
  char* mc = (char*)a.dst[rank];  // multicast view of the destination
  const char* src = (const char*)a.src[rank];
  const size_t V = a.count / 16;
  constexpr uint32_t tv = 32 * kNvlsU;
  const uint32_t nt = (uint32_t)((V + tv - 1) / tv);
  const int lane = threadIdx.x & 31;
  rp_trace(a, 0);
  const PhaseBase pb = phase_begin(a, rank);
  if (!phase_end(a, rank, 0, pb)) return;
  if (rank == a.root) {
    uint32_t j = claim_tile(a, rank, 1);
    while (j < nt) {
      const uint32_t next = claim_tile(a, rank, 1);
      const size_t lo = (size_t)j * tv + lane;
      uint4 r[kNvlsU];
#pragma unroll
      for (int u = 0; u < kNvlsU; ++u) {
        const size_t v = lo + (size_t)u * 32;
        if (v < V) r[u] = ld128_stream(src + v * 16);
      }
#pragma unroll
      for (int u = 0; u < kNvlsU; ++u) {
        const size_t v = lo + (size_t)u * 32;
        if (v < V) mc_st(mc + v * 16, r[u]);
      }
      j = next;
    }
  }
  if (!phase_end(a, rank, 1, pb)) return;
  dyn_finish(a, rank, 2, pb);
  rp_trace(a, 7);
}


// ===========================================================================
// K4r: pipelined relay broadcast (multi-process, large messages)
// The message is cut into tiles; tile i belongs to non-root "owner" i mod (N-1).
//   root : src tile -> owner's landing area (NVLink store), own dst; flag owner
//   owner: waits for its flag, landing -> every other non-root's landing (NVLink)
//          and its own dst; flags them
//   other: waits for its flag, landing -> own dst
// Every rank claims tiles in index order (per-warp claims), so a tile's chain
// root -> owner -> others only ever waits on work of the same tile that was
// claimed earlier -- no deadlock with any number of resident warps. The root's
// egress carries S once, every non-root's ingress S and egress (N-2)/(N-1)*S:
// the broadcast bound with P2P stores (no multicast protocol overhead), and the
// tiles pipeline the two hops. Flags are per-tile epochs (this call's phase-0
// base + 1, equal on every rank) in a region only this kernel writes, so they
// never need resetting. One trailing rank barrier: the next call may write the
// landing areas only after every rank has copied out of them.
// a.write_off = landing offset (staging, or the dst itself when it is
// pool-resident: copy_out = 0), a.read_off = flag-region offset, a.tile_v =
// 16-byte vectors per tile.
// ===========================================================================
// Block-wide copy of bytes [lo, hi) from s to nd destinations (16-byte vectors,
// kRelayU in flight per thread; bytes when a pointer is misaligned).
template <int kRelayU>
__device__ __forceinline__ void relay_copy(const char* s, char* const* d, int nd, size_t lo, size_t hi) {
  bool al = (((uintptr_t)s) & 15u) == 0;
  for (int k = 0; k < nd; ++k) al = al && ((((uintptr_t)d[k]) & 15u) == 0);
  if (al) {
    const size_t step = (size_t)blockDim.x * 16 * kRelayU;
    for (size_t base = lo + (size_t)threadIdx.x * 16; base < hi; base += step) {
      uint4 r[kRelayU];
#pragma unroll
      for (int u = 0; u < kRelayU; ++u) {
        const size_t o = base + (size_t)u * blockDim.x * 16;
        if (o < hi) r[u] = ld128(s + o);
      }
#pragma unroll
      for (int u = 0; u < kRelayU; ++u) {
        const size_t o = base + (size_t)u * blockDim.x * 16;
        if (o < hi)
          for (int k = 0; k < nd; ++k) st128(d[k] + o, r[u]);
      }
    }
  } else {  // a misaligned user pointer on this rank: bytes
    for (size_t o = lo + threadIdx.x; o < hi; o += blockDim.x) {
      const char v = s[o];
      for (int k = 0; k < nd; ++k) d[k][o] = v;
    }
  }
}

// Publish this block's tile: every thread's stores happen-before thread 0's
// system fence (bar.sync orders them), then the flag stores.
__device__ __forceinline__ void relay_publish(const CollArgs& a, const int* q, int nq, uint32_t i, uint32_t epoch) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    for (int k = 0; k < nq; ++k) st_relaxed_sys((uint32_t*)(a.t.data[q[k]] + a.read_off) + i, epoch);
  }
}

// Claim the next tile index of `counter` (one atomic per block, index order).
__device__ __forceinline__ uint32_t relay_claim(const CollArgs& a, int rank, int counter) {
  __shared__ uint32_t s_tile;
  __syncthreads();
  if (threadIdx.x == 0) s_tile = atomicAdd(a.t.sig[rank] + (size_t)RP_CTR_ROW * RP_MAX_RANKS + counter, 1u);
  __syncthreads();
  return s_tile;
}

// Block-wide wait for tile i's flag (thread 0 spins; every thread then acquires it).
__device__ __forceinline__ bool relay_wait(const CollArgs& a, int rank, const uint32_t* f, uint32_t epoch) {
  __shared__ int s_ok;
  if (threadIdx.x == 0) s_ok = wait_reach(a.t, a.world, a.timeout_ns, rank, f, epoch) ? 1 : 0;
  __syncthreads();
  if (!s_ok) return false;
  (void)ld_acquire_sys(f);
  return true;
}

// Roles: the root pushes every tile (claim counter 1). A non-root's blocks split:
// even blocks FORWARD the tiles it owns (wait for the root's flag, store to the
// other non-roots and its own dst, publish) on counter 1, odd blocks RECEIVE the
// tiles others own (wait for the owner's flag, copy the landing area to dst) on
// counter 2. Forwarding never waits on receiving, so blocks parked on flags never
// starve the relays (one role for every block left them ~1/(N-1) of the SMs).
// Landing in a pool-resident dst there is nothing to receive: all blocks forward.
template <int MINB>
__global__ void __launch_bounds__(kThreads, MINB) bcast_relay(const CollArgs a) {
  constexpr int kU = MINB > 1 ? 4 : 8;  // 16-byte vectors in flight per thread
  const int rank = a.rank, W = a.world, root = a.root;
  if (rp_aborted(a.t, rank)) return;
  const size_t B = a.count;
  const size_t tb = (size_t)a.tile_v * 16;
  const uint32_t nt = (uint32_t)((B + tb - 1) / tb);
  rp_trace(a, 0);
  const PhaseBase pb = phase_begin(a, rank);
  // landing straight in a pool-resident dst: every receiver must have entered the
  // call (its earlier writes to dst are done) before anyone stores into it
  if (a.copy_in && !phase_end(a, rank, 0, pb)) return;
  const uint32_t epoch = pb.seen[1] + 1u;  // equal on every rank
  uint32_t* myflags = (uint32_t*)(a.t.data[rank] + a.read_off);
  const char* land = a.t.data[rank] + a.write_off;
  char* dst = (char*)a.dst[rank];
  const char* src = (const char*)a.src[rank];
  const uint32_t W1 = (uint32_t)(W - 1);
  const int me = rank < root ? rank : rank - 1;  // this non-root's owner index
  const bool split = rank != root && a.copy_out && W > 2 && gridDim.x > 1;
  // a.relay_root_blocks > 0 caps the blocks the root pushes with (A/B knob: fewer
  // tiles in progress start the relays earlier, but each SM's NVLink stores
  // sustain only ~5 GB/s, so the root needs every block -- 64 blocks: 786 vs 433 us
  // at 256 MiB, N=4; profiles/r01_relay_ab.txt)
  const bool fwd = rank == root ? (a.relay_root_blocks <= 0 || (int)blockIdx.x < a.relay_root_blocks)
                                : (!split || (blockIdx.x & 1) == 0);
  const bool recv = rank != root && a.copy_out && W > 2 && (!split || (blockIdx.x & 1) == 1);
  bool ok = true;
  char* d[RP_MAX_RANKS];
  int q[RP_MAX_RANKS];
  if (fwd) {
    for (uint32_t k = relay_claim(a, rank, 1);; k = relay_claim(a, rank, 1)) {
      int nd = 0, nq = 0;
      if (rank == root) {
        const uint32_t i = k;
        if (i >= nt) break;
        const size_t lo = (size_t)i * tb, hi = std::min(lo + tb, B);
        const int o = (int)(i % W1);
        const int owner = o < root ? o : o + 1;
        d[nd++] = a.t.data[owner] + a.write_off;
        if (dst != src) d[nd++] = dst;
        relay_copy<kU>(src, d, nd, lo, hi);
        q[nq++] = owner;
        relay_publish(a, q, nq, i, epoch);
        continue;
      }
      const uint32_t i = (uint32_t)me + k * W1;  // the k-th tile this rank owns
      if (i >= nt) break;
      const size_t lo = (size_t)i * tb, hi = std::min(lo + tb, B);
      if (!(ok = relay_wait(a, rank, myflags + i, epoch))) break;
      for (int p = 0; p < W; ++p)
        if (p != root && p != rank) {
          d[nd++] = a.t.data[p] + a.write_off;
          q[nq++] = p;
        }
      if (a.copy_out) d[nd++] = dst;
      if (nd) relay_copy<kU>(land, d, nd, lo, hi);
      if (nq) relay_publish(a, q, nq, i, epoch);
    }
  }
  if (recv && ok) {
    const uint32_t W2 = (uint32_t)(W - 2);
    for (uint32_t j = relay_claim(a, rank, 2);; j = relay_claim(a, rank, 2)) {
      const uint32_t r = j % W2;
      const uint32_t i = (j / W2) * W1 + (r < (uint32_t)me ? r : r + 1);  // j-th tile owned by others
      if (i >= nt) break;
      const size_t lo = (size_t)i * tb, hi = std::min(lo + tb, B);
      if (!(ok = relay_wait(a, rank, myflags + i, epoch))) break;
      d[0] = dst;
      relay_copy<kU>(land, d, 1, lo, hi);
    }
  }
  if (!ok) return;  // the abort word is set: every rank leaves its waits
  if (!phase_end(a, rank, 1, pb)) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) {  // dyn_finish for the phases this call used
    if (a.copy_in) state_store(a.t, rank, RP_ST_PH_SEEN + 0, pb.seen[0] + 1u);
    state_store(a.t, rank, RP_ST_PH_SEEN + 1, pb.seen[1] + 1u);
    for (int k = 0; k < 3; ++k) {
      state_store(a.t, rank, RP_CTR_ROW * RP_MAX_RANKS + k, 0u);
      state_store(a.t, rank, RP_CTR_ROW * RP_MAX_RANKS + 4 + k, 0u);
    }
  }
  rp_trace(a, 7);
}

}  // namespace rp

using namespace rp;

int rp_relay_bcast_launch(rp_comm* c, const void* src, void* dst, size_t bytes, int root, bool land_in_dst,
                          size_t land_off, cudaStream_t stream,
                          int (*dyn)(rp_comm*, const void*, CollArgs&, cudaStream_t, const char*, int, int, uint32_t),
                          CollArgs& a) {
  if (bytes % 16) return rp_fail(RP_ERR_INVALID, "broadcast(relay): bytes must be a multiple of 16");
  const size_t V = bytes / 16;
  // one tile per block at a time (one system fence per tile published); 64 KiB
  // by default, RP_RELAY_TILE_KB overrides (A/B)
  size_t tmin = 4096;
  if (const char* e = getenv("RP_RELAY_TILE_KB")) tmin = std::max<size_t>(512, (size_t)atoi(e) * 64);
  size_t tv = std::max<size_t>(tmin, (V + RP_FLAG_WORDS - 1) / RP_FLAG_WORDS);
  tv = (tv + 511) / 512 * 512;
  a.count = bytes;
  a.root = root;
  a.chunk = V;
  a.src[c->rank] = src;
  a.dst[c->rank] = dst;
  a.write_off = land_off;
  a.read_off = c->tile_flags();
  a.copy_in = land_in_dst ? 1 : 0;  // entry barrier (see the kernel)
  a.relay_root_blocks = 0;  // all
  if (const char* e = getenv("RP_RELAY_ROOT_BLOCKS")) a.relay_root_blocks = std::max(0, atoi(e));
  a.copy_out = land_in_dst ? 0 : 1;
  const char* occ = getenv("RP_RELAY_OCC");
  // 2 blocks per SM (4 vectors in flight per thread) measured best: N=4 256 MiB
  // 432 vs 539 us at 1 block per SM (profiles/r01_relay_ab.txt)
  const void* fn = (occ && occ[0] == '1') ? (const void*)bcast_relay<1> : (const void*)bcast_relay<2>;
  return dyn(c, fn, a, stream, "bcast_relay", 0, kThreads, (uint32_t)tv);
}

int rp_nvls_bcast_launch(rp_comm* c, const void* src, void* dst, size_t bytes, int root, cudaStream_t stream,
                         int (*dyn)(rp_comm*, const void*, CollArgs&, cudaStream_t, const char*, int, int, uint32_t),
                         CollArgs& a) {
  NvlsState* s = nvls_of(c);
  if (!s || !s->bound) return rp_fail(RP_ERR_CONFIG, "broadcast(nvls): NVLS region not set up");
  if (!rp_nvls_covers(c, dst, bytes) || bytes % 16)
    return rp_fail(RP_ERR_INVALID, "broadcast(nvls): dst must be a 16-byte multiple inside the NVLS region");
  if (c->rank == root && ((uintptr_t)src % 16)) {  // misaligned source: multicast from dst
    RP_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, stream));
    src = dst;
  }
  const size_t off = (size_t)((const char*)dst - (const char*)s->uc_va);
  a.count = bytes;
  a.root = root;
  a.chunk = bytes / 16;
  a.src[c->rank] = src;
  a.dst[c->rank] = (void*)(s->mc_va + off);
  a.copy_in = a.copy_out = 0;
  return dyn(c, (const void*)bcast_nvls<false>, a, stream, "bcast_nvls", c->num_sms, kNvlsThreads, 32 * kNvlsU);
}

int rp_nvls_launch(rp_comm* c, const void* buf, size_t count, int dtype, int op, cudaStream_t stream,
                   int (*dyn)(rp_comm*, const void*, CollArgs&, cudaStream_t, const char*, int, int, uint32_t), CollArgs& a) {
  NvlsState* s = nvls_of(c);
  if (!s || !s->bound) return rp_fail(RP_ERR_CONFIG, "all_reduce(nvls): NVLS region not set up");
  const char* p = (const char*)buf;
  const char* base = (const char*)s->uc_va;
  const size_t esz = rp_dtype_size(dtype);
  if (p < base || p + count * esz > base + s->size)
    return rp_fail(RP_ERR_INVALID, "all_reduce(nvls): buffer must live in the NVLS region (in place)");
  if (dtype != RP_F32 && dtype != RP_BF16 && dtype != RP_F16)
    return rp_fail(RP_ERR_INVALID, "all_reduce(nvls): f32 / bf16 / f16 only");
  if (op == RP_MAX) return rp_fail(RP_ERR_INVALID, "all_reduce(nvls): sum / mean / premean only");
  const size_t off = (size_t)(p - base);
  if (off % 16) return rp_fail(RP_ERR_INVALID, "all_reduce(nvls): buffer must be 16-byte aligned");
  const size_t V = (count + (16 / esz) - 1) / (16 / esz);
  if (off + V * 16 > s->size) return rp_fail(RP_ERR_INVALID, "all_reduce(nvls): buffer tail exceeds the region");
  a.count = count;
  a.chunk = (V + c->world - 1) / c->world;
  const void* fn = nullptr;
#define RP_N(DT)                                                                       \
  if (dtype == DT) {                                                                   \
    if (op == RP_SUM) fn = (const void*)ar_nvls<DT, RP_SUM>;                            \
    else if (op == RP_MEAN) fn = (const void*)ar_nvls<DT, RP_MEAN>;                     \
    else fn = (const void*)ar_nvls<DT, RP_PREMEAN>;                                    \
  }
  RP_N(RP_F32)
  RP_N(RP_BF16)
  RP_N(RP_F16)
#undef RP_N
  a.src[c->rank] = (const void*)(s->mc_va + off);  // the kernel's multicast view
  a.copy_in = a.copy_out = 0;
  return dyn(c, fn, a, stream, "nvls", c->num_sms, kNvlsThreads, 32 * kNvlsU);
}

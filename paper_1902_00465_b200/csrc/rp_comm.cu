// Communicator lifecycle, topology discovery, the exported C ABI (include/rp.h)
// and the K6 fusion-buffer pack/unpack kernels.
//
// Bootstrap: each rank allocates one device region [signals | data pool], exports
// a CUDA IPC handle, and the caller exchanges the blobs (torch.distributed over
// NCCL/gloo, used ONLY for this). rp_comm_import maps every peer's region into
// this process, so kernels address peers' pools as plain device pointers that
// resolve over NVLink/NVSwitch. Replaces the reference's transport layer
// and its communicator (graph.py:565-583).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvml.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <string>

#include "rp_device.cuh"

static thread_local std::string g_last_error;

void rp_set_error(const std::string& msg) { g_last_error = msg; }
int rp_fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

size_t rp_dtype_size(int dtype) {
  switch (dtype) {
    case RP_F32: return 4;
    case RP_F64: return 8;
    case RP_BF16: return 2;
    case RP_F16: return 2;
  }
  return 0;
}
bool rp_dtype_valid(int dtype) { return rp_dtype_size(dtype) != 0; }

int rp_set_device_from_ptr(const void* p) {
  cudaPointerAttributes at;
  RP_CUDA_CHECK(cudaPointerGetAttributes(&at, p));
  if (at.type != cudaMemoryTypeDevice && at.type != cudaMemoryTypeManaged)
    return rp_fail(RP_ERR_INVALID, "expected a device pointer");
  RP_CUDA_CHECK(cudaSetDevice(at.device));
  return RP_OK;
}

static const uint64_t kMagic = 0x52505f434f4d4d31ull;  // "RP_COMM1"

int rp_blocks_per_rank(rp_comm* c, const void* func, int threads, int want) {
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, func, threads, 0) != cudaSuccess || occ < 1) occ = 1;
  // Every block of every (virtual) rank must be co-resident: blocks wait on
  // their peers' blocks of the same index.
  int cap = occ * c->num_sms;
  if (c->is_virtual) cap /= c->world;
  cap = std::min(cap, RP_MAX_BLOCKS);
  if (c->cap() > 0) cap = std::min(cap, c->cap());
  return std::max(1, std::min(want, cap));
}

int64_t rp_wave_per_rank(rp_comm* c, int per_sm) {
  int64_t w = (int64_t)std::max(per_sm, 1) * c->num_sms;
  if (c->is_virtual) w /= c->world;
  if (c->cap() > 0) w = std::min<int64_t>(w, c->cap());
  return std::max<int64_t>(w, 1);
}

int rp_launch(rp_comm* c, const void* func, dim3 grid, dim3 block, void** args, size_t smem,
              cudaStream_t stream, bool coop) {
  cudaError_t e;
  if (coop && c->is_virtual && c->world > 1)
    e = cudaLaunchCooperativeKernel(func, grid, block, args, smem, stream);
  else
    e = cudaLaunchKernel(func, grid, block, args, smem, stream);
  if (e != cudaSuccess) return rp_fail(RP_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
  return RP_OK;
}

// ---------------------------------------------------------------------------
// K6: multi-tensor pack / unpack with fused cast (one launch per <=96 tensors)
// ---------------------------------------------------------------------------
namespace rp {

constexpr int kPackMax = 96;
constexpr int kPackThreads = 256;
constexpr int kPackElemsPerBlock = 8192;

struct PackTable {
  const void* ptr[kPackMax];  // tensor data (src for pack, dst for unpack)
  int64_t count[kPackMax];
  int64_t off[kPackMax];      // element offset in the flat buffer
  int32_t block0[kPackMax + 1];
  int n;
};

template <typename S, typename D>
__device__ __forceinline__ void copy_cast(D* dst, const S* src, int64_t n) {
  // 8 elements per step; vector path when both sides are 16-byte aligned
  const bool al = ((((uintptr_t)dst) | ((uintptr_t)src)) & 15u) == 0;
  int64_t i = 0;
  if (al) {
    const int64_t nv = n / 8;
    for (int64_t v = threadIdx.x; v < nv; v += blockDim.x) {
      S s[8];
      D d[8];
      if constexpr (sizeof(S) == 2) {
        *(uint4*)s = ld128_stream(src + v * 8);
      } else if constexpr (sizeof(S) == 4) {
        *(uint4*)s = ld128_stream(src + v * 8);
        *(uint4*)(s + 4) = ld128_stream(src + v * 8 + 4);
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) *(uint4*)(s + 2 * k) = ld128_stream(src + v * 8 + 2 * k);
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) d[k] = convert<D>(s[k]);
      if constexpr (sizeof(D) == 2) {
        st128(dst + v * 8, *(uint4*)d);
      } else if constexpr (sizeof(D) == 4) {
        st128(dst + v * 8, *(uint4*)d);
        st128(dst + v * 8 + 4, *(uint4*)(d + 4));
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) st128(dst + v * 8 + 2 * k, *(uint4*)(d + 2 * k));
      }
    }
    i = nv * 8;
  }
  for (int64_t j = i + threadIdx.x; j < n; j += blockDim.x) dst[j] = convert<D>(src[j]);
}

template <typename S, typename D, bool PACK>
__global__ void __launch_bounds__(kPackThreads) pack_kernel(const PackTable t, void* flat) {
  // locate this block's tensor (block0 is a prefix sum of blocks per tensor)
  int lo = 0, hi = t.n - 1;
  const int b = blockIdx.x;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (t.block0[mid] <= b) lo = mid;
    else hi = mid - 1;
  }
  const int i = lo;
  const int64_t start = (int64_t)(b - t.block0[i]) * kPackElemsPerBlock;
  const int64_t n = std::min<int64_t>(kPackElemsPerBlock, t.count[i] - start);
  if (n <= 0) return;
  if (PACK) {
    copy_cast<S, D>((D*)flat + t.off[i] + start, (const S*)t.ptr[i] + start, n);
  } else {
    copy_cast<S, D>((D*)t.ptr[i] + start, (const S*)flat + t.off[i] + start, n);
  }
}

template <bool PACK>
const void* pick_pack(int s, int d) {
#define RP_P(SD, ST, DD, DT) \
  if (s == SD && d == DD) return (const void*)pack_kernel<ST, DT, PACK>;
  RP_P(RP_F32, float, RP_F32, float)
  RP_P(RP_F32, float, RP_BF16, __nv_bfloat16)
  RP_P(RP_F32, float, RP_F16, __half)
  RP_P(RP_BF16, __nv_bfloat16, RP_F32, float)
  RP_P(RP_F16, __half, RP_F32, float)
  RP_P(RP_BF16, __nv_bfloat16, RP_BF16, __nv_bfloat16)
  RP_P(RP_F16, __half, RP_F16, __half)
  RP_P(RP_F64, double, RP_F64, double)
#undef RP_P
  return nullptr;
}

}  // namespace rp

using namespace rp;

static int pack_common(bool pack, void* flat, int dtype_flat, const void* const* ptrs, const int64_t* counts,
                       const int64_t* offs, int n, int dtype_t, cudaStream_t stream) {
  const void* fn = pack ? pick_pack<true>(dtype_t, dtype_flat) : pick_pack<false>(dtype_flat, dtype_t);
  if (!fn) return rp_fail(RP_ERR_INVALID, "pack/unpack: unsupported dtype pair");
  if (n <= 0) return RP_OK;
  int rc = rp_set_device_from_ptr(flat);
  if (rc) return rc;
  for (int base = 0; base < n; base += kPackMax) {
    PackTable t;
    memset(&t, 0, sizeof(t));
    t.n = std::min(kPackMax, n - base);
    int blocks = 0;
    for (int i = 0; i < t.n; ++i) {
      t.ptr[i] = ptrs[base + i];
      t.count[i] = counts[base + i];
      t.off[i] = offs[base + i];
      t.block0[i] = blocks;
      blocks += (int)((counts[base + i] + kPackElemsPerBlock - 1) / kPackElemsPerBlock);
    }
    t.block0[t.n] = blocks;
    if (blocks == 0) continue;
    void* args[] = {&t, &flat};
    cudaError_t e = cudaLaunchKernel(fn, dim3(blocks), dim3(kPackThreads), args, 0, stream);
    if (e != cudaSuccess) return rp_fail(RP_ERR_CUDA, std::string("pack launch: ") + cudaGetErrorString(e));
  }
  return RP_OK;
}

// ---------------------------------------------------------------------------
// topology discovery
// ---------------------------------------------------------------------------

// NVML, loaded at run time (no link-time dependency).
typedef nvmlReturn_t (*nvml_by_pci_t)(const char*, nvmlDevice_t*);
typedef nvmlReturn_t (*nvml_p2p_t)(nvmlDevice_t, nvmlDevice_t, nvmlGpuP2PCapsIndex_t, nvmlGpuP2PStatus_t*);
typedef nvmlReturn_t (*nvml_link_state_t)(nvmlDevice_t, unsigned int, nvmlEnableState_t*);
struct NvmlApi {
  nvml_by_pci_t by_pci = nullptr;
  nvml_p2p_t p2p = nullptr;
  nvml_link_state_t link_state = nullptr;
};
static const NvmlApi& nvml() {
  static std::mutex mu;
  static NvmlApi api;
  static bool tried = false;
  std::lock_guard<std::mutex> g(mu);
  if (!tried) {
    tried = true;
    if (void* h = dlopen("libnvidia-ml.so.1", RTLD_NOW | RTLD_LOCAL)) {
      typedef nvmlReturn_t (*init_t)(void);
      init_t init = (init_t)dlsym(h, "nvmlInit_v2");
      if (init && init() == NVML_SUCCESS) {
        api.by_pci = (nvml_by_pci_t)dlsym(h, "nvmlDeviceGetHandleByPciBusId_v2");
        api.p2p = (nvml_p2p_t)dlsym(h, "nvmlDeviceGetP2PStatus");
        api.link_state = (nvml_link_state_t)dlsym(h, "nvmlDeviceGetNvLinkState");
      }
    }
  }
  return api;
}
static bool nvml_device(int dev, nvmlDevice_t* out) {
  char bus[32];
  return nvml().by_pci && cudaDeviceGetPCIBusId(bus, sizeof(bus), dev) == cudaSuccess &&
         nvml().by_pci(bus, out) == NVML_SUCCESS;
}

// NVLink P2P status of a pair: 1 (NVLink P2P), 0 (no NVLink between them) or -1
// (NVML unavailable).
static int nvml_nvlink_p2p(int dev_a, int dev_b, std::string* why) {
  nvmlDevice_t na, nb;
  if (!nvml().p2p || !nvml_device(dev_a, &na) || !nvml_device(dev_b, &nb)) {
    *why = "NVML unavailable: cannot confirm NVLink";
    return -1;
  }
  nvmlGpuP2PStatus_t st = NVML_P2P_STATUS_UNKNOWN;
  if (nvml().p2p(na, nb, NVML_P2P_CAPS_INDEX_NVLINK, &st) != NVML_SUCCESS) {
    *why = "nvmlDeviceGetP2PStatus failed";
    return -1;
  }
  if (st != NVML_P2P_STATUS_OK) *why = "NVML reports no NVLink P2P (status " + std::to_string((int)st) + ")";
  return st == NVML_P2P_STATUS_OK ? 1 : 0;
}

// Active NVLink links of a device (an NVSwitch B200 has 18), -1 when unknown.
static int nvml_active_links(int dev) {
  nvmlDevice_t d;
  if (!nvml().link_state || !nvml_device(dev, &d)) return -1;
  int n = 0;
  for (unsigned l = 0; l < NVML_NVLINK_MAX_LINKS; ++l) {
    nvmlEnableState_t st = NVML_FEATURE_DISABLED;
    if (nvml().link_state(d, l, &st) == NVML_SUCCESS && st == NVML_FEATURE_ENABLED) ++n;
  }
  return n;
}

// Link from this rank to peer `me_or_peer` (include/rp.h RP_LINK_*).
int rp_classify_link(rp_comm* c, const RpExport& me, const RpExport& peer, bool self, std::string* why) {
  if (self) return RP_LINK_SELF;
  if (memcmp(peer.uuid, me.uuid, 16) == 0) {
    if (peer.pid == me.pid && peer.loopback && me.loopback) return RP_LINK_LOOPBACK;
    *why = "shares this rank's GPU (use a virtual communicator, or a loopback world in one process)";
    return RP_LINK_SAME_DEVICE;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess) ndev = 0;
  for (int d = 0; d < ndev; ++d) {
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, d) != cudaSuccess) continue;
    if (memcmp(&prop.uuid, peer.uuid, 16) != 0) continue;
    int ok = 0, acc = 0;
    cudaDeviceCanAccessPeer(&ok, c->device, d);
    cudaDeviceGetP2PAttribute(&acc, cudaDevP2PAttrAccessSupported, c->device, d);
    if (!ok || !acc) {
      *why = "no CUDA peer access to device " + std::to_string(d);
      return RP_LINK_NONE;
    }
    const int nv = nvml_nvlink_p2p(c->device, d, why);
    if (nv == 1) return RP_LINK_NVLINK;
    return nv == 0 ? RP_LINK_PCIE : RP_LINK_UNKNOWN;
  }
  *why = "peer GPU is not visible to this process (CUDA_VISIBLE_DEVICES?)";
  return RP_LINK_UNKNOWN;
}

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

int rp_topology_check(int world, int rank, const int* links, int allow_pcie, int loopback) {
  if (!links || world < 1 || world > RP_MAX_RANKS || rank < 0 || rank >= world)
    return rp_fail(RP_ERR_INVALID, "rp_topology_check: bad arguments");
  static const char* names[] = {"self", "NVLink", "PCIe peer access only", "no peer access", "unknown",
                                "same device", "loopback"};
  for (int p = 0; p < world; ++p) {
    const int l = links[p];
    bool ok;
    switch (l) {
      case RP_LINK_SELF: ok = p == rank; break;
      case RP_LINK_NVLINK: ok = true; break;
      case RP_LINK_PCIE: ok = allow_pcie != 0; break;
      case RP_LINK_LOOPBACK: ok = loopback != 0; break;
      default: ok = false;
    }
    if (!ok) {
      const char* n = (l >= 0 && l <= RP_LINK_LOOPBACK) ? names[l] : "invalid";
      return rp_fail(RP_ERR_CONFIG, "topology: rank " + std::to_string(rank) + " -> rank " + std::to_string(p) +
                                        " link is '" + n +
                                        "'; an NVLink/NVSwitch all-to-all is required (no fallback; "
                                        "RP_ALLOW_PCIE=1 accepts PCIe peer access for tests)");
    }
  }
  return RP_OK;
}

const char* rp_last_error(void) { return g_last_error.c_str(); }

const char* rp_version(void) { return "rp 0.1.0 sm_100a"; }

static int init_device(rp_comm* c) {
  RP_CUDA_CHECK(cudaSetDevice(c->device));
  cudaDeviceProp prop;
  RP_CUDA_CHECK(cudaGetDeviceProperties(&prop, c->device));
  c->num_sms = prop.multiProcessorCount;
  if (prop.major < 10)
    return rp_fail(RP_ERR_CONFIG, "device " + std::to_string(c->device) + " (" + prop.name +
                                      ") is not sm_100-class; this library is built for sm_100a only");
  return RP_OK;
}

static int alloc_region(rp_comm* c, int r) {
  char* base = nullptr;
  if (!c->aux) RP_CUDA_CHECK(cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking));
  RP_CUDA_CHECK(cudaMalloc(&base, RP_SIGNAL_BYTES + c->pool_bytes));
  c->alloc[r] = base;
  c->table.sig[r] = (uint32_t*)base;
  c->table.data[r] = base + RP_SIGNAL_BYTES;
  RP_CUDA_CHECK(cudaMemsetAsync(base, 0, RP_SIGNAL_BYTES, c->aux));
  RP_CUDA_CHECK(cudaMemsetAsync(c->table.data[r] + c->tile_flags(), 0, RP_FLAG_BYTES, c->aux));
  RP_CUDA_CHECK(cudaStreamSynchronize(c->aux));
  return RP_OK;
}

int rp_comm_create(int rank, int world, int device, size_t pool_bytes, rp_comm_t* out) {
  if (!out) return rp_fail(RP_ERR_INVALID, "rp_comm_create: out is NULL");
  if (world < 1 || world > RP_MAX_RANKS || rank < 0 || rank >= world)
    return rp_fail(RP_ERR_CONFIG, "rp_comm_create: need 1 <= world <= 8 and 0 <= rank < world");
  if (pool_bytes < RP_MIN_POOL) return rp_fail(RP_ERR_INVALID, "rp_comm_create: pool_bytes must be >= 16 MiB");
  rp_comm* c = new rp_comm();
  c->rank = rank;
  c->world = world;
  c->device = device;
  c->pool_bytes = (pool_bytes + RP_ALIGN - 1) / RP_ALIGN * RP_ALIGN;
  int rc = init_device(c);
  if (!rc) rc = alloc_region(c, rank);
  if (rc) {
    delete c;
    return rc;
  }
  if (world == 1) c->imported = true;
  *out = c;
  return RP_OK;
}

int rp_comm_create_virtual(int world, int device, size_t pool_bytes, rp_comm_t* out) {
  if (!out) return rp_fail(RP_ERR_INVALID, "rp_comm_create_virtual: out is NULL");
  if (world < 1 || world > RP_MAX_RANKS) return rp_fail(RP_ERR_CONFIG, "virtual world must be 1..8");
  if (pool_bytes < RP_MIN_POOL) return rp_fail(RP_ERR_INVALID, "rp_comm_create_virtual: pool_bytes must be >= 16 MiB");
  rp_comm* c = new rp_comm();
  c->world = world;
  c->device = device;
  c->is_virtual = true;
  c->pool_bytes = (pool_bytes + RP_ALIGN - 1) / RP_ALIGN * RP_ALIGN;
  int rc = init_device(c);
  for (int r = 0; r < world && !rc; ++r) rc = alloc_region(c, r);
  if (!rc && world > 1) {
    int coop = 0;
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device);
    if (!coop) rc = rp_fail(RP_ERR_CONFIG, "device lacks cooperative launch (needed by virtual replicas)");
  }
  if (rc) {
    for (int r = 0; r < world; ++r)
      if (c->alloc[r]) cudaFree(c->alloc[r]);
    if (c->aux) cudaStreamDestroy(c->aux);
    delete c;
    return rc;
  }
  c->imported = true;
  *out = c;
  return RP_OK;
}

size_t rp_comm_export_size(void) { return sizeof(RpExport); }

int rp_comm_export(rp_comm_t c, void* buf, size_t* len) {
  if (!c || !buf || !len) return rp_fail(RP_ERR_INVALID, "rp_comm_export: NULL argument");
  if (c->is_virtual) return rp_fail(RP_ERR_INVALID, "rp_comm_export: virtual communicators need no export");
  if (*len < sizeof(RpExport)) return rp_fail(RP_ERR_INVALID, "rp_comm_export: buffer too small");
  RP_CUDA_CHECK(cudaSetDevice(c->device));
  RpExport e;
  memset(&e, 0, sizeof(e));
  e.magic = kMagic;
  e.rank = c->rank;
  e.world = c->world;
  e.pool_bytes = c->pool_bytes;
  RP_CUDA_CHECK(cudaIpcGetMemHandle(&e.handle, c->alloc[c->rank]));
  cudaDeviceProp prop;
  RP_CUDA_CHECK(cudaGetDeviceProperties(&prop, c->device));
  memcpy(e.uuid, &prop.uuid, 16);
  e.pci_bus = prop.pciBusID;
  e.pci_device = prop.pciDeviceID;
  e.pci_domain = prop.pciDomainID;
  e.base = (uint64_t)(uintptr_t)c->alloc[c->rank];
  e.pid = (int32_t)getpid();
  e.loopback = c->loopback ? 1 : 0;
  e.nvlinks = c->loopback ? -1 : nvml_active_links(c->device);
  memcpy(buf, &e, sizeof(e));
  *len = sizeof(e);
  return RP_OK;
}

// Loopback regions are plain pointers shared by the ranks of one process, so a
// region may be freed only once EVERY rank that mapped it has destroyed its
// communicator: a rank that finished (or failed) early must not free memory a
// peer's kernel may still store into (that was an illegal-address fault).
static std::mutex g_lb_mu;
static std::map<char*, int> g_lb_refs;

static void lb_ref(char* base) {
  std::lock_guard<std::mutex> g(g_lb_mu);
  ++g_lb_refs[base];
}
// Drop one reference; true when the caller must free the region.
static bool lb_unref(char* base) {
  std::lock_guard<std::mutex> g(g_lb_mu);
  auto it = g_lb_refs.find(base);
  if (it == g_lb_refs.end()) return false;
  if (--it->second > 0) return false;
  g_lb_refs.erase(it);
  return true;
}

int rp_comm_import(rp_comm_t c, const void* all, size_t len) {
  if (!c || !all) return rp_fail(RP_ERR_INVALID, "rp_comm_import: NULL argument");
  if (c->is_virtual || c->world == 1) return RP_OK;
  if (len != sizeof(RpExport) * (size_t)c->world)
    return rp_fail(RP_ERR_PROTOCOL, "rp_comm_import: expected world export blobs");
  RP_CUDA_CHECK(cudaSetDevice(c->device));
  const RpExport* ex = (const RpExport*)all;
  for (int p = 0; p < c->world; ++p) {
    if (ex[p].magic != kMagic || ex[p].rank != p || ex[p].world != c->world)
      return rp_fail(RP_ERR_PROTOCOL, "rp_comm_import: blob " + std::to_string(p) + " is not rank " +
                                          std::to_string(p) + " of this world");
    if (ex[p].pool_bytes != c->pool_bytes)
      return rp_fail(RP_ERR_PROTOCOL, "rp_comm_import: ranks disagree on pool_bytes");
    if (ex[p].loopback != (c->loopback ? 1 : 0))
      return rp_fail(RP_ERR_PROTOCOL, "rp_comm_import: ranks disagree on loopback mode");
  }
  // topology discovered at init: classify the link to every peer, then apply the
  // policy (rp_topology_check) -- NVLink P2P to every peer, or a loopback world
  int links[RP_MAX_RANKS];
  std::string why[RP_MAX_RANKS];
  for (int p = 0; p < c->world; ++p) links[p] = rp_classify_link(c, ex[c->rank], ex[p], p == c->rank, &why[p]);
  const char* pe = getenv("RP_ALLOW_PCIE");
  const int allow = (pe && pe[0] == '1') ? 1 : 0;
  int rc = rp_topology_check(c->world, c->rank, links, allow, c->loopback ? 1 : 0);
  int nvl[RP_MAX_RANKS];
  for (int p = 0; p < c->world; ++p) nvl[p] = ex[p].nvlinks;
  if (!rc && !c->loopback && !allow) rc = rp_topology_uniform(c->world, nvl);
  if (rc) {
    for (int p = 0; p < c->world; ++p)
      if (!why[p].empty()) rp_set_error(rp_last_error() + std::string("; rank ") + std::to_string(p) + ": " + why[p]);
    return rc;
  }
  for (int p = 0; p < c->world; ++p) {
    c->links[p] = links[p];
    c->nvlinks[p] = nvl[p];
  }
  if (c->loopback) {
    for (int p = 0; p < c->world; ++p) lb_ref(p == c->rank ? c->alloc[c->rank] : (char*)(uintptr_t)ex[p].base);
    c->lb_refs = true;
  }
  for (int p = 0; p < c->world; ++p) {
    if (p == c->rank) continue;
    char* ptr = nullptr;
    if (links[p] == RP_LINK_LOOPBACK) {
      ptr = (char*)(uintptr_t)ex[p].base;  // same process, same device: a plain pointer (not owned)
    } else {
      void* vp = nullptr;
      cudaError_t e = cudaIpcOpenMemHandle(&vp, ex[p].handle, cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess)
        return rp_fail(RP_ERR_CONFIG, "cudaIpcOpenMemHandle(rank " + std::to_string(p) + "): " + cudaGetErrorString(e));
      c->ipc_opened[p] = true;
      c->alloc[p] = (char*)vp;
      ptr = (char*)vp;
    }
    c->table.sig[p] = (uint32_t*)ptr;
    c->table.data[p] = ptr + RP_SIGNAL_BYTES;
  }
  c->imported = true;
  return RP_OK;
}

int rp_loopback_prepare(int device) {
  // The stream-ordered allocator may hand one rank's stream memory another rank's
  // stream freed, inserting a wait on that stream (internal dependency). In a
  // loopback world that wait can close a cycle -- stream A waits for B's free
  // point, queued behind B's collective kernel, which waits for A's next kernel --
  // so cross-stream reuse is limited to frees that already completed
  // (opportunistic) or that the caller ordered (event dependencies).
  RP_CUDA_CHECK(cudaSetDevice(device));
  cudaMemPool_t pools[2] = {nullptr, nullptr};
  RP_CUDA_CHECK(cudaDeviceGetDefaultMemPool(&pools[0], device));
  RP_CUDA_CHECK(cudaDeviceGetMemPool(&pools[1], device));
  for (cudaMemPool_t p : pools) {
    int off = 0;
    RP_CUDA_CHECK(cudaMemPoolSetAttribute(p, cudaMemPoolReuseAllowInternalDependencies, &off));
  }
  return RP_OK;
}

int rp_topology_uniform(int world, const int* nvlinks) {
  if (!nvlinks || world < 1 || world > RP_MAX_RANKS) return rp_fail(RP_ERR_INVALID, "rp_topology_uniform: bad arguments");
  for (int p = 0; p < world; ++p) {
    if (nvlinks[p] < 0) continue;  // NVML could not count (the P2P check already required NVLink)
    for (int q = 0; q < p; ++q) {
      if (nvlinks[q] >= 0 && nvlinks[q] != nvlinks[p])
        return rp_fail(RP_ERR_CONFIG, "topology: non-uniform NVLink -- rank " + std::to_string(q) + " has " +
                                          std::to_string(nvlinks[q]) + " active links, rank " + std::to_string(p) +
                                          " has " + std::to_string(nvlinks[p]) +
                                          " (an NVSwitch all-to-all gives every GPU the same links)");
    }
    if (nvlinks[p] == 0)
      return rp_fail(RP_ERR_CONFIG, "topology: rank " + std::to_string(p) + " has no active NVLink link");
  }
  return RP_OK;
}

int rp_comm_topology(rp_comm_t c, int* links, int* nvlinks) {
  if (!c || !links || !nvlinks) return rp_fail(RP_ERR_INVALID, "rp_comm_topology: NULL argument");
  for (int p = 0; p < c->world; ++p) {
    links[p] = c->is_virtual ? RP_LINK_SELF : (c->world == 1 ? RP_LINK_SELF : c->links[p]);
    nvlinks[p] = c->is_virtual || c->world == 1 ? -1 : c->nvlinks[p];
  }
  return RP_OK;
}

int rp_comm_set_loopback(rp_comm_t c, int on) {
  if (!c) return rp_fail(RP_ERR_INVALID, "rp_comm_set_loopback: NULL comm");
  if (c->is_virtual) return rp_fail(RP_ERR_INVALID, "rp_comm_set_loopback: virtual communicators are already local");
  if (c->imported && c->world > 1) return rp_fail(RP_ERR_INVALID, "rp_comm_set_loopback: call before rp_comm_import");
  c->loopback = on != 0;
  // every rank's blocks must be co-resident with every other rank's: at most
  // num_sms / world blocks per rank, each at most one SM, so an empty SM always
  // exists while any block of the world is still unscheduled
  c->loopback_cap = c->loopback ? std::max(1, c->num_sms / c->world) : 0;
  return RP_OK;
}

int rp_comm_destroy(rp_comm_t c) {
  if (!c) return RP_OK;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  rp_release_registrations(c);
  rp_nvls_destroy(c);
  if (c->lb_refs) {
    // every rank's region, freed by whichever rank lets go of it last
    for (int r = 0; r < c->world; ++r) {
      char* base = (char*)c->table.sig[r];
      if (base && lb_unref(base)) cudaFree(base);
    }
  } else {
    for (int r = 0; r < RP_MAX_RANKS; ++r) {
      if (!c->alloc[r]) continue;
      if (c->ipc_opened[r]) cudaIpcCloseMemHandle(c->alloc[r]);
      else if (r == c->rank || c->is_virtual) cudaFree(c->alloc[r]);
    }
  }
  if (c->aux) cudaStreamDestroy(c->aux);
  if (c->bn_partials) cudaFree(c->bn_partials);
  for (double* p : c->bn_retired) cudaFree(p);
  delete c;
  return RP_OK;
}

int rp_comm_pool(rp_comm_t c, int rank, void** base, size_t* bytes) {
  if (!c || !base || !bytes) return rp_fail(RP_ERR_INVALID, "rp_comm_pool: NULL argument");
  const int r = rank < 0 ? c->rank : rank;
  if (r < 0 || r >= c->world || (!c->is_virtual && r != c->rank))
    return rp_fail(RP_ERR_INVALID, "rp_comm_pool: rank not local to this process");
  *base = c->table.data[r];
  *bytes = c->pool_bytes;
  return RP_OK;
}

int rp_comm_info(rp_comm_t c, int* rank, int* world, int* is_virtual, int* num_sms, size_t* scratch_off) {
  if (!c) return rp_fail(RP_ERR_INVALID, "rp_comm_info: NULL comm");
  if (rank) *rank = c->rank;
  if (world) *world = c->world;
  if (is_virtual) *is_virtual = c->is_virtual ? 1 : 0;
  if (num_sms) *num_sms = c->num_sms;
  if (scratch_off) *scratch_off = (c->reserved + RP_ALIGN - 1) / RP_ALIGN * RP_ALIGN;
  return RP_OK;
}

int rp_comm_reserve(rp_comm_t c, size_t bytes) {
  if (!c) return rp_fail(RP_ERR_INVALID, "rp_comm_reserve: NULL comm");
  if (bytes > c->scratch_end()) return rp_fail(RP_ERR_INVALID, "rp_comm_reserve: exceeds pool");
  c->reserved = bytes;
  return RP_OK;
}

int rp_comm_set_timeout(rp_comm_t c, uint64_t ns) {
  if (!c) return rp_fail(RP_ERR_INVALID, "rp_comm_set_timeout: NULL comm");
  c->timeout_ns = ns;
  return RP_OK;
}

int rp_comm_set_block_cap(rp_comm_t c, int blocks) {
  if (!c) return rp_fail(RP_ERR_INVALID, "rp_comm_set_block_cap: NULL comm");
  if (blocks < 0) return rp_fail(RP_ERR_INVALID, "rp_comm_set_block_cap: negative");
  c->block_cap = blocks;
  return RP_OK;
}

int rp_comm_check(rp_comm_t c) {
  if (!c) return rp_fail(RP_ERR_INVALID, "rp_comm_check: NULL comm");
  RP_CUDA_CHECK(cudaSetDevice(c->device));
  // a loopback world shares the device with its peers: a device-wide sync could
  // wait on a peer kernel that waits for this rank's next launch; the caller syncs
  // the streams it launched on instead
  if (!c->loopback) RP_CUDA_CHECK(cudaDeviceSynchronize());
  uint32_t worst = 0, info[3] = {0, 0, 0};
  for (int r = 0; r < c->world; ++r) {
    if (!c->is_virtual && r != c->rank) continue;
    uint32_t w[4] = {0, 0, 0, 0};
    RP_CUDA_CHECK(cudaMemcpyAsync(w, c->table.sig[r] + RP_ABORT_WORD, 16, cudaMemcpyDeviceToHost, c->aux));
    RP_CUDA_CHECK(cudaStreamSynchronize(c->aux));
    if (w[0] > worst || (w[0] == RP_ABORT_TIMEOUT && worst != RP_ABORT_TIMEOUT)) {
      worst = w[0];
      memcpy(info, w + 1, sizeof(info));
    }
  }
  if (worst == RP_ABORT_TIMEOUT) {
    // which signal word the wait was on: row (block index / BN row / phase row) and source rank
    const uint32_t row = info[0] / RP_MAX_RANKS, src = info[0] % RP_MAX_RANKS;
    std::string where = row >= (uint32_t)RP_PH_ROW0 && row < (uint32_t)RP_CTR_ROW
                            ? "phase row " + std::to_string(row - RP_PH_ROW0)
                            : (row >= (uint32_t)RP_BN_ROW0 ? "BN row " : "block row ") + std::to_string(row);
    return rp_fail(RP_ERR_ABORTED, "collective timed out waiting for a peer (dead or diverged rank): " + where +
                                       ", source rank " + std::to_string(src) + ", waited for " +
                                       std::to_string(info[1]) + ", saw " + std::to_string(info[2]));
  }
  if (worst == RP_ABORT_PEER) return rp_fail(RP_ERR_ABORTED, "collective aborted by another rank");
  return RP_OK;
}

static bool ready(rp_comm_t c) { return c && c->imported; }

#define RP_REQUIRE_READY(c, name)                                                        \
  do {                                                                                   \
    if (!ready(c)) return rp_fail(RP_ERR_INVALID, std::string(name) + ": communicator not imported"); \
    cudaSetDevice((c)->device);                                                          \
  } while (0)

int rp_all_reduce(rp_comm_t c, const void* src, void* dst, size_t count, int dtype_in, int dtype_comm,
                  int dtype_out, int op, int algo, void* stream) {
  RP_REQUIRE_READY(c, "rp_all_reduce");
  if (c->is_virtual) return rp_fail(RP_ERR_INVALID, "rp_all_reduce: virtual communicator needs rp_all_reduce_v");
  const void* s[1] = {src};
  void* d[1] = {dst};
  return rp_launch_all_reduce(c, s, d, count, dtype_in, dtype_comm, dtype_out, op, algo, (cudaStream_t)stream);
}

int rp_all_reduce_apply(rp_comm_t c, const void* grad, void* param, size_t count, int dtype_grad, int opt,
                        const double* hyper, float* state0, float* state1, int32_t* step, void* stream) {
  RP_REQUIRE_READY(c, "rp_all_reduce_apply");
  if (c->is_virtual) return rp_fail(RP_ERR_INVALID, "rp_all_reduce_apply: virtual communicator needs rp_all_reduce_apply_v");
  const void* g[1] = {grad};
  void* p[1] = {param};
  float* s0[1] = {state0};
  float* s1[1] = {state1};
  int32_t* st[1] = {step};
  return rp_launch_apply(c, g, p, count, dtype_grad, opt, hyper, s0, s1, st, (cudaStream_t)stream);
}

int rp_all_reduce_apply_v(rp_comm_t c, const void* const* grad, void* const* param, size_t count, int dtype_grad,
                          int opt, const double* hyper, float* const* state0, float* const* state1,
                          int32_t* const* step, void* stream) {
  RP_REQUIRE_READY(c, "rp_all_reduce_apply_v");
  if (!c->is_virtual) return rp_fail(RP_ERR_INVALID, "rp_all_reduce_apply_v: needs a virtual communicator");
  if (!grad || !param) return rp_fail(RP_ERR_INVALID, "rp_all_reduce_apply_v: NULL argument");
  return rp_launch_apply(c, grad, param, count, dtype_grad, opt, hyper, state0, state1, step, (cudaStream_t)stream);
}

int rp_all_reduce_algo(rp_comm_t c, const void* src, const void* dst, size_t count, int dtype_in, int dtype_comm,
                       int dtype_out, int op, int algo, int* chosen) {
  RP_REQUIRE_READY(c, "rp_all_reduce_algo");
  if (!chosen) return rp_fail(RP_ERR_INVALID, "rp_all_reduce_algo: NULL argument");
  if (!rp_dtype_valid(dtype_comm)) return rp_fail(RP_ERR_INVALID, "rp_all_reduce_algo: unknown dtype");
  const void* s[RP_MAX_RANKS] = {src};
  const void* d[RP_MAX_RANKS] = {dst};
  *chosen = rp_resolve_ar_algo(c, s, d, count, dtype_in, dtype_comm, dtype_out, op, algo);
  return RP_OK;
}

int rp_all_reduce_plan(rp_comm_t c, const void* src, const void* dst, size_t count, int dtype_in, int dtype_comm,
                       int dtype_out, int op, int algo, int64_t* plan) {
  RP_REQUIRE_READY(c, "rp_all_reduce_plan");
  if (!plan) return rp_fail(RP_ERR_INVALID, "rp_all_reduce_plan: NULL argument");
  if (!rp_dtype_valid(dtype_in) || !rp_dtype_valid(dtype_comm) || !rp_dtype_valid(dtype_out))
    return rp_fail(RP_ERR_INVALID, "rp_all_reduce_plan: unknown dtype");
  const void* s[RP_MAX_RANKS] = {src};
  const void* d[RP_MAX_RANKS] = {dst};
  rp_plan_all_reduce(c, s, d, count, dtype_in, dtype_comm, dtype_out, op, algo, plan);
  return RP_OK;
}

int rp_all_reduce_v(rp_comm_t c, const void* const* src, void* const* dst, size_t count, int dtype_in,
                    int dtype_comm, int dtype_out, int op, int algo, void* stream) {
  RP_REQUIRE_READY(c, "rp_all_reduce_v");
  if (!c->is_virtual) return rp_fail(RP_ERR_INVALID, "rp_all_reduce_v: needs a virtual communicator");
  return rp_launch_all_reduce(c, src, dst, count, dtype_in, dtype_comm, dtype_out, op, algo, (cudaStream_t)stream);
}

int rp_all_gather(rp_comm_t c, const void* src, void* dst, size_t bytes, void* stream) {
  RP_REQUIRE_READY(c, "rp_all_gather");
  if (c->is_virtual) return rp_fail(RP_ERR_INVALID, "rp_all_gather: virtual communicator needs rp_all_gather_v");
  const void* s[1] = {src};
  void* d[1] = {dst};
  if (c->world == 1) {
    if (dst != src) RP_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
    return RP_OK;
  }
  return rp_launch_all_gather(c, s, d, bytes, (cudaStream_t)stream);
}

int rp_all_gather_v(rp_comm_t c, const void* const* src, void* const* dst, size_t bytes, void* stream) {
  RP_REQUIRE_READY(c, "rp_all_gather_v");
  if (!c->is_virtual) return rp_fail(RP_ERR_INVALID, "rp_all_gather_v: needs a virtual communicator");
  if (c->world == 1) {
    if (dst[0] != src[0])
      RP_CUDA_CHECK(cudaMemcpyAsync(dst[0], src[0], bytes, cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
    return RP_OK;
  }
  return rp_launch_all_gather(c, src, dst, bytes, (cudaStream_t)stream);
}

int rp_broadcast(rp_comm_t c, const void* src, void* dst, size_t bytes, int root, int algo, void* stream) {
  RP_REQUIRE_READY(c, "rp_broadcast");
  if (c->is_virtual) return rp_fail(RP_ERR_INVALID, "rp_broadcast: virtual communicator needs rp_broadcast_v");
  if (c->world == 1) {
    if (dst != src && src) RP_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
    return RP_OK;
  }
  const void* s[1] = {src ? src : dst};
  void* d[1] = {dst};
  return rp_launch_broadcast(c, s, d, bytes, root, algo, (cudaStream_t)stream);
}

int rp_broadcast_v(rp_comm_t c, const void* const* src, void* const* dst, size_t bytes, int root, int algo,
                   void* stream) {
  RP_REQUIRE_READY(c, "rp_broadcast_v");
  if (!c->is_virtual) return rp_fail(RP_ERR_INVALID, "rp_broadcast_v: needs a virtual communicator");
  if (c->world == 1) {
    if (dst[0] != src[0])
      RP_CUDA_CHECK(cudaMemcpyAsync(dst[0], src[0], bytes, cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
    return RP_OK;
  }
  return rp_launch_broadcast(c, src, dst, bytes, root, algo, (cudaStream_t)stream);
}

int rp_bn_stats(rp_comm_t c, const void* x, int dtype, int64_t rows, int64_t ch, int64_t hw, int layout,
                float eps, float* mean, float* var, float* invstd, double* count, void* stream) {
  RP_REQUIRE_READY(c, "rp_bn_stats");
  return rp_launch_bn_stats(c, x, dtype, rows, ch, hw, layout, eps, mean, var, invstd, count, (cudaStream_t)stream);
}

int rp_bn_bwd_stats(rp_comm_t c, const void* x, const void* dy, int dtype, int64_t rows, int64_t ch, int64_t hw,
                    int layout, const float* mean, float* sum_dy, float* sum_dy_xmu, float* local_sum_dy,
                    float* local_sum_dy_xmu, void* stream) {
  RP_REQUIRE_READY(c, "rp_bn_bwd_stats");
  return rp_launch_bn_bwd_stats(c, x, dy, dtype, rows, ch, hw, layout, mean, sum_dy, sum_dy_xmu, local_sum_dy,
                                local_sum_dy_xmu, (cudaStream_t)stream);
}

int rp_pack(void* dst, int dtype_dst, const void* const* ptrs, const int64_t* counts, const int64_t* offs, int n,
            int dtype_src, void* stream) {
  return pack_common(true, dst, dtype_dst, ptrs, counts, offs, n, dtype_src, (cudaStream_t)stream);
}

int rp_unpack(const void* src, int dtype_src, void* const* ptrs, const int64_t* counts, const int64_t* offs, int n,
              int dtype_dst, void* stream) {
  return pack_common(false, (void*)src, dtype_src, (const void* const*)ptrs, counts, offs, n, dtype_dst,
                     (cudaStream_t)stream);
}

}  // extern "C"

// User-buffer registration: a caller-owned buffer (e.g. a torch tensor) mapped on
// every peer once, so in-place all-reduces of it take the zero-copy pull two-shot
// (loads from every peer's copy, stores of the folded chunk into every peer's copy)
// instead of the push form with staging -- the path pool-resident buckets take.
// Multi-process: the buffer's allocation is exported with cudaIpcGetMemHandle (the
// allocation base from cuMemGetAddressRange, plus the buffer's offset in it) and
// opened once per peer allocation (refcounted); a loopback world exchanges plain
// pointers. Collective: every rank registers its corresponding buffer, in the same
// order, so registration indices agree.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <string.h>
#include <unistd.h>

#include <string>

#include "rp_device.cuh"

namespace {

const uint64_t kRegMagic = 0x52505f5245473031ull;  // "RP_REG01"

struct RpRegExport {
  uint64_t magic;
  int32_t rank, pid;
  uint64_t bytes;
  uint64_t ptr;     // the buffer in the exporting process
  uint64_t offset;  // buffer - allocation base
  int32_t has_handle, loopback;
  cudaIpcMemHandle_t handle;  // of the allocation base
};

PFN_cuMemGetAddressRange g_range = nullptr;

int address_range(const void* p, char** base, size_t* size) {
  if (!g_range) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
      return rp_fail(RP_ERR_CONFIG, "CUDA driver entry point cuMemGetAddressRange unavailable");
    g_range = (PFN_cuMemGetAddressRange)fn;
  }
  CUdeviceptr b = 0;
  size_t sz = 0;
  if (g_range(&b, &sz, (CUdeviceptr)(uintptr_t)p) != CUDA_SUCCESS)
    return rp_fail(RP_ERR_INVALID, "register: not a device allocation");
  *base = (char*)(uintptr_t)b;
  *size = sz;
  return RP_OK;
}

}  // namespace

bool rp_registered(rp_comm* c, const void* p, size_t bytes, int* reg, size_t* off) {
  const char* q = (const char*)p;
  for (size_t i = 0; i < c->regs.size(); ++i) {
    const RpReg& r = c->regs[i];
    const char* b = r.ptr[c->rank];
    if (r.live && q >= b && q + bytes <= b + r.bytes) {
      *reg = (int)i;
      *off = (size_t)(q - b);
      return true;
    }
  }
  return false;
}

static void unmap_peer(rp_comm* c, const std::string& key) {
  auto it = c->ipc_cache.find(key);
  if (it == c->ipc_cache.end()) return;
  if (--it->second.second == 0) {
    cudaIpcCloseMemHandle(it->second.first);
    c->ipc_cache.erase(it);
  }
}

void rp_release_registrations(rp_comm* c) {
  for (RpReg& r : c->regs) {
    if (!r.live) continue;
    for (int p = 0; p < RP_MAX_RANKS; ++p)
      if (!r.ipc_key[p].empty()) unmap_peer(c, r.ipc_key[p]);
    r.live = false;
  }
}

extern "C" {

size_t rp_register_export_size(void) { return sizeof(RpRegExport); }

int rp_register_export(rp_comm_t c, const void* ptr, size_t bytes, void* blob, size_t* len) {
  if (!c || !ptr || !blob || !len) return rp_fail(RP_ERR_INVALID, "rp_register_export: NULL argument");
  if (c->is_virtual) return rp_fail(RP_ERR_INVALID, "rp_register_export: virtual replicas share one GPU's memory");
  if (*len < sizeof(RpRegExport)) return rp_fail(RP_ERR_INVALID, "rp_register_export: buffer too small");
  RP_CUDA_CHECK(cudaSetDevice(c->device));
  RpRegExport e;
  memset(&e, 0, sizeof(e));
  e.magic = kRegMagic;
  e.rank = c->rank;
  e.pid = (int32_t)getpid();
  e.bytes = bytes;
  e.ptr = (uint64_t)(uintptr_t)ptr;
  e.loopback = c->loopback ? 1 : 0;
  if (!c->loopback && c->world > 1) {
    char* base = nullptr;
    size_t size = 0;
    int rc = address_range(ptr, &base, &size);
    if (rc) return rc;
    if ((const char*)ptr + bytes > base + size) return rp_fail(RP_ERR_INVALID, "register: buffer exceeds its allocation");
    cudaError_t err = cudaIpcGetMemHandle(&e.handle, base);
    if (err != cudaSuccess)
      return rp_fail(RP_ERR_CONFIG, std::string("register: the buffer's allocation cannot be shared over CUDA IPC (") +
                                        cudaGetErrorString(err) +
                                        "; stream-ordered pool and expandable-segment memory are not IPC-shareable)");
    e.has_handle = 1;
    e.offset = (uint64_t)((const char*)ptr - base);
  }
  memcpy(blob, &e, sizeof(e));
  *len = sizeof(e);
  return RP_OK;
}

int rp_register_import(rp_comm_t c, const void* all, size_t len, int* reg) {
  if (!c || !all || !reg) return rp_fail(RP_ERR_INVALID, "rp_register_import: NULL argument");
  if (!c->imported) return rp_fail(RP_ERR_INVALID, "rp_register_import: communicator not imported");
  if (len != sizeof(RpRegExport) * (size_t)c->world)
    return rp_fail(RP_ERR_PROTOCOL, "rp_register_import: expected world registration blobs");
  RP_CUDA_CHECK(cudaSetDevice(c->device));
  const RpRegExport* ex = (const RpRegExport*)all;
  for (int p = 0; p < c->world; ++p) {
    if (ex[p].magic != kRegMagic || ex[p].rank != p)
      return rp_fail(RP_ERR_PROTOCOL, "rp_register_import: blob " + std::to_string(p) + " is not rank " +
                                          std::to_string(p) + "'s registration");
    if (ex[p].bytes != ex[c->rank].bytes)
      return rp_fail(RP_ERR_PROTOCOL, "rp_register_import: ranks registered buffers of different sizes");
  }
  RpReg r;
  r.bytes = ex[c->rank].bytes;
  for (int p = 0; p < c->world; ++p) {
    if (p == c->rank || (ex[p].loopback && ex[p].pid == (int32_t)getpid())) {
      r.ptr[p] = (char*)(uintptr_t)ex[p].ptr;
      continue;
    }
    if (!ex[p].has_handle) return rp_fail(RP_ERR_PROTOCOL, "rp_register_import: peer exported no IPC handle");
    const std::string key((const char*)&ex[p].handle, sizeof(cudaIpcMemHandle_t));
    auto it = c->ipc_cache.find(key);
    char* base = nullptr;
    if (it != c->ipc_cache.end()) {
      base = it->second.first;
      ++it->second.second;
    } else {
      void* vp = nullptr;
      cudaError_t err = cudaIpcOpenMemHandle(&vp, ex[p].handle, cudaIpcMemLazyEnablePeerAccess);
      if (err != cudaSuccess) {
        for (int q = 0; q < p; ++q)
          if (!r.ipc_key[q].empty()) unmap_peer(c, r.ipc_key[q]);
        return rp_fail(RP_ERR_CONFIG, "register: cudaIpcOpenMemHandle(rank " + std::to_string(p) + "): " +
                                          cudaGetErrorString(err));
      }
      base = (char*)vp;
      c->ipc_cache[key] = {base, 1};
    }
    r.ipc_key[p] = key;
    r.ptr[p] = base + ex[p].offset;
  }
  r.live = true;
  c->regs.push_back(r);
  *reg = (int)c->regs.size() - 1;
  return RP_OK;
}

int rp_unregister(rp_comm_t c, int reg) {
  if (!c || reg < 0 || (size_t)reg >= c->regs.size() || !c->regs[reg].live)
    return rp_fail(RP_ERR_INVALID, "rp_unregister: no such registration");
  RP_CUDA_CHECK(cudaSetDevice(c->device));
  RpReg& r = c->regs[reg];
  for (int p = 0; p < RP_MAX_RANKS; ++p)
    if (!r.ipc_key[p].empty()) unmap_peer(c, r.ipc_key[p]);
  r.live = false;
  return RP_OK;
}

}  // extern "C"

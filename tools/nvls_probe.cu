// NVLS microbenchmark (single process, all visible GPUs): multicast object bound
// to every GPU; measures multimem.ld_reduce (in-switch sum) and multimem.st
// bandwidth per GPU with different unroll depths and grids. Design evidence for
// the RP_ALGO_NVLS kernel.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/nvls_probe tools/nvls_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>
#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); printf("%s:%d %s -> %s\n", __FILE__, __LINE__, #x, s); exit(1);} } while (0)
#define RK(x) do { cudaError_t r = (x); if (r != cudaSuccess) { printf("%s:%d %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(r)); exit(1);} } while (0)

template <int U>
__global__ void k_ldred(char* mc, size_t lo, size_t hi, float4* sink) {
  float acc = 0.f;
  for (size_t base = lo + ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 16; base < hi;
       base += (size_t)gridDim.x * blockDim.x * 16 * U) {
    float4 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      size_t o = base + (size_t)u * gridDim.x * blockDim.x * 16;
      if (o < hi)
        asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(r[u].x), "=f"(r[u].y), "=f"(r[u].z), "=f"(r[u].w) : "l"(mc + o) : "memory");
      else r[u] = make_float4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += r[u].x + r[u].y + r[u].z + r[u].w;
  }
  if (acc == 12345.f) sink[0] = make_float4(acc, 0, 0, 0);
}
template <int U>
__global__ void k_st(char* mc, size_t lo, size_t hi) {
  for (size_t base = lo + ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 16; base < hi;
       base += (size_t)gridDim.x * blockDim.x * 16 * U) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      size_t o = base + (size_t)u * gridDim.x * blockDim.x * 16;
      if (o < hi)
        asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc + o), "f"(1.f), "f"(2.f),
                     "f"(3.f), "f"(4.f) : "memory");
    }
  }
}
template <int U>
__global__ void k_both(char* mc, size_t lo, size_t hi) {
  for (size_t base = lo + ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 16; base < hi;
       base += (size_t)gridDim.x * blockDim.x * 16 * U) {
    float4 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      size_t o = base + (size_t)u * gridDim.x * blockDim.x * 16;
      if (o < hi)
        asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(r[u].x), "=f"(r[u].y), "=f"(r[u].z), "=f"(r[u].w) : "l"(mc + o) : "memory");
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      size_t o = base + (size_t)u * gridDim.x * blockDim.x * 16;
      if (o < hi)
        asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc + o), "f"(r[u].x),
                     "f"(r[u].y), "f"(r[u].z), "f"(r[u].w) : "memory");
    }
  }
}

int main(int argc, char** argv) {
  size_t bytes = (size_t)(argc > 1 ? atoi(argv[1]) : 256) << 20;
  CK(cuInit(0));
  int n = 0;
  RK(cudaGetDeviceCount(&n));
  if (n < 2) { printf("need >= 2 GPUs\n"); return 0; }
  CUmulticastObjectProp mp = {};
  mp.numDevices = n;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t g = 0;
  CK(cuMulticastGetGranularity(&g, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  bytes = (bytes + g - 1) / g * g;
  mp.size = bytes;
  CUmemGenericAllocationHandle mc;
  RK(cudaSetDevice(0));
  RK(cudaFree(0));
  CK(cuMulticastCreate(&mc, &mp));
  for (int d = 0; d < n; ++d) { CUdevice dev; CK(cuDeviceGet(&dev, d)); CK(cuMulticastAddDevice(mc, dev)); }
  std::vector<CUdeviceptr> mcva(n);
  for (int d = 0; d < n; ++d) {
    RK(cudaSetDevice(d));
    RK(cudaFree(0));
    CUmemAllocationProp ap = {};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = d;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    CUmemGenericAllocationHandle ph;
    CK(cuMemCreate(&ph, bytes, &ap, 0));
    CK(cuMulticastBindMem(mc, 0, ph, 0, bytes, 0));
    CUmemAccessDesc acc = {};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = d;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CK(cuMemAddressReserve(&mcva[d], bytes, g, 0, 0));
    CK(cuMemMap(mcva[d], bytes, 0, mc, 0));
    CK(cuMemSetAccess(mcva[d], bytes, &acc, 1));
  }
  float4* sink[8];
  cudaStream_t st[8];
  for (int d = 0; d < n; ++d) { RK(cudaSetDevice(d)); RK(cudaMalloc(&sink[d], 64)); RK(cudaStreamCreate(&st[d])); }
  printf("%d GPUs, %zu MiB, per-GPU chunk %zu MiB (GB/s per GPU of chunk bytes)\n", n, bytes >> 20, (bytes / n) >> 20);
  auto run = [&](const char* name, auto launch) {
    for (int w = 0; w < 2; ++w)
      for (int d = 0; d < n; ++d) { RK(cudaSetDevice(d)); launch(d); }
    for (int d = 0; d < n; ++d) { RK(cudaSetDevice(d)); RK(cudaDeviceSynchronize()); }
    cudaEvent_t e0[8], e1[8];
    const int it = 5;
    for (int d = 0; d < n; ++d) {
      RK(cudaSetDevice(d)); RK(cudaEventCreate(&e0[d])); RK(cudaEventCreate(&e1[d]));
      RK(cudaEventRecord(e0[d], st[d]));
      for (int i = 0; i < it; ++i) launch(d);
      RK(cudaEventRecord(e1[d], st[d]));
    }
    float worst = 0;
    for (int d = 0; d < n; ++d) {
      RK(cudaSetDevice(d)); RK(cudaDeviceSynchronize());
      float ms; RK(cudaEventElapsedTime(&ms, e0[d], e1[d])); if (ms > worst) worst = ms;
    }
    printf("%-36s %8.1f us  %7.1f GB/s/GPU(chunk)\n", name, worst * 1e3 / it, (bytes / n) / (worst / it * 1e-3) / 1e9);
  };
  const size_t chunk = bytes / n;
  for (int grid : {148, 296, 592, 1184})
    for (int thr : {256, 512}) {
      char nm[64];
      snprintf(nm, 64, "ld_reduce U4 grid %d x %d", grid, thr);
      run(nm, [&](int d) { k_ldred<4><<<grid, thr, 0, st[d]>>>((char*)mcva[d], d * chunk, (d + 1) * chunk, sink[d]); });
      snprintf(nm, 64, "ld_reduce U8 grid %d x %d", grid, thr);
      run(nm, [&](int d) { k_ldred<8><<<grid, thr, 0, st[d]>>>((char*)mcva[d], d * chunk, (d + 1) * chunk, sink[d]); });
      snprintf(nm, 64, "st U4 grid %d x %d", grid, thr);
      run(nm, [&](int d) { k_st<4><<<grid, thr, 0, st[d]>>>((char*)mcva[d], d * chunk, (d + 1) * chunk); });
      snprintf(nm, 64, "ld_reduce+st U4 grid %d x %d", grid, thr);
      run(nm, [&](int d) { k_both<4><<<grid, thr, 0, st[d]>>>((char*)mcva[d], d * chunk, (d + 1) * chunk); });
    }
  return 0;
}

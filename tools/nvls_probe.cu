// NVLS microbenchmark (single process, all visible GPUs): a multicast object bound
// to every GPU; times multimem.ld_reduce (in-switch sum), multimem.st, and the
// fused ld_reduce -> st all-reduce body, each iteration after an L2 flush (as in
// bench.py), as max over GPUs. Sweeps unroll, grid, block size and memory
// semantics (weak vs .relaxed.sys). Design evidence for the RP_ALGO_NVLS kernel.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/nvls_probe tools/nvls_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <algorithm>
#include <vector>
#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); printf("%s:%d %s -> %s\n", __FILE__, __LINE__, #x, s); exit(1);} } while (0)
#define RK(x) do { cudaError_t r = (x); if (r != cudaSuccess) { printf("%s:%d %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(r)); exit(1);} } while (0)

template <bool WEAK>
__device__ __forceinline__ float4 ldr(const char* p) {
  float4 r;
  if (WEAK)
    asm volatile("multimem.ld_reduce.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p) : "memory");
  else
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p) : "memory");
  return r;
}
template <bool WEAK>
__device__ __forceinline__ void mst(char* p, float4 v) {
  if (WEAK)
    asm volatile("multimem.st.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
                 : "memory");
  else
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
                 "f"(v.w) : "memory");
}

// MODE 0: ld_reduce only, 1: st only, 2: ld_reduce -> st (the all-reduce body)
template <int MODE, int U, bool WEAK>
__global__ void k_body(char* mc, size_t lo, size_t hi, float4* sink) {
  const size_t stride = (size_t)gridDim.x * blockDim.x * 16;
  float acc = 0.f;
  for (size_t base = lo + ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 16; base < hi; base += stride * U) {
    float4 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t o = base + (size_t)u * stride;
      r[u] = make_float4(1.f, 2.f, 3.f, 4.f);
      if (MODE != 1 && o < hi) r[u] = ldr<WEAK>(mc + o);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t o = base + (size_t)u * stride;
      if (MODE == 0) acc += r[u].x + r[u].y + r[u].z + r[u].w;
      else if (o < hi) mst<WEAK>(mc + o, r[u]);
    }
  }
  if (acc == 12345.f) sink[0] = make_float4(acc, 0, 0, 0);
}

__global__ void k_flush(float4* p, size_t n, float v) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_float4(v, v, v, v);
}

int main(int argc, char** argv) {
  size_t bytes = (size_t)(argc > 1 ? atoi(argv[1]) : 64) << 20;
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
  const size_t flush_n = (256u << 20) / 16;
  float4* sink[8];
  float4* fl[8];
  cudaStream_t st[8];
  for (int d = 0; d < n; ++d) {
    RK(cudaSetDevice(d));
    RK(cudaMalloc(&sink[d], 64));
    RK(cudaMalloc(&fl[d], flush_n * 16));
    RK(cudaStreamCreate(&st[d]));
  }
  printf("%d GPUs, message %zu MiB, chunk %zu MiB; L2 flushed before each iteration; time = max over GPUs, median of 7\n",
         n, bytes >> 20, (bytes / n) >> 20);
  printf("%-44s %9s %10s %10s\n", "kernel", "us", "busBW", "link/dir");
  const size_t chunk = bytes / n;
  auto run = [&](const char* name, int mode, auto launch) {
    std::vector<float> ts;
    cudaEvent_t e0[8], e1[8];
    for (int d = 0; d < n; ++d) { RK(cudaSetDevice(d)); RK(cudaEventCreate(&e0[d])); RK(cudaEventCreate(&e1[d])); }
    for (int it = 0; it < 9; ++it) {
      for (int d = 0; d < n; ++d) { RK(cudaSetDevice(d)); k_flush<<<592, 512, 0, st[d]>>>(fl[d], flush_n, (float)it); }
      for (int d = 0; d < n; ++d) { RK(cudaSetDevice(d)); RK(cudaStreamSynchronize(st[d])); }
      for (int d = 0; d < n; ++d) {
        RK(cudaSetDevice(d));
        RK(cudaEventRecord(e0[d], st[d]));
        launch(d);
        RK(cudaEventRecord(e1[d], st[d]));
      }
      float worst = 0;
      for (int d = 0; d < n; ++d) {
        RK(cudaSetDevice(d)); RK(cudaStreamSynchronize(st[d]));
        float ms; RK(cudaEventElapsedTime(&ms, e0[d], e1[d])); worst = std::max(worst, ms);
      }
      if (it >= 2) ts.push_back(worst);
    }
    std::sort(ts.begin(), ts.end());
    const double t = ts[ts.size() / 2] * 1e-3;
    // all-reduce busBW convention 2(N-1)/N * S / t; per-direction link bytes of the body (N+1)/N * S
    const double bus = (mode == 2 ? 2.0 * (n - 1) / n * bytes / t : 0) / 1e9;
    const double link = (mode == 0 ? bytes : mode == 1 ? bytes : (double)(n + 1) / n * bytes) / t / 1e9;
    printf("%-44s %9.1f %10.1f %10.1f\n", name, t * 1e6, bus, link);
  };
#define RUN(MODE, U, WEAK, G, T)                                                                       \
  {                                                                                                    \
    char nm[64];                                                                                       \
    snprintf(nm, 64, "%s U%d %s grid %dx%d", MODE == 0 ? "ld_reduce" : MODE == 1 ? "st" : "ldred+st", U, \
             WEAK ? "weak" : "sys", G, T);                                                             \
    run(nm, MODE, [&](int d) {                                                                         \
      k_body<MODE, U, WEAK><<<G, T, 0, st[d]>>>((char*)mcva[d], d * chunk, (d + 1) * chunk, sink[d]); \
    });                                                                                                \
  }
  RUN(0, 4, false, 148, 512) RUN(1, 4, false, 148, 512)
  RUN(2, 1, true, 148, 128) RUN(2, 2, true, 148, 128) RUN(2, 4, true, 148, 128)
  RUN(2, 1, true, 148, 256) RUN(2, 2, true, 148, 256)
  RUN(2, 1, true, 148, 384) RUN(2, 1, true, 148, 512) RUN(2, 1, true, 148, 768) RUN(2, 1, true, 148, 1024)
  RUN(2, 1, true, 74, 512) RUN(2, 1, true, 74, 1024) RUN(2, 1, true, 296, 256) RUN(2, 1, true, 296, 128)
  RUN(2, 2, true, 74, 512) RUN(2, 4, true, 74, 256) RUN(2, 1, true, 444, 256)
  return 0;
}

// NVLink data-movement probe (design evidence for the collective kernels).
// One process drives 2 GPUs with peer access enabled; measures GPU0<->GPU1
// bandwidth of: LDG.128 pull, STG.128 push, TMA bulk pull/push (cp.async.bulk via
// shared memory), uni- and bi-directional, over grid/unroll/tile variants.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/nvlink_probe tools/nvlink_probe.cu
//   ./tools/nvlink_probe [MiB]
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e = (x);                                                                   \
    if (e != cudaSuccess) {                                                                \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e));     \
      exit(1);                                                                             \
    }                                                                                      \
  } while (0)

__device__ __forceinline__ uint4 ld128(const void* p) {
  uint4 r;
  asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void st128(void* p, uint4 v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

template <int U>
__global__ void k_copy(uint4* __restrict__ dst, const uint4* __restrict__ src, size_t n) {
  const size_t stride = (size_t)gridDim.x * blockDim.x * U;
  for (size_t i = (size_t)blockIdx.x * blockDim.x * U + threadIdx.x; i < n; i += stride) {
    uint4 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i + (size_t)u * blockDim.x < n) r[u] = ld128(src + i + (size_t)u * blockDim.x);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i + (size_t)u * blockDim.x < n) st128(dst + i + (size_t)u * blockDim.x, r[u]);
  }
}

// --- TMA bulk: global -> smem (mbarrier) -> global (bulk_group) ----------------
__device__ __forceinline__ void mbar_init(uint64_t* m, int cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(m)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect(uint64_t* m, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(m)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n LAB_WAIT:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra LAB_WAIT;\n}\n" ::"r"((uint32_t)__cvta_generic_to_shared(m)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* smem, const void* g, uint32_t bytes, uint64_t* m) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(smem)),
               "l"(g), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(m))
               : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* g, const void* smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g),
               "r"((uint32_t)__cvta_generic_to_shared(smem)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

template <int STAGES>
__global__ void k_tma(char* dst, const char* src, size_t bytes, uint32_t tile) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t bar[STAGES];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < STAGES; ++s) mbar_init(&bar[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const size_t ntiles = (bytes + tile - 1) / tile;
  // tiles owned by this block: b, b+G, b+2G ...
  size_t first = blockIdx.x;
  int issued = 0;
  size_t t_issue = first;
  // prologue
  for (int s = 0; s < STAGES && t_issue < ntiles; ++s, t_issue += gridDim.x, ++issued) {
    const uint32_t nb = (uint32_t)((t_issue * tile + tile <= bytes) ? tile : bytes - t_issue * tile);
    mbar_expect(&bar[s], nb);
    bulk_g2s(smem + (size_t)s * tile, src + t_issue * tile, nb, &bar[s]);
  }
  int k = 0;
  for (size_t t = first; t < ntiles; t += gridDim.x, ++k) {
    const int s = k % STAGES;
    const uint32_t parity = (k / STAGES) & 1;
    mbar_wait(&bar[s], parity);
    const uint32_t nb = (uint32_t)((t * tile + tile <= bytes) ? tile : bytes - t * tile);
    bulk_s2g(dst + t * tile, smem + (size_t)s * tile, nb);
    bulk_commit();
    if (t_issue < ntiles) {
      // stage s is refilled once its store has read smem
      bulk_wait_read<0>();
      const uint32_t nb2 = (uint32_t)((t_issue * tile + tile <= bytes) ? tile : bytes - t_issue * tile);
      mbar_expect(&bar[s], nb2);
      bulk_g2s(smem + (size_t)s * tile, src + t_issue * tile, nb2, &bar[s]);
      t_issue += gridDim.x;
    }
  }
  bulk_wait_all();
}

struct Res {
  float ms0, ms1;
};

typedef void (*Launch)(int dev, char* dst, const char* src, size_t bytes, cudaStream_t s, int a, int b);

template <int U>
void launch_copy(int dev, char* dst, const char* src, size_t bytes, cudaStream_t s, int blocks, int threads) {
  k_copy<U><<<blocks, threads, 0, s>>>((uint4*)dst, (const uint4*)src, bytes / 16);
}
template <int ST>
void launch_tma(int dev, char* dst, const char* src, size_t bytes, cudaStream_t s, int blocks, int tile) {
  size_t sm = (size_t)ST * tile;
  static bool set[8] = {};
  if (!set[dev]) {
    CK(cudaFuncSetAttribute(k_tma<ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    set[dev] = true;
  }
  k_tma<ST><<<blocks, 32, sm, s>>>(dst, src, bytes, (uint32_t)tile);
}

// bytes moved over the link per direction / time
float run(Launch fn0, int a, int b, char* d0, const char* s0, char* d1, const char* s1, size_t bytes, bool bidir,
          cudaStream_t st0, cudaStream_t st1, int iters = 10) {
  cudaEvent_t e0[2], e1[2];
  CK(cudaSetDevice(0));
  CK(cudaEventCreate(&e0[0]));
  CK(cudaEventCreate(&e0[1]));
  CK(cudaSetDevice(1));
  CK(cudaEventCreate(&e1[0]));
  CK(cudaEventCreate(&e1[1]));
  for (int w = 0; w < 2; ++w) {
    CK(cudaSetDevice(0));
    fn0(0, d0, s0, bytes, st0, a, b);
    if (bidir) {
      CK(cudaSetDevice(1));
      fn0(1, d1, s1, bytes, st1, a, b);
    }
  }
  CK(cudaSetDevice(0));
  CK(cudaDeviceSynchronize());
  CK(cudaSetDevice(1));
  CK(cudaDeviceSynchronize());
  CK(cudaSetDevice(0));
  CK(cudaEventRecord(e0[0], st0));
  for (int i = 0; i < iters; ++i) fn0(0, d0, s0, bytes, st0, a, b);
  CK(cudaEventRecord(e0[1], st0));
  if (bidir) {
    CK(cudaSetDevice(1));
    CK(cudaEventRecord(e1[0], st1));
    for (int i = 0; i < iters; ++i) fn0(1, d1, s1, bytes, st1, a, b);
    CK(cudaEventRecord(e1[1], st1));
  }
  CK(cudaSetDevice(0));
  CK(cudaDeviceSynchronize());
  CK(cudaSetDevice(1));
  CK(cudaDeviceSynchronize());
  float ms = 0, ms1 = 0;
  CK(cudaEventElapsedTime(&ms, e0[0], e0[1]));
  if (bidir) CK(cudaEventElapsedTime(&ms1, e1[0], e1[1]));
  ms /= iters;
  ms1 /= iters;
  return (float)(bytes / (double)(bidir ? fmaxf(ms, ms1) : ms) / 1e6);  // GB/s
}

int main(int argc, char** argv) {
  size_t mib = argc > 1 ? atoi(argv[1]) : 256;
  size_t bytes = mib << 20;
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) {
    printf("need 2 GPUs\n");
    return 0;
  }
  char *a0, *b0, *a1, *b1;
  cudaStream_t st0, st1;
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  CK(cudaMalloc(&a0, bytes));
  CK(cudaMalloc(&b0, bytes));
  CK(cudaMemset(a0, 1, bytes));
  CK(cudaStreamCreateWithFlags(&st0, cudaStreamNonBlocking));
  CK(cudaSetDevice(1));
  CK(cudaDeviceEnablePeerAccess(0, 0));
  CK(cudaMalloc(&a1, bytes));
  CK(cudaMalloc(&b1, bytes));
  CK(cudaMemset(a1, 2, bytes));
  CK(cudaStreamCreateWithFlags(&st1, cudaStreamNonBlocking));
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);

  printf("bytes=%zu MiB  (GB/s per direction; bidir = both GPUs moving at once)\n", mib);
  // local HBM copy reference
  printf("local copy  LDG/STG U4 148x512: %.1f GB/s (r+w counted once)\n",
         run(launch_copy<4>, sms, 512, b0, a0, b1, a1, bytes, false, st0, st1));
  const int grids[] = {sms, 2 * sms, 4 * sms};
  const int thr[] = {256, 512, 1024};
  for (int bidir = 0; bidir < 2; ++bidir) {
    for (int g : grids)
      for (int t : thr) {
        if (g * t > sms * 2048) continue;
        float pull = run(launch_copy<4>, g, t, b0, a1, b1, a0, bytes, bidir, st0, st1);  // GPU0 reads GPU1
        float push = run(launch_copy<4>, g, t, a1 /*peer dst*/, b0, a0, b1, bytes, bidir, st0, st1);
        printf("%s LDG/STG U4 grid %4d x %4d: pull %6.1f  push %6.1f GB/s\n", bidir ? "bidir" : "uni  ", g, t, pull,
               push);
      }
    for (int g : grids)
      for (int tile : {16384, 32768, 65536}) {
        if ((size_t)tile * 3 > 200 * 1024) continue;
        float pull = run(launch_tma<3>, g, tile, b0, a1, b1, a0, bytes, bidir, st0, st1);
        float push = run(launch_tma<3>, g, tile, a1, b0, a0, b1, bytes, bidir, st0, st1);
        printf("%s TMA bulk 3-stage grid %4d tile %6d: pull %6.1f  push %6.1f GB/s\n", bidir ? "bidir" : "uni  ", g,
               tile, pull, push);
      }
  }
  return 0;
}

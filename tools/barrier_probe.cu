// Cross-GPU barrier latency microbenchmark (one process, 2..8 GPUs with peer
// access; one kernel per GPU, so waiting kernels are on DIFFERENT devices).
// Each kernel runs ITERS barriers back to back; reports us per barrier for:
//   flat_st   per-block pairwise flags: st.release.sys to peer slot, ld.acquire.sys poll (rank_barrier)
//   flat_red  every block red.release.sys.add into one word per (peer, src rank), poll for count
//   hier      local atom.acq_rel.gpu count-in, last block red.release.sys to peers, poll
//   relaxed   fence.acq_rel.sys by thread 0 then st.relaxed.sys flags, ld.relaxed poll + fence
//   hier1f    hier, but the last block issues ONE fence.acq_rel.sys then red.relaxed.sys to every
//             peer (a release pattern; red.release.sys per peer costs one system fence each)
// Design evidence for the phase barriers of the collectives.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/barrier_probe tools/barrier_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>
#define RK(x) do { cudaError_t r = (x); if (r != cudaSuccess) { printf("%s:%d %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(r)); exit(1);} } while (0)

struct Tab { uint32_t* sig[8]; };
__device__ __forceinline__ uint32_t ld_acq(const uint32_t* p) { uint32_t v; asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ uint32_t ld_rlx(const uint32_t* p) { uint32_t v; asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }

// sig layout: [0, 1024*8) flat_st slots row*8+src; [8192, 8200) counters [src]; [8200] local arrival
template <int MODE>
__global__ void k_bar(Tab t, int world, int rank, int iters, uint32_t base) {
  __shared__ int dummy;
  for (int it = 1; it <= iters; ++it) {
    const uint32_t v = base + it;
    __syncthreads();
    if (MODE == 0) {
      if (threadIdx.x < world) {
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(t.sig[threadIdx.x] + blockIdx.x * 8 + rank), "r"(v) : "memory");
        while ((int32_t)(ld_acq(t.sig[rank] + blockIdx.x * 8 + threadIdx.x) - v) < 0) {}
      }
    } else if (MODE == 1) {
      if (threadIdx.x < world) {
        asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(t.sig[threadIdx.x] + 8192 + rank) : "memory");
        const uint32_t tgt = base * gridDim.x + it * gridDim.x;
        while ((int32_t)(ld_acq(t.sig[rank] + 8192 + threadIdx.x) - tgt) < 0) {}
      }
    } else if (MODE == 2) {
      if (threadIdx.x == 0) {
        uint32_t old;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(t.sig[rank] + 8200) : "memory");
        if (old == (base + it) * gridDim.x - 1)
          for (int p = 0; p < world; ++p)
            asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(t.sig[p] + 8192 + rank) : "memory");
      }
      if (threadIdx.x < world)
        while ((int32_t)(ld_acq(t.sig[rank] + 8192 + threadIdx.x) - v) < 0) {}
    } else if (MODE == 4) {
      if (threadIdx.x == 0) {
        uint32_t old;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(t.sig[rank] + 8200) : "memory");
        if (old == (base + it) * gridDim.x - 1) {
          asm volatile("fence.acq_rel.sys;" ::: "memory");
          for (int p = 0; p < world; ++p)
            asm volatile("red.relaxed.sys.global.add.u32 [%0], 1;" ::"l"(t.sig[p] + 8192 + rank) : "memory");
        }
      }
      if (threadIdx.x < world)
        while ((int32_t)(ld_acq(t.sig[rank] + 8192 + threadIdx.x) - v) < 0) {}
    } else {
      if (threadIdx.x == 0) asm volatile("fence.acq_rel.sys;" ::: "memory");
      __syncthreads();
      if (threadIdx.x < world) {
        asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(t.sig[threadIdx.x] + blockIdx.x * 8 + rank), "r"(v) : "memory");
        while ((int32_t)(ld_rlx(t.sig[rank] + blockIdx.x * 8 + threadIdx.x) - v) < 0) {}
        asm volatile("fence.acq_rel.sys;" ::: "memory");
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && blockIdx.x == 1000000) dummy = 0;
}

int main() {
  int n = 0;
  RK(cudaGetDeviceCount(&n));
  if (n > 8) n = 8;
  Tab t;
  for (int d = 0; d < n; ++d) {
    RK(cudaSetDevice(d));
    for (int e = 0; e < n; ++e) if (e != d) RK(cudaDeviceEnablePeerAccess(e, 0));
    RK(cudaMalloc(&t.sig[d], 64 << 10));
    RK(cudaMemset(t.sig[d], 0, 64 << 10));
  }
  const char* names[5] = {"flat_st (rank_barrier)", "flat_red (old phase)", "hier (red.release/peer)", "relaxed+fence", "hier1f (1 fence)"};
  for (int world = 2; world <= n; world *= 2) {
    for (int grid : {1, 148, 296}) {
      for (int mode = 0; mode < 5; ++mode) {
        for (int d = 0; d < world; ++d) { RK(cudaSetDevice(d)); RK(cudaMemset(t.sig[d], 0, 64 << 10)); RK(cudaDeviceSynchronize()); }
        const int iters = 2000;
        cudaEvent_t e0[8], e1[8];
        float worst = 0;
        for (int rep = 0; rep < 2; ++rep) {
          for (int d = 0; d < world; ++d) {
            RK(cudaSetDevice(d)); RK(cudaEventCreate(&e0[d])); RK(cudaEventCreate(&e1[d]));
            RK(cudaEventRecord(e0[d]));
            uint32_t base = rep * iters;
            if (mode == 0) k_bar<0><<<grid, 256>>>(t, world, d, iters, base);
            if (mode == 1) k_bar<1><<<grid, 256>>>(t, world, d, iters, base);
            if (mode == 2) k_bar<2><<<grid, 256>>>(t, world, d, iters, base);
            if (mode == 3) k_bar<3><<<grid, 256>>>(t, world, d, iters, base);
            if (mode == 4) k_bar<4><<<grid, 256>>>(t, world, d, iters, base);
            RK(cudaEventRecord(e1[d]));
          }
          worst = 0;
          for (int d = 0; d < world; ++d) {
            RK(cudaSetDevice(d)); RK(cudaDeviceSynchronize());
            float ms; RK(cudaEventElapsedTime(&ms, e0[d], e1[d])); if (ms > worst) worst = ms;
          }
        }
        printf("world %d grid %4d %-24s %7.2f us/barrier\n", world, grid, names[mode], worst * 1e3 / iters);
      }
    }
  }
  return 0;
}

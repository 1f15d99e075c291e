// Device-side building blocks: cross-GPU signalling, 128-bit vector access,
// element conversions and the rank-ordered fold.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "rp_internal.h"

namespace rp {

// ---------------------------------------------------------------------------
// memory-model primitives (system scope: peers are other GPUs over NVLink)
// ---------------------------------------------------------------------------

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_relaxed_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// 128-bit loads/stores. Peer data is read with plain weak loads after an
// acquire (never .nc: peers write these buffers during the kernel).
__device__ __forceinline__ uint4 ld128(const void* p) {
  uint4 r;
  asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint4 ld128_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st128(void* p, uint4 v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

// ---------------------------------------------------------------------------
// cross-rank barrier: block b of every rank meets block b of every other rank
// ---------------------------------------------------------------------------

// Slot layout in each rank's signal region: sig[row * RP_MAX_RANKS + src_rank].
// Thread p < world stores `value` into peer p's slot (row, rank) with release
// semantics, then spins (acquire) until its own slot (row, p) reaches `value`.
// Values are monotone per slot, so "reached" is a wrap-safe >= test.
// Returns false if the wait timed out or a peer aborted (the block must bail).
__device__ __forceinline__ void red_release_sys_add(uint32_t* p, uint32_t v) {
  asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Spin (acquire) until *p reaches `target` (wrap-safe >=). Bounded by %globaltimer:
// on timeout the abort word of every rank is set; a set abort word ends the wait.
// Returns false on abort/timeout.
__device__ __forceinline__ bool wait_reach(const RankTable& t, int world, uint64_t timeout_ns, int rank,
                                           const uint32_t* p, uint32_t target) {
  uint32_t* abort_word = t.sig[rank] + RP_ABORT_WORD;
  uint64_t t0 = 0;
  uint32_t spins = 0;
  while ((int32_t)(ld_acquire_sys(p) - target) < 0) {
    if ((++spins & 255u) == 0) {
      if (ld_relaxed_sys(abort_word) != 0) return false;  // a peer gave up: leave quickly
      const uint64_t now = globaltimer();
      if (t0 == 0) t0 = now;
      else if (now - t0 > timeout_ns) {
        // record the timeout locally (with the word, target and value seen, for
        // rp_comm_check's message) and tell every peer to stop waiting
        if (atomicCAS(abort_word, 0u, RP_ABORT_TIMEOUT) == 0u) {
          abort_word[1] = (uint32_t)(p - t.sig[rank]);
          abort_word[2] = target;
          abort_word[3] = ld_relaxed_sys(p);
        }
        for (int q = 0; q < world; ++q)
          if (q != rank) atomicCAS(t.sig[q] + RP_ABORT_WORD, 0u, RP_ABORT_PEER);
        return false;
      }
    }
  }
  return true;
}

// A communicator that aborted stays aborted (rp_comm_check): every later kernel
// returns at once, so nothing is stored into a peer's pool after an abort (in a
// loopback world a peer that gave up may be tearing its region down).
__device__ __forceinline__ bool rp_aborted(const RankTable& t, int rank) {
  return ld_relaxed_sys(t.sig[rank] + RP_ABORT_WORD) != 0u;
}

__device__ __forceinline__ bool rank_barrier(const RankTable& t, int world, uint64_t timeout_ns, int rank,
                                             int row, uint32_t value) {
  __shared__ int s_ok;
  __syncthreads();  // all of this block's prior writes happen-before the release below
  if (threadIdx.x == 0) s_ok = 1;
  __syncthreads();
  if (threadIdx.x < (unsigned)world) {
    const int p = threadIdx.x;
    st_release_sys(t.sig[p] + (size_t)row * RP_MAX_RANKS + rank, value);
    if (!wait_reach(t, world, timeout_ns, rank, t.sig[rank] + (size_t)row * RP_MAX_RANKS + p, value)) s_ok = 0;
  }
  __syncthreads();
  return s_ok != 0;
}

// Rank-level phase barrier for dynamically scheduled kernels (any block may have
// touched any tile, so every block of every rank must be counted). Hierarchical:
// each block counts itself in on a LOCAL arrival counter (RP_CTR_ROW word
// 4 + phase, zeroed by dyn_finish) with a gpu-scope acq_rel atomic; the block
// that completes the count has thereby acquired every block's writes, issues ONE
// fence.acq_rel.sys (cumulative: it covers those writes) and then a relaxed
// increment of counter [phase row][rank] on every rank -- a release pattern
// with a single system fence (red.release.sys per peer costs one fence each,
// ~1.5 us apiece, tools/barrier_probe). Wait: every block spins (locally) until its
// counters [phase row][p] reach `target` = calls already seen + 1. One remote
// atomic and one system-scope fence per rank instead of per block: with every
// block of every rank hitting the same peer word, the flat form cost 5-8 us per
// barrier at 148-296 blocks (RP_TRACE, profiles/r01_trace_nvls.txt).
__device__ __forceinline__ void phase_arrive(const RankTable& t, int world, int rank, int phase) {
  __syncthreads();  // the block's writes happen-before thread 0's release
  if (threadIdx.x == 0) {
    uint32_t old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;"
                 : "=r"(old)
                 : "l"(t.sig[rank] + (size_t)RP_CTR_ROW * RP_MAX_RANKS + 4 + phase)
                 : "memory");
    if (old == gridDim.x - 1) {  // last block of this rank
      asm volatile("fence.acq_rel.sys;" ::: "memory");
      for (int p = 0; p < world; ++p)
        asm volatile("red.relaxed.sys.global.add.u32 [%0], 1;" ::"l"(t.sig[p] + (size_t)(RP_PH_ROW0 + phase) * RP_MAX_RANKS + rank)
                     : "memory");
    }
  }
}
__device__ __forceinline__ bool phase_wait(const RankTable& t, int world, uint64_t timeout_ns, int rank, int phase,
                                           uint32_t target) {
  __shared__ int s_ok;
  if (threadIdx.x == 0) s_ok = 1;
  __syncthreads();
  if (threadIdx.x < (unsigned)world &&
      !wait_reach(t, world, timeout_ns, rank, t.sig[rank] + (size_t)(RP_PH_ROW0 + phase) * RP_MAX_RANKS + threadIdx.x,
                  target))
    s_ok = 0;
  __syncthreads();
  return s_ok != 0;
}
// RP_TRACE analysis stamps: 8 u64 per block -- [0] start, [2k-1]/[2k] enter/leave
// barrier k (k = 1..3), [7] end.
__device__ __forceinline__ void rp_trace(const CollArgs& a, int slot) {
  if (a.trace != nullptr && threadIdx.x == 0)
    a.trace[((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 8 + slot] = globaltimer();
}
// Barrier k (1..3) of this call for the current block: value e0 + k, where e0 is
// the block's epoch read at kernel start (epoch_begin).
__device__ __forceinline__ bool rank_barrier(const CollArgs& a, int rank, int row, uint32_t e0, int k) {
  rp_trace(a, 2 * k - 1);
  const bool ok = rank_barrier(a.t, a.world, a.timeout_ns, rank, row, e0 + (uint32_t)k);
  rp_trace(a, 2 * k);
  return ok;
}

// ---------------------------------------------------------------------------
// device-side sequencing state (rp_internal.h RP_ST_*): local to each rank
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t state_load(const RankTable& t, int rank, int idx) {
  return *((volatile const uint32_t*)(t.sig[rank] + idx));
}
__device__ __forceinline__ void state_store(const RankTable& t, int rank, int idx, uint32_t v) {
  *((volatile uint32_t*)(t.sig[rank] + idx)) = v;
}
// Epoch of barrier row `row` for this block (collective rows or BN rows).
__device__ __forceinline__ uint32_t epoch_begin(const RankTable& t, int rank, int state_idx) {
  return state_load(t, rank, state_idx);
}
// Advance the block's epoch by the number of barriers the call used (thread 0,
// after the block's last barrier; every rank advances identically).
__device__ __forceinline__ void epoch_end(const RankTable& t, int rank, int state_idx, uint32_t v) {
  if (threadIdx.x == 0) state_store(t, rank, state_idx, v);
}
// Call-wide one-shot landing-zone parity: every block reads it at start and
// counts itself in; the last block of the call flips it (all reads precede the
// flip) and resets the counter. The same for every block of a call, which the
// zone-reuse argument needs (rp_allreduce.cuh K1p).
__device__ __forceinline__ uint32_t zone_parity_begin(const RankTable& t, int rank) {
  __shared__ uint32_t s_par;
  if (threadIdx.x == 0) {
    s_par = state_load(t, rank, RP_ST_ZONE_PAR) & 1u;
    __threadfence();
    const uint32_t n = atomicAdd(t.sig[rank] + RP_ST_ZONE_PAR + 1, 1u);
    if (n == gridDim.x - 1) {  // last reader of this call
      state_store(t, rank, RP_ST_ZONE_PAR + 1, 0u);
      state_store(t, rank, RP_ST_ZONE_PAR, s_par ^ 1u);
    }
  }
  __syncthreads();
  return s_par;
}

// ---------------------------------------------------------------------------
// element types
// ---------------------------------------------------------------------------

template <int DT> struct DType;
template <> struct DType<RP_F32> { using T = float;          using Acc = float;  static constexpr int kVec = 4; };
template <> struct DType<RP_F64> { using T = double;         using Acc = double; static constexpr int kVec = 2; };
template <> struct DType<RP_BF16> { using T = __nv_bfloat16; using Acc = float;  static constexpr int kVec = 8; };
template <> struct DType<RP_F16> { using T = __half;         using Acc = float;  static constexpr int kVec = 8; };

__device__ __forceinline__ float to_acc(float x) { return x; }
__device__ __forceinline__ double to_acc(double x) { return x; }
__device__ __forceinline__ float to_acc(__nv_bfloat16 x) { return __bfloat162float(x); }
__device__ __forceinline__ float to_acc(__half x) { return __half2float(x); }

template <typename T> __device__ __forceinline__ T from_f32(float x);
template <> __device__ __forceinline__ float from_f32<float>(float x) { return x; }
template <> __device__ __forceinline__ double from_f32<double>(float x) { return (double)x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }
template <> __device__ __forceinline__ __half from_f32<__half>(float x) { return __float2half_rn(x); }

template <typename T> __device__ __forceinline__ T from_acc(float x) { return from_f32<T>(x); }
template <typename T> __device__ __forceinline__ T from_acc(double x) { return (T)x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_acc<__nv_bfloat16>(double x) { return __double2bfloat16(x); }
template <> __device__ __forceinline__ __half from_acc<__half>(double x) { return __double2half(x); }

// generic scalar conversion between any two element types (exact widening,
// round-to-nearest-even narrowing)
template <typename D, typename S> __device__ __forceinline__ D convert(S x) { return from_acc<D>(to_acc(x)); }
template <> __device__ __forceinline__ float convert<float, double>(double x) { return __double2float_rn(x); }
template <> __device__ __forceinline__ double convert<double, float>(float x) { return (double)x; }

// IEEE ops with contraction disabled (bit-exact with numpy's elementwise ops)
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float div_rn(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }
// np.maximum(a, b): a if (a > b or a is NaN) else b
template <typename A> __device__ __forceinline__ A np_max(A a, A b) { return (a > b || a != a) ? a : b; }

__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }

// x / NR correctly rounded. For a power-of-two NR the exact quotient equals the
// exact product x * (1/NR), so the (correctly rounded) multiply is bit-identical to
// the division -- subnormals included -- at a fraction of the instructions.
template <int NR, typename A>
__device__ __forceinline__ A div_count(A x) {
  if constexpr ((NR & (NR - 1)) == 0) return mul_rn(x, (A)1 / (A)NR);
  else return div_rn(x, (A)NR);
}

// Rank-ordered fold of OP over NR operands, one element (graph.py:514-528,
// SPEC.md:406): first() takes rank 0's operand, next() ranks 1..NR-1 in order.
template <int OP, typename A, int NR>
struct Fold {
  A acc;
  __device__ __forceinline__ void first(A x) { acc = (OP == RP_PREMEAN) ? div_count<NR>(x) : x; }
  __device__ __forceinline__ void next(A x) {
    if (OP == RP_MAX) acc = np_max(acc, x);
    else if (OP == RP_PREMEAN) acc = add_rn(acc, div_count<NR>(x));
    else acc = add_rn(acc, x);
  }
  __device__ __forceinline__ A result() const { return (OP == RP_MEAN) ? div_count<NR>(acc) : acc; }
};

// Vector view of a 16-byte packet.
template <typename T>
union Pack16 {
  uint4 u;
  T e[16 / sizeof(T)];
};

}  // namespace rp

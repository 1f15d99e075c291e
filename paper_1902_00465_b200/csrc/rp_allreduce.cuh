// All-reduce kernels K1 (one-shot) and K2 (two-shot) plus the single-replica
// fold; templated on the exchange dtype, the op and the rank count. Included by
// one translation unit per dtype (rp_ar_<dtype>.cu) so they compile in parallel.
#pragma once
#include <algorithm>
#include <type_traits>

#include "rp_device.cuh"

namespace rp {

constexpr int kThreads = 512;
constexpr int kUnroll = 2;

__device__ __forceinline__ bool aligned16(const void* p) { return (((uintptr_t)p) & 15u) == 0; }

// --- user-buffer staging (fused cast) ---------------------------------------

// Tc-vector v of a user array of S (count elements), converted to Tc; padding 0.
template <typename Tc, typename S>
__device__ __forceinline__ uint4 load_user(const S* src, size_t v, size_t count, bool al) {
  constexpr int VEC = 16 / sizeof(Tc);
  Pack16<Tc> r;
  const size_t e0 = v * VEC;
  if (al && e0 + VEC <= count) {
    if constexpr (sizeof(S) == sizeof(Tc)) {
      r.u = ld128_stream(src + e0);
    } else {
      static_assert(sizeof(S) == 2 * sizeof(Tc), "only f32 -> 16-bit narrowing");
      Pack16<S> lo, hi;
      lo.u = ld128_stream(src + e0);
      hi.u = ld128_stream(src + e0 + VEC / 2);
#pragma unroll
      for (int e = 0; e < VEC / 2; ++e) {
        r.e[e] = convert<Tc>(lo.e[e]);
        r.e[e + VEC / 2] = convert<Tc>(hi.e[e]);
      }
    }
  } else {
#pragma unroll
    for (int e = 0; e < VEC; ++e)
      r.e[e] = (e0 + e < count) ? convert<Tc>(src[e0 + e]) : convert<Tc>(0.0f);
  }
  return r.u;
}

// Store Tc-vector v (converted to D) into a user array of D (count elements).
template <typename Tc, typename D>
__device__ __forceinline__ void store_user(D* dst, size_t v, size_t count, bool al, uint4 val) {
  constexpr int VEC = 16 / sizeof(Tc);
  Pack16<Tc> r;
  r.u = val;
  const size_t e0 = v * VEC;
  if (al && e0 + VEC <= count) {
    if constexpr (sizeof(D) == sizeof(Tc)) {
      st128(dst + e0, r.u);
    } else {
      static_assert(sizeof(D) == 2 * sizeof(Tc), "only 16-bit -> f32 widening");
      Pack16<D> lo, hi;
#pragma unroll
      for (int e = 0; e < VEC / 2; ++e) {
        lo.e[e] = convert<D>(r.e[e]);
        hi.e[e] = convert<D>(r.e[e + VEC / 2]);
      }
      st128(dst + e0, lo.u);
      st128(dst + e0 + VEC / 2, hi.u);
    }
  } else {
#pragma unroll
    for (int e = 0; e < VEC; ++e)
      if (e0 + e < count) dst[e0 + e] = convert<D>(r.e[e]);
  }
}

// Stage vectors [lo, hi) of the user src into the pool (as Tc).
template <typename Tc>
__device__ void stage_in(const CollArgs& a, int rank, char* pool, size_t lo, size_t hi) {
  const void* src = a.src[rank];
  const bool al = aligned16(src);
  for (size_t v = lo + threadIdx.x; v < hi; v += blockDim.x) {
    uint4 x;
    if (a.dtype_in == RP_F32 && !std::is_same<Tc, float>::value) {
      if constexpr (sizeof(Tc) == 2) x = load_user<Tc>((const float*)src, v, a.count, al);
      else x = load_user<Tc>((const Tc*)src, v, a.count, al);
    } else {
      x = load_user<Tc>((const Tc*)src, v, a.count, al);
    }
    st128(pool + v * 16, x);
  }
}

// Copy vectors [lo, hi) of the pool result (Tc) out to the user dst.
template <typename Tc>
__device__ void stage_out(const CollArgs& a, int rank, const char* pool, size_t lo, size_t hi) {
  void* dst = a.dst[rank];
  const bool al = aligned16(dst);
  for (size_t v = lo + threadIdx.x; v < hi; v += blockDim.x) {
    uint4 x = ld128(pool + v * 16);
    if (a.dtype_out == RP_F32 && !std::is_same<Tc, float>::value) {
      if constexpr (sizeof(Tc) == 2) store_user<Tc>((float*)dst, v, a.count, al, x);
      else store_user<Tc>((Tc*)dst, v, a.count, al, x);
    } else {
      store_user<Tc>((Tc*)dst, v, a.count, al, x);
    }
  }
}

// Fold one 16-byte packet position across NR ranks (rank order) and round to T.
template <typename T, typename A, int OP, int NR>
__device__ __forceinline__ uint4 fold_packet(const uint4 (&x)[NR]) {
  constexpr int VEC = 16 / sizeof(T);
  Pack16<T> out;
#pragma unroll
  for (int e = 0; e < VEC; ++e) {
    Fold<OP, A, NR> f;
    Pack16<T> p0;
    p0.u = x[0];
    f.first(to_acc(p0.e[e]));
#pragma unroll
    for (int p = 1; p < NR; ++p) {
      Pack16<T> pp;
      pp.u = x[p];
      f.next(to_acc(pp.e[e]));
    }
    out.e[e] = from_acc<T>(f.result());
  }
  return out.u;
}

// ---------------------------------------------------------------------------
// K2: two-shot all-reduce
// ---------------------------------------------------------------------------
template <int DT, int OP, int NR>
__global__ void __launch_bounds__(kThreads) ar_twoshot(const CollArgs a) {
  using T = typename DType<DT>::T;
  using A = typename DType<DT>::Acc;
  const int rank = a.rank >= 0 ? a.rank : (int)blockIdx.y;
  const size_t V = (a.count + (16 / sizeof(T)) - 1) / (16 / sizeof(T));
  const size_t Vc = a.chunk;
  const size_t sub = (Vc + gridDim.x - 1) / gridDim.x;
  const size_t b0 = (size_t)blockIdx.x * sub;
  const size_t b1 = std::min(b0 + sub, Vc);
  rp_trace(a, 0);

  if (a.copy_in && b0 < b1) {
    char* mine = a.t.data[rank] + a.read_off;
#pragma unroll 1
    for (int c = 0; c < NR; ++c) {
      const size_t lo = c * Vc + b0, hi = std::min(c * Vc + b1, V);
      if (lo < hi) stage_in<T>(a, rank, mine, lo, hi);
    }
  }
  if (!rank_barrier(a, rank, blockIdx.x, a.epoch + 1)) return;

  const char* in[NR];
  char* out[NR];
#pragma unroll
  for (int p = 0; p < NR; ++p) {
    in[p] = a.t.data[p] + a.read_off;
    out[p] = a.t.data[p] + a.write_off;
  }
  const size_t lo = rank * Vc + b0;
  const size_t hi = std::min(rank * Vc + b1, V);
  const size_t stride = (size_t)blockDim.x * kUnroll;
  for (size_t base = lo + threadIdx.x; base < hi; base += stride) {
    uint4 x[kUnroll][NR];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const size_t v = base + (size_t)u * blockDim.x;
      if (v < hi) {
#pragma unroll
        for (int p = 0; p < NR; ++p) x[u][p] = ld128(in[p] + v * 16);
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const size_t v = base + (size_t)u * blockDim.x;
      if (v < hi) {
        const uint4 r = fold_packet<T, A, OP, NR>(x[u]);
#pragma unroll
        for (int p = 0; p < NR; ++p) st128(out[p] + v * 16, r);
      }
    }
  }
  if (!rank_barrier(a, rank, blockIdx.x, a.epoch + 2)) return;

  if (a.copy_out) {
    if (b0 < b1) {
      const char* mine = a.t.data[rank] + a.write_off;
#pragma unroll 1
      for (int c = 0; c < NR; ++c) {
        const size_t l = c * Vc + b0, h = std::min(c * Vc + b1, V);
        if (l < h) stage_out<T>(a, rank, mine, l, h);
      }
    }
    // staging is read after the last barrier above: hold peers until we are done
    rank_barrier(a, rank, blockIdx.x, a.epoch + 3);
  }
  rp_trace(a, 7);
}

// Element-type plumbing shared by the push kernels: user src -> exchange T,
// exchange T -> user dst (fused casts, tails and misalignment handled).
template <typename T>
__device__ __forceinline__ uint4 load_src(const CollArgs& a, const void* src, size_t v, bool al) {
  if constexpr (sizeof(T) == 2) {
    if (a.dtype_in == RP_F32) return load_user<T>((const float*)src, v, a.count, al);
  }
  return load_user<T>((const T*)src, v, a.count, al);
}
template <typename T>
__device__ __forceinline__ void store_dst(const CollArgs& a, void* dst, size_t v, bool al, uint4 r) {
  if constexpr (sizeof(T) == 2) {
    if (a.dtype_out == RP_F32) {
      store_user<T>((float*)dst, v, a.count, al, r);
      return;
    }
  }
  store_user<T>((T*)dst, v, a.count, al, r);
}

// ---------------------------------------------------------------------------
// K2p: two-shot all-reduce, push form (the NVLink path). Only stores cross the
// links; every reduction reads local HBM.
//   phase 1: rank r pushes chunk c of its src into rank c's landing slot Q_c[r]
//   barrier
//   phase 2: rank r folds chunk r: its own src plus Q_r[p] for p != r, ascending
//            rank order, and pushes the rounded result into every rank's output
//            (the pool dst region, or the pool W region when dst is a user buffer)
//   barrier ; [copy W -> user dst ; barrier]
// No start barrier: a peer's Q region is only read between that peer's two
// barriers of the same call (see rp_internal.h pool layout).
// a.read_off = Q offset (slots of a.chunk vectors per source rank),
// a.write_off = output offset, a.copy_out = output is W (user dst elsewhere).
// ---------------------------------------------------------------------------
template <int DT, int OP, int NR>
__global__ void __launch_bounds__(kThreads) ar_twoshot_push(const CollArgs a) {
  using T = typename DType<DT>::T;
  using A = typename DType<DT>::Acc;
  const int rank = a.rank >= 0 ? a.rank : (int)blockIdx.y;
  const size_t V = (a.count + (16 / sizeof(T)) - 1) / (16 / sizeof(T));
  const size_t Vc = a.chunk;
  const size_t sub = (Vc + gridDim.x - 1) / gridDim.x;
  const size_t b0 = (size_t)blockIdx.x * sub;
  const size_t b1 = std::min(b0 + sub, Vc);
  const void* src = a.src[rank];
  const bool ali = aligned16(src);
  rp_trace(a, 0);

  // phase 1: scatter my chunks to their owners (stagger targets across ranks)
#pragma unroll 1
  for (int i = 1; i < NR; ++i) {
    const int c = (rank + i) % NR;
    const size_t lo = c * Vc + b0, hi = std::min(c * Vc + b1, V);
    char* slot = a.t.data[c] + a.read_off + (size_t)rank * Vc * 16;  // Q_c[rank]
    const size_t c0 = c * Vc;
    constexpr int U = 4;
    for (size_t base = lo + threadIdx.x; base < hi; base += (size_t)blockDim.x * U) {
      uint4 x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const size_t v = base + (size_t)u * blockDim.x;
        if (v < hi) x[u] = load_src<T>(a, src, v, ali);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const size_t v = base + (size_t)u * blockDim.x;
        if (v < hi) st128(slot + (v - c0) * 16, x[u]);
      }
    }
  }
  if (!rank_barrier(a, rank, blockIdx.x, a.epoch + 1)) return;

  // phase 2: fold my chunk in rank order, push the result everywhere
  {
    const size_t lo = rank * Vc + b0, hi = std::min(rank * Vc + b1, V);
    const char* q = a.t.data[rank] + a.read_off;  // Q_rank[p] at q + (p*Vc + v - rank*Vc)*16
    const size_t r0 = rank * Vc;
    void* dst = a.dst[rank];
    const bool alo = aligned16(dst);
    constexpr int U = NR > 4 ? 1 : 2;
    for (size_t base = lo + threadIdx.x; base < hi; base += (size_t)blockDim.x * U) {
      uint4 x[U][NR];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const size_t v = base + (size_t)u * blockDim.x;
        if (v < hi) {
#pragma unroll
          for (int p = 0; p < NR; ++p)
            x[u][p] = (p == rank) ? load_src<T>(a, src, v, ali) : ld128(q + ((size_t)p * Vc + (v - r0)) * 16);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const size_t v = base + (size_t)u * blockDim.x;
        if (v < hi) {
          const uint4 r = fold_packet<T, A, OP, NR>(x[u]);
#pragma unroll
          for (int i = 1; i < NR; ++i) {
            const int p = (rank + i) % NR;
            st128(a.t.data[p] + a.write_off + v * 16, r);
          }
          if (a.copy_out) store_dst<T>(a, dst, v, alo, r);
          else st128(a.t.data[rank] + a.write_off + v * 16, r);
        }
      }
    }
  }
  if (!rank_barrier(a, rank, blockIdx.x, a.epoch + 2)) return;

  if (a.copy_out) {  // peers' results landed in W: copy them to the user dst
    if (b0 < b1) {
      const char* w = a.t.data[rank] + a.write_off;
      void* dst = a.dst[rank];
      const bool alo = aligned16(dst);
#pragma unroll 1
      for (int c = 0; c < NR; ++c) {
        if (c == rank) continue;
        const size_t lo = c * Vc + b0, hi = std::min(c * Vc + b1, V);
        for (size_t v = lo + threadIdx.x; v < hi; v += blockDim.x) store_dst<T>(a, dst, v, alo, ld128(w + v * 16));
      }
    }
    rank_barrier(a, rank, blockIdx.x, a.epoch + 3);
  }
  rp_trace(a, 7);
}

// ---------------------------------------------------------------------------
// K1p: one-shot all-reduce, push form (latency regime, ONE barrier).
//   rank r pushes its whole src into every peer's landing zone slot Z_p[r];
//   barrier; every rank folds its own src and the N-1 received slots (local
//   reads, ascending rank order) straight into its dst.
// The landing zone alternates between two fixed regions by call parity
// (a.read_off), so no trailing barrier is needed: a peer can only push into a
// zone of the same parity after passing a barrier of the next call, i.e. after
// we finished reading this one.
// ---------------------------------------------------------------------------
template <int DT, int OP, int NR>
__global__ void __launch_bounds__(kThreads) ar_oneshot_push(const CollArgs a) {
  using T = typename DType<DT>::T;
  using A = typename DType<DT>::Acc;
  const int rank = a.rank >= 0 ? a.rank : (int)blockIdx.y;
  const size_t V = (a.count + (16 / sizeof(T)) - 1) / (16 / sizeof(T));
  const size_t sub = (V + gridDim.x - 1) / gridDim.x;
  const size_t lo = (size_t)blockIdx.x * sub;
  const size_t hi = std::min(lo + sub, V);
  const void* src = a.src[rank];
  const bool ali = aligned16(src);
  for (size_t v = lo + threadIdx.x; v < hi; v += blockDim.x) {
    const uint4 x = load_src<T>(a, src, v, ali);
#pragma unroll
    for (int i = 1; i < NR; ++i) {
      const int p = (rank + i) % NR;
      st128(a.t.data[p] + a.read_off + ((size_t)rank * V + v) * 16, x);
    }
  }
  if (!rank_barrier(a, rank, blockIdx.x, a.epoch + 1)) return;
  const char* z = a.t.data[rank] + a.read_off;
  void* dst = a.dst[rank];
  const bool alo = aligned16(dst);
  for (size_t v = lo + threadIdx.x; v < hi; v += blockDim.x) {
    uint4 x[NR];
#pragma unroll
    for (int p = 0; p < NR; ++p) x[p] = (p == rank) ? load_src<T>(a, src, v, ali) : ld128(z + ((size_t)p * V + v) * 16);
    store_dst<T>(a, dst, v, alo, fold_packet<T, A, OP, NR>(x));
  }
}

// ---------------------------------------------------------------------------
// K1: one-shot all-reduce (result written locally: user dst or own pool)
// ---------------------------------------------------------------------------
template <int DT, int OP, int NR>
__global__ void __launch_bounds__(kThreads) ar_oneshot(const CollArgs a) {
  using T = typename DType<DT>::T;
  using A = typename DType<DT>::Acc;
  constexpr int kUnroll = NR > 4 ? 1 : 2;  // latency regime: keep registers for NR loads
  const int rank = a.rank >= 0 ? a.rank : (int)blockIdx.y;
  const size_t V = (a.count + (16 / sizeof(T)) - 1) / (16 / sizeof(T));
  const size_t sub = (V + gridDim.x - 1) / gridDim.x;
  const size_t lo = (size_t)blockIdx.x * sub;
  const size_t hi = std::min(lo + sub, V);

  if (a.copy_in && lo < hi) stage_in<T>(a, rank, a.t.data[rank] + a.read_off, lo, hi);
  if (!rank_barrier(a, rank, blockIdx.x, a.epoch + 1)) return;

  const char* in[NR];
#pragma unroll
  for (int p = 0; p < NR; ++p) in[p] = a.t.data[p] + a.read_off;
  char* own_out = a.t.data[rank] + a.write_off;
  void* dst = a.dst[rank];
  const bool al = aligned16(dst);
  const size_t stride = (size_t)blockDim.x * kUnroll;
  for (size_t base = lo + threadIdx.x; base < hi; base += stride) {
    uint4 x[kUnroll][NR];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const size_t v = base + (size_t)u * blockDim.x;
      if (v < hi) {
#pragma unroll
        for (int p = 0; p < NR; ++p) x[u][p] = ld128(in[p] + v * 16);
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const size_t v = base + (size_t)u * blockDim.x;
      if (v < hi) {
        const uint4 r = fold_packet<T, A, OP, NR>(x[u]);
        if (a.copy_out) {
          if (a.dtype_out == RP_F32 && !std::is_same<T, float>::value) {
            if constexpr (sizeof(T) == 2) store_user<T>((float*)dst, v, a.count, al, r);
            else store_user<T>((T*)dst, v, a.count, al, r);
          } else {
            store_user<T>((T*)dst, v, a.count, al, r);
          }
        } else {
          st128(own_out + v * 16, r);
        }
      }
    }
  }
  rank_barrier(a, rank, blockIdx.x, a.epoch + 2);  // peers done reading our input
}

// ---------------------------------------------------------------------------
// world == 1: local op (identity fold) with the same conversion rules
// ---------------------------------------------------------------------------
template <int DT, int OP>
__global__ void __launch_bounds__(kThreads) ar_single(const CollArgs a) {
  using T = typename DType<DT>::T;
  using A = typename DType<DT>::Acc;
  const size_t V = (a.count + (16 / sizeof(T)) - 1) / (16 / sizeof(T));
  const void* src = a.src[0];
  void* dst = a.dst[0];
  const bool ali = aligned16(src), alo = aligned16(dst);
  for (size_t v = blockIdx.x * (size_t)blockDim.x + threadIdx.x; v < V; v += (size_t)gridDim.x * blockDim.x) {
    uint4 x;
    if (a.dtype_in == RP_F32 && !std::is_same<T, float>::value) {
      if constexpr (sizeof(T) == 2) x = load_user<T>((const float*)src, v, a.count, ali);
      else x = load_user<T>((const T*)src, v, a.count, ali);
    } else {
      x = load_user<T>((const T*)src, v, a.count, ali);
    }
    uint4 xs[1] = {x};
    const uint4 r = fold_packet<T, A, OP, 1>(xs);
    if (a.dtype_out == RP_F32 && !std::is_same<T, float>::value) {
      if constexpr (sizeof(T) == 2) store_user<T>((float*)dst, v, a.count, alo, r);
      else store_user<T>((T*)dst, v, a.count, alo, r);
    } else {
      store_user<T>((T*)dst, v, a.count, alo, r);
    }
  }
}


// pick a kernel for (op, algo, world, push); world == 1 -> single-replica fold
template <int DT, int OP>
const void* pick_ar(int algo, int world, int push) {
#define RP_CASE(NR)                                                                             \
  case NR:                                                                                      \
    if (push)                                                                                   \
      return algo == RP_ALGO_ONESHOT ? (const void*)ar_oneshot_push<DT, OP, NR>                 \
                                     : (const void*)ar_twoshot_push<DT, OP, NR>;                \
    return algo == RP_ALGO_ONESHOT ? (const void*)ar_oneshot<DT, OP, NR>                        \
                                   : (const void*)ar_twoshot<DT, OP, NR>;
  switch (world) {
    case 1: return (const void*)ar_single<DT, OP>;
    RP_CASE(2) RP_CASE(3) RP_CASE(4) RP_CASE(5) RP_CASE(6) RP_CASE(7) RP_CASE(8)
    default: return nullptr;
  }
#undef RP_CASE
}

template <int DT>
const void* pick_ar_op(int op, int algo, int world, int push) {
  switch (op) {
    case RP_SUM: return pick_ar<DT, RP_SUM>(algo, world, push);
    case RP_MEAN: return pick_ar<DT, RP_MEAN>(algo, world, push);
    case RP_MAX: return pick_ar<DT, RP_MAX>(algo, world, push);
    case RP_PREMEAN: return pick_ar<DT, RP_PREMEAN>(algo, world, push);
  }
  return nullptr;
}

}  // namespace rp

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

  if (a.copy_out && b0 < b1) {
    const char* mine = a.t.data[rank] + a.write_off;
#pragma unroll 1
    for (int c = 0; c < NR; ++c) {
      const size_t l = c * Vc + b0, h = std::min(c * Vc + b1, V);
      if (l < h) stage_out<T>(a, rank, mine, l, h);
    }
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


// pick a kernel for (op, algo, world); world == 1 -> single-replica fold
template <int DT, int OP>
const void* pick_ar(int algo, int world) {
#define RP_CASE(NR)                                                                   \
  case NR:                                                                            \
    return algo == RP_ALGO_ONESHOT ? (const void*)ar_oneshot<DT, OP, NR>              \
                                   : (const void*)ar_twoshot<DT, OP, NR>;
  switch (world) {
    case 1: return (const void*)ar_single<DT, OP>;
    RP_CASE(2) RP_CASE(3) RP_CASE(4) RP_CASE(5) RP_CASE(6) RP_CASE(7) RP_CASE(8)
    default: return nullptr;
  }
#undef RP_CASE
}

template <int DT>
const void* pick_ar_op(int op, int algo, int world) {
  switch (op) {
    case RP_SUM: return pick_ar<DT, RP_SUM>(algo, world);
    case RP_MEAN: return pick_ar<DT, RP_MEAN>(algo, world);
    case RP_MAX: return pick_ar<DT, RP_MAX>(algo, world);
    case RP_PREMEAN: return pick_ar<DT, RP_PREMEAN>(algo, world);
  }
  return nullptr;
}

}  // namespace rp

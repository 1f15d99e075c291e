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
// Minimum resident blocks per SM for the two-shot. ncu shows 1 block/SM (68-84
// registers, 25% occupancy, long-scoreboard bound), but forcing 2 (<= 64
// registers, a few spills on odd rank counts) measured no better: N=1 184.7 vs
// 183.9 us, N=2 124.8 vs 121.1 us, N=4 P2P 172.8 vs 175 us
// (profiles/r01_twoshot_occupancy.txt) -- the tile loop keeps enough bytes in
// flight at one block per SM.
#ifndef RP_TWOSHOT_MIN_BLOCKS
#define RP_TWOSHOT_MIN_BLOCKS 1
#endif
constexpr int kTwoshotMinBlocks = RP_TWOSHOT_MIN_BLOCKS;
// 16-byte packets per lane per step of the two-shot fold (each loads NR operands):
// 2 x 8 operands at NR > 4 (122 registers; N=1 bench 179.4 vs 183.3 us with 1),
// 4 x NR at NR <= 4 (93-120 registers; N=2 117.7 vs 121.1 us, N=4 P2P 169.7 vs
// 172.8 us with 2) -- profiles/r01_twoshot_occupancy.txt
#ifndef RP_TWOSHOT_U
#define RP_TWOSHOT_U(NR) ((NR) > 4 ? 2 : 4)
#endif

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

// Claim the next tile of `phase` from this rank's local counter: one atomic per
// WARP per tile, broadcast by shuffle -- no block-wide barrier in the main loop
// (per-block claims cost two __syncthreads per tile: ~1/3 of the stall samples,
// profiles/r01_ncu_ar_twoshot_dyn_n1.txt). The counters start every call at 0
// (dyn_finish resets them), so nothing per call comes from the host.
__device__ __forceinline__ uint32_t claim_tile(const CollArgs& a, int rank, int phase) {
  uint32_t t = 0;
  if ((threadIdx.x & 31) == 0) t = atomicAdd(a.t.sig[rank] + (size_t)RP_CTR_ROW * RP_MAX_RANKS + phase, 1u);
  return __shfl_sync(0xffffffffu, t, 0);
}

// The same per-warp claim on an explicit counter.
__device__ __forceinline__ uint32_t claim_ctr(uint32_t* ctr) {
  uint32_t t = 0;
  if ((threadIdx.x & 31) == 0) t = atomicAdd(ctr, 1u);
  return __shfl_sync(0xffffffffu, t, 0);
}

// Per-call phase-barrier bases, read by every block at kernel start: rank p's
// counter on phase row k must reach seen[k] + 1 (one arrival per rank per call).
struct PhaseBase {
  uint32_t seen[3];
};
__device__ __forceinline__ PhaseBase phase_begin(const CollArgs& a, int rank) {
  PhaseBase b;
#pragma unroll
  for (int k = 0; k < 3; ++k) b.seen[k] = state_load(a.t, rank, RP_ST_PH_SEEN + k);
  return b;
}

// Phase end for the dynamically scheduled kernels: count this block in, wait for
// every block of every rank (trace slots 2p+1 / 2p+2).
__device__ __forceinline__ bool phase_end(const CollArgs& a, int rank, int phase, const PhaseBase& pb) {
  phase_arrive(a.t, a.world, rank, phase);
  rp_trace(a, 2 * phase + 1);
  const bool ok = phase_wait(a.t, a.world, a.timeout_ns, rank, phase, pb.seen[phase] + 1u);
  rp_trace(a, 2 * phase + 2);
  return ok;
}

// After the call's last phase barrier (every block of this rank has read the
// bases, made its last claim and arrived everywhere): advance the bases of the
// phases used and zero the tile and arrival counters for the next call. One
// thread of the rank's block 0.
__device__ __forceinline__ void dyn_finish(const CollArgs& a, int rank, int phases, const PhaseBase& pb) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    for (int k = 0; k < phases; ++k) state_store(a.t, rank, RP_ST_PH_SEEN + k, pb.seen[k] + 1u);
    for (int k = 0; k < 3; ++k) {
      state_store(a.t, rank, RP_CTR_ROW * RP_MAX_RANKS + k, 0u);
      state_store(a.t, rank, RP_CTR_ROW * RP_MAX_RANKS + 4 + k, 0u);
    }
  }
}

// ---------------------------------------------------------------------------
// K2d: two-shot all-reduce, dynamically scheduled (the default large-message
// kernel, both data-movement forms). Warps claim tiles of tile_v vectors from a
// per-rank atomic counter and phases are separated by rank-level counter
// barriers, so no block waits on one particular peer block and the tail is one
// tile (static per-block partitioning left a 20-60 us end spread, RP_TRACE).
//
// PULL (PUSH = false; src pool-resident, or staged by phase 0):
//   P0  [copy_in] stage every chunk's tiles of src into pool[read_off]   | barrier 0
//   P1  tiles of chunk `rank`: load all N operands (N-1 over NVLink), fold in
//       rank order, store the result into every rank's pool[write_off]   | barrier 1
//   P2  [copy_out] pool[write_off] -> user dst, all chunks                | barrier 2
// PUSH (PUSH = true; src anywhere):
//   P0  tiles of chunks c != rank: src -> Q_c[rank] (stores over NVLink)  | barrier 0
//   P1  tiles of chunk `rank`: own src + Q_rank[p], fold, store result to
//       every rank's pool[write_off] (dst region, or W)                   | barrier 1
//   P2  [copy_out] W -> user dst for chunks c != rank                     | barrier 2
// Barrier 0 also orders the start: no rank writes into a peer before that peer
// entered the call (the peer's previous use of its pool is complete).
// ---------------------------------------------------------------------------
template <int DT, int OP, int NR, bool PUSH>
__global__ void __launch_bounds__(kThreads, kTwoshotMinBlocks) ar_twoshot_dyn(const CollArgs a) {
  using T = typename DType<DT>::T;
  using A = typename DType<DT>::Acc;
  const int rank = a.rank >= 0 ? a.rank : (int)blockIdx.y;
  if (rp_aborted(a.t, rank)) return;
  const size_t V = (a.count + (16 / sizeof(T)) - 1) / (16 / sizeof(T));
  const size_t Vc = a.chunk;
  const uint32_t tv = a.tile_v;
  const uint32_t tpc = (uint32_t)((Vc + tv - 1) / tv);  // tiles per chunk
  const void* src = a.src[rank];
  const bool ali = aligned16(src);
  void* dst = a.dst[rank];
  const bool alo = aligned16(dst);
  // [lo, hi) vectors of tile j of chunk c
  auto tile_range = [&](int c, uint32_t j, size_t& lo, size_t& hi) {
    lo = (size_t)c * Vc + (size_t)j * tv;
    hi = std::min(std::min(lo + tv, (size_t)(c + 1) * Vc), V);
  };
  rp_trace(a, 0);
  const PhaseBase pb = phase_begin(a, rank);
  const int lane = threadIdx.x & 31;

  // ---- phase 0 --------------------------------------------------------------
  if (PUSH) {
    const uint32_t n0 = tpc * (NR - 1);
    for (uint32_t i = claim_tile(a, rank, 0); i < n0; i = claim_tile(a, rank, 0)) {
      const int c = (rank + 1 + (int)(i / tpc)) % NR;
      size_t lo, hi;
      tile_range(c, i % tpc, lo, hi);
      char* slot = a.t.data[c] + a.read_off + ((ptrdiff_t)rank - (ptrdiff_t)c) * (ptrdiff_t)Vc * 16;  // + v*16
      constexpr int U = 4;
      for (size_t base = lo + lane; base < hi; base += 32 * U) {
        uint4 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const size_t v = base + (size_t)u * 32;
          if (v < hi) x[u] = load_src<T>(a, src, v, ali);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const size_t v = base + (size_t)u * 32;
          if (v < hi) st128(slot + v * 16, x[u]);
        }
      }
    }
  } else if (a.copy_in) {
    const uint32_t n0 = tpc * NR;
    char* mine = a.t.data[rank] + a.read_off;
    for (uint32_t i = claim_tile(a, rank, 0); i < n0; i = claim_tile(a, rank, 0)) {
      size_t lo, hi;
      tile_range((int)(i / tpc), i % tpc, lo, hi);
      for (size_t v = lo + lane; v < hi; v += 32) st128(mine + v * 16, load_src<T>(a, src, v, ali));
    }
  }
  if (!phase_end(a, rank, 0, pb)) return;

  // ---- phase 1: fold my chunk, store the result on every rank ---------------
  {
    const char* in[NR];
#pragma unroll
    for (int p = 0; p < NR; ++p) {
      if (PUSH) in[p] = a.t.data[rank] + a.read_off + ((ptrdiff_t)p - (ptrdiff_t)rank) * (ptrdiff_t)Vc * 16;  // Q_rank[p]
      else in[p] = a.t.data[p] + a.read_off;
    }
    constexpr int U = RP_TWOSHOT_U(NR);
    for (uint32_t j = claim_tile(a, rank, 1); j < tpc; j = claim_tile(a, rank, 1)) {
      size_t lo, hi;
      tile_range(rank, j, lo, hi);
      for (size_t base = lo + lane; base < hi; base += 32 * U) {
        uint4 x[U][NR];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const size_t v = base + (size_t)u * 32;
          if (v < hi) {
#pragma unroll
            for (int p = 0; p < NR; ++p)
              x[u][p] = (PUSH && p == rank) ? load_src<T>(a, src, v, ali) : ld128(in[p] + v * 16);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const size_t v = base + (size_t)u * 32;
          if (v < hi) {
            const uint4 r = fold_packet<T, A, OP, NR>(x[u]);
#pragma unroll
            for (int i = 1; i < NR; ++i) {
              const int p = (rank + i) % NR;
              st128(a.t.data[p] + a.write_off + v * 16, r);
            }
            if (PUSH && a.copy_out) store_dst<T>(a, dst, v, alo, r);
            else st128(a.t.data[rank] + a.write_off + v * 16, r);
          }
        }
      }
    }
  }
  if (!phase_end(a, rank, 1, pb)) return;

  // ---- phase 2: results that landed in staging -> user dst ------------------
  if (a.copy_out) {
    const char* w = a.t.data[rank] + a.write_off;
    const uint32_t n2 = tpc * (PUSH ? NR - 1 : NR);
    for (uint32_t i = claim_tile(a, rank, 2); i < n2; i = claim_tile(a, rank, 2)) {
      const int c = PUSH ? (rank + 1 + (int)(i / tpc)) % NR : (int)(i / tpc);
      size_t lo, hi;
      tile_range(c, i % tpc, lo, hi);
      for (size_t v = lo + lane; v < hi; v += 32) store_dst<T>(a, dst, v, alo, ld128(w + v * 16));
    }
    if (!phase_end(a, rank, 2, pb)) return;  // staging is read after barrier 1: hold peers until done
  }
  dyn_finish(a, rank, a.copy_out ? 3 : 2, pb);
  rp_trace(a, 7);
}

// ---------------------------------------------------------------------------
// K1p: one-shot all-reduce, push form (latency regime, ONE barrier).
//   rank r pushes its whole src into every peer's landing zone slot Z_p[r];
//   barrier; every rank folds its own src and the N-1 received slots (local
//   reads, ascending rank order) straight into its dst.
// The landing zone alternates between two fixed regions by call parity (kept on
// the device, zone_parity_begin), so no trailing barrier is needed: a peer can
// only push into a zone of the same parity after passing a barrier of the next
// call, whose kernel cannot start before this one completed everywhere.
// a.read_off = parity-0 zone; parity 1 lies RP_OS_REGION above it.
// ---------------------------------------------------------------------------
template <int DT, int OP, int NR>
__global__ void __launch_bounds__(kThreads) ar_oneshot_push(const CollArgs a) {
  using T = typename DType<DT>::T;
  using A = typename DType<DT>::Acc;
  const int rank = a.rank >= 0 ? a.rank : (int)blockIdx.y;
  if (rp_aborted(a.t, rank)) return;
  const size_t V = (a.count + (16 / sizeof(T)) - 1) / (16 / sizeof(T));
  const size_t sub = (V + gridDim.x - 1) / gridDim.x;
  const size_t lo = (size_t)blockIdx.x * sub;
  const size_t hi = std::min(lo + sub, V);
  const void* src = a.src[rank];
  const bool ali = aligned16(src);
  const int es = RP_ST_BLK_EPOCH + blockIdx.x;
  const uint32_t e0 = epoch_begin(a.t, rank, es);
  const size_t zone = a.read_off + (size_t)zone_parity_begin(a.t, rank) * RP_OS_REGION;
  for (size_t v = lo + threadIdx.x; v < hi; v += blockDim.x) {
    const uint4 x = load_src<T>(a, src, v, ali);
#pragma unroll
    for (int i = 1; i < NR; ++i) {
      const int p = (rank + i) % NR;
      st128(a.t.data[p] + zone + ((size_t)rank * V + v) * 16, x);
    }
  }
  if (!rank_barrier(a, rank, blockIdx.x, e0, 1)) return;
  epoch_end(a.t, rank, es, e0 + 1);
  const char* z = a.t.data[rank] + zone;
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
  if (rp_aborted(a.t, rank)) return;
  const size_t V = (a.count + (16 / sizeof(T)) - 1) / (16 / sizeof(T));
  const size_t sub = (V + gridDim.x - 1) / gridDim.x;
  const size_t lo = (size_t)blockIdx.x * sub;
  const size_t hi = std::min(lo + sub, V);
  const int es = RP_ST_BLK_EPOCH + blockIdx.x;
  const uint32_t e0 = epoch_begin(a.t, rank, es);

  if (a.copy_in && lo < hi) stage_in<T>(a, rank, a.t.data[rank] + a.read_off, lo, hi);
  if (!rank_barrier(a, rank, blockIdx.x, e0, 1)) return;

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
  rank_barrier(a, rank, blockIdx.x, e0, 2);  // peers done reading our input
  epoch_end(a.t, rank, es, e0 + 2);
}

// ---------------------------------------------------------------------------
// K2v: flat all-reduce for VIRTUAL replicas (all NR replicas' buffers in this
// GPU's HBM). Nothing crosses a link, so nothing needs partitioning by rank:
// every warp claims tiles of the flat vector range from one counter and, per
// 16-byte position, loads all NR operands, folds them in rank order and stores
// the result into all NR outputs -- each buffer read once and written once (the
// HBM minimum, 2*NR*S), with no barrier at all. The two-shot's rank chunks, two
// phase barriers and one-rank-per-blockIdx.y grid (144 of 148 SMs at NR=8) were
// pure overhead here. In place is safe: a position's NR loads precede its NR
// stores in the same thread. The last block to finish zeroes the counters.
// ---------------------------------------------------------------------------
#ifndef RP_VFLAT_U
#define RP_VFLAT_U(NR) ((NR) > 4 ? 2 : 4)
#endif
template <int DT, int OP, int NR>
__global__ void __launch_bounds__(kThreads, 1) ar_virtual_flat(const CollArgs a) {
  using T = typename DType<DT>::T;
  using A = typename DType<DT>::Acc;
  if (rp_aborted(a.t, 0)) return;
  const size_t V = (a.count + (16 / sizeof(T)) - 1) / (16 / sizeof(T));
  const uint32_t tv = a.tile_v;
  const uint32_t ntiles = (uint32_t)((V + tv - 1) / tv);
  uint32_t* ctr = a.t.sig[0] + RP_ST_VFLAT_CTR;
  const int lane = threadIdx.x & 31;
  bool ali = true, alo = true;
#pragma unroll
  for (int p = 0; p < NR; ++p) {
    ali = ali && aligned16(a.src[p]);
    alo = alo && aligned16(a.dst[p]);
  }
  constexpr int U = RP_VFLAT_U(NR);
  for (uint32_t t = claim_ctr(ctr); t < ntiles; t = claim_ctr(ctr)) {
    const size_t lo = (size_t)t * tv;
    const size_t hi = std::min(lo + tv, V);
    for (size_t base = lo + lane; base < hi; base += 32 * U) {
      uint4 x[U][NR];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const size_t v = base + (size_t)u * 32;
        if (v < hi) {
#pragma unroll
          for (int p = 0; p < NR; ++p) x[u][p] = load_src<T>(a, a.src[p], v, ali);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const size_t v = base + (size_t)u * 32;
        if (v < hi) {
          const uint4 r = fold_packet<T, A, OP, NR>(x[u]);
#pragma unroll
          for (int p = 0; p < NR; ++p) store_dst<T>(a, a.dst[p], v, alo, r);
        }
      }
    }
  }
  // last block out resets the counters for the next call (all claims are done)
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(a.t.sig[0] + RP_ST_VFLAT_DONE, 1u) == gridDim.x - 1) {
      state_store(a.t, 0, RP_ST_VFLAT_CTR, 0u);
      state_store(a.t, 0, RP_ST_VFLAT_DONE, 0u);
    }
  }
}

// ---------------------------------------------------------------------------
// K2v-bulk: the same flat fold with the operands staged by the bulk-copy engine
// (cp.async.bulk global->shared, completion counted on an mbarrier) instead of
// 16-byte register loads -- the Blackwell data-movement path, A/B against the
// register form (RP_VFLAT_BULK=1). Every warp runs its own 2-stage ring: lane 0
// arms the stage's mbarrier with the byte count and issues NR bulk copies of one
// 32*kBulkU-vector slice each; the warp waits on the phase, folds from shared
// memory (lane-contiguous 16-byte reads, conflict-free) and stores the result to
// all NR outputs; meanwhile the next stage's copies are in flight. Bytes in flight
// no longer cost registers. Only the whole, 16-byte-aligned vectors go through the
// bulk engine (the host checks alignment and that no cast is fused); a partial
// last vector is folded by one warp on the register path, so no copy ever reads
// past a buffer's end.
// ---------------------------------------------------------------------------
constexpr int kBulkThreads = 256;
constexpr int kBulkU = 2;                     // 16-byte packets per lane per operand per stage
constexpr int kBulkSlice = 32 * kBulkU;       // vectors per operand slice
constexpr int kBulkStages = 2;
__host__ __device__ constexpr size_t bulk_smem_bytes(int nr) {
  return (size_t)(kBulkThreads / 32) * kBulkStages * nr * kBulkSlice * 16;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "RP_MBAR_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra RP_MBAR_DONE;\n"
      "bra RP_MBAR_WAIT;\n"
      "RP_MBAR_DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(smem)),
               "l"(gmem), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

template <int DT, int OP, int NR>
__global__ void __launch_bounds__(kBulkThreads, 1) ar_virtual_flat_bulk(const CollArgs a) {
  using T = typename DType<DT>::T;
  using A = typename DType<DT>::Acc;
  constexpr int VEC = 16 / sizeof(T);
  extern __shared__ __align__(128) uint4 ring[];  // [warp][stage][NR][kBulkSlice]
  __shared__ __align__(8) uint64_t bars[kBulkThreads / 32][kBulkStages];
  if (rp_aborted(a.t, 0)) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t Vfull = a.count / VEC;  // whole vectors: every byte of them lies inside the buffers
  const uint32_t tv = a.tile_v;
  const uint32_t ntiles = (uint32_t)((Vfull + tv - 1) / tv);
  uint32_t* ctr = a.t.sig[0] + RP_ST_VFLAT_CTR;
  uint4* mine = ring + (size_t)warp * kBulkStages * NR * kBulkSlice;
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < kBulkStages; ++s) mbar_init(&bars[warp][s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  // the partial last vector (count % VEC elements): one warp, register path
  if (blockIdx.x == 0 && warp == 0 && Vfull * VEC < a.count && lane == 0) {
    uint4 x[NR];
#pragma unroll
    for (int p = 0; p < NR; ++p) x[p] = load_src<T>(a, a.src[p], Vfull, false);
    const uint4 r = fold_packet<T, A, OP, NR>(x);
#pragma unroll
    for (int p = 0; p < NR; ++p) store_dst<T>(a, a.dst[p], Vfull, false, r);
  }
  // warp-uniform producer state: the next slice to issue
  uint32_t tile = claim_ctr(ctr);
  size_t nxt = (size_t)tile * tv;
  size_t tile_hi = tile < ntiles ? std::min(nxt + tv, Vfull) : 0;
  size_t st_v0[kBulkStages];
  uint32_t st_n[kBulkStages];
  uint32_t parity = 0;  // bit s: phase of stage s
  int inflight = 0, s_issue = 0, s_cons = 0;
  auto issue = [&]() {  // one slice of the current tile into stage s_issue (tile < ntiles)
    const uint32_t n = (uint32_t)std::min<size_t>(kBulkSlice, tile_hi - nxt);
    st_v0[s_issue] = nxt;
    st_n[s_issue] = n;
    if (lane == 0) {
      uint64_t* bar = &bars[warp][s_issue];
      mbar_arrive_expect_tx(bar, n * 16u * NR);
#pragma unroll
      for (int p = 0; p < NR; ++p)
        bulk_g2s(mine + ((size_t)s_issue * NR + p) * kBulkSlice, (const char*)a.src[p] + nxt * 16, n * 16u, bar);
    }
    nxt += n;
    if (nxt >= tile_hi) {  // next tile
      tile = claim_ctr(ctr);
      nxt = (size_t)tile * tv;
      tile_hi = tile < ntiles ? std::min(nxt + tv, Vfull) : 0;
    }
    s_issue ^= 1;
    ++inflight;
  };
  while (true) {
    while (inflight < kBulkStages && tile < ntiles) issue();
    if (inflight == 0) break;
    mbar_wait(&bars[warp][s_cons], (parity >> s_cons) & 1u);
    parity ^= 1u << s_cons;
    const uint4* stage = mine + (size_t)s_cons * NR * kBulkSlice;
    const size_t v0 = st_v0[s_cons];
    const uint32_t n = st_n[s_cons];
#pragma unroll
    for (int u = 0; u < kBulkU; ++u) {
      const uint32_t i = lane + 32u * u;
      if (i < n) {
        uint4 x[NR];
#pragma unroll
        for (int p = 0; p < NR; ++p) x[p] = stage[(size_t)p * kBulkSlice + i];
        const uint4 r = fold_packet<T, A, OP, NR>(x);
#pragma unroll
        for (int p = 0; p < NR; ++p) st128((char*)a.dst[p] + (v0 + i) * 16, r);
      }
    }
    __syncwarp();  // every lane's reads of this stage precede its refill
    s_cons ^= 1;
    --inflight;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(a.t.sig[0] + RP_ST_VFLAT_DONE, 1u) == gridDim.x - 1) {
      state_store(a.t, 0, RP_ST_VFLAT_CTR, 0u);
      state_store(a.t, 0, RP_ST_VFLAT_DONE, 0u);
    }
  }
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
                                     : (const void*)ar_twoshot_dyn<DT, OP, NR, true>;           \
    return algo == RP_ALGO_ONESHOT ? (const void*)ar_oneshot<DT, OP, NR>                        \
                                   : (const void*)ar_twoshot_dyn<DT, OP, NR, false>;
  if (algo == RP_ALGO_FLAT_BULK) {  // bulk-copy form of the flat kernel (internal selector)
    switch (world) {
      case 2: return (const void*)ar_virtual_flat_bulk<DT, OP, 2>;
      case 3: return (const void*)ar_virtual_flat_bulk<DT, OP, 3>;
      case 4: return (const void*)ar_virtual_flat_bulk<DT, OP, 4>;
      case 5: return (const void*)ar_virtual_flat_bulk<DT, OP, 5>;
      case 6: return (const void*)ar_virtual_flat_bulk<DT, OP, 6>;
      case 7: return (const void*)ar_virtual_flat_bulk<DT, OP, 7>;
      case 8: return (const void*)ar_virtual_flat_bulk<DT, OP, 8>;
      default: return nullptr;
    }
  }
  if (algo == RP_ALGO_FLAT) {
    switch (world) {
      case 2: return (const void*)ar_virtual_flat<DT, OP, 2>;
      case 3: return (const void*)ar_virtual_flat<DT, OP, 3>;
      case 4: return (const void*)ar_virtual_flat<DT, OP, 4>;
      case 5: return (const void*)ar_virtual_flat<DT, OP, 5>;
      case 6: return (const void*)ar_virtual_flat<DT, OP, 6>;
      case 7: return (const void*)ar_virtual_flat<DT, OP, 7>;
      case 8: return (const void*)ar_virtual_flat<DT, OP, 8>;
      default: return nullptr;
    }
  }
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

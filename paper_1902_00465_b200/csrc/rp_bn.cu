// Cross-replica batch-norm statistics (K5 forward, K5b backward) and the
// elementwise BN apply kernels.
//
// Reference: the cross-replica BN listing PAPER.md:213-219 (mean = all_sum(mean/R),
// mean_sq = all_sum(mean(h^2)/R)) with SPEC.md:530's corrected variance
// E[h^2]-E[h]^2 and eps=1e-5 inside the sqrt, generalised to per-channel
// statistics. The reference cannot differentiate through its collectives
// (graph.py:562, :585); K5b supplies the backward reduction.
//
// Two launches per statistics call:
//   bn_partial_*  : HBM-bound local pass. Every thread accumulates its channels
//                   in f64 over a slice of rows and the block folds its rows in a
//                   fixed order -> per-split partials P[split][c] (sum, sumsq).
//   bn_exchange   : one thread per channel folds P over splits (fixed order),
//                   publishes (sum, sumsq, count) in its pool's BN records,
//                   meets its peers on a BN signal row, folds all ranks' records
//                   in ascending rank order (f64) and writes the outputs.
#include <algorithm>

#include "rp_device.cuh"

namespace rp {

constexpr int kBnThreads = 256;
constexpr int kExThreads = 256;

struct BnArgs {
  const void* x[RP_MAX_RANKS];
  const void* dy[RP_MAX_RANKS];
  const float* mean[RP_MAX_RANKS];
  double* part[RP_MAX_RANKS];  // per local replica: [S][C][2]
  int64_t rows, C, hw;
  int S;
};

struct ExArgs {
  RankTable t;
  double* part[RP_MAX_RANKS];
  float* out0[RP_MAX_RANKS];
  float* out1[RP_MAX_RANKS];
  float* out2[RP_MAX_RANKS];
  float* out3[RP_MAX_RANKS];
  double* count[RP_MAX_RANKS];
  size_t bn_off;  // pool offset of the BN records
  int64_t C;
  int cpb;        // channels per exchange block (power of two, 1..256)
  double local_count[RP_MAX_RANKS];
  int S;
  int world;
  int rank;  // -1: virtual (rank = blockIdx.y)
  int bwd;
  float eps;
  uint64_t timeout_ns;
};

template <typename T>
__device__ __forceinline__ double ld_as_f64(const T* p) {
  return (double)to_acc(*p);
}

// f64 block reduction of NV values per thread over threadIdx.y (fixed order).
template <int NV>
__device__ __forceinline__ void reduce_rows_y(double (&v)[NV], double* smem) {
  // smem: [blockDim.y][blockDim.x][NV]
  const int tx = threadIdx.x, ty = threadIdx.y, bx = blockDim.x;
#pragma unroll
  for (int k = 0; k < NV; ++k) smem[(ty * bx + tx) * NV + k] = v[k];
  __syncthreads();
  if (ty == 0) {
    for (int y = 1; y < (int)blockDim.y; ++y)
#pragma unroll
      for (int k = 0; k < NV; ++k) v[k] += smem[(y * bx + tx) * NV + k];
  }
}

// NV elements of T starting at p (16-byte vector when NV*sizeof(T) == 16)
template <typename T, int NV>
__device__ __forceinline__ void load_nv(const T* p, double (&out)[NV]) {
  if constexpr (NV * sizeof(T) == 16) {
    Pack16<T> v;
    v.u = ld128_stream(p);
#pragma unroll
    for (int k = 0; k < NV; ++k) out[k] = (double)to_acc(v.e[k]);
  } else {
#pragma unroll
    for (int k = 0; k < NV; ++k) out[k] = (double)to_acc(p[k]);
  }
}

// --- NHWC / NC: x is [rows, C], channels innermost ---------------------------
// 1-D block of 256 threads over a column block of up to 256 channel-vectors (NV
// channels each): thread t owns channel-vector t % CVB and rows t / CVB + k*RY
// (RY = 256 / CVB rows per sweep), so narrow layers (C = 64) still keep every
// thread busy. U rows are loaded before any is accumulated (U x 16 B in flight
// per thread), accumulation is f64, and the RY row-partials of a channel are
// folded in a fixed order through shared memory.
template <typename T, bool BWD, int NV>
__device__ __forceinline__ void nhwc_partial(const BnArgs& a, int rep, double* smem) {
  // raw 16-byte packets stay in registers until accumulated (4 regs per packet)
  constexpr bool kPacked = NV * sizeof(T) == 16;
  // packed: x2 with the prefetch buffer; f32 forward is latency-bound at 4 rows
  // (16-bit types: 8/4 rows need 150-160 registers, 1 block per SM: slower, measured)
  constexpr int U = kPacked ? (sizeof(T) == 4 ? (BWD ? 4 : 8) : (BWD ? 2 : 4)) : 4;
  const T* x = (const T*)a.x[rep];
  const T* dy = BWD ? (const T*)a.dy[rep] : nullptr;
  const int64_t C = a.C, M = a.rows;
  const int64_t CVt = C / NV;
  const int64_t cvb0 = (int64_t)blockIdx.x * kBnThreads;
  const int CVB = (int)std::min<int64_t>(CVt - cvb0, kBnThreads);
  const int RY = kBnThreads / CVB;
  const int t = threadIdx.x;
  const int cv = t % CVB, ry = t / CVB;
  const bool active = ry < RY;
  const int64_t c0 = (cvb0 + cv) * NV;
  const int64_t rps = (M + a.S - 1) / a.S;
  const int64_t r0 = (int64_t)blockIdx.y * rps, r1 = std::min(r0 + rps, M);
  double s1[NV], s2[NV], mu[NV];
  float muf[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    s1[k] = 0.0;
    s2[k] = 0.0;
    muf[k] = BWD ? a.mean[rep][c0 + k] : 0.0f;
    mu[k] = (double)muf[k];
  }
  if (active && kPacked) {
    // software pipeline: the next U rows are requested before the current U are
    // accumulated, so every warp always has U x 16 B in flight (single-buffered,
    // a warp stopped loading while it accumulated in f64: ~half the bytes in
    // flight, 53% of HBM, ncu profiles/r01_ncu_bn.txt)
    const int64_t step = (int64_t)RY * U;
    uint4 px[U], pd[U];
    auto load = [&](int64_t r, uint4 (&bx)[U], uint4 (&bd)[U]) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t rr = r + (int64_t)u * RY;
        if (rr < r1) {
          bx[u] = ld128_stream(x + rr * C + c0);
          if (BWD) bd[u] = ld128_stream(dy + rr * C + c0);
        }
      }
    };
    int64_t r = r0 + ry;
    if (r < r1) load(r, px, pd);
    for (; r < r1; r += step) {
      uint4 nx[U], nd[U];
      if (r + step < r1) load(r + step, nx, nd);
      if constexpr (sizeof(T) <= 4) {
        // 32-bit-or-narrower inputs: the U rows of one step are summed in f32 (at most
        // U = 8 terms: relative error <= 8u = 4.8e-7 per chunk, independent across
        // chunks) and each chunk enters the f64 accumulators once -- one f32->f64
        // conversion and one f64 op per U elements instead of three per element, which
        // kept the FP64 pipe ~70% busy at the HBM rate (the forward stopped at 57-82%)
        float f1[NV], f2[NV];
#pragma unroll
        for (int k = 0; k < NV; ++k) f1[k] = f2[k] = 0.0f;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (r + (int64_t)u * RY < r1) {
            Pack16<T> vx, vd;
            vx.u = px[u];
            if (BWD) vd.u = pd[u];
#pragma unroll
            for (int k = 0; k < NV; ++k) {
              const float xk = to_acc(vx.e[k]);
              if (BWD) {
                const float dk = to_acc(vd.e[k]);
                f1[k] += dk;
                f2[k] = fmaf(dk, xk - muf[k], f2[k]);
              } else {
                f1[k] += xk;
                f2[k] = fmaf(xk, xk, f2[k]);
              }
            }
          }
        }
#pragma unroll
        for (int k = 0; k < NV; ++k) {
          s1[k] += (double)f1[k];
          s2[k] += (double)f2[k];
        }
      } else {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (r + (int64_t)u * RY < r1) {
            Pack16<T> vx, vd;
            vx.u = px[u];
            if (BWD) vd.u = pd[u];
#pragma unroll
            for (int k = 0; k < NV; ++k) {
              const double xk = (double)to_acc(vx.e[k]);
              if (BWD) {
                const double dk = (double)to_acc(vd.e[k]);
                s1[k] += dk;
                s2[k] = fma(dk, xk - mu[k], s2[k]);
              } else {
                s1[k] += xk;
                s2[k] = fma(xk, xk, s2[k]);
              }
            }
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        px[u] = nx[u];
        if (BWD) pd[u] = nd[u];
      }
    }
  } else if (active) {
    const int64_t step = (int64_t)RY * U;
    for (int64_t r = r0 + ry; r < r1; r += step) {
      double xv[U][NV], dv[U][NV];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t rr = r + (int64_t)u * RY;
        if (rr < r1) {
          load_nv<T, NV>(x + rr * C + c0, xv[u]);
          if (BWD) load_nv<T, NV>(dy + rr * C + c0, dv[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (r + (int64_t)u * RY < r1) {
#pragma unroll
          for (int k = 0; k < NV; ++k) {
            if (BWD) {
              s1[k] += dv[u][k];
              s2[k] = fma(dv[u][k], xv[u][k] - mu[k], s2[k]);
            } else {
              s1[k] += xv[u][k];
              s2[k] = fma(xv[u][k], xv[u][k], s2[k]);
            }
          }
        }
      }
    }
  }
  // fold the RY row-partials of each channel-vector in row-group order
  if (active) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      smem[((size_t)ry * CVB + cv) * 2 * NV + 2 * k] = s1[k];
      smem[((size_t)ry * CVB + cv) * 2 * NV + 2 * k + 1] = s2[k];
    }
  }
  __syncthreads();
  if (ry == 0) {
    for (int y = 1; y < RY; ++y)
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        s1[k] += smem[((size_t)y * CVB + cv) * 2 * NV + 2 * k];
        s2[k] += smem[((size_t)y * CVB + cv) * 2 * NV + 2 * k + 1];
      }
    double* P = a.part[rep] + ((int64_t)blockIdx.y * C) * 2;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      P[(c0 + k) * 2] = s1[k];
      P[(c0 + k) * 2 + 1] = s2[k];
    }
  }
}

template <typename T, bool BWD, int NV>
__global__ void __launch_bounds__(kBnThreads) bn_partial_nhwc(const BnArgs a) {
  extern __shared__ double smem[];
  nhwc_partial<T, BWD, NV>(a, blockIdx.z, smem);
}

// --- NCHW: x is [n, C, hw] ---------------------------------------------------
// block (c, split): 8 warps take samples round-robin, lanes stride the hw plane.
template <typename T, bool BWD>
__global__ void __launch_bounds__(kBnThreads) bn_partial_nchw(const BnArgs a) {
  constexpr int VEC = 16 / sizeof(T);
  __shared__ double red[kBnThreads / 32][2];
  const int rep = blockIdx.z;
  const T* x = (const T*)a.x[rep];
  const T* dy = BWD ? (const T*)a.dy[rep] : nullptr;
  const int64_t C = a.C, N = a.rows, HW = a.hw;
  const int64_t c = blockIdx.x;
  const int64_t nps = (N + a.S - 1) / a.S;
  const int64_t n0 = (int64_t)blockIdx.y * nps, n1 = std::min(n0 + nps, N);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  const double mu = BWD ? (double)a.mean[rep][c] : 0.0;
  const bool vec = (HW % VEC == 0) && ((((uintptr_t)x) & 15u) == 0) &&
                   (!BWD || ((((uintptr_t)dy) & 15u) == 0));
  double s1 = 0.0, s2 = 0.0;
  for (int64_t n = n0 + warp; n < n1; n += nwarps) {
    const int64_t base = (n * C + c) * HW;
    if (vec) {
#pragma unroll 4
      for (int64_t j = (int64_t)lane * VEC; j < HW; j += 32 * VEC) {
        Pack16<T> px;
        px.u = ld128_stream(x + base + j);
        if (BWD) {
          Pack16<T> pd;
          pd.u = ld128_stream(dy + base + j);
#pragma unroll
          for (int k = 0; k < VEC; ++k) {
            const double d = (double)to_acc(pd.e[k]);
            s1 += d;
            s2 = fma(d, (double)to_acc(px.e[k]) - mu, s2);
          }
        } else {
#pragma unroll
          for (int k = 0; k < VEC; ++k) {
            const double v = (double)to_acc(px.e[k]);
            s1 += v;
            s2 = fma(v, v, s2);
          }
        }
      }
    } else {
      for (int64_t j = lane; j < HW; j += 32) {
        const double v = ld_as_f64(x + base + j);
        if (BWD) {
          const double d = ld_as_f64(dy + base + j);
          s1 += d;
          s2 = fma(d, v - mu, s2);
        } else {
          s1 += v;
          s2 = fma(v, v, s2);
        }
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s1 += __shfl_down_sync(0xffffffffu, s1, o);
    s2 += __shfl_down_sync(0xffffffffu, s2, o);
  }
  if (lane == 0) {
    red[warp][0] = s1;
    red[warp][1] = s2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < nwarps; ++w) {
      s1 += red[w][0];
      s2 += red[w][1];
    }
    double* P = a.part[rep] + ((int64_t)blockIdx.y * C + c) * 2;
    P[0] = s1;
    P[1] = s2;
  }
}

// --- exchange: fold splits, publish, fold ranks ------------------------------
// Block = a.cpb channels x (256 / cpb) threads per channel: thread j of a channel
// folds splits j, j+tpc, ... (independent accumulators, fixed assignment), the tpc
// partial sums are then folded in lane order through shared memory -- a
// deterministic order, parallel over the S split partials (a serial loop over S at
// L2 latency dominated small layers).
// Rank-level barrier of the nblk exchange blocks of this rank, hierarchical like
// the collectives' phase barriers (rp_device.cuh phase_arrive): every block counts
// itself in on a LOCAL counter (gpu-scope acq_rel atomic); the last one resets it,
// issues ONE fence.acq_rel.sys and a relaxed increment of its slot on every rank's
// BN phase row; all blocks then wait for every rank's slot to reach `target`.
// The flat form (a release store per block per peer) cost two system-scope fences
// per block per call: ~27 us for a 4 MiB layer, ncu gpu__time_duration
// (profiles/r01_bn_bench_clean.txt, before this change).
__device__ __forceinline__ bool bn_barrier(const ExArgs& a, int rank, int nblk, uint32_t target) {
  __syncthreads();  // the block's record writes happen-before thread 0's arrival
  if (threadIdx.x == 0) {
    uint32_t* ctr = a.t.sig[rank] + (size_t)RP_CTR_ROW * RP_MAX_RANKS + 4 + RP_BN_PHASE;
    uint32_t old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(ctr) : "memory");
    if (old == (uint32_t)nblk - 1) {  // last exchange block of this rank
      atomicExch(ctr, 0u);            // next barrier counts from 0 (ordered by the fence)
      asm volatile("fence.acq_rel.sys;" ::: "memory");
      for (int p = 0; p < a.world; ++p)
        asm volatile("red.relaxed.sys.global.add.u32 [%0], 1;" ::"l"(
                         a.t.sig[p] + (size_t)(RP_PH_ROW0 + RP_BN_PHASE) * RP_MAX_RANKS + rank)
                     : "memory");
    }
  }
  return phase_wait(a.t, a.world, a.timeout_ns, rank, RP_BN_PHASE, target);
}

// The rank-level part of a statistics call, for channel c whose local sums (s1, s2)
// this thread owns (owner): publish the record, meet the peers once (hierarchical
// barrier over the nblk blocks of every rank), fold every rank's record in rank
// order and write the outputs; advance the call count.
__device__ __forceinline__ void finish_exchange(const ExArgs& a, int rank, int blk, int nblk, uint32_t seen,
                                                int64_t c, bool owner, double s1, double s2) {
  const size_t bn_off = a.bn_off + (size_t)(seen & 1u) * RP_BN_HALF;
  const int rep = a.rank >= 0 ? 0 : rank;  // local replica index
  if (owner) {
    if (a.bwd) {  // this replica's own sums (weight / bias gradients)
      if (a.out2[rep]) a.out2[rep][c] = (float)s1;
      if (a.out3[rep]) a.out3[rep][c] = (float)s2;
    }
    double* rec = (double*)(a.t.data[rank] + bn_off) + c * 3;
    rec[0] = s1;
    rec[1] = s2;
    rec[2] = a.local_count[rep];
  }
  // one rank, one replica: every thread reads back only its own records -- no barrier
  const bool sync = a.world > 1;
  if (sync && !bn_barrier(a, rank, nblk, seen + 1u)) return;
  if (owner) {
    // every rank's record is requested before any is added (one NVLink round trip,
    // not world of them), then folded in ascending rank order
    double r0[RP_MAX_RANKS], r1[RP_MAX_RANKS], r2[RP_MAX_RANKS];
#pragma unroll
    for (int p = 0; p < RP_MAX_RANKS; ++p) {
      if (p < a.world) {
        const double* rec = (const double*)(a.t.data[p] + bn_off) + c * 3;
        r0[p] = rec[0];
        r1[p] = rec[1];
        r2[p] = rec[2];
      }
    }
    double A1 = 0.0, A2 = 0.0, Mt = 0.0;
#pragma unroll
    for (int p = 0; p < RP_MAX_RANKS; ++p) {
      if (p < a.world) {
        A1 += r0[p];
        A2 += r1[p];
        Mt += r2[p];
      }
    }
    if (a.bwd) {
      a.out0[rep][c] = (float)A1;
      a.out1[rep][c] = (float)A2;
    } else {
      const double mean = A1 / Mt;
      double var = A2 / Mt - mean * mean;
      var = var < 0.0 ? 0.0 : var;
      a.out0[rep][c] = (float)mean;
      a.out1[rep][c] = (float)var;
      a.out2[rep][c] = (float)(1.0 / sqrt(var + (double)a.eps));
    }
    if (c == 0 && a.count[rep]) *a.count[rep] = Mt;
  }
  // advance the call count (after this block's barrier every block of this rank has
  // read `seen`; the state is local). One rank: the count still flips the parity.
  if (blk == 0 && threadIdx.x == 0) state_store(a.t, rank, RP_ST_PH_SEEN + RP_BN_PHASE, seen + 1u);
}

__device__ __forceinline__ void exchange_body(const ExArgs& a, int rank, int blk, int nblk) {
  __shared__ double red[kExThreads][2];
  // BN calls completed so far (one barrier each, equal on every rank); the record
  // set alternates with its parity, so the next call can write its records while a
  // slow peer may still be reading this one's: a rank reuses a set only after the
  // following call's barrier, which every peer reaches after its reads
  const uint32_t seen = state_load(a.t, rank, RP_ST_PH_SEEN + RP_BN_PHASE);
  const int rep = a.rank >= 0 ? 0 : rank;  // local replica index
  const int tpc = kExThreads / a.cpb;      // threads per channel
  const int lane = threadIdx.x % tpc;
  const int64_t c = (int64_t)blk * a.cpb + threadIdx.x / tpc;
  const int64_t C = a.C;
  // fold the S split partials of channel c: thread `lane` of the channel's tpc
  // threads sums splits lane, lane + tpc, ...; the tpc sums are then combined by a
  // fixed shuffle tree (warp) and a fixed-order pass over warp sums -- deterministic,
  // and log-depth (a serial pass over 256 values cost ~4 us at C = 128)
  double s1 = 0.0, s2 = 0.0;
  if (c < C) {
    const double* P = a.part[rep];
#pragma unroll 4
    for (int s = lane; s < a.S; s += tpc) {
      s1 += P[((int64_t)s * C + c) * 2];
      s2 += P[((int64_t)s * C + c) * 2 + 1];
    }
  }
  const int width = tpc < 32 ? tpc : 32;
  for (int o = width >> 1; o > 0; o >>= 1) {
    s1 += __shfl_down_sync(0xffffffffu, s1, o, width);
    s2 += __shfl_down_sync(0xffffffffu, s2, o, width);
  }
  if (tpc > 32) {  // one partial per warp, folded in warp order by the channel's first thread
    if ((threadIdx.x & 31) == 0) {
      red[threadIdx.x >> 5][0] = s1;
      red[threadIdx.x >> 5][1] = s2;
    }
    __syncthreads();
    if (lane == 0) {
      const int w0 = threadIdx.x >> 5;
      for (int w = 1; w < tpc / 32; ++w) {
        s1 += red[w0 + w][0];
        s2 += red[w0 + w][1];
      }
    }
  }
  finish_exchange(a, rank, blk, nblk, seen, c, lane == 0 && c < C, s1, s2);
}

// --- K5s: small layers (NHWC) in ONE pass with no split partials ---------------
// Block b owns channel-vectors [b*cvb, (b+1)*cvb) over ALL rows: thread t takes
// channel-vector t % cvb and rows t / cvb + k*RY (RY = 256 / cvb), sums them (f32
// chunks of U rows into f64, as nhwc_partial), the RY row groups are folded by a
// fixed shared-memory tree, and the block publishes its channels' records and meets
// its peers directly (finish_exchange). No split partials in global memory, no
// device-wide barrier, no separate exchange blocks: a small layer (a 4 MiB SN-GAN
// layer took 16.4 us at one rank, 25.6 us at two, against 8.1 us for the apply on
// the same tensor) is then one short pass plus one rank-level meeting.
struct BnSmallArgs {
  const void* x[RP_MAX_RANKS];
  const void* dy[RP_MAX_RANKS];
  const float* mean[RP_MAX_RANKS];
  int64_t rows, C, hw;
  int cvb;  // NHWC: channel-vectors per block; NCHW: channels per block (powers of two)
};

template <typename T, bool BWD, int NV>
__global__ void __launch_bounds__(kBnThreads) bn_stats_small(const ExArgs e, const BnSmallArgs b) {
  extern __shared__ double sm[];  // [RY][cvb][NV][2]
  const int rank = e.rank >= 0 ? e.rank : (int)blockIdx.y;
  if (rp_aborted(e.t, rank)) return;
  const int rep = e.rank >= 0 ? 0 : rank;
  const int cvb = b.cvb, RY = kBnThreads / cvb;
  const int t = threadIdx.x, cv = t % cvb, ry = t / cvb;
  const int64_t C = b.C, M = b.rows;
  const int64_t c0 = ((int64_t)blockIdx.x * cvb + cv) * NV;
  const bool active = c0 < C;
  const T* x = (const T*)b.x[rep];
  const T* dy = BWD ? (const T*)b.dy[rep] : nullptr;
  const uint32_t seen = state_load(e.t, rank, RP_ST_PH_SEEN + RP_BN_PHASE);
  double s1[NV], s2[NV];
  float muf[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    s1[k] = s2[k] = 0.0;
    muf[k] = (BWD && active) ? b.mean[rep][c0 + k] : 0.0f;
  }
  if (active) {
    constexpr int U = 4;
    for (int64_t r = ry; r < M; r += (int64_t)RY * U) {
      uint4 px[U], pd[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t rr = r + (int64_t)u * RY;
        if (rr < M) {
          px[u] = ld128_stream(x + rr * C + c0);
          if (BWD) pd[u] = ld128_stream(dy + rr * C + c0);
        }
      }
      float f1[NV], f2[NV];
#pragma unroll
      for (int k = 0; k < NV; ++k) f1[k] = f2[k] = 0.0f;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (r + (int64_t)u * RY < M) {
          Pack16<T> vx, vd;
          vx.u = px[u];
          if (BWD) vd.u = pd[u];
#pragma unroll
          for (int k = 0; k < NV; ++k) {
            const float xk = to_acc(vx.e[k]);
            if (BWD) {
              const float dk = to_acc(vd.e[k]);
              f1[k] += dk;
              f2[k] = fmaf(dk, xk - muf[k], f2[k]);
            } else {
              f1[k] += xk;
              f2[k] = fmaf(xk, xk, f2[k]);
            }
          }
        }
      }
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        s1[k] += (double)f1[k];
        s2[k] += (double)f2[k];
      }
    }
  }
  // fixed-order tree over the RY row groups (RY is a power of two)
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    sm[(((size_t)ry * cvb + cv) * NV + k) * 2] = s1[k];
    sm[(((size_t)ry * cvb + cv) * NV + k) * 2 + 1] = s2[k];
  }
  __syncthreads();
  for (int h = RY >> 1; h > 0; h >>= 1) {
    if (ry < h) {
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        const size_t i = (((size_t)ry * cvb + cv) * NV + k) * 2, j = (((size_t)(ry + h) * cvb + cv) * NV + k) * 2;
        sm[i] += sm[j];
        sm[i + 1] += sm[j + 1];
      }
    }
    __syncthreads();
  }
  // one thread per channel of this block publishes and folds
  const int j = threadIdx.x;  // channel j of the block's cvb * NV
  const int64_t c = (int64_t)blockIdx.x * cvb * NV + j;
  const bool owner = j < cvb * NV && c < C;
  const double v1 = owner ? sm[(size_t)j * 2] : 0.0, v2 = owner ? sm[(size_t)j * 2 + 1] : 0.0;
  finish_exchange(e, rank, blockIdx.x, gridDim.x, seen, c, owner, v1, v2);
}

// K5s for NCHW [n, C, hw]: block b owns channels [b*cpb, (b+1)*cpb), all n x hw
// elements of each (thread t takes elements t, t+256, ... of the channel's n runs of
// hw), one f64 partial per (thread, channel), a fixed shared-memory tree over the
// 256 threads, then the block's rank-level exchange (finish_exchange).
template <typename T, bool BWD>
__global__ void __launch_bounds__(kBnThreads) bn_stats_small_nchw(const ExArgs e, const BnSmallArgs b) {
  constexpr int VEC = 16 / sizeof(T);
  extern __shared__ double sm[];  // [256][cpb][2]
  const int rank = e.rank >= 0 ? e.rank : (int)blockIdx.y;
  if (rp_aborted(e.t, rank)) return;
  const int rep = e.rank >= 0 ? 0 : rank;
  const int cpb = b.cvb, t = threadIdx.x;
  const int64_t C = b.C, N = b.rows, HW = b.hw;
  const T* x = (const T*)b.x[rep];
  const T* dy = BWD ? (const T*)b.dy[rep] : nullptr;
  const uint32_t seen = state_load(e.t, rank, RP_ST_PH_SEEN + RP_BN_PHASE);
  const bool vec = (HW % VEC == 0) && ((((uintptr_t)x) & 15u) == 0) && (!BWD || ((((uintptr_t)dy) & 15u) == 0));
  for (int j = 0; j < cpb; ++j) {
    const int64_t c = (int64_t)blockIdx.x * cpb + j;
    double s1 = 0.0, s2 = 0.0;
    if (c < C) {
      const float mu = BWD ? b.mean[rep][c] : 0.0f;
      if (vec) {
        const int64_t vpr = HW / VEC;  // vectors per (n, c) run
        for (int64_t q = t; q < N * vpr; q += kBnThreads) {
          const int64_t n = q / vpr, i = q - n * vpr;
          const int64_t off = (n * C + c) * HW + i * VEC;
          Pack16<T> px, pd;
          px.u = ld128_stream(x + off);
          if (BWD) pd.u = ld128_stream(dy + off);
          float f1 = 0.0f, f2 = 0.0f;  // one 16-byte vector in f32, then into f64
#pragma unroll
          for (int k = 0; k < VEC; ++k) {
            const float xk = to_acc(px.e[k]);
            if (BWD) {
              const float dk = to_acc(pd.e[k]);
              f1 += dk;
              f2 = fmaf(dk, xk - mu, f2);
            } else {
              f1 += xk;
              f2 = fmaf(xk, xk, f2);
            }
          }
          s1 += (double)f1;
          s2 += (double)f2;
        }
      } else {
        for (int64_t q = t; q < N * HW; q += kBnThreads) {
          const int64_t n = q / HW, i = q - n * HW;
          const int64_t off = (n * C + c) * HW + i;
          const double xk = ld_as_f64(x + off);
          if (BWD) {
            const double dk = ld_as_f64(dy + off);
            s1 += dk;
            s2 = fma(dk, xk - (double)mu, s2);
          } else {
            s1 += xk;
            s2 = fma(xk, xk, s2);
          }
        }
      }
    }
    sm[((size_t)t * cpb + j) * 2] = s1;
    sm[((size_t)t * cpb + j) * 2 + 1] = s2;
  }
  __syncthreads();
  for (int h = kBnThreads >> 1; h > 0; h >>= 1) {  // fixed-order tree over the threads
    if (t < h) {
      for (int j = 0; j < cpb; ++j) {
        sm[((size_t)t * cpb + j) * 2] += sm[((size_t)(t + h) * cpb + j) * 2];
        sm[((size_t)t * cpb + j) * 2 + 1] += sm[((size_t)(t + h) * cpb + j) * 2 + 1];
      }
    }
    __syncthreads();
  }
  const int64_t c = (int64_t)blockIdx.x * cpb + t;
  const bool owner = t < cpb && c < C;
  const double v1 = owner ? sm[(size_t)t * 2] : 0.0, v2 = owner ? sm[(size_t)t * 2 + 1] : 0.0;
  finish_exchange(e, rank, blockIdx.x, gridDim.x, seen, c, owner, v1, v2);
}

__global__ void __launch_bounds__(kExThreads) bn_exchange(const ExArgs a) {
  const int rank = a.rank >= 0 ? a.rank : (int)blockIdx.y;
  if (rp_aborted(a.t, rank)) return;
  exchange_body(a, rank, blockIdx.x, gridDim.x);
}

// --- fused statistics (NHWC): the local pass and the cross-replica reduction in
// ONE cooperative launch (one wave of co-resident blocks per replica):
//   every block: its split's per-channel partials (nhwc_partial)
//   device-wide barrier (monotone counter; the consumed base lives in the local
//     sequencing state, so graph replays stay in step)
//   blocks 0..ex_blocks-1: fold the split partials of their channels (fixed
//     order), publish, meet the peers on their BN row, fold ranks in ascending
//     order, write the outputs (exchange_body)
// Saves the second launch and lets up to 256 blocks fold the partials.
struct FusedBnArgs {
  BnArgs b;
  ExArgs e;
  int ex_blocks;
};

template <typename T, bool BWD, int NV>
__global__ void __launch_bounds__(kBnThreads) bn_stats_fused(const FusedBnArgs f) {
  extern __shared__ double smem[];
  const int rank = f.e.rank >= 0 ? f.e.rank : (int)blockIdx.z;
  const int rep = f.e.rank >= 0 ? 0 : rank;
  const uint32_t total = gridDim.x * gridDim.y;
  const uint32_t bid = blockIdx.y * gridDim.x + blockIdx.x;
  const uint32_t base = state_load(f.e.t, rank, RP_ST_BN_GRID_BASE);
  nhwc_partial<T, BWD, NV>(f.b, rep, smem);
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t* ctr = f.e.t.sig[rank] + RP_ST_BN_GRID_CTR;
    __threadfence();
    atomicAdd(ctr, 1u);
    // bounded like every other wait: a grid that could not become co-resident
    // aborts (rp_comm_check reports it) instead of spinning forever
    wait_reach(f.e.t, f.e.world, f.e.timeout_ns, rank, ctr, base + total);
  }
  __syncthreads();
  if ((int)bid >= f.ex_blocks || rp_aborted(f.e.t, rank)) return;
  exchange_body(f.e, rank, (int)bid, f.ex_blocks);
  if (bid == 0 && threadIdx.x == 0) state_store(f.e.t, rank, RP_ST_BN_GRID_BASE, base + total);
}

// --- elementwise apply ----------------------------------------------------------
// chan(i) for element i: NHWC -> i % C ; NCHW -> (i / hw) % C
template <typename T, bool BWD>
__global__ void __launch_bounds__(kBnThreads) bn_apply_kernel(const T* __restrict__ x, const T* __restrict__ dy,
                                                              T* __restrict__ y, int64_t total, int64_t C,
                                                              int64_t hw, int nchw, const float* __restrict__ mean,
                                                              const float* __restrict__ invstd,
                                                              const float* __restrict__ w, const float* __restrict__ b,
                                                              const float* __restrict__ sum_dy,
                                                              const float* __restrict__ sum_dy_xmu,
                                                              const double* __restrict__ count, float inv_m) {
  constexpr int VEC = 16 / sizeof(T);
  if (BWD && count) inv_m = (float)(1.0 / *count);  // M on the device: no host sync
  const bool vec = (((((uintptr_t)x) | ((uintptr_t)y) | (BWD ? (uintptr_t)dy : 0)) & 15u) == 0) &&
                   (nchw ? (hw % VEC == 0) : (C % VEC == 0));
  auto coef = [&](int64_t ch, float& m, float& s, float& k1, float& k2) {
    m = mean[ch];
    s = invstd[ch];
    const float g = w ? w[ch] : 1.0f;
    if (BWD) {
      k1 = sum_dy[ch] * inv_m;
      k2 = s * s * sum_dy_xmu[ch] * inv_m;
      s = s * g;  // final multiplier
    } else {
      k1 = s * g;                 // scale
      k2 = b ? b[ch] : 0.0f;      // shift
    }
  };
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (vec) {
    constexpr int U = 4;  // U independent 16-byte loads in flight per thread
    const int64_t nv = total / VEC;
    for (int64_t v0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v0 < nv; v0 += stride * U) {
      Pack16<T> px[U], pd[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t v = v0 + u * stride;
        if (v < nv) {
          px[u].u = ld128_stream(x + v * VEC);
          if (BWD) pd[u].u = ld128_stream(dy + v * VEC);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t v = v0 + u * stride;
        if (v >= nv) break;
        const int64_t i0 = v * VEC;
        Pack16<T> py;
        if (nchw) {
          float m, s, k1, k2;
          coef((i0 / hw) % C, m, s, k1, k2);
#pragma unroll
          for (int k = 0; k < VEC; ++k) {
            const float xv = to_acc(px[u].e[k]);
            float r;
            if (BWD) r = (to_acc(pd[u].e[k]) - k1 - (xv - m) * k2) * s;
            else r = (xv - m) * k1 + k2;
            py.e[k] = from_f32<T>(r);
          }
        } else {
          const int64_t c0 = i0 % C;
#pragma unroll
          for (int k = 0; k < VEC; ++k) {
            float m, s, k1, k2;
            coef(c0 + k, m, s, k1, k2);
            const float xv = to_acc(px[u].e[k]);
            float r;
            if (BWD) r = (to_acc(pd[u].e[k]) - k1 - (xv - m) * k2) * s;
            else r = (xv - m) * k1 + k2;
            py.e[k] = from_f32<T>(r);
          }
        }
        st128(y + i0, py.u);
      }
    }
  } else {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
      const int64_t ch = nchw ? (i / hw) % C : i % C;
      float m, s, k1, k2;
      coef(ch, m, s, k1, k2);
      const float xv = to_acc(x[i]);
      float r;
      if (BWD) r = (to_acc(dy[i]) - k1 - (xv - m) * k2) * s;
      else r = (xv - m) * k1 + k2;
      y[i] = from_f32<T>(r);
    }
  }
}

// NHWC apply with per-thread coefficients in registers. The host picks the grid
// so that the packet stride (blocks x threads x VEC elements) is a multiple of C:
// every packet a thread touches then covers the same VEC channels, so mean /
// invstd / weight / bias (or the backward terms) are loaded ONCE per thread
// instead of per element (the generic kernel issues VEC x 4 scalar loads per
// 16-byte packet: bf16 apply ran at 30% of HBM).
template <typename T, bool BWD>
__global__ void __launch_bounds__(kBnThreads) bn_apply_nhwc_rc(
    const T* __restrict__ x, const T* __restrict__ dy, T* __restrict__ y, int64_t total, int64_t C,
    const float* __restrict__ mean, const float* __restrict__ invstd, const float* __restrict__ w,
    const float* __restrict__ b, const float* __restrict__ sum_dy, const float* __restrict__ sum_dy_xmu,
    const double* __restrict__ count, float inv_m) {
  constexpr int VEC = 16 / sizeof(T);
  if (BWD && count) inv_m = (float)(1.0 / *count);
  constexpr int U = 4;
  const int64_t nv = total / VEC;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t c0 = (gt * VEC) % C;
  float m[VEC], k1[VEC], k2[VEC], sc[VEC];
#pragma unroll
  for (int k = 0; k < VEC; ++k) {
    const int64_t ch = c0 + k;
    m[k] = mean[ch];
    const float s = invstd[ch];
    const float g = w ? w[ch] : 1.0f;
    if (BWD) {
      k1[k] = sum_dy[ch] * inv_m;
      k2[k] = s * s * sum_dy_xmu[ch] * inv_m;
      sc[k] = s * g;
    } else {
      k1[k] = s * g;
      k2[k] = b ? b[ch] : 0.0f;
    }
  }
  for (int64_t v0 = gt; v0 < nv; v0 += stride * U) {
    Pack16<T> px[U], pd[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t v = v0 + u * stride;
      if (v < nv) {
        px[u].u = ld128_stream(x + v * VEC);
        if (BWD) pd[u].u = ld128_stream(dy + v * VEC);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t v = v0 + u * stride;
      if (v >= nv) break;
      Pack16<T> py;
#pragma unroll
      for (int k = 0; k < VEC; ++k) {
        const float xv = to_acc(px[u].e[k]);
        float r;
        if (BWD) r = (to_acc(pd[u].e[k]) - k1[k] - (xv - m[k]) * k2[k]) * sc[k];
        else r = (xv - m[k]) * k1[k] + k2[k];
        py.e[k] = from_f32<T>(r);
      }
      st128(y + v * VEC, py.u);
    }
  }
}

}  // namespace rp

using namespace rp;

namespace {

// Per-split f64 partials. Grown geometrically and never freed before the
// communicator (an earlier launch on another stream may still read the old
// buffer), so no device-wide synchronisation: it would deadlock a loopback world,
// whose peers wait on this rank's next kernel. Growing inside a CUDA-graph capture
// is refused (run the step once eagerly first, as graph capture requires anyway).
int ensure_partials(rp_comm* c, size_t bytes, cudaStream_t stream) {
  if (bytes <= c->bn_partials_bytes) return RP_OK;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(stream, &cs);
  if (cs != cudaStreamCaptureStatusNone)
    return rp_fail(RP_ERR_INVALID, "bn: statistics scratch must grow (" + std::to_string(bytes) +
                                       " bytes) during CUDA-graph capture; run the step once before capturing");
  size_t want = std::max<size_t>(bytes, std::max<size_t>(2 * c->bn_partials_bytes, (size_t)4 << 20));
  double* p = nullptr;
  // stream-ordered: no implicit device-wide wait (cudaMalloc may wait for the
  // whole device, i.e. for a loopback peer's kernel waiting on this rank)
  RP_CUDA_CHECK(cudaMallocAsync((void**)&p, want, stream));
  if (c->bn_partials) c->bn_retired.push_back(c->bn_partials);
  c->bn_partials = p;
  c->bn_partials_bytes = want;
  return RP_OK;
}

// NHWC kernels come in a 16-byte-vector form (NV = 16/sizeof(T); C % NV == 0 and
// aligned pointers) and a scalar form (NV = 1).
template <bool BWD>
const void* pick_partial(int dtype, int layout, bool vec) {
  const bool nchw = layout == RP_LAYOUT_NCHW;
#define RP_B(DT, T)                                                                    \
  if (dtype == DT) {                                                                   \
    if (nchw) return (const void*)bn_partial_nchw<T, BWD>;                              \
    return vec ? (const void*)bn_partial_nhwc<T, BWD, 16 / sizeof(T)>                  \
               : (const void*)bn_partial_nhwc<T, BWD, 1>;                              \
  }
  RP_B(RP_F32, float)
  RP_B(RP_BF16, __nv_bfloat16)
  RP_B(RP_F16, __half)
  RP_B(RP_F64, double)
#undef RP_B
  return nullptr;
}

template <bool BWD>
const void* pick_fused(int dtype, bool vec) {
#define RP_F(DT, T)                                                                    \
  if (dtype == DT)                                                                     \
    return vec ? (const void*)bn_stats_fused<T, BWD, 16 / sizeof(T)> : (const void*)bn_stats_fused<T, BWD, 1>;
  RP_F(RP_F32, float)
  RP_F(RP_BF16, __nv_bfloat16)
  RP_F(RP_F16, __half)
  RP_F(RP_F64, double)
#undef RP_F
  return nullptr;
}

// The exchange arguments of one statistics call (outputs, records, counts).
void fill_ex(rp_comm* c, bool bwd, float eps, int64_t rows, int64_t hw, int64_t ch, float* o0, float* o1, float* o2,
             float* o3, double* count, ExArgs& e) {
  const int W = c->world;
  const int nrep = c->is_virtual ? W : 1;
  memset(&e, 0, sizeof(e));
  e.t = c->table;
  e.bn_off = c->bn_records();
  e.C = ch;
  e.world = W;
  e.rank = c->is_virtual ? -1 : c->rank;
  e.bwd = bwd ? 1 : 0;
  e.eps = eps;
  e.timeout_ns = c->timeout_ns;
  for (int i = 0; i < nrep; ++i) {
    e.local_count[i] = (double)rows * (double)hw;
    if (c->is_virtual) {
      e.out0[i] = ((float* const*)o0)[i];
      e.out1[i] = ((float* const*)o1)[i];
      e.out2[i] = o2 ? ((float* const*)o2)[i] : nullptr;
      e.out3[i] = o3 ? ((float* const*)o3)[i] : nullptr;
      e.count[i] = count ? ((double* const*)count)[i] : nullptr;
    } else {
      e.out0[i] = o0;
      e.out1[i] = o1;
      e.out2[i] = o2;
      e.out3[i] = o3;
      e.count[i] = count;
    }
  }
}

const void* small_kernel(bool bwd, int dtype) {
#define RP_S(DT, T)                                                                        \
  if (dtype == DT) return bwd ? (const void*)bn_stats_small<T, true, 16 / sizeof(T)>       \
                              : (const void*)bn_stats_small<T, false, 16 / sizeof(T)>;
  RP_S(RP_F32, float)
  RP_S(RP_BF16, __nv_bfloat16)
  RP_S(RP_F16, __half)
#undef RP_S
  return nullptr;  // f64: the split path
}

const void* small_nchw_kernel(bool bwd, int dtype) {
#define RP_S(DT, T) \
  if (dtype == DT) return bwd ? (const void*)bn_stats_small_nchw<T, true> : (const void*)bn_stats_small_nchw<T, false>;
  RP_S(RP_F32, float)
  RP_S(RP_BF16, __nv_bfloat16)
  RP_S(RP_F16, __half)
#undef RP_S
  return nullptr;
}

int bn_common(rp_comm* c, bool bwd, const void* x, const void* dy, int dtype, int64_t rows, int64_t ch, int64_t hw,
              int layout, float eps, const float* mean, float* o0, float* o1, float* o2, float* o3, double* count,
              cudaStream_t stream) {
  if (ch <= 0 || rows < 0 || hw <= 0) return rp_fail(RP_ERR_INVALID, "bn: bad shape");
  if (ch > (int64_t)RP_BN_ROWS * kExThreads) return rp_fail(RP_ERR_INVALID, "bn: too many channels (max 65536)");
  if (layout != RP_LAYOUT_NHWC && layout != RP_LAYOUT_NCHW) return rp_fail(RP_ERR_INVALID, "bn: unknown layout");
  if (layout == RP_LAYOUT_NHWC && hw != 1) return rp_fail(RP_ERR_INVALID, "bn: NHWC/NC layout takes hw == 1");
  if (!rp_dtype_valid(dtype)) return rp_fail(RP_ERR_INVALID, "bn: unsupported dtype");
  const int W = c->world;
  const int nrep = c->is_virtual ? W : 1;
  const size_t esz = rp_dtype_size(dtype);
  const int vec = (int)(16 / esz);
  bool vecok = (ch % vec) == 0;
  for (int i = 0; i < nrep; ++i) {
    const void* xi = c->is_virtual ? ((const void* const*)x)[i] : x;
    const void* di = bwd ? (c->is_virtual ? ((const void* const*)dy)[i] : dy) : nullptr;
    vecok = vecok && ((uintptr_t)xi % 16 == 0) && (!bwd || (uintptr_t)di % 16 == 0);
  }
  const int nv = vecok ? vec : 1;
  const void* fn = bwd ? pick_partial<true>(dtype, layout, vecok) : pick_partial<false>(dtype, layout, vecok);
  if (!fn) return rp_fail(RP_ERR_INVALID, "bn: unsupported dtype");

  BnArgs a;
  memset(&a, 0, sizeof(a));
  a.rows = rows;
  a.C = ch;
  a.hw = hw;
  // pointer plumbing: virtual communicators pass host arrays of per-replica pointers
  for (int i = 0; i < nrep; ++i) {
    a.x[i] = c->is_virtual ? ((const void* const*)x)[i] : x;
    if (bwd) {
      a.dy[i] = c->is_virtual ? ((const void* const*)dy)[i] : dy;
      a.mean[i] = c->is_virtual ? ((const float* const*)mean)[i] : mean;
    }
  }
  // K5s: small layers in one pass (bn_stats_small / bn_stats_small_nchw), opt-in with
  // RP_BN_SMALL=1 until it has been measured on the GPU (round 2 lost GPU access
  // before it could be); the split path below is the default
  {
    const char* se = getenv("RP_BN_SMALL");
    const bool small_on = se && se[0] == '1';
    const void* sf = small_kernel(bwd, dtype);
    if (layout == RP_LAYOUT_NHWC && vecok && sf && rows > 0 && small_on) {
      const int64_t CVt = ch / nv;
      const size_t ssm = (size_t)kBnThreads * nv * 2 * sizeof(double);
      int occ = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sf, kBnThreads, ssm) != cudaSuccess || occ < 1) occ = 1;
      const int64_t wave = rp_wave_per_rank(c, occ);
      int cvb = 1;  // >= 128 blocks when C allows, one co-resident wave, <= 16 channel-vectors per block
      while (cvb < 16 && CVt / (cvb * 2) >= 128) cvb *= 2;
      while (cvb < 16 && (CVt + cvb - 1) / cvb > wave) cvb *= 2;
      const int RY = kBnThreads / cvb;
      const int64_t blocks = (CVt + cvb - 1) / cvb;
      if (rows <= (int64_t)32 * RY && blocks <= wave) {
        BnSmallArgs b;
        memset(&b, 0, sizeof(b));
        for (int i = 0; i < nrep; ++i) {
          b.x[i] = a.x[i];
          b.dy[i] = a.dy[i];
          b.mean[i] = a.mean[i];
        }
        b.rows = rows;
        b.C = ch;
        b.hw = 1;
        b.cvb = cvb;
        ExArgs e;
        fill_ex(c, bwd, eps, rows, hw, ch, o0, o1, o2, o3, count, e);
        void* args[] = {&e, &b};
        return rp_launch(c, sf, dim3((unsigned)blocks, nrep), dim3(kBnThreads), args, ssm, stream);
      }
    }
    const void* nf = small_nchw_kernel(bwd, dtype);
    if (layout == RP_LAYOUT_NCHW && nf && rows > 0 && small_on) {
      int occ = 0;
      const size_t ssm8 = (size_t)kBnThreads * 8 * 2 * sizeof(double);
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, nf, kBnThreads, ssm8) != cudaSuccess || occ < 1) occ = 1;
      const int64_t wave = rp_wave_per_rank(c, occ);
      int cpb = 1;  // channels per block: the fewest that fit one co-resident wave
      while (cpb < 8 && (ch + cpb - 1) / cpb > wave) cpb *= 2;
      const int64_t blocks = (ch + cpb - 1) / cpb;
      // bounded work per thread: <= 256 elements over the block's channels
      if (blocks <= wave && rows * hw * cpb <= (int64_t)256 * kBnThreads) {
        BnSmallArgs b;
        memset(&b, 0, sizeof(b));
        for (int i = 0; i < nrep; ++i) {
          b.x[i] = a.x[i];
          b.dy[i] = a.dy[i];
          b.mean[i] = a.mean[i];
        }
        b.rows = rows;
        b.C = ch;
        b.hw = hw;
        b.cvb = cpb;
        ExArgs e;
        fill_ex(c, bwd, eps, rows, hw, ch, o0, o1, o2, o3, count, e);
        void* args[] = {&e, &b};
        const size_t ssm = (size_t)kBnThreads * cpb * 2 * sizeof(double);
        return rp_launch(c, nf, dim3((unsigned)blocks, nrep), dim3(kBnThreads), args, ssm, stream);
      }
    }
  }
  dim3 grid, block;
  size_t smem = 0;
  // one full wave of co-resident blocks: bytes in flight on every SM and no
  // partial last wave (444 blocks at 2 resident per SM ran 1.5 waves, ncu)
  int per_sm = 0;
  {
    const size_t smem0 = layout == RP_LAYOUT_NHWC ? (size_t)kBnThreads * 2 * nv * sizeof(double) : 0;
    if (smem0 > 48 * 1024) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem0);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kBnThreads, smem0) != cudaSuccess || per_sm < 1)
      per_sm = 2;
  }
  const int target = (int)rp_wave_per_rank(c, per_sm);
  if (layout == RP_LAYOUT_NHWC) {
    block = dim3(kBnThreads);
    const int64_t cvt = ch / nv;  // channel-vectors per row
    const int cb = (int)((cvt + kBnThreads - 1) / kBnThreads);
    const int64_t ry = kBnThreads / std::min<int64_t>(cvt, kBnThreads);  // rows per sweep
    int S = (int)std::max<int64_t>(1, std::min<int64_t>((rows + ry * 16 - 1) / (ry * 16), (target + cb - 1) / cb));
    S = std::min(S, 65535);
    a.S = S;
    grid = dim3(cb, S, nrep);
    smem = (size_t)kBnThreads * 2 * nv * sizeof(double);
  } else {
    block = dim3(kBnThreads);
    int S = (int)std::max<int64_t>(1, std::min<int64_t>(rows, (target + ch - 1) / ch));
    S = std::min(S, 65535);
    a.S = S;
    grid = dim3((unsigned)ch, S, nrep);
  }
  // Fused single launch (NHWC): the grid must be one co-resident wave per replica
  // set and hold at least one block per exchange group (<= 256 BN rows); when it
  // cannot (huge C with many virtual replicas) the two-kernel path runs instead.
  bool fused = layout == RP_LAYOUT_NHWC && getenv("RP_BN_UNFUSED") == nullptr;
  const void* ff = nullptr;
  int fcpb = 1, fex = 0;
  if (fused) {
    ff = bwd ? pick_fused<true>(dtype, vecok) : pick_fused<false>(dtype, vecok);
    if (smem > 48 * 1024)
      RP_CUDA_CHECK(cudaFuncSetAttribute(ff, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int fper = 0;
    RP_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&fper, ff, kBnThreads, smem));
    const int64_t wave = rp_wave_per_rank(c, fper);  // co-resident blocks per replica
    if ((int64_t)grid.x * grid.y > wave) grid.y = (unsigned)std::max<int64_t>(1, wave / grid.x);
    const int64_t emax = std::min<int64_t>(RP_BN_ROWS, wave);
    // exchange blocks: as many as the partial pass's grid already has (never more
    // splits than the local pass wants: a 4 MiB layer at 64 splits would otherwise
    // be cut into 256 splits of 4 rows -- 4x the partial traffic and the fold work),
    // unless C needs more blocks even at 256 channels per block
    const int64_t egrid = std::min<int64_t>(emax, (int64_t)grid.x * grid.y);
    while (fcpb < kExThreads && (ch + fcpb - 1) / fcpb > egrid) fcpb *= 2;
    while (fcpb < kExThreads && (ch + fcpb - 1) / fcpb > emax) fcpb *= 2;
    fex = (int)((ch + fcpb - 1) / fcpb);
    if ((int64_t)grid.x * grid.y < fex) grid.y = (unsigned)((fex + grid.x - 1) / grid.x);  // empty splits: zeros
    fused = fex <= emax && (int64_t)grid.x * grid.y <= wave;
    if (fused) a.S = (int)grid.y;
  }
  const size_t per_rep = (size_t)a.S * ch * 2 * sizeof(double);
  int rc = ensure_partials(c, per_rep * nrep, stream);
  if (rc) return rc;
  for (int i = 0; i < nrep; ++i) a.part[i] = c->bn_partials + (per_rep / sizeof(double)) * i;
  if (smem > 48 * 1024) {
    RP_CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  }
  if (!fused && rows > 0) {
    void* args[] = {&a};
    RP_CUDA_CHECK(cudaLaunchKernel(fn, grid, block, args, smem, stream));
  } else if (!fused) {
    RP_CUDA_CHECK(cudaMemsetAsync(c->bn_partials, 0, per_rep * nrep, stream));
  }

  ExArgs e;
  fill_ex(c, bwd, eps, rows, hw, ch, o0, o1, o2, o3, count, e);
  e.S = a.S;
  for (int i = 0; i < nrep; ++i) e.part[i] = a.part[i];
  if (fused) {  // one launch: partials, device-wide barrier, exchange (bn_stats_fused)
    e.cpb = fcpb;
    FusedBnArgs fa;
    fa.b = a;
    fa.e = e;
    fa.ex_blocks = fex;
    void* fargs[] = {&fa};
    // the grid is one co-resident wave (checked above); a loopback world shares the
    // device with its peers' kernels, so it relies on the block cap instead of the
    // cooperative launch's whole-device guarantee
    if (c->loopback) RP_CUDA_CHECK(cudaLaunchKernel(ff, grid, block, fargs, smem, stream));
    else RP_CUDA_CHECK(cudaLaunchCooperativeKernel(ff, grid, block, fargs, smem, stream));
    return RP_OK;
  }
  // exchange geometry: as many blocks as the BN signal rows and co-residency allow,
  // >= 16 channels per block, the rest of the 256 threads fold split partials
  const int max_blocks = std::min(RP_BN_ROWS, rp_blocks_per_rank(c, (const void*)bn_exchange, kExThreads, RP_BN_ROWS));
  int cpb = 16;
  while (cpb < kExThreads && (ch + cpb - 1) / cpb > max_blocks) cpb *= 2;
  e.cpb = cpb;
  const int blocks = (int)((ch + cpb - 1) / cpb);
  if (blocks > max_blocks) return rp_fail(RP_ERR_INVALID, "bn: too many channels for the exchange");
  void* args[] = {&e};
  return rp_launch(c, (const void*)bn_exchange, dim3(blocks, c->is_virtual ? W : 1), dim3(kExThreads), args, 0,
                   stream);
}

}  // namespace

int rp_launch_bn_stats(rp_comm* c, const void* x, int dtype, int64_t rows, int64_t ch, int64_t hw, int layout,
                       float eps, float* mean, float* var, float* invstd, double* count, cudaStream_t stream) {
  if (!mean || !var || !invstd) return rp_fail(RP_ERR_INVALID, "bn_stats: NULL output");
  return bn_common(c, false, x, nullptr, dtype, rows, ch, hw, layout, eps, nullptr, mean, var, invstd, nullptr,
                   count, stream);
}

int rp_launch_bn_bwd_stats(rp_comm* c, const void* x, const void* dy, int dtype, int64_t rows, int64_t ch,
                           int64_t hw, int layout, const float* mean, float* sum_dy, float* sum_dy_xmu,
                           float* local_sum_dy, float* local_sum_dy_xmu, cudaStream_t stream) {
  if (!mean || !sum_dy || !sum_dy_xmu) return rp_fail(RP_ERR_INVALID, "bn_bwd_stats: NULL argument");
  return bn_common(c, true, x, dy, dtype, rows, ch, hw, layout, 0.0f, mean, sum_dy, sum_dy_xmu, local_sum_dy,
                   local_sum_dy_xmu, nullptr, stream);
}

namespace {

int64_t gcd64(int64_t a, int64_t b) {
  while (b) {
    const int64_t t = a % b;
    a = b;
    b = t;
  }
  return a;
}

// Register-cached NHWC apply when the layout allows it; returns false to fall
// back to the generic kernel.
template <bool BWD>
bool launch_apply_rc(int dtype, const void* x, const void* dy, void* y, int64_t total, int64_t C, const float* mean,
                     const float* invstd, const float* w, const float* b, const float* sdy, const float* sdx,
                     const double* cnt, float inv_m, int sms, cudaStream_t stream) {
  const int vec = (int)(16 / rp_dtype_size(dtype));
  if (C % vec || total % vec) return false;
  if ((((uintptr_t)x) | ((uintptr_t)y) | (BWD ? (uintptr_t)dy : 0)) & 15u) return false;
  const int64_t period = C / gcd64(C, (int64_t)kBnThreads * vec);  // blocks per channel cycle
  const int64_t want = std::max<int64_t>(1, std::min<int64_t>((total / vec + kBnThreads * 4 - 1) / (kBnThreads * 4),
                                                             (int64_t)sms * 8));
  if (period > want && period > (int64_t)sms * 8) return false;
  const int64_t blocks = std::max<int64_t>(period, want / period * period);
  const void* fn = nullptr;
  switch (dtype) {
    case RP_F32: fn = (const void*)bn_apply_nhwc_rc<float, BWD>; break;
    case RP_BF16: fn = (const void*)bn_apply_nhwc_rc<__nv_bfloat16, BWD>; break;
    case RP_F16: fn = (const void*)bn_apply_nhwc_rc<__half, BWD>; break;
    default: return false;
  }
  void* args[] = {(void*)&x, (void*)&dy, (void*)&y, (void*)&total, (void*)&C, (void*)&mean, (void*)&invstd,
                  (void*)&w, (void*)&b, (void*)&sdy, (void*)&sdx, (void*)&cnt, (void*)&inv_m};
  return cudaLaunchKernel(fn, dim3((unsigned)blocks), dim3(kBnThreads), args, 0, stream) == cudaSuccess;
}

}  // namespace

extern "C" {

int rp_bn_apply(const void* x, void* y, int dtype, int64_t rows, int64_t ch, int64_t hw, int layout,
                const float* mean, const float* invstd, const float* weight, const float* bias, void* stream) {
  const int64_t total = rows * ch * hw;
  if (total == 0) return RP_OK;
  const int nchw = layout == RP_LAYOUT_NCHW;
  const float* none = nullptr;
  const void* fn = nullptr;
  switch (dtype) {
    case RP_F32: fn = (const void*)bn_apply_kernel<float, false>; break;
    case RP_BF16: fn = (const void*)bn_apply_kernel<__nv_bfloat16, false>; break;
    case RP_F16: fn = (const void*)bn_apply_kernel<__half, false>; break;
    default: return rp_fail(RP_ERR_INVALID, "bn_apply: dtype must be f32/bf16/f16");
  }
  const void* dy = nullptr;
  const double* no_count = nullptr;
  float inv_m = 0.0f;
  int64_t C = ch, HW = hw;
  void* args[] = {(void*)&x, (void*)&dy, (void*)&y, (void*)&total, (void*)&C, (void*)&HW, (void*)&nchw,
                  (void*)&mean, (void*)&invstd, (void*)&weight, (void*)&bias, (void*)&none, (void*)&none,
                  (void*)&no_count, (void*)&inv_m};
  int rc = rp_set_device_from_ptr(x);
  if (rc) return rc;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (!nchw && launch_apply_rc<false>(dtype, x, nullptr, y, total, ch, mean, invstd, weight, bias, nullptr, nullptr,
                                      nullptr, 0.0f, sms, (cudaStream_t)stream))
    return RP_OK;
  const int blocks = (int)std::min<int64_t>((total / 8 + kBnThreads - 1) / kBnThreads + 1, (int64_t)sms * 8);
  RP_CUDA_CHECK(cudaLaunchKernel(fn, dim3(blocks), dim3(kBnThreads), args, 0, (cudaStream_t)stream));
  return RP_OK;
}

int rp_bn_bwd_apply(const void* x, const void* dy, void* dx, int dtype, int64_t rows, int64_t ch, int64_t hw,
                    int layout, const float* mean, const float* invstd, const float* weight, const float* sum_dy,
                    const float* sum_dy_xmu, double count_total, const double* count_device, void* stream) {
  const int64_t total = rows * ch * hw;
  if (total == 0) return RP_OK;
  const int nchw = layout == RP_LAYOUT_NCHW;
  const float* none = nullptr;
  const void* fn = nullptr;
  switch (dtype) {
    case RP_F32: fn = (const void*)bn_apply_kernel<float, true>; break;
    case RP_BF16: fn = (const void*)bn_apply_kernel<__nv_bfloat16, true>; break;
    case RP_F16: fn = (const void*)bn_apply_kernel<__half, true>; break;
    default: return rp_fail(RP_ERR_INVALID, "bn_bwd_apply: dtype must be f32/bf16/f16");
  }
  if (!count_device && !(count_total > 0)) return rp_fail(RP_ERR_INVALID, "bn_bwd_apply: count must be > 0");
  float inv_m = count_device ? 0.0f : (float)(1.0 / count_total);
  int64_t C = ch, HW = hw;
  void* args[] = {(void*)&x, (void*)&dy, (void*)&dx, (void*)&total, (void*)&C, (void*)&HW, (void*)&nchw,
                  (void*)&mean, (void*)&invstd, (void*)&weight, (void*)&none, (void*)&sum_dy, (void*)&sum_dy_xmu,
                  (void*)&count_device, (void*)&inv_m};
  int rc = rp_set_device_from_ptr(x);
  if (rc) return rc;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (!nchw && launch_apply_rc<true>(dtype, x, dy, dx, total, ch, mean, invstd, weight, nullptr, sum_dy, sum_dy_xmu,
                                     count_device, inv_m, sms, (cudaStream_t)stream))
    return RP_OK;
  const int blocks = (int)std::min<int64_t>((total / 8 + kBnThreads - 1) / kBnThreads + 1, (int64_t)sms * 8);
  RP_CUDA_CHECK(cudaLaunchKernel(fn, dim3(blocks), dim3(kBnThreads), args, 0, (cudaStream_t)stream));
  return RP_OK;
}

}  // extern "C"

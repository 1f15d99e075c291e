// Cross-replica collectives over NVLink/NVSwitch peer memory (sm_100a).
//
//   K1 ar_oneshot  : every rank folds all N inputs (ascending rank) for its block's
//                    slice and writes the result locally. Latency regime.
//   K2 ar_twoshot  : reduce-scatter by pulling chunk `rank` from every peer, fold in
//                    rank order, push the rounded result into every peer's buffer
//                    (all-gather by stores). In-place safe: the only reader of
//                    chunk r of any buffer is rank r itself, before it writes it.
//   K3 allgather   : pull every peer's slot into dst in rank order.
//   K4 broadcast   : direct pull from root, or scatter from root + all-gather.
//
// Every kernel partitions work so that block b of rank r depends only on block
// b of its peers; one signal row per block index carries the barrier (see
// rp_device.cuh). Replaces the reference's in-process folds (graph.py:506-540),
// the mesh seam's communicator calls (graph.py:565-583) and the SPEC ring
// (SPEC.md:188-222).
#include <stdlib.h>

#include <stdio.h>

#include <algorithm>
#include <vector>

#include "rp_device.cuh"

const void* rp_pick_ar_f32(int op, int algo, int world, int push);
const void* rp_pick_ar_f64(int op, int algo, int world, int push);
const void* rp_pick_ar_bf16(int op, int algo, int world, int push);
const void* rp_pick_ar_f16(int op, int algo, int world, int push);
size_t rp_bulk_smem_bytes(int nr);
int rp_bulk_threads();

static const void* pick_ar_any(int dtype, int op, int algo, int world, int push) {
  switch (dtype) {
    case RP_F32: return rp_pick_ar_f32(op, algo, world, push);
    case RP_F64: return rp_pick_ar_f64(op, algo, world, push);
    case RP_BF16: return rp_pick_ar_bf16(op, algo, world, push);
    case RP_F16: return rp_pick_ar_f16(op, algo, world, push);
  }
  return nullptr;
}

struct CollArgs;
static int launch_push(rp_comm* c, const void* const* src, void* const* dst, size_t count, int dtype_in,
                       int dtype_comm, int dtype_out, int op, int algo, cudaStream_t stream, CollArgs a);

namespace rp {

constexpr int kThreads = 512;

__device__ __forceinline__ bool aligned16(const void* p) { return (((uintptr_t)p) & 15u) == 0; }

// ---------------------------------------------------------------------------
// byte copies (all_gather / broadcast)
// ---------------------------------------------------------------------------

__device__ __forceinline__ void copy_bytes(char* dst, const char* src, size_t lo, size_t hi, bool vec) {
  if (vec) {  // lo, hi multiples of 16, pointers 16-aligned
    const size_t step = (size_t)blockDim.x * 16 * 4;
    for (size_t o = lo + threadIdx.x * 16; o < hi; o += step) {
      uint4 r[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const size_t oo = o + (size_t)u * blockDim.x * 16;
        if (oo < hi) r[u] = ld128(src + oo);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const size_t oo = o + (size_t)u * blockDim.x * 16;
        if (oo < hi) st128(dst + oo, r[u]);
      }
    }
  } else {
    for (size_t o = lo + threadIdx.x; o < hi; o += blockDim.x) dst[o] = src[o];
  }
}

// K3: all_gather. Rank p's contribution lives at pool_p[read_off + p*read_stride].
// a.count = bytes per rank, a.chunk = per-block byte slice (multiple of 16).
__global__ void __launch_bounds__(kThreads) allgather_kernel(const CollArgs a, size_t read_stride, int vec) {
  const int rank = a.rank >= 0 ? a.rank : (int)blockIdx.y;
  if (rp_aborted(a.t, rank)) return;
  const size_t B = a.count;
  const size_t lo = (size_t)blockIdx.x * a.chunk;
  const size_t hi = std::min(lo + a.chunk, B);
  const int es = RP_ST_BLK_EPOCH + blockIdx.x;
  const uint32_t e0 = epoch_begin(a.t, rank, es);
  if (a.copy_in && lo < hi)
    copy_bytes(a.t.data[rank] + a.read_off + rank * read_stride, (const char*)a.src[rank], lo, hi, vec);
  if (!rank_barrier(a, rank, blockIdx.x, e0, 1)) return;
  char* dst = (char*)a.dst[rank];
  if (lo < hi) {
    for (int i = 0; i < a.world; ++i) {
      const int p = (rank + i) % a.world;  // stagger peers to spread NVLink load
      const char* src = a.t.data[p] + a.read_off + p * read_stride;
      char* d = dst + (size_t)p * B;
      if (d == src) continue;  // in-place slot already holds our data
      copy_bytes(d, src, lo, hi, vec);
    }
  }
  rank_barrier(a, rank, blockIdx.x, e0, 2);
  epoch_end(a.t, rank, es, e0 + 2);
}

// K3p: one-shot all_gather, push form (multi-process, small messages, ONE barrier):
// every rank stores its src into slot [rank] of every peer's one-shot landing zone
// (and straight into its own dst slot), meets its peers once, then copies the
// received slots into dst locally. The zone alternates by call parity exactly as
// for the push one-shot all-reduce (same zones, same parity state), so no trailing
// barrier is needed. a.read_off = parity-0 zone, a.chunk = slot stride (16-B
// multiple, slots * world <= RP_OS_REGION), a.write_off = per-block byte slice.
__global__ void __launch_bounds__(kThreads) allgather_push_kernel(const CollArgs a, int vec) {
  const int rank = a.rank;
  if (rp_aborted(a.t, rank)) return;
  const size_t B = a.count;
  const size_t lo = (size_t)blockIdx.x * a.write_off;
  const size_t hi = std::min(lo + a.write_off, B);
  const int es = RP_ST_BLK_EPOCH + blockIdx.x;
  const uint32_t e0 = epoch_begin(a.t, rank, es);
  const size_t zone = a.read_off + (size_t)zone_parity_begin(a.t, rank) * RP_OS_REGION;
  const char* src = (const char*)a.src[rank];
  char* dst = (char*)a.dst[rank];
  if (lo < hi) {
    for (int i = 1; i < a.world; ++i) {
      const int p = (rank + i) % a.world;
      copy_bytes(a.t.data[p] + zone + (size_t)rank * a.chunk, src, lo, hi, vec);
    }
    if (dst + (size_t)rank * B != src) copy_bytes(dst + (size_t)rank * B, src, lo, hi, vec);
  }
  if (!rank_barrier(a, rank, blockIdx.x, e0, 1)) return;
  epoch_end(a.t, rank, es, e0 + 1);
  if (lo < hi) {
    const char* z = a.t.data[rank] + zone;
    for (int i = 1; i < a.world; ++i) {
      const int p = (rank + i) % a.world;
      copy_bytes(dst + (size_t)p * B, z + (size_t)p * a.chunk, lo, hi, vec);
    }
  }
}

// K4p: one-shot broadcast, push form (multi-process, small messages, ONE barrier):
// the root stores its src into every peer's one-shot landing zone (and its own
// dst), all ranks meet once, every non-root copies the zone into its dst. Same
// zones and parity protocol as K1p / K3p. a.write_off = per-block byte slice.
__global__ void __launch_bounds__(kThreads) bcast_push_kernel(const CollArgs a, int vec) {
  const int rank = a.rank;
  if (rp_aborted(a.t, rank)) return;
  const size_t B = a.count;
  const size_t lo = (size_t)blockIdx.x * a.write_off;
  const size_t hi = std::min(lo + a.write_off, B);
  const int es = RP_ST_BLK_EPOCH + blockIdx.x;
  const uint32_t e0 = epoch_begin(a.t, rank, es);
  const size_t zone = a.read_off + (size_t)zone_parity_begin(a.t, rank) * RP_OS_REGION;
  char* dst = (char*)a.dst[rank];
  if (rank == a.root && lo < hi) {
    const char* src = (const char*)a.src[rank];
    for (int i = 1; i < a.world; ++i) copy_bytes(a.t.data[(rank + i) % a.world] + zone, src, lo, hi, vec);
    if (dst != src) copy_bytes(dst, src, lo, hi, vec);
  }
  if (!rank_barrier(a, rank, blockIdx.x, e0, 1)) return;
  epoch_end(a.t, rank, es, e0 + 1);
  if (rank != a.root && lo < hi) copy_bytes(dst, a.t.data[rank] + zone, lo, hi, vec);
}

// K4a: direct broadcast: every rank pulls root's pool copy.
__global__ void __launch_bounds__(kThreads) bcast_direct_kernel(const CollArgs a, int vec) {
  const int rank = a.rank >= 0 ? a.rank : (int)blockIdx.y;
  if (rp_aborted(a.t, rank)) return;
  const size_t B = a.count;
  const size_t lo = (size_t)blockIdx.x * a.chunk;
  const size_t hi = std::min(lo + a.chunk, B);
  const int es = RP_ST_BLK_EPOCH + blockIdx.x;
  const uint32_t e0 = epoch_begin(a.t, rank, es);
  if (rank == a.root && a.copy_in && lo < hi)
    copy_bytes(a.t.data[rank] + a.read_off, (const char*)a.src[rank], lo, hi, vec);
  if (!rank_barrier(a, rank, blockIdx.x, e0, 1)) return;
  const char* src = a.t.data[a.root] + a.read_off;
  char* dst = (char*)a.dst[rank];
  if (lo < hi && dst != src) copy_bytes(dst, src, lo, hi, vec);
  rank_barrier(a, rank, blockIdx.x, e0, 2);
  epoch_end(a.t, rank, es, e0 + 2);
}

// K4b: scatter + all-gather broadcast. The message is cut into `world` chunks
// of a.chunk*gridDim.x bytes... precisely: chunk c = [c*C, (c+1)*C), C = per-rank
// bytes (multiple of 16*gridDim.x); block b owns slice b of every chunk.
__global__ void __launch_bounds__(kThreads) bcast_scatter_kernel(const CollArgs a, size_t C, int vec) {
  const int rank = a.rank >= 0 ? a.rank : (int)blockIdx.y;
  if (rp_aborted(a.t, rank)) return;
  const size_t B = a.count;
  const size_t s0 = (size_t)blockIdx.x * a.chunk;
  const size_t s1 = std::min(s0 + a.chunk, C);
  char* root_pool = a.t.data[a.root] + a.read_off;
  const int es = RP_ST_BLK_EPOCH + blockIdx.x;
  const uint32_t e0 = epoch_begin(a.t, rank, es);
  if (rank == a.root && a.copy_in && s0 < s1) {
    for (int c = 0; c < a.world; ++c) {
      const size_t lo = c * C + s0, hi = std::min(c * C + s1, B);
      if (lo < hi) copy_bytes(root_pool, (const char*)a.src[rank], lo, hi, vec);
    }
  }
  if (!rank_barrier(a, rank, blockIdx.x, e0, 1)) return;
  // scatter: pull my chunk from root into my pool staging (root keeps its own)
  char* my_stage = a.t.data[rank] + a.write_off;
  {
    const size_t lo = rank * C + s0, hi = std::min(rank * C + s1, B);
    if (lo < hi && rank != a.root) copy_bytes(my_stage, root_pool, lo, hi, vec);
  }
  if (!rank_barrier(a, rank, blockIdx.x, e0, 2)) return;
  // all-gather: pull chunk c from its owner's staging (root's chunks from root_pool)
  char* dst = (char*)a.dst[rank];
  for (int i = 0; i < a.world; ++i) {
    const int c = (rank + i) % a.world;
    const size_t lo = c * C + s0, hi = std::min(c * C + s1, B);
    if (lo >= hi) continue;
    const char* src = (c == a.root) ? root_pool : (a.t.data[c] + a.write_off);
    if (dst + 0 == src) continue;
    copy_bytes(dst, src, lo, hi, vec);
  }
  rank_barrier(a, rank, blockIdx.x, e0, 3);
  epoch_end(a.t, rank, es, e0 + 3);
}

}  // namespace rp

// ===========================================================================
// host launchers
// ===========================================================================
using namespace rp;

namespace {

// Find which pool offset (if any) a pointer of rank r lies in.
bool in_pool(rp_comm* c, int r, const void* p, size_t bytes, size_t* off) {
  const char* base = c->table.data[r];
  const char* q = (const char*)p;
  if (q >= base && q + bytes <= base + c->pool_bytes) {
    *off = (size_t)(q - base);
    return true;
  }
  return false;
}

// Every replica's pointer at the same pool offset (symmetric allocation).
bool symmetric_in_pool(rp_comm* c, const void* const* ptrs, size_t bytes, size_t* off) {
  const int n = c->is_virtual ? c->world : 1;
  size_t o0 = 0;
  for (int i = 0; i < n; ++i) {
    const int r = c->is_virtual ? i : c->rank;
    size_t o;
    if (!in_pool(c, r, ptrs[i], bytes, &o)) return false;
    if (i == 0) o0 = o;
    else if (o != o0) return false;
  }
  *off = o0;
  return true;
}

size_t round_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

void fill_ptrs(rp_comm* c, CollArgs& a, const void* const* src, void* const* dst) {
  const int n = c->is_virtual ? c->world : 1;
  for (int i = 0; i < RP_MAX_RANKS; ++i) {
    a.src[i] = nullptr;
    a.dst[i] = nullptr;
  }
  for (int i = 0; i < n; ++i) {
    const int r = c->is_virtual ? i : c->rank;
    a.src[r] = src ? src[i] : nullptr;
    a.dst[r] = dst ? dst[i] : nullptr;
  }
}

// Launch a collective kernel; with RP_TRACE=<file> (analysis only) also collect
// the per-block %globaltimer stamps (rp_device.cuh rp_trace) and append them as
// one JSON line per launch. Tracing synchronises the stream.
int launch_coll(rp_comm* c, const void* fn, dim3 grid, CollArgs& a, cudaStream_t stream, const char* tag,
                int threads = kThreads, bool coop = true) {
  const char* path = getenv("RP_TRACE");
  const size_t n = (size_t)grid.x * grid.y * 8;
  unsigned long long* buf = nullptr;
  a.trace = nullptr;
  if (path) {
    RP_CUDA_CHECK(cudaMalloc(&buf, n * 8));
    RP_CUDA_CHECK(cudaMemsetAsync(buf, 0, n * 8, stream));
    a.trace = buf;
  }
  void* args[] = {&a};
  const int rc = rp_launch(c, fn, grid, dim3(threads), args, 0, stream, coop);
  if (path) {
    std::vector<unsigned long long> h(n);
    cudaStreamSynchronize(stream);
    cudaMemcpy(h.data(), buf, n * 8, cudaMemcpyDeviceToHost);
    cudaFree(buf);
    a.trace = nullptr;
    char fname[1024];
    snprintf(fname, sizeof(fname), "%s.rank%d", path, c->rank);
    if (FILE* f = fopen(fname, "a")) {
      fprintf(f, "{\"tag\":\"%s\",\"rank\":%d,\"world\":%d,\"grid\":[%u,%u],\"count\":%zu,\"stamps\":[", tag, c->rank,
              c->world, grid.x, grid.y, a.count);
      for (size_t i = 0; i < n; ++i) fprintf(f, "%s%llu", i ? "," : "", h[i]);
      fprintf(f, "]}\n");
      fclose(f);
    }
  }
  return rc;
}

// Launch a dynamically scheduled two-shot (ar_twoshot_dyn): pick the grid and the
// tile size and launch. Everything per call that must agree across ranks (phase
// barrier targets, tile counters) lives on the device (rp_internal.h RP_ST_*),
// so the launch is the same every time and can be captured in a CUDA graph.
int dyn_launch(rp_comm* c, const void* fn, CollArgs& a, cudaStream_t stream, const char* tag, int max_blocks,
               int threads, uint32_t tile_v) {
  const int W = c->world;
  const size_t Vc = a.chunk;
  int blocks = (int)std::min<size_t>((Vc + (size_t)threads * 2 - 1) / ((size_t)threads * 2),
                                     (size_t)(max_blocks > 0 ? max_blocks : RP_MAX_BLOCKS));
  blocks = rp_blocks_per_rank(c, fn, threads, std::max(blocks, 1));
  // tiles are claimed per warp: >= 4 per warp so the tail is short, 4..64 KiB
  if (tile_v == 0) {
    const uint32_t warps = (uint32_t)blocks * (threads / 32);
    size_t tv = Vc / ((size_t)warps * 4);
    tile_v = (uint32_t)std::min<size_t>(std::max<size_t>(round_up(tv, 256), 256), 4096);
  }
  a.tile_v = tile_v;
  return launch_coll(c, fn, dim3(blocks, c->is_virtual ? W : 1), a, stream, tag, threads);
}

void base_args(rp_comm* c, CollArgs& a) {
  a.trace = nullptr;
  a.tile_v = 0;
  a.relay_root_blocks = 0;
  a.t = c->table;
  a.world = c->world;
  a.rank = c->is_virtual ? -1 : c->rank;
  a.timeout_ns = c->timeout_ns;
}

// An in-place all-reduce of a registered user buffer (rp_register_*), no cast:
// every peer's copy is addressable, so the zero-copy pull two-shot applies.
bool registered_in_place(rp_comm* c, const void* const* src, const void* const* dst, size_t count, int dtype_in,
                         int dtype_comm, int dtype_out, int* reg, size_t* off) {
  if (c->is_virtual || c->regs.empty() || src[0] != dst[0] || dtype_in != dtype_comm || dtype_out != dtype_comm)
    return false;
  return rp_registered(c, src[0], count * rp_dtype_size(dtype_comm), reg, off);
}

}  // namespace

// shared with rp_apply.cu (fused optimizer apply)
bool rp_symmetric_in_pool(rp_comm* c, const void* const* ptrs, size_t bytes, size_t* off) {
  return symmetric_in_pool(c, ptrs, bytes, off);
}
void rp_base_args(rp_comm* c, CollArgs& a) { base_args(c, a); }
int rp_dyn_launch(rp_comm* c, const void* fn, CollArgs& a, cudaStream_t stream, const char* tag) {
  return dyn_launch(c, fn, a, stream, tag, 0, kThreads, 0);
}

// Algorithm choice: deterministic in (arguments, world, NVLS placement), hence
// identical on every rank (NVLS buffers are allocated symmetrically).
int rp_resolve_ar_algo(rp_comm* c, const void* const* src, const void* const* dst, size_t count, int dtype_in,
                       int dtype_comm, int dtype_out, int op, int algo) {
  if (algo != RP_ALGO_AUTO) return algo;
  const int W = c->world;
  // virtual replicas share one GPU's HBM: the flat kernel reads and writes every
  // buffer once with no barrier (RP_VIRTUAL_ALGO=rank restores the rank-partitioned
  // one-shot / two-shot below, for A/B)
  if (c->is_virtual && W > 1) {
    const char* va = getenv("RP_VIRTUAL_ALGO");
    if (!(va && va[0] == 'r')) return RP_ALGO_FLAT;
  }
  const size_t bytes = count * rp_dtype_size(dtype_comm);
  // NVLS (in-switch reduce + multicast store) moves (N+1)/N of the message per
  // link direction against 2(N-1)/N for the two-shot: it wins from N=4 on, above
  // the one-shot regime (tools/sweep.py, profiles/r01_sweep_nvls_n4.txt: 22.6 vs
  // 38 us at 2 MiB, 168 vs 201 us at 64 MiB). The caller opts in by placing the
  // buffer in the NVLS region; RP_NVLS=0 disables the automatic choice.
  const char* ne = getenv("RP_NVLS");
  if (!c->is_virtual && W >= 4 && !(ne && ne[0] == '0') && src[0] == dst[0] && dtype_in == dtype_comm &&
      dtype_out == dtype_comm && op != RP_MAX &&
      (dtype_comm == RP_F32 || dtype_comm == RP_BF16 || dtype_comm == RP_F16) && bytes >= ((size_t)512 << 10) &&
      rp_nvls_covers(c, dst[0], bytes))
    return RP_ALGO_NVLS;
  // crossover from tools/sweep.py: the push one-shot (multi-process, one barrier,
  // ~8-12 us) beats the two-phase two-shot (~20-30 us floor) up to ~2 MiB at
  // N=2 and the landing zone bounds it at RP_OS_REGION/N; virtual replicas use
  // the pull forms, whose one-shot reads N times the message from HBM
  size_t oneshot_max;
  if (c->is_virtual) oneshot_max = W <= 2 ? ((size_t)512 << 10) : (W <= 4 ? ((size_t)256 << 10) : ((size_t)128 << 10));
  else oneshot_max = std::min(RP_OS_REGION / (size_t)W, W <= 2 ? ((size_t)2 << 20) : ((size_t)1 << 20));
  return bytes <= oneshot_max ? RP_ALGO_ONESHOT : RP_ALGO_TWOSHOT;
}

// What rp_launch_all_reduce will do with these arguments, for cross-rank agreement
// checks: every rank must pick the same algorithm, data-movement form and pool
// placement (a rank passing a pool view where a peer passes a plain tensor would
// launch a different kernel against the shared barrier state).
void rp_plan_all_reduce(rp_comm* c, const void* const* src, const void* const* dst, size_t count, int dtype_in,
                        int dtype_comm, int dtype_out, int op, int algo, int64_t* plan) {
  const int a = rp_resolve_ar_algo(c, src, dst, count, dtype_in, dtype_comm, dtype_out, op, algo);
  size_t so = 0, doff = 0;
  const bool sp = symmetric_in_pool(c, src, count * rp_dtype_size(dtype_in), &so);
  const bool dp = symmetric_in_pool(c, dst, count * rp_dtype_size(dtype_out), &doff);
  int reg = -1;
  size_t roff = 0;
  const bool rg = registered_in_place(c, src, dst, count, dtype_in, dtype_comm, dtype_out, &reg, &roff);
  int push = 0;
  if (!c->is_virtual && a != RP_ALGO_NVLS)
    push = (a == RP_ALGO_ONESHOT || !((sp || rg) && dtype_in == dtype_comm)) ? 1 : 0;
  if (const char* e = getenv("RP_AR_IMPL")) push = (e[0] == 'p' && e[1] == 'u' && e[2] == 's') ? 1 : 0;
  plan[0] = a;
  plan[1] = push;
  plan[2] = sp ? (int64_t)so : (rg ? -2 : -1);
  plan[3] = dp ? (int64_t)doff : (rg ? -2 : -1);
}

int rp_launch_all_reduce(rp_comm* c, const void* const* src, void* const* dst, size_t count,
                         int dtype_in, int dtype_comm, int dtype_out, int op, int algo,
                         cudaStream_t stream) {
  if (count == 0) return RP_OK;
  if (!rp_dtype_valid(dtype_in) || !rp_dtype_valid(dtype_comm) || !rp_dtype_valid(dtype_out))
    return rp_fail(RP_ERR_INVALID, "all_reduce: unknown dtype");
  if (op < RP_SUM || op > RP_PREMEAN) return rp_fail(RP_ERR_INVALID, "all_reduce: unknown op");
  auto pair_ok = [&](int user) {
    return user == dtype_comm ||
           (user == RP_F32 && (dtype_comm == RP_BF16 || dtype_comm == RP_F16));
  };
  if (!pair_ok(dtype_in) || !pair_ok(dtype_out))
    return rp_fail(RP_ERR_INVALID, "all_reduce: dtype_in/dtype_out must equal dtype_comm "
                                   "or be f32 with a 16-bit dtype_comm");
  const size_t esz = rp_dtype_size(dtype_comm);
  const size_t vec = 16 / esz;
  const size_t V = (count + vec - 1) / vec;
  const int W = c->world;
  const int nrep = c->is_virtual ? W : 1;

  CollArgs a;
  base_args(c, a);
  fill_ptrs(c, a, src, dst);
  a.count = count;
  a.dtype_in = dtype_in;
  a.dtype_out = dtype_out;
  a.root = 0;
  a.chunk = 0;
  a.read_off = a.write_off = 0;
  a.copy_in = a.copy_out = 0;

  if (W == 1) {  // a single replica: the fold of one operand (identity / x/1)
    const void* fn = pick_ar_any(dtype_comm, op, RP_ALGO_TWOSHOT, 1, 0);
    a.src[0] = src[0];
    a.dst[0] = dst[0];
    const int blocks = (int)std::min<size_t>((V + kThreads - 1) / kThreads, (size_t)c->num_sms * 4);
    void* args[] = {&a};
    RP_CUDA_CHECK(cudaLaunchKernel(fn, dim3(std::max(blocks, 1)), dim3(kThreads), args, 0, stream));
    return RP_OK;
  }

  const size_t bytes = count * esz;
  algo = rp_resolve_ar_algo(c, src, (const void* const*)dst, count, dtype_in, dtype_comm, dtype_out, op, algo);
  if (algo == RP_ALGO_NVLS) {  // in-switch reduction, in place in the NVLS region
    if (c->is_virtual) return rp_fail(RP_ERR_CONFIG, "all_reduce(nvls): needs a multi-process communicator");
    if (src[0] != dst[0] || dtype_in != dtype_comm || dtype_out != dtype_comm)
      return rp_fail(RP_ERR_INVALID, "all_reduce(nvls): in place, without a cast");
    return rp_nvls_launch(c, dst[0], count, dtype_comm, op, stream, dyn_launch, a);
  }
  if (algo == RP_ALGO_FLAT) {
    if (!c->is_virtual) return rp_fail(RP_ERR_INVALID, "all_reduce(flat): needs a virtual communicator");
    // A/B: the bulk-copy (cp.async.bulk + mbarrier) staging of the same fold, for
    // aligned buffers without a fused cast
    if (const char* be = getenv("RP_VFLAT_BULK")) {
      bool ok = be[0] == '1' && dtype_in == dtype_comm && dtype_out == dtype_comm;
      for (int i = 0; i < W && ok; ++i) ok = ((((uintptr_t)src[i]) | ((uintptr_t)dst[i])) & 15u) == 0;
      if (ok) {
        const void* fb = pick_ar_any(dtype_comm, op, RP_ALGO_FLAT_BULK, W, 0);
        if (!fb) return rp_fail(RP_ERR_INVALID, "all_reduce(flat bulk): unsupported replica count (2..8)");
        const size_t smem = rp_bulk_smem_bytes(W);
        RP_CUDA_CHECK(cudaFuncSetAttribute(fb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int occ = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fb, rp_bulk_threads(), smem) != cudaSuccess || occ < 1)
          occ = 1;
        int blocks = occ * c->num_sms;
        if (c->cap() > 0) blocks = std::min(blocks, c->cap());
        const size_t warps = (size_t)blocks * (rp_bulk_threads() / 32);
        size_t tv = V / (warps * 8);  // ~8 tiles per warp: the tail is one small tile
        if (const char* e = getenv("RP_VFLAT_TILE")) tv = (size_t)atoi(e);
        a.tile_v = (uint32_t)std::min<size_t>(std::max<size_t>(round_up(tv, 256), 256), 4096);
        void* args[] = {&a};
        return rp_launch(c, fb, dim3(std::max(blocks, 1)), dim3(rp_bulk_threads()), args, smem, stream, false);
      }
    }
    const void* fn = pick_ar_any(dtype_comm, op, RP_ALGO_FLAT, W, 0);
    if (!fn) return rp_fail(RP_ERR_INVALID, "all_reduce(flat): unsupported replica count (2..8)");
    // one co-resident wave on EVERY SM; tiles of 256..4096 vectors
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kThreads, 0) != cudaSuccess || occ < 1) occ = 1;
    int blocks = (int)std::min<size_t>((size_t)occ * c->num_sms, (V + 31) / 32);
    if (c->cap() > 0) blocks = std::min(blocks, c->cap());
    blocks = std::max(blocks, 1);
    const size_t warps = (size_t)blocks * (kThreads / 32);
    size_t tv = V / (warps * 8);  // ~8 tiles per warp: the tail is one small tile
    if (const char* e = getenv("RP_VFLAT_TILE")) tv = (size_t)atoi(e);
    a.tile_v = (uint32_t)std::min<size_t>(std::max<size_t>(round_up(tv, 256), 256), 4096);
    return launch_coll(c, fn, dim3(blocks), a, stream, "virtual_flat", kThreads, /*coop=*/false);
  }
  if (algo != RP_ALGO_ONESHOT && algo != RP_ALGO_TWOSHOT)
    return rp_fail(RP_ERR_INVALID, "all_reduce: unknown algorithm");

  // Data-movement form (measured): for one-process-per-GPU
  // communicators the one-shot is the push form (reads src in place, ONE barrier:
  // 8 us vs 16 us at 1 KiB, N=2); the two-shot is the pull form when the source is
  // pool-resident (zero-copy: 628 vs 512 GB/s at 256 MiB, N=2) and the push form
  // when it would need staging (it reads src in place: 465 vs 376 GB/s at 64 MiB).
  // Virtual replicas share one GPU's HBM: the pull form, which reads and writes
  // every buffer exactly once. RP_AR_IMPL=push|pull overrides (tests, A/B).
  int push;
  if (c->is_virtual) {
    push = 0;
  } else if (algo == RP_ALGO_ONESHOT) {
    push = 1;
  } else {
    size_t off0;
    int reg0;
    push = (dtype_in == dtype_comm &&
            (symmetric_in_pool(c, src, count * rp_dtype_size(dtype_in), &off0) ||
             registered_in_place(c, src, (const void* const*)dst, count, dtype_in, dtype_comm, dtype_out, &reg0, &off0)))
               ? 0 : 1;
  }
  if (const char* e = getenv("RP_AR_IMPL")) push = (e[0] == 'p' && e[1] == 'u' && e[2] == 's') ? 1 : 0;
  if (push) return launch_push(c, src, dst, count, dtype_in, dtype_comm, dtype_out, op, algo, stream, a);

  // a registered user buffer, in place: the pool two-shot with every rank's copy
  // of the buffer as the data table (read_off = write_off = the offset inside it)
  {
    int reg = -1;
    size_t roff = 0;
    if (algo == RP_ALGO_TWOSHOT &&
        registered_in_place(c, src, (const void* const*)dst, count, dtype_in, dtype_comm, dtype_out, &reg, &roff)) {
      const void* fn = pick_ar_any(dtype_comm, op, RP_ALGO_TWOSHOT, W, 0);
      if (!fn) return rp_fail(RP_ERR_INVALID, "all_reduce: unsupported world size (1..8)");
      for (int p = 0; p < W; ++p) a.t.data[p] = c->regs[reg].ptr[p];
      a.read_off = a.write_off = roff;
      a.copy_in = a.copy_out = 0;
      a.chunk = (V + W - 1) / W;
      return dyn_launch(c, fn, a, stream, "twoshot_registered", 0, kThreads, 0);
    }
  }

  // Placement. Pool-resident buffers (symmetric offsets, allocated identically on
  // every rank) are exchanged zero-copy; anything else is staged through scratch.
  const size_t padded = round_up(V * 16, RP_ALIGN);
  size_t src_off = 0, dst_off = 0;
  const bool src_pool = dtype_in == dtype_comm &&
                        symmetric_in_pool(c, src, count * rp_dtype_size(dtype_in), &src_off);
  const bool dst_pool = dtype_out == dtype_comm &&
                        symmetric_in_pool(c, (const void* const*)dst, count * rp_dtype_size(dtype_out), &dst_off);
  if (src_pool && dst_pool && src_off != dst_off &&
      !(dst_off + padded <= src_off || src_off + padded <= dst_off))
    return rp_fail(RP_ERR_INVALID, "all_reduce: partially overlapping pool buffers");
  if (algo == RP_ALGO_ONESHOT && src_pool && dst_pool && src_off == dst_off)
    algo = RP_ALGO_TWOSHOT;  // in-place: peers are still reading our input

  const size_t scratch = round_up(c->reserved, RP_ALIGN);
  const size_t scratch_end = c->scratch_end();
  size_t need_scratch = 0;
  if (algo == RP_ALGO_ONESHOT) {
    a.copy_in = !src_pool;
    a.read_off = src_pool ? src_off : scratch;
    a.copy_out = 1;  // every rank writes its own dst directly (with the output cast)
    need_scratch = src_pool ? 0 : padded;
  } else if (src_pool && dst_pool) {
    a.read_off = src_off;
    a.write_off = dst_off;
  } else if (src_pool) {          // keep src intact: push into scratch, copy out
    a.read_off = src_off;
    a.write_off = scratch;
    a.copy_out = 1;
    need_scratch = padded;
  } else if (dst_pool) {          // stage in, push straight into the dst region
    a.copy_in = 1;
    a.read_off = scratch;
    a.write_off = dst_off;
    need_scratch = padded;
  } else {                        // stage in, reduce in place in scratch, copy out
    a.copy_in = 1;
    a.copy_out = 1;
    a.read_off = a.write_off = scratch;
    need_scratch = padded;
  }

  if (scratch + need_scratch > scratch_end) {
    // Stage in pieces that fit the scratch window (each piece is a full collective).
    const size_t avail = scratch_end > scratch ? scratch_end - scratch : 0;
    size_t piece = (avail / 16) * vec;
    piece -= piece % ((size_t)W * vec * 64);
    if (piece == 0) return rp_fail(RP_ERR_INVALID, "all_reduce: pool too small to stage the message");
    for (size_t off = 0; off < count; off += piece) {
      const size_t n = std::min(piece, count - off);
      const void* s2[RP_MAX_RANKS];
      void* d2[RP_MAX_RANKS];
      for (int i = 0; i < nrep; ++i) {
        s2[i] = (const char*)src[i] + off * rp_dtype_size(dtype_in);
        d2[i] = (char*)dst[i] + off * rp_dtype_size(dtype_out);
      }
      const int rc = rp_launch_all_reduce(c, s2, d2, n, dtype_in, dtype_comm, dtype_out, op, algo, stream);
      if (rc) return rc;
    }
    return RP_OK;
  }

  const void* fn = pick_ar_any(dtype_comm, op, algo, W, 0);
  if (!fn) return rp_fail(RP_ERR_INVALID, "all_reduce: unsupported world size (1..8)");
  if (algo == RP_ALGO_TWOSHOT) {
    a.chunk = (V + W - 1) / W;
    return dyn_launch(c, fn, a, stream, "twoshot_pull", 0, kThreads, 0);
  }
  const size_t per_block = (size_t)kThreads * 2;
  int blocks = (int)std::min<size_t>((V + per_block - 1) / per_block, (size_t)RP_MAX_BLOCKS);
  blocks = rp_blocks_per_rank(c, fn, kThreads, std::max(blocks, 1));
  return launch_coll(c, fn, dim3(blocks, c->is_virtual ? W : 1), a, stream, "oneshot_pull");
}

// Push-form all-reduce (K1p one-shot / K2p two-shot, rp_allreduce.cuh).
static int launch_push(rp_comm* c, const void* const* src, void* const* dst, size_t count, int dtype_in,
                       int dtype_comm, int dtype_out, int op, int algo, cudaStream_t stream, CollArgs a) {
  const int W = c->world;
  const int nrep = c->is_virtual ? W : 1;
  const size_t vec = 16 / rp_dtype_size(dtype_comm);
  const size_t V = (count + vec - 1) / vec;
  // one-shot landing zone: W slots of V vectors must fit one parity region
  if (algo == RP_ALGO_ONESHOT && (size_t)W * V * 16 > RP_OS_REGION) algo = RP_ALGO_TWOSHOT;
  const size_t scratch = round_up(c->reserved, RP_ALIGN);
  const size_t scratch_end = c->scratch_end();
  size_t work;
  if (algo == RP_ALGO_ONESHOT) {
    a.read_off = c->oneshot_zone(0);  // the kernel adds the device-side parity
    a.copy_out = 1;
    a.chunk = 0;
    work = V;
  } else {
    const size_t Vc = (V + W - 1) / W;
    const size_t qbytes = round_up((size_t)W * Vc * 16, RP_ALIGN);
    size_t dst_off = 0;
    const bool dst_pool = dtype_out == dtype_comm &&
                          symmetric_in_pool(c, (const void* const*)dst, count * rp_dtype_size(dtype_out), &dst_off) &&
                          dst_off + round_up(V * 16, RP_ALIGN) <= scratch;
    const size_t need = qbytes + (dst_pool ? 0 : qbytes);
    if (scratch + need > scratch_end) {
      // pieces that fit the staging window (each piece is a full collective)
      const size_t avail = scratch_end > scratch ? scratch_end - scratch : 0;
      size_t piece = (avail / (dst_pool ? 1 : 2) / 16) * vec;
      piece -= piece % ((size_t)W * vec * 64);
      if (piece == 0) return rp_fail(RP_ERR_INVALID, "all_reduce: pool too small to stage the message");
      for (size_t off = 0; off < count; off += piece) {
        const size_t n = std::min(piece, count - off);
        const void* s2[RP_MAX_RANKS];
        void* d2[RP_MAX_RANKS];
        for (int i = 0; i < nrep; ++i) {
          s2[i] = (const char*)src[i] + off * rp_dtype_size(dtype_in);
          d2[i] = (char*)dst[i] + off * rp_dtype_size(dtype_out);
        }
        CollArgs a2 = a;
        fill_ptrs(c, a2, s2, d2);
        const int rc = launch_push(c, s2, d2, n, dtype_in, dtype_comm, dtype_out, op, algo, stream, a2);
        if (rc) return rc;
      }
      return RP_OK;
    }
    a.chunk = Vc;
    a.read_off = scratch;
    a.write_off = dst_pool ? dst_off : scratch + qbytes;
    a.copy_out = dst_pool ? 0 : 1;
    a.copy_in = 0;
    a.count = count;
    const void* fn = pick_ar_any(dtype_comm, op, algo, W, 1);
    if (!fn) return rp_fail(RP_ERR_INVALID, "all_reduce: unsupported world size (1..8)");
    return dyn_launch(c, fn, a, stream, "twoshot_push", 0, kThreads, 0);
  }
  a.count = count;
  const void* fn = pick_ar_any(dtype_comm, op, algo, W, 1);
  if (!fn) return rp_fail(RP_ERR_INVALID, "all_reduce: unsupported world size (1..8)");
  const size_t per_block = (size_t)kThreads * 2;
  int blocks = (int)std::min<size_t>((work + per_block - 1) / per_block, (size_t)RP_MAX_BLOCKS);
  blocks = rp_blocks_per_rank(c, fn, kThreads, std::max(blocks, 1));
  return launch_coll(c, fn, dim3(blocks, c->is_virtual ? W : 1), a, stream,
                     algo == RP_ALGO_TWOSHOT ? "twoshot_push" : "oneshot_push");
}

// All-gather: rank order (graph.py:575-579). Inputs are read from the peers'
// pools: in place (src == dst + rank*bytes, dst in the pool) or staged.
int rp_launch_all_gather(rp_comm* c, const void* const* src, void* const* dst, size_t bytes,
                         cudaStream_t stream) {
  if (bytes == 0) return RP_OK;
  const int W = c->world;
  const int nrep = c->is_virtual ? W : 1;
  CollArgs a;
  base_args(c, a);
  fill_ptrs(c, a, src, dst);
  a.count = bytes;
  a.copy_out = 0;
  a.write_off = 0;
  a.root = 0;
  bool vec = (bytes % 16) == 0;
  for (int i = 0; i < nrep; ++i)
    vec = vec && ((uintptr_t)src[i] % 16 == 0) && ((uintptr_t)dst[i] % 16 == 0);
  const size_t scratch = round_up(c->reserved, RP_ALIGN);
  const size_t scratch_end = c->scratch_end();
  // small messages between processes: push into the peers' landing zones, one
  // barrier (K3p); the bound keeps world slots inside one zone
  const size_t slot = round_up(bytes, 16);
  if (!c->is_virtual && W > 1 && slot * W <= RP_OS_REGION && slot <= ((size_t)1 << 20) &&
      getenv("RP_AG_PULL") == nullptr) {
    a.read_off = c->oneshot_zone(0);
    a.chunk = slot;
    const size_t per_block_min = (size_t)16 * kThreads * 2;
    const int want = (int)std::min<size_t>((bytes + per_block_min - 1) / per_block_min, (size_t)RP_MAX_BLOCKS);
    const int blocks = rp_blocks_per_rank(c, (const void*)allgather_push_kernel, kThreads, std::max(want, 1));
    a.write_off = round_up((bytes + blocks - 1) / blocks, 16);
    int ivec = vec ? 1 : 0;
    void* args[] = {&a, &ivec};
    return rp_launch(c, (const void*)allgather_push_kernel, dim3(blocks), dim3(kThreads), args, 0, stream);
  }
  bool in_place = true;
  for (int i = 0; i < nrep && in_place; ++i) {
    const int r = c->is_virtual ? i : c->rank;
    in_place = (const char*)src[i] == (const char*)dst[i] + (size_t)r * bytes;
  }
  size_t read_stride = 0, doff = 0;
  if (in_place && symmetric_in_pool(c, (const void* const*)dst, bytes * W, &doff)) {
    a.copy_in = 0;
    a.read_off = doff;
    read_stride = bytes;
  } else {
    if (scratch + round_up(bytes, RP_ALIGN) > scratch_end)
      return rp_fail(RP_ERR_INVALID, "all_gather: per-rank message exceeds the staging pool");
    a.copy_in = 1;
    a.read_off = scratch;
  }
  const size_t per_block_min = (size_t)16 * kThreads * 4;
  const int want = (int)std::min<size_t>((bytes + per_block_min - 1) / per_block_min, (size_t)RP_MAX_BLOCKS);
  const int blocks = rp_blocks_per_rank(c, (const void*)allgather_kernel, kThreads, std::max(want, 1));
  a.chunk = round_up((bytes + blocks - 1) / blocks, 16);
  int ivec = vec ? 1 : 0;
  void* args[] = {&a, &read_stride, &ivec};
  return rp_launch(c, (const void*)allgather_kernel, dim3(blocks, c->is_virtual ? W : 1), dim3(kThreads),
                   args, 0, stream);
}

// Broadcast from `root` (the reference always uses rank 0, graph.py:581).
// In place (src == dst on every rank, dst in the pool) the root's buffer is read
// directly; otherwise the root stages its src into scratch.
int rp_launch_broadcast(rp_comm* c, const void* const* src, void* const* dst, size_t bytes, int root,
                        int algo, cudaStream_t stream) {
  if (bytes == 0) return RP_OK;
  const int W = c->world;
  if (root < 0 || root >= W) return rp_fail(RP_ERR_INVALID, "broadcast: root out of range");
  const int nrep = c->is_virtual ? W : 1;
  CollArgs a;
  base_args(c, a);
  fill_ptrs(c, a, src, dst);
  a.count = bytes;
  a.root = root;
  a.copy_out = 0;
  const size_t scratch = round_up(c->reserved, RP_ALIGN);
  const size_t scratch_end = c->scratch_end();
  const size_t pb = round_up(bytes, RP_ALIGN);
  bool vec = (bytes % 16) == 0;
  bool in_place = true;
  for (int i = 0; i < nrep; ++i) {
    const int r = c->is_virtual ? i : c->rank;
    if (r == root) vec = vec && ((uintptr_t)src[i] % 16 == 0);
    vec = vec && ((uintptr_t)dst[i] % 16 == 0);
    in_place = in_place && (src[i] == dst[i]);
  }
  // NVLS: destination placed in the multicast region (symmetric on every rank, so
  // every rank makes the same choice); the root multicasts from any local source
  if (!c->is_virtual && W >= 2 && (algo == RP_ALGO_NVLS || algo == RP_ALGO_AUTO)) {
    const char* ne = getenv("RP_NVLS");
    // (a property of dst alone, which is symmetric: every rank decides alike)
    const bool nvls_ok = rp_nvls_covers(c, dst[0], bytes) && bytes % 16 == 0;
    if (algo == RP_ALGO_NVLS || (nvls_ok && !(ne && ne[0] == '0')))
      return rp_nvls_bcast_launch(c, src[0], dst[0], bytes, root, stream, dyn_launch, a);
  } else if (algo == RP_ALGO_NVLS) {
    return rp_fail(RP_ERR_CONFIG, "broadcast(nvls): needs a multi-process communicator");
  }
  // small messages between processes: the root pushes into the peers' landing zones
  // (K4p), one barrier
  if (!c->is_virtual && W > 1 && algo == RP_ALGO_AUTO && bytes <= std::min(RP_OS_REGION, (size_t)1 << 20) &&
      getenv("RP_BCAST_PULL") == nullptr) {
    a.read_off = c->oneshot_zone(0);
    const size_t per_block_min = (size_t)16 * kThreads * 2;
    const int want = (int)std::min<size_t>((bytes + per_block_min - 1) / per_block_min, (size_t)RP_MAX_BLOCKS);
    const int blocks = rp_blocks_per_rank(c, (const void*)bcast_push_kernel, kThreads, std::max(want, 1));
    a.write_off = round_up((bytes + blocks - 1) / blocks, 16);
    int ivec = vec ? 1 : 0;
    void* args[] = {&a, &ivec};
    return rp_launch(c, (const void*)bcast_push_kernel, dim3(blocks), dim3(kThreads), args, 0, stream);
  }
  // large messages between processes: the pipelined relay (K4r) from 32 MiB, where
  // its pipeline fill is amortised (below, direct pull / scatter are faster:
  // profiles/r01_sweep_nccl_final_n4.txt). It lands in the dst itself when that is
  // pool-resident (symmetric), else in staging
  if (!c->is_virtual && W > 1 && bytes % 16 == 0 &&
      (algo == RP_ALGO_RELAY || (algo == RP_ALGO_AUTO && bytes >= ((size_t)32 << 20) &&
                                 getenv("RP_BCAST_PULL") == nullptr))) {
    size_t loff = 0;
    const bool land_dst = symmetric_in_pool(c, (const void* const*)dst, bytes, &loff);
    if (!land_dst) loff = scratch;
    if (land_dst || scratch + pb <= scratch_end)
      return rp_relay_bcast_launch(c, src[0], dst[0], bytes, root, land_dst, loff, stream, dyn_launch, a);
    if (algo == RP_ALGO_RELAY) return rp_fail(RP_ERR_INVALID, "broadcast(relay): message exceeds the staging pool");
  } else if (algo == RP_ALGO_RELAY) {
    return rp_fail(RP_ERR_INVALID, "broadcast(relay): multi-process, 16-byte multiple sizes only");
  }
  size_t doff = 0;
  if (in_place && symmetric_in_pool(c, (const void* const*)dst, bytes, &doff)) {
    a.copy_in = 0;
    a.read_off = doff;
  } else {
    a.copy_in = 1;
    a.read_off = scratch;
  }
  // scatter + all-gather from 8 MiB at N > 2 (2-4 MiB: direct pull is faster, sweep)
  if (algo == RP_ALGO_AUTO)
    algo = (bytes >= ((size_t)8 << 20) && W > 2 && !c->is_virtual) || (bytes >= ((size_t)1 << 20) && W > 2 && c->is_virtual)
               ? RP_ALGO_SCATTER
               : RP_ALGO_DIRECT;
  if (algo == RP_ALGO_SCATTER) {
    a.write_off = a.copy_in ? scratch + pb : scratch;  // per-rank staging of its chunk
    if (a.write_off + pb > scratch_end) algo = RP_ALGO_DIRECT;
  }
  if (a.copy_in && scratch + pb > scratch_end)
    return rp_fail(RP_ERR_INVALID, "broadcast: message exceeds the staging pool");
  int ivec = vec ? 1 : 0;
  const size_t per_block_min = (size_t)16 * kThreads * 4;
  if (algo == RP_ALGO_SCATTER) {
    const int want = (int)std::min<size_t>((bytes / W + per_block_min - 1) / per_block_min, (size_t)RP_MAX_BLOCKS);
    const int blocks = rp_blocks_per_rank(c, (const void*)bcast_scatter_kernel, kThreads, std::max(want, 1));
    size_t C = round_up((bytes + W - 1) / W, (size_t)16 * blocks);
    a.chunk = C / blocks;
    void* args[] = {&a, &C, &ivec};
    return rp_launch(c, (const void*)bcast_scatter_kernel, dim3(blocks, c->is_virtual ? W : 1),
                     dim3(kThreads), args, 0, stream);
  }
  a.write_off = 0;
  const int want = (int)std::min<size_t>((bytes + per_block_min - 1) / per_block_min, (size_t)RP_MAX_BLOCKS);
  const int blocks = rp_blocks_per_rank(c, (const void*)bcast_direct_kernel, kThreads, std::max(want, 1));
  a.chunk = round_up((bytes + blocks - 1) / blocks, 16);
  void* args[] = {&a, &ivec};
  return rp_launch(c, (const void*)bcast_direct_kernel, dim3(blocks, c->is_virtual ? W : 1), dim3(kThreads),
                   args, 0, stream);
}

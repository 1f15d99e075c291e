// Fused optimizer apply: the wrap_optimizer step as ONE kernel.
//
// The reference's wrapped optimizer averages every gradient with
// all_sum(g / R) and then applies the base rule on every replica
// (PAPER.md:196-206); all replicas compute the same update on
// the same averaged gradient ("mirrored" variables). Here the
// gradient bucket is folded two-shot style and the update is applied by the rank
// that owns each chunk, which then stores the UPDATED PARAMETERS into every
// rank's parameter bucket -- the all-gather phase carries parameters instead of
// averaged gradients, so the traffic equals one all-reduce of the bucket, the
// optimizer reads/writes 1/N of the parameters per rank, and optimizer state is
// kept for the owned shard only. Every replica receives the same bits (one
// writer per element), so mirrored semantics hold exactly.
//
//   P0  barrier 0: every rank's gradient bucket is packed (pool, symmetric)
//   P1  tiles of chunk `rank` (per-warp claims): pull the N gradient packets,
//       fold premean in rank order (bit-identical to the unfused path's averaged
//       gradient), apply SGD / Adam / AdamW in f32 to the owned parameters and
//       state, store the new parameters into every rank's parameter bucket
//   P1  barrier 1: every rank's parameter bucket holds the updated parameters
//
// The per-replica step counter lives on the device (read at start, advanced by
// block 0 after the last barrier), so a captured CUDA graph replays correctly.
#include <algorithm>

#include "rp_allreduce.cuh"

namespace rp {

struct ApplyArgs {
  CollArgs a;  // MUST be first (rp_dyn_launch passes &a): read_off = grad bucket, write_off = param bucket
  float* s0[RP_MAX_RANKS];   // SGD momentum / Adam exp_avg, owned shard, per local replica
  float* s1[RP_MAX_RANKS];   // Adam exp_avg_sq
  int32_t* step[RP_MAX_RANKS];
  float lr, h1, h2, wd, eps;  // SGD: h1 momentum, h2 dampening; Adam: h1 beta1, h2 beta2
  double beta1, beta2;        // bias corrections in double (as torch computes them in Python)
  int nesterov;
};

template <int OPT>
__device__ __forceinline__ void apply_one(const ApplyArgs& x, int32_t step, float g, float& p, float& m, float& v,
                                          float step_size, float bc2_sqrt) {
  if (OPT == RP_OPT_SGD) {
    // torch.optim.SGD (_single_tensor_sgd / _multi_tensor_sgd)
    if (x.wd != 0.f) g = g + x.wd * p;
    if (x.h1 != 0.f) {
      m = (step == 0) ? g : m * x.h1 + (1.f - x.h2) * g;
      g = x.nesterov ? g + x.h1 * m : m;
    }
    p = p - x.lr * g;
  } else {
    // torch.optim.Adam / AdamW (non-amsgrad, not maximize)
    if (OPT == RP_OPT_ADAMW) p = p * (1.f - x.lr * x.wd);
    else if (x.wd != 0.f) g = g + x.wd * p;
    m = m + (1.f - x.h1) * (g - m);          // exp_avg.lerp_(g, 1 - beta1)
    v = v * x.h2 + (1.f - x.h2) * (g * g);   // exp_avg_sq.mul_(beta2).addcmul_(g, g, 1 - beta2)
    const float denom = sqrtf(v) / bc2_sqrt + x.eps;
    p = p - step_size * (m / denom);
  }
}

template <int GT, int OPT, int NR>
__global__ void __launch_bounds__(kThreads) ar_apply(const ApplyArgs x) {
  using T = typename DType<GT>::T;
  using A = typename DType<GT>::Acc;
  constexpr int E = 16 / sizeof(T);  // elements per gradient packet (f32 params: E floats)
  const CollArgs& a = x.a;
  const int rank = a.rank >= 0 ? a.rank : (int)blockIdx.y;
  if (rp_aborted(a.t, rank)) return;
  const int local = a.rank >= 0 ? 0 : rank;  // index into the per-local-replica pointer arrays
  const size_t V = (a.count + E - 1) / E;
  const size_t Vc = a.chunk;
  const uint32_t tv = a.tile_v;
  const uint32_t tpc = (uint32_t)((Vc + tv - 1) / tv);
  const int lane = threadIdx.x & 31;
  const int32_t step = *((volatile const int32_t*)x.step[local]);
  float step_size = 0.f, bc2_sqrt = 1.f;
  if (OPT != RP_OPT_SGD) {
    const double t = (double)step + 1.0;
    step_size = (float)((double)x.lr / (1.0 - pow(x.beta1, t)));
    bc2_sqrt = (float)sqrt(1.0 - pow(x.beta2, t));
  }
  rp_trace(a, 0);
  const PhaseBase pb = phase_begin(a, rank);
  if (!phase_end(a, rank, 0, pb)) return;

  const char* in[NR];
#pragma unroll
  for (int p = 0; p < NR; ++p) in[p] = a.t.data[p] + a.read_off;
  const float* pmine = (const float*)(a.t.data[rank] + a.write_off);
  float* s0 = x.s0[local];
  float* s1 = x.s1[local];
  const size_t shard0 = (size_t)rank * Vc;  // first packet of the owned chunk
  for (uint32_t j = claim_tile(a, rank, 1); j < tpc; j = claim_tile(a, rank, 1)) {
    const size_t lo = shard0 + (size_t)j * tv;
    const size_t hi = std::min(std::min(lo + tv, shard0 + Vc), V);
    for (size_t v = lo + lane; v < hi; v += 32) {
      uint4 g16[NR];
#pragma unroll
      for (int p = 0; p < NR; ++p) g16[p] = ld128(in[p] + v * 16);
      Pack16<T> gp;
      gp.u = fold_packet<T, A, RP_PREMEAN, NR>(g16);  // the averaged gradient, rounded to T as unfused
      const size_t e0 = v * E;
      const size_t s_at = (v - shard0) * E;
      const bool full = e0 + E <= a.count;
      float pv[E], mv[E], vv[E];
#pragma unroll
      for (int q = 0; q < E / 4; ++q) {
        const float4 p4 = *(const float4*)(pmine + e0 + 4 * q);
        pv[4 * q] = p4.x; pv[4 * q + 1] = p4.y; pv[4 * q + 2] = p4.z; pv[4 * q + 3] = p4.w;
        if (OPT != RP_OPT_SGD || x.h1 != 0.f) {
          const float4 m4 = *(const float4*)(s0 + s_at + 4 * q);
          mv[4 * q] = m4.x; mv[4 * q + 1] = m4.y; mv[4 * q + 2] = m4.z; mv[4 * q + 3] = m4.w;
        }
        if (OPT != RP_OPT_SGD) {
          const float4 v4 = *(const float4*)(s1 + s_at + 4 * q);
          vv[4 * q] = v4.x; vv[4 * q + 1] = v4.y; vv[4 * q + 2] = v4.z; vv[4 * q + 3] = v4.w;
        }
      }
#pragma unroll
      for (int e = 0; e < E; ++e)
        if (full || e0 + e < a.count) apply_one<OPT>(x, step, to_acc(gp.e[e]), pv[e], mv[e], vv[e], step_size, bc2_sqrt);
#pragma unroll
      for (int q = 0; q < E / 4; ++q) {
        const float4 p4 = make_float4(pv[4 * q], pv[4 * q + 1], pv[4 * q + 2], pv[4 * q + 3]);
        uint4 pu;
        memcpy(&pu, &p4, 16);
#pragma unroll
        for (int i = 0; i < NR; ++i) {  // every replica's parameter bucket, own rank last
          const int p = (rank + 1 + i) % NR;
          st128(a.t.data[p] + a.write_off + (e0 + 4 * q) * 4, pu);
        }
        if (OPT != RP_OPT_SGD || x.h1 != 0.f)
          *(float4*)(s0 + s_at + 4 * q) = make_float4(mv[4 * q], mv[4 * q + 1], mv[4 * q + 2], mv[4 * q + 3]);
        if (OPT != RP_OPT_SGD)
          *(float4*)(s1 + s_at + 4 * q) = make_float4(vv[4 * q], vv[4 * q + 1], vv[4 * q + 2], vv[4 * q + 3]);
      }
    }
  }
  if (!phase_end(a, rank, 1, pb)) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) *((volatile int32_t*)x.step[local]) = step + 1;
  dyn_finish(a, rank, 2, pb);
  rp_trace(a, 7);
}

template <int GT, int OPT>
const void* pick_apply_nr(int world) {
  switch (world) {
    case 1: return (const void*)ar_apply<GT, OPT, 1>;
    case 2: return (const void*)ar_apply<GT, OPT, 2>;
    case 3: return (const void*)ar_apply<GT, OPT, 3>;
    case 4: return (const void*)ar_apply<GT, OPT, 4>;
    case 5: return (const void*)ar_apply<GT, OPT, 5>;
    case 6: return (const void*)ar_apply<GT, OPT, 6>;
    case 7: return (const void*)ar_apply<GT, OPT, 7>;
    case 8: return (const void*)ar_apply<GT, OPT, 8>;
  }
  return nullptr;
}

template <int GT>
const void* pick_apply(int opt, int world) {
  if (opt == RP_OPT_SGD) return pick_apply_nr<GT, RP_OPT_SGD>(world);
  if (opt == RP_OPT_ADAM) return pick_apply_nr<GT, RP_OPT_ADAM>(world);
  return pick_apply_nr<GT, RP_OPT_ADAMW>(world);
}

}  // namespace rp

using namespace rp;

// Owned shard of the optimizer state: packets are split in rank order, chunk =
// ceil(packets / world); the state arrays hold chunk * E floats per rank.
static void apply_geometry(rp_comm* c, size_t count, int dtype_grad, size_t* chunk_packets, size_t* elems_per_packet) {
  const size_t E = 16 / rp_dtype_size(dtype_grad);
  const size_t V = (count + E - 1) / E;
  *chunk_packets = (V + c->world - 1) / c->world;
  *elems_per_packet = E;
}

int rp_launch_apply(rp_comm* c, const void* const* grad, void* const* param, size_t count, int dtype_grad, int opt,
                    const double* hyper, float* const* state0, float* const* state1, int32_t* const* step,
                    cudaStream_t stream) {
  if (count == 0) return RP_OK;
  if (dtype_grad != RP_F32 && dtype_grad != RP_BF16)
    return rp_fail(RP_ERR_INVALID, "all_reduce_apply: gradient bucket must be f32 or bf16");
  if (opt != RP_OPT_SGD && opt != RP_OPT_ADAM && opt != RP_OPT_ADAMW)
    return rp_fail(RP_ERR_INVALID, "all_reduce_apply: unknown optimizer");
  if (!hyper) return rp_fail(RP_ERR_INVALID, "all_reduce_apply: NULL hyperparameters");
  const int n = c->is_virtual ? c->world : 1;
  const bool need_s0 = opt != RP_OPT_SGD || hyper[1] != 0.0;
  for (int i = 0; i < n; ++i) {
    if (!step || !step[i]) return rp_fail(RP_ERR_INVALID, "all_reduce_apply: NULL step counter");
    if (need_s0 && (!state0 || !state0[i])) return rp_fail(RP_ERR_INVALID, "all_reduce_apply: NULL state0");
    if (opt != RP_OPT_SGD && (!state1 || !state1[i])) return rp_fail(RP_ERR_INVALID, "all_reduce_apply: NULL state1");
    if ((need_s0 && ((uintptr_t)state0[i] & 15)) || (opt != RP_OPT_SGD && ((uintptr_t)state1[i] & 15)))
      return rp_fail(RP_ERR_INVALID, "all_reduce_apply: state must be 16-byte aligned");
  }
  size_t chunk, E;
  apply_geometry(c, count, dtype_grad, &chunk, &E);
  const size_t gbytes = ((count + E - 1) / E) * 16;
  size_t goff = 0, poff = 0;
  if (!rp_symmetric_in_pool(c, grad, gbytes, &goff))
    return rp_fail(RP_ERR_INVALID, "all_reduce_apply: gradient bucket must be pool-resident (symmetric)");
  if (!rp_symmetric_in_pool(c, (const void* const*)param, ((count + E - 1) / E) * E * 4, &poff))
    return rp_fail(RP_ERR_INVALID, "all_reduce_apply: parameter bucket must be pool-resident (symmetric)");
  if (goff % 16 || poff % 16) return rp_fail(RP_ERR_INVALID, "all_reduce_apply: buckets must be 16-byte aligned");
  if (goff < poff + ((count + E - 1) / E) * E * 4 && poff < goff + gbytes)
    return rp_fail(RP_ERR_INVALID, "all_reduce_apply: gradient and parameter buckets overlap");
  const void* fn = dtype_grad == RP_F32 ? pick_apply<RP_F32>(opt, c->world) : pick_apply<RP_BF16>(opt, c->world);
  if (!fn) return rp_fail(RP_ERR_INVALID, "all_reduce_apply: unsupported world size (1..8)");

  ApplyArgs x;
  memset(&x, 0, sizeof(x));
  rp_base_args(c, x.a);
  x.a.count = count;
  x.a.chunk = chunk;
  x.a.read_off = goff;
  x.a.write_off = poff;
  x.a.dtype_in = x.a.dtype_out = dtype_grad;
  for (int i = 0; i < n; ++i) {
    x.s0[i] = need_s0 ? state0[i] : nullptr;
    x.s1[i] = opt != RP_OPT_SGD ? state1[i] : nullptr;
    x.step[i] = step[i];
  }
  x.lr = (float)hyper[0];
  x.h1 = (float)hyper[1];
  x.h2 = (float)hyper[2];
  x.wd = (float)hyper[3];
  x.eps = (float)hyper[4];
  x.nesterov = hyper[5] != 0.0;
  x.beta1 = hyper[1];
  x.beta2 = hyper[2];
  if (opt == RP_OPT_SGD && x.nesterov && (x.h1 == 0.f || x.h2 != 0.f))
    return rp_fail(RP_ERR_INVALID, "all_reduce_apply: Nesterov momentum requires a momentum and zero dampening");
  static_assert(offsetof(ApplyArgs, a) == 0, "CollArgs must lead ApplyArgs");
  return rp_dyn_launch(c, fn, x.a, stream, "apply");
}

extern "C" {

int rp_apply_shard(rp_comm_t c, size_t count, int dtype_grad, size_t* first, size_t* len) {
  if (!c || !first || !len) return rp_fail(RP_ERR_INVALID, "rp_apply_shard: NULL argument");
  if (dtype_grad != RP_F32 && dtype_grad != RP_BF16)
    return rp_fail(RP_ERR_INVALID, "rp_apply_shard: gradient bucket must be f32 or bf16");
  size_t chunk, E;
  apply_geometry(c, count, dtype_grad, &chunk, &E);
  *first = (size_t)(c->is_virtual ? 0 : c->rank) * chunk * E;  // virtual: replica r owns [r*len, (r+1)*len)
  *len = chunk * E;
  return RP_OK;
}

}  // extern "C"

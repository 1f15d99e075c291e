/*
 * rp.h -- C ABI of the B200-native TF-Replicator data-parallel hot path.
 *
 * Plain pointers, sizes and int status codes; no torch or C++ types cross this
 * boundary. Every collective is enqueued on the caller's CUDA stream and returns
 * immediately (the host never blocks), which is how a Graph kernel or an
 * optimizer wrapper calls it. One issuing host thread per communicator.
 *
 * Reference interfaces each entry point replaces (paths under /root/reference):
 *   - the duck-typed communicator consumed by the mesh seam
 *       pkg/src/replicator/graph.py:565-583 (_mesh_collective_kernel):
 *         comm.all_reduce(local, kind in {sum,mean,max}, label)  graph.py:573-574
 *         comm.all_gather(local, label) -> list in rank order    graph.py:575-579
 *         comm.broadcast(root_value|None, label, shape, dtype)   graph.py:580-582
 *   - the in-process stitched folds the MultiDevice replicator rewrites each
 *     collective placeholder into (graph.py:506-540: nary_sum/nary_mean/nary_max,
 *     concat/pack, pick0), served here by a *virtual* communicator whose ranks
 *     are replicas resident on one GPU;
 *   - the absent SPEC collectives module: ring_all_reduce / all_sum / all_reduce /
 *     all_gather / broadcast, and the absent wrap_optimizer
 *      and cross-replica batch norm
 *     (PAPER.md:213-219).
 *
 * Status codes map one-to-one onto the reference's exception classes
 * (pkg/src/replicator/errors.py), see RP_ERR_* below.
 */
#ifndef RP_H_
#define RP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define RP_API __attribute__((visibility("default")))
#else
#define RP_API
#endif

typedef struct rp_comm* rp_comm_t;

/* Element types. 0/1 are the reference's DTYPE_CODES (tensor.py:16-21). */
enum {
  RP_F32 = 0,
  RP_F64 = 1,
  RP_BF16 = 2,
  RP_F16 = 3,
};

/* Reduction kinds (graph.py:514-533 and SPEC.md:406). */
enum {
  RP_SUM = 0,     /* nary_sum: ((x0+x1)+x2)+... ascending rank           */
  RP_MEAN = 1,    /* nary_mean: fold_sum / N (sum, then divide)           */
  RP_MAX = 2,     /* nary_max: np.maximum left fold                       */
  RP_PREMEAN = 3, /* wrap_optimizer all_sum(g/R): divide, then sum        */
};

/* Algorithm selection for rp_all_reduce / rp_broadcast. */
enum {
  RP_ALGO_AUTO = 0,
  RP_ALGO_ONESHOT = 1, /* every rank folds all N inputs (latency regime)      */
  RP_ALGO_TWOSHOT = 2, /* reduce-scatter (pull) + all-gather (push)           */
  RP_ALGO_DIRECT = 1,  /* broadcast: every rank pulls from root              */
  RP_ALGO_SCATTER = 2, /* broadcast: scatter from root + all-gather           */
  RP_ALGO_NVLS = 3,    /* all_reduce in the NVSwitch (multimem), in place in the NVLS
                          region; NOT rank-ordered: ~1e-6 relative. AUTO picks it
                          for in-place f32/bf16/f16 sum/mean/premean of >= 512 KiB
                          inside the NVLS region at world >= 4 (RP_NVLS=0: never).
                          broadcast: dst inside the NVLS region (16-byte multiple):
                          the root's multicast store reaches every rank (bit-exact);
                          AUTO picks it whenever dst lies in the region */
  RP_ALGO_RELAY = 4,   /* broadcast, multi-process: pipelined tiles root -> owner ->
                          peers over NVLink (P2P stores); AUTO above 1 MiB */
  RP_ALGO_FLAT = 5,    /* all_reduce, virtual communicator: one barrier-free kernel over
                          the flat range -- per 16-byte position all R operands loaded,
                          folded in rank order, stored to all R outputs (every buffer
                          read and written once). AUTO picks it for virtual replicas */
};

/* Status codes -> reference exception (errors.py). */
enum {
  RP_OK = 0,
  RP_ERR_INVALID = 1,  /* bad argument / shape        -> ShapeError (errors.py:12)          */
  RP_ERR_CONFIG = 2,   /* topology / deployment        -> ConfigurationError (errors.py:32)  */
  RP_ERR_CUDA = 3,     /* CUDA runtime failure         -> CollectiveError (errors.py:60)     */
  RP_ERR_ABORTED = 4,  /* a rank aborted / timed out   -> CollectiveAbortedError (errors.py:68) */
  RP_ERR_PROTOCOL = 5, /* ranks disagree               -> ProtocolError (errors.py:64)       */
};

/* Human-readable description of the last failure on the calling thread. */
RP_API const char* rp_last_error(void);

/* ---- lifecycle ---------------------------------------------------------- */

/* Multi-process communicator: one rank per process/GPU. Allocates this rank's
 * registered pool (pool_bytes of data + a signal region) on `device`. */
RP_API int rp_comm_create(int rank, int world, int device, size_t pool_bytes, rp_comm_t* out);

/* Virtual communicator: `world` replicas resident on ONE device (the reference's
 * in-process MultiDevice replication, graph.py:506-540). Collectives on it take
 * per-replica pointer arrays (the *_v entry points) and run as one cooperative
 * kernel over all replicas' data. Usable immediately (no export/import). */
RP_API int rp_comm_create_virtual(int world, int device, size_t pool_bytes, rp_comm_t* out);

/* Size of this rank's export blob (opaque; exchanged by the caller, e.g. an
 * all_gather over torch.distributed). */
RP_API size_t rp_comm_export_size(void);
RP_API int rp_comm_export(rp_comm_t comm, void* buf, size_t* len);

/* `all` = world export blobs concatenated in rank order. Discovers the topology
 * (replaces the reference's MultiGpu device assignment): every
 * peer's GPU must be visible, CUDA peer access must work, and NVML must report
 * NVLink P2P to it (NVSwitch gives every pair NVLink) -- rp_topology_check's
 * policy -- and every rank's GPU must have the same number of active NVLink links
 * (rp_topology_uniform); RP_ERR_CONFIG (-> ConfigurationError, errors.py:32) otherwise, naming
 * the pair and the link found. RP_ALLOW_PCIE=1 in the environment accepts PCIe
 * peer access (tests only). Then opens every peer's pool over CUDA IPC (loopback
 * peers: the plain pointer). */
RP_API int rp_comm_import(rp_comm_t comm, const void* all, size_t len);

/* Link kinds rp_comm_import classifies each peer into. */
enum {
  RP_LINK_SELF = 0,
  RP_LINK_NVLINK = 1,      /* CUDA peer access + NVML NVLink P2P                  */
  RP_LINK_PCIE = 2,        /* peer access, but NVML reports no NVLink              */
  RP_LINK_NONE = 3,        /* no CUDA peer access                                 */
  RP_LINK_UNKNOWN = 4,     /* peer not visible, or NVML unavailable               */
  RP_LINK_SAME_DEVICE = 5, /* another process on this GPU                          */
  RP_LINK_LOOPBACK = 6,    /* a rank of this process's loopback world (same GPU)  */
};

/* The topology policy rp_comm_import applies to this rank's row of links
 * (links[p] = RP_LINK_* to rank p): NVLINK everywhere; PCIE only with
 * allow_pcie; LOOPBACK only in a loopback world. RP_ERR_CONFIG with the offending
 * pair in rp_last_error() otherwise. Pure host logic (no device needed). */
RP_API int rp_topology_check(int world, int rank, const int* links, int allow_pcie, int loopback);

/* Uniformity of the NVLink fabric rp_comm_import also requires (unless
 * RP_ALLOW_PCIE=1): every rank's GPU has the same number of active NVLink links
 * (nvlinks[p], from NVML; -1 = unknown, skipped) and none has zero -- what an
 * NVSwitch all-to-all gives (18 links per B200). RP_ERR_CONFIG otherwise, naming
 * the ranks. Pure host logic. */
RP_API int rp_topology_uniform(int world, const int* nvlinks);

/* The topology rp_comm_import discovered: links[p] (RP_LINK_* from this rank to
 * rank p) and nvlinks[p] (active NVLink links of rank p's GPU, -1 unknown), world
 * entries each. */
RP_API int rp_comm_topology(rp_comm_t comm, int* links, int* nvlinks);

/* Loopback world (testing the multi-process kernels on ONE GPU): `world`
 * non-virtual communicators created in ONE process on the same device, each
 * driven from its own host thread and stream, exchange blobs in-process and set
 * this BEFORE rp_comm_import. Peers' regions are then plain pointers (no IPC) and
 * every rank's grids are capped at num_sms / world blocks so all ranks' blocks
 * are co-resident. Same kernels, same barriers, same pool layout as one process
 * per GPU; the NVLink hop is replaced by local HBM. */
RP_API int rp_comm_set_loopback(rp_comm_t comm, int on);

/* Make `device`'s stream-ordered memory pools safe for a loopback world (call once,
 * before the ranks allocate): no cross-stream reuse through inserted waits
 * (cudaMemPoolReuseAllowInternalDependencies = 0), which could make one rank's
 * stream wait behind a peer's collective kernel that waits for this rank. */
RP_API int rp_loopback_prepare(int device);

RP_API int rp_comm_destroy(rp_comm_t comm);

/* Registered data region of replica `rank` (multi-process: only this rank;
 * virtual: any replica). Buffers inside it are exchanged zero-copy. */
RP_API int rp_comm_pool(rp_comm_t comm, int rank, void** base, size_t* bytes);

/* Scratch window used to stage non-pool buffers: [scratch_off, pool_bytes). */
RP_API int rp_comm_info(rp_comm_t comm, int* rank, int* world, int* is_virtual, int* num_sms,
                 size_t* scratch_off);

/* Reserve the first `bytes` of the pool for caller buffers (fusion buckets);
 * staging uses the rest. Must be called identically on every rank. */
RP_API int rp_comm_reserve(rp_comm_t comm, size_t bytes);

/* Synchronise the device (a loopback rank does not: its caller synchronises the
 * streams it launched on, since a device-wide sync could wait on a peer kernel
 * that waits for this rank's next launch) and report a collective abort/timeout
 * recorded by the kernels (RP_ERR_ABORTED with the reason). The abort is sticky:
 * a communicator that aborted stays aborted. */
RP_API int rp_comm_check(rp_comm_t comm);

/* Spin timeout for cross-rank waits, nanoseconds (default 20 s). */
RP_API int rp_comm_set_timeout(rp_comm_t comm, uint64_t ns);

/* Cap the grid of every later collective launch at `blocks` blocks per rank (0 =
 * no cap: as many co-resident blocks as the kernel allows). Used while a
 * collective runs beside compute kernels (wrap_optimizer overlap: the exchange
 * leaves the other SMs to backward). Kernels whose blocks pair up by index across
 * ranks rely on equal grids: set it identically on every rank, at the same point
 * of the collective sequence. No reference counterpart (the reference's
 * collectives run after the whole backward). */
RP_API int rp_comm_set_block_cap(rp_comm_t comm, int blocks);

/* ---- NVLS (NVLink SHARP) region ------------------------------------------ */
/* A multicast object spanning all ranks' GPUs with `bytes` of each rank's memory
 * bound to it (RP_ALGO_NVLS reduces inside the NVSwitch). Bootstrap order, every
 * step on every rank unless noted:
 *   rp_nvls_create (rank 0 creates + listens; returns a socket name in `name`)
 *   [exchange `name`]  rp_nvls_serve (rank 0)  ||  rp_nvls_join(name) (others)
 *   rp_nvls_add  [barrier]  rp_nvls_bind  [barrier]
 * The handle travels as a POSIX fd over an abstract Unix socket (same host). */
RP_API int rp_nvls_create(rp_comm_t comm, size_t bytes, char* name, size_t name_cap);
RP_API int rp_nvls_serve(rp_comm_t comm);
RP_API int rp_nvls_join(rp_comm_t comm, const char* name);
RP_API int rp_nvls_add(rp_comm_t comm);
RP_API int rp_nvls_bind(rp_comm_t comm);
/* This rank's (unicast) view of the region: allocate fusion buckets here. */
RP_API int rp_nvls_pool(rp_comm_t comm, void** base, size_t* bytes);

/* ---- collectives (multi-process form: this rank's buffers) ---------------- */

/* dst[i] = OP over ranks of src[i], i < count. dtype_in / dtype_out are the
 * element types of src / dst; the exchange dtype is dtype_comm (the fused cast:
 * e.g. f32 grads exchanged as bf16 with dtype_comm=RP_BF16). Accumulation is in
 * f32 (f32/bf16/f16) or f64 (f64), ascending rank order, rounded once.
 * src == dst is allowed. */
RP_API int rp_all_reduce(rp_comm_t comm, const void* src, void* dst, size_t count, int dtype_in,
                  int dtype_comm, int dtype_out, int op, int algo, void* stream);

/* ---- fused optimizer apply (wrap_optimizer as one kernel) ------------------- */
/* The wrapped optimizer's step in ONE
 * kernel: the gradient bucket `grad` (count elements of dtype_grad, f32|bf16) is
 * averaged with the rank-ordered premean fold (bit-identical to rp_all_reduce
 * RP_PREMEAN), the rank owning each chunk applies the optimizer update to the f32
 * parameter bucket `param` (count elements) in f32, and stores the updated values
 * into every rank's `param` -- every replica ends with the same bits (mirrored
 * variables). Both buckets are pool-resident at symmetric offsets.
 * Optimizer state covers this rank's shard only (rp_apply_shard); `step` is a
 * device int32 the kernel reads and advances (graph-replay safe).
 * hyper[6] = {lr, momentum | beta1, dampening | beta2, weight_decay, eps, nesterov}
 * with torch.optim.SGD / Adam / AdamW semantics (non-amsgrad, not maximize). */
enum { RP_OPT_SGD = 0, RP_OPT_ADAM = 1, RP_OPT_ADAMW = 2 };
RP_API int rp_apply_shard(rp_comm_t comm, size_t count, int dtype_grad, size_t* first, size_t* len);
RP_API int rp_all_reduce_apply(rp_comm_t comm, const void* grad, void* param, size_t count, int dtype_grad, int opt,
                               const double* hyper, float* state0, float* state1, int32_t* step, void* stream);
RP_API int rp_all_reduce_apply_v(rp_comm_t comm, const void* const* grad, void* const* param, size_t count,
                                 int dtype_grad, int opt, const double* hyper, float* const* state0,
                                 float* const* state1, int32_t* const* step, void* stream);

/* The algorithm rp_all_reduce would run for these arguments (RP_ALGO_ONESHOT,
 * RP_ALGO_TWOSHOT, RP_ALGO_NVLS or, virtual, RP_ALGO_FLAT) in *chosen; nothing is
 * launched. */
RP_API int rp_all_reduce_algo(rp_comm_t comm, const void* src, const void* dst, size_t count, int dtype_in,
                              int dtype_comm, int dtype_out, int op, int algo, int* chosen);

/* The plan rp_all_reduce would follow, for cross-rank agreement checks
 * (Replicator(check_protocol=True) digests it): plan[0] = algorithm (AUTO
 * resolved), plan[1] = 1 for the push data-movement form, plan[2] / plan[3] = pool
 * offset of src / dst, -2 for a registered user buffer (rp_register_*), -1 for
 * any other buffer. Ranks MUST agree on all four
 * (symmetric placement): a rank passing a pool view where a peer passes a plain
 * tensor would launch a different kernel against the shared barrier state.
 * Multi-process communicators only look at this rank's pointers. */
RP_API int rp_all_reduce_plan(rp_comm_t comm, const void* src, const void* dst, size_t count, int dtype_in,
                              int dtype_comm, int dtype_out, int op, int algo, int64_t* plan);

/* ---- user-buffer registration -------------------------------------------
 * Collective: every rank registers its corresponding buffer (same size, same
 * order). rp_register_export fills this rank's blob (the buffer's allocation
 * exported with cudaIpcGetMemHandle, plus its offset; a loopback world: the plain
 * pointer); the caller exchanges the blobs (rank order) and passes them all to
 * rp_register_import, which maps every peer's copy (each peer allocation opened
 * once, refcounted) and returns the registration index. Afterwards an in-place
 * rp_all_reduce of the buffer (or of a sub-range at the same offset on every rank),
 * without a cast, takes the zero-copy pull two-shot -- the path pool buckets take
 * -- instead of the push form with staging (rp_all_reduce_plan reports -2 as its
 * placement). Stream-ordered-pool and expandable-segment memory cannot be shared
 * over CUDA IPC (RP_ERR_CONFIG). The caller keeps the buffers alive until
 * rp_unregister (collective) or rp_comm_destroy. */
RP_API size_t rp_register_export_size(void);
RP_API int rp_register_export(rp_comm_t comm, const void* ptr, size_t bytes, void* blob, size_t* len);
RP_API int rp_register_import(rp_comm_t comm, const void* all, size_t len, int* reg);
RP_API int rp_unregister(rp_comm_t comm, int reg);

/* dst[r*bytes_per_rank ...] = src of rank r (rank order, graph.py:575-579). */
RP_API int rp_all_gather(rp_comm_t comm, const void* src, void* dst, size_t bytes_per_rank, void* stream);

/* dst = root's src on every rank (graph.py:580-582; the reference root is 0). */
RP_API int rp_broadcast(rp_comm_t comm, const void* src, void* dst, size_t bytes, int root, int algo,
                 void* stream);

/* ---- collectives (virtual form: one pointer per replica) ----------------- */

RP_API int rp_all_reduce_v(rp_comm_t comm, const void* const* src, void* const* dst, size_t count,
                    int dtype_in, int dtype_comm, int dtype_out, int op, int algo, void* stream);
RP_API int rp_all_gather_v(rp_comm_t comm, const void* const* src, void* const* dst,
                    size_t bytes_per_rank, void* stream);
RP_API int rp_broadcast_v(rp_comm_t comm, const void* const* src, void* const* dst, size_t bytes, int root,
                   int algo, void* stream);

/* ---- cross-replica batch norm statistics --------------------------------- */

/* Layouts of x / dy. */
enum {
  RP_LAYOUT_NC = 0,   /* [n, c]          (channels innermost)  */
  RP_LAYOUT_NHWC = 0, /* [n, h, w, c] == [n*h*w, c]            */
  RP_LAYOUT_NCHW = 1, /* [n, c, hw]                            */
};

/* Per-channel cross-replica statistics of x (forward, K5):
 *   sum_c = sum over all replicas' elements of channel c, sumsq_c likewise;
 *   mean = sum/M, var = sumsq/M - mean^2 (biased), invstd = 1/sqrt(var+eps)
 * with M the global element count per channel (replicas may differ in batch).
 * Local partials and the cross-replica fold are f64. Outputs (device, length c,
 * f32): mean, var, invstd; `count` (device f64 scalar, may be NULL) receives M.
 * `rows` = n (NCHW) or n*h*w (NHWC); `hw` = spatial size (NCHW) or 1.
 * On a virtual communicator x/outputs are host arrays of per-replica device
 * pointers (cast to the pointer types below). */
RP_API int rp_bn_stats(rp_comm_t comm, const void* x, int dtype, int64_t rows, int64_t c, int64_t hw,
                int layout, float eps, float* mean, float* var, float* invstd, double* count,
                void* stream);

/* Backward statistics (K5b): sum_dy_c and sum_dy_xmu_c = sum dy*(x-mean_c),
 * cross-replica summed in f64, written as f32. local_sum_dy / local_sum_dy_xmu
 * (may be NULL) receive this replica's own sums (for the weight/bias grads, which
 * the wrapped optimizer then averages across replicas). */
RP_API int rp_bn_bwd_stats(rp_comm_t comm, const void* x, const void* dy, int dtype, int64_t rows,
                    int64_t c, int64_t hw, int layout, const float* mean, float* sum_dy,
                    float* sum_dy_xmu, float* local_sum_dy, float* local_sum_dy_xmu, void* stream);

/* Elementwise BN apply (forward): y = (x-mean)*invstd*w + b   (w/b may be NULL). */
RP_API int rp_bn_apply(const void* x, void* y, int dtype, int64_t rows, int64_t c, int64_t hw, int layout,
                const float* mean, const float* invstd, const float* weight, const float* bias,
                void* stream);

/* Elementwise BN backward: dx = (dy - sum_dy/M - (x-mean)*invstd^2*sum_dy_xmu/M)*invstd*w.
 * M = *count_device (the device f64 scalar rp_bn_stats wrote; no host sync) when
 * count_device is non-NULL, else count_total. */
RP_API int rp_bn_bwd_apply(const void* x, const void* dy, void* dx, int dtype, int64_t rows, int64_t c,
                    int64_t hw, int layout, const float* mean, const float* invstd,
                    const float* weight, const float* sum_dy, const float* sum_dy_xmu,
                    double count_total, const double* count_device, void* stream);

/* ---- fusion-buffer packing (K6) ------------------------------------------ */

/* Gather `n` tensors (ptrs[i], counts[i] elements of dtype_src) into the flat
 * buffer dst (dtype_dst) at element offsets offs[i], casting (RNE) on the fly;
 * one launch for all tensors. Host arrays. */
RP_API int rp_pack(void* dst, int dtype_dst, const void* const* ptrs, const int64_t* counts,
            const int64_t* offs, int n, int dtype_src, void* stream);
/* Inverse of rp_pack: scatter the flat buffer back into the tensors. */
RP_API int rp_unpack(const void* src, int dtype_src, void* const* ptrs, const int64_t* counts,
              const int64_t* offs, int n, int dtype_dst, void* stream);

/* Library build id / version string. */
RP_API const char* rp_version(void);

#ifdef __cplusplus
}
#endif

#endif /* RP_H_ */

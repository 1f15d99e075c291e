// Internal definitions shared by the rp_* translation units (not part of the ABI).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include <map>
#include <string>
#include <vector>

#include "../../include/rp.h"

#define RP_MAX_RANKS 8
// internal kernel selector (not an ABI algorithm): the bulk-copy form of RP_ALGO_FLAT
#define RP_ALGO_FLAT_BULK 105
// Signal slots: one row of RP_MAX_RANKS u32 per block index. Rows
// [0, RP_MAX_BLOCKS) carry the per-block barriers of the collectives; rows
// [RP_BN_ROW0, RP_BN_ROW0 + RP_BN_ROWS) those of the BN statistics exchange.
#define RP_MAX_BLOCKS 1024
#define RP_BN_ROW0 (RP_MAX_BLOCKS)
#define RP_BN_ROWS 256
// rank-level phase counters of the dynamically scheduled kernels, and the
// per-rank tile-claim counters (local atomics), one per phase
#define RP_PH_ROW0 (RP_BN_ROW0 + RP_BN_ROWS)
#define RP_PH_ROWS 4
#define RP_CTR_ROW (RP_PH_ROW0 + RP_PH_ROWS)
// phase row 3 (and local arrival word 4 + 3) belongs to the BN exchange barrier
#define RP_BN_PHASE 3
#define RP_ABORT_WORD ((RP_CTR_ROW + 4) * RP_MAX_RANKS)  // u32 index
// Device-side sequencing state, local to each rank (never written by peers), in
// the last 16 KiB of the signal region. Kernels read it at start and advance it
// at the end, so launches carry no per-call host state and a captured CUDA graph
// replays correctly (every rank runs the same sequence, so the copies agree):
//   blk_epoch[b]  barrier epoch of block index b (collective rows 0..1023)
//   bn_epoch[b]   same for the BN exchange rows
//   zone_par[b]   one-shot landing-zone parity of block b
//   ph_seen[k]    arrivals already consumed per source rank on phase row k
//   bn_grid       fused BN kernel's device-wide barrier (counter, consumed base)
#define RP_STATE_WORD (12 * 1024)
#define RP_ST_BLK_EPOCH (RP_STATE_WORD)
#define RP_ST_BN_EPOCH (RP_ST_BLK_EPOCH + RP_MAX_BLOCKS)
#define RP_ST_ZONE_PAR (RP_ST_BN_EPOCH + 256)
#define RP_ST_PH_SEEN (RP_ST_ZONE_PAR + RP_MAX_BLOCKS)
// fused BN statistics kernel: device-wide barrier (monotone arrival counter and
// the count already consumed by earlier calls)
#define RP_ST_BN_GRID_CTR (RP_ST_PH_SEEN + 8)
#define RP_ST_BN_GRID_BASE (RP_ST_PH_SEEN + 9)
// flat virtual all-reduce (ar_virtual_flat): tile-claim counter and blocks-done
// counter, zeroed by the call's last block (so a launch carries no host state)
#define RP_ST_VFLAT_CTR (RP_ST_PH_SEEN + 10)
#define RP_ST_VFLAT_DONE (RP_ST_PH_SEEN + 11)
#define RP_SIGNAL_BYTES (64 * 1024)  // signal region ahead of the data
#define RP_ALIGN 256
// Pool layout (every rank identical):
//   [0, reserved)                          caller buffers (fusion buckets), zero-copy
//   [reserved, scratch_end)                general staging (two-shot Q / W, pull staging)
//   [scratch_end, +2*RP_OS_REGION)         one-shot push landing zones, parity 0 / 1
//   [pool_bytes - RP_BN_BYTES, pool_bytes) BN per-channel exchange records
// Kernels may read their pool after their LAST barrier only from the one-shot
// landing zones (double-buffered by call parity); everything else is protected
// by a trailing barrier, so a peer that already started the next call and
// pushes without a start barrier can never clobber data still being read.
// The BN records hold (sum, sumsq, count) as f64 for up to RP_BN_ROWS*256 channels.
#define RP_BN_HALF ((size_t)RP_BN_ROWS * 256 * 3 * 8)
#define RP_BN_BYTES (2 * RP_BN_HALF)  // two record sets, alternating by call parity
#define RP_OS_REGION ((size_t)4 << 20)
// Per-tile ready flags of the relay broadcast (u32 epochs, zeroed at creation,
// written only by that kernel): one per tile, at most RP_FLAG_WORDS tiles.
#define RP_FLAG_WORDS 65536
#define RP_FLAG_BYTES ((size_t)RP_FLAG_WORDS * 4)
#define RP_MIN_POOL ((size_t)16 << 20)

// Abort reasons written into the abort word (first writer wins).
#define RP_ABORT_TIMEOUT 1u
#define RP_ABORT_PEER 2u

struct RankTable {
  char* data[RP_MAX_RANKS];       // data region base of every rank (peer-mapped)
  uint32_t* sig[RP_MAX_RANKS];    // signal region base of every rank (peer-mapped)
};

// A user buffer registered with every peer (rp_register_*): the base pointer of
// the same buffer on every rank (IPC-mapped, or loopback plain pointers).
struct RpReg {
  char* ptr[RP_MAX_RANKS] = {};
  size_t bytes = 0;
  bool live = false;
  std::string ipc_key[RP_MAX_RANKS];  // opened IPC handle per peer ("" = not IPC)
};

struct rp_comm {
  int rank = 0;
  int world = 1;
  int device = 0;
  bool is_virtual = false;
  bool imported = false;
  size_t pool_bytes = 0;   // data bytes per rank
  size_t reserved = 0;     // [0, reserved) belongs to the caller (fusion buckets)
  char* alloc[RP_MAX_RANKS] = {};   // allocations owned by this process
  bool ipc_opened[RP_MAX_RANKS] = {};
  RankTable table{};
  uint64_t timeout_ns = 20ull * 1000ull * 1000ull * 1000ull;
  int num_sms = 148;
  int max_coresident = 0;
  int block_cap = 0;       // >0: at most this many blocks per rank (rp_comm_set_block_cap)
  // loopback world (rp_comm_set_loopback): several non-virtual ranks in ONE process
  // on ONE device, each driven from its own host thread and stream. Peers' regions
  // are plain pointers of this process (no IPC), and every rank's grids are capped
  // at num_sms / world blocks so all ranks' blocks are co-resident.
  bool loopback = false;
  int loopback_cap = 0;    // num_sms / world in a loopback world
  bool lb_refs = false;    // holds a reference on every rank's region (loopback registry)
  // registered user buffers and the peer IPC mappings they hold (refcounted by handle)
  std::vector<RpReg> regs;
  std::map<std::string, std::pair<char*, int>> ipc_cache;
  // topology discovered by rp_comm_import (rp_comm_topology)
  int links[RP_MAX_RANKS] = {};
  int nvlinks[RP_MAX_RANKS] = {};
  // effective per-rank block cap (0: none): the caller's cap and the loopback cap
  int cap() const {
    if (loopback_cap > 0) return block_cap > 0 ? (block_cap < loopback_cap ? block_cap : loopback_cap) : loopback_cap;
    return block_cap;
  }
  // BN scratch: per-split f64 partials (device memory, all local replicas)
  double* bn_partials = nullptr;
  size_t bn_partials_bytes = 0;
  std::vector<double*> bn_retired;  // outgrown partials, freed with the communicator
  void* nvls = nullptr;    // NvlsState (rp_nvls.cu): multicast-bound region, or NULL
  // private non-blocking stream for the library's own small copies (signal-region
  // init, rp_comm_check's abort read): never the legacy default stream, which
  // waits for every blocking stream -- in a loopback world, for a peer's kernel
  // that waits for this rank (measured: a 5 s stall until the spin timeout)
  cudaStream_t aux = nullptr;
  // end of the general staging window (see the layout above)
  size_t scratch_end() const { return pool_bytes - RP_BN_BYTES - RP_FLAG_BYTES - 2 * RP_OS_REGION; }
  size_t oneshot_zone(int parity) const { return scratch_end() + (size_t)parity * RP_OS_REGION; }
  size_t tile_flags() const { return pool_bytes - RP_BN_BYTES - RP_FLAG_BYTES; }
  size_t bn_records() const { return pool_bytes - RP_BN_BYTES; }
};

// Export blob exchanged between ranks.
struct RpExport {
  uint64_t magic;
  int32_t rank, world;
  uint64_t pool_bytes;
  cudaIpcMemHandle_t handle;
  unsigned char uuid[16];
  int32_t pci_bus, pci_device, pci_domain;
  uint64_t base;     // region base in the exporting process (loopback peers only)
  int32_t pid;       // exporting process
  int32_t loopback;  // exporter runs a loopback world
  int32_t nvlinks;   // active NVLink links of the exporter's GPU (NVML), -1 unknown
};

// Kernel argument block for the collectives (by value, < 4 KB).
struct CollArgs {
  RankTable t;
  const void* src[RP_MAX_RANKS];
  void* dst[RP_MAX_RANKS];
  size_t read_off;      // pool offset holding (or receiving) each rank's input
  size_t write_off;     // pool offset receiving the pushed result (two-shot)
  size_t count;         // elements (all_reduce) or bytes (copy collectives)
  size_t chunk;         // per-rank chunk (vectors or bytes) for partitioned phases
  int world;
  int rank;             // -1: virtual communicator, rank = blockIdx.y
  int copy_in;          // stage src -> pool[read_off] inside the kernel
  int copy_out;         // pool[write_off] -> dst inside the kernel
  int dtype_in, dtype_out;
  int root;
  uint64_t timeout_ns;
  unsigned long long* trace;  // RP_TRACE analysis: per-block %globaltimer stamps, or NULL
  uint32_t tile_v;            // dynamically scheduled kernels: vectors (16 B) per tile
  int relay_root_blocks;      // relay broadcast: blocks the root pushes with
};

int rp_classify_link(rp_comm* c, const RpExport& me, const RpExport& peer, bool self, std::string* why);

// [p, p + bytes) lies inside one live registration: its index and the offset
bool rp_registered(rp_comm* c, const void* p, size_t bytes, int* reg, size_t* off);
void rp_release_registrations(rp_comm* c);

// error plumbing
void rp_set_error(const std::string& msg);
int rp_fail(int code, const std::string& msg);
#define RP_CUDA_CHECK(expr)                                                        \
  do {                                                                             \
    cudaError_t e_ = (expr);                                                       \
    if (e_ != cudaSuccess)                                                         \
      return rp_fail(RP_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

size_t rp_dtype_size(int dtype);
// Make the device owning `p` current (entry points without a communicator).
int rp_set_device_from_ptr(const void* p);
bool rp_dtype_valid(int dtype);

// launchers (defined in the .cu files)
int rp_launch_all_reduce(rp_comm* c, const void* const* src, void* const* dst, size_t count,
                         int dtype_in, int dtype_comm, int dtype_out, int op, int algo,
                         cudaStream_t stream);
int rp_launch_all_gather(rp_comm* c, const void* const* src, void* const* dst, size_t bytes,
                         cudaStream_t stream);
int rp_launch_broadcast(rp_comm* c, const void* const* src, void* const* dst, size_t bytes,
                        int root, int algo, cudaStream_t stream);
int rp_launch_bn_stats(rp_comm* c, const void* x, int dtype, int64_t rows, int64_t ch, int64_t hw,
                       int layout, float eps, float* mean, float* var, float* invstd, double* count,
                       cudaStream_t stream);
int rp_launch_bn_bwd_stats(rp_comm* c, const void* x, const void* dy, int dtype, int64_t rows,
                           int64_t ch, int64_t hw, int layout, const float* mean, float* sum_dy,
                           float* sum_dy_xmu, float* local_sum_dy, float* local_sum_dy_xmu,
                           cudaStream_t stream);

// Launch helper: cooperative launch for virtual communicators (all replicas'
// blocks must be co-resident because they wait on one another), plain launch
// otherwise (one rank per process; blocks only wait on peers' blocks).
int rp_launch(rp_comm* c, const void* func, dim3 grid, dim3 block, void** args, size_t smem,
              cudaStream_t stream, bool coop = true);
// Blocks per rank for a collective kernel given its per-block occupancy.
int rp_blocks_per_rank(rp_comm* c, const void* func, int threads, int want);
// Co-resident block budget per rank for kernels that size their own grid (BN):
// occupancy x SMs, divided among virtual replicas, and at most the block cap.
int64_t rp_wave_per_rank(rp_comm* c, int per_sm);

// shared collective plumbing (rp_collectives.cu), used by rp_apply.cu. The
// dynamically scheduled launch passes &a as the kernel's only parameter: a kernel
// taking a larger struct whose FIRST member is the CollArgs gets the whole struct.
bool rp_symmetric_in_pool(rp_comm* c, const void* const* ptrs, size_t bytes, size_t* off);
void rp_base_args(rp_comm* c, CollArgs& a);
int rp_dyn_launch(rp_comm* c, const void* fn, CollArgs& a, cudaStream_t stream, const char* tag);
int rp_launch_apply(rp_comm* c, const void* const* grad, void* const* param, size_t count, int dtype_grad, int opt,
                    const double* hyper, float* const* state0, float* const* state1, int32_t* const* step,
                    cudaStream_t stream);

// NVLS (rp_nvls.cu)
void rp_nvls_destroy(rp_comm* c);
// [p, p + bytes) lies in this rank's bound NVLS region, 16-byte aligned
bool rp_nvls_covers(rp_comm* c, const void* p, size_t bytes);
// Algorithm rp_all_reduce runs (AUTO resolved): RP_ALGO_ONESHOT / TWOSHOT / NVLS
int rp_resolve_ar_algo(rp_comm* c, const void* const* src, const void* const* dst, size_t count, int dtype_in,
                       int dtype_comm, int dtype_out, int op, int algo);
void rp_plan_all_reduce(rp_comm* c, const void* const* src, const void* const* dst, size_t count, int dtype_in,
                        int dtype_comm, int dtype_out, int op, int algo, int64_t* plan);
int rp_relay_bcast_launch(rp_comm* c, const void* src, void* dst, size_t bytes, int root, bool land_in_dst,
                          size_t land_off, cudaStream_t stream,
                          int (*dyn)(rp_comm*, const void*, CollArgs&, cudaStream_t, const char*, int, int, uint32_t),
                          CollArgs& a);
int rp_nvls_bcast_launch(rp_comm* c, const void* src, void* dst, size_t bytes, int root, cudaStream_t stream,
                         int (*dyn)(rp_comm*, const void*, CollArgs&, cudaStream_t, const char*, int, int, uint32_t),
                         CollArgs& a);
int rp_nvls_launch(rp_comm* c, const void* buf, size_t count, int dtype, int op, cudaStream_t stream,
                   int (*dyn)(rp_comm*, const void*, CollArgs&, cudaStream_t, const char*, int, int, uint32_t), CollArgs& a);

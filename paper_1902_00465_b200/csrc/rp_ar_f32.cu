// Instantiates the all-reduce kernels for the f32 exchange dtype.
#include "rp_allreduce.cuh"

const void* rp_pick_ar_f32(int op, int algo, int world, int push) {
  return rp::pick_ar_op<RP_F32>(op, algo, world, push);
}

size_t rp_bulk_smem_bytes(int nr) { return rp::bulk_smem_bytes(nr); }
int rp_bulk_threads() { return rp::kBulkThreads; }

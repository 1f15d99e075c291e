// Instantiates the all-reduce kernels for the f16 exchange dtype.
#include "rp_allreduce.cuh"

const void* rp_pick_ar_f16(int op, int algo, int world, int push) {
  return rp::pick_ar_op<RP_F16>(op, algo, world, push);
}

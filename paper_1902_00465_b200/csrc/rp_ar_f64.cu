// Instantiates the all-reduce kernels for the f64 exchange dtype.
#include "rp_allreduce.cuh"

const void* rp_pick_ar_f64(int op, int algo, int world, int push) {
  return rp::pick_ar_op<RP_F64>(op, algo, world, push);
}

// spmm_mean.cu -- SpMM worker kernels for ReduceOp::Mean (types.hpp:116).
#include "spmm_inst.cuh"

namespace sgnn {
SGNN_DEFINE_SPMM_LOOKUP(spmm_lookup_mean, SGNN_REDUCE_MEAN)
}  // namespace sgnn

// spmm_mean.cu -- SpMM worker kernels for ReduceOp::mean (types.hpp:116).
#include "spmm_inst.cuh"

namespace sgnn {
SGNN_DEFINE_SPMM_LOOKUP(spmm_lookup_mean, SGNN_REDUCE_MEAN, SGNN_SPMM_OCC_CONFIGS)
}  // namespace sgnn

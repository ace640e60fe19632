// spmm_sum.cu -- SpMM worker kernels for ReduceOp::sum (types.hpp:116).
#include "spmm_inst.cuh"

namespace sgnn {
SGNN_DEFINE_SPMM_LOOKUP(spmm_lookup_sum, SGNN_REDUCE_SUM, SGNN_SPMM_OCC_CONFIGS)
}  // namespace sgnn

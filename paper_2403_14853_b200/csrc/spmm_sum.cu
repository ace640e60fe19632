// spmm_sum.cu -- SpMM worker kernels for ReduceOp::Sum (types.hpp:116).
#include "spmm_inst.cuh"

namespace sgnn {
SGNN_DEFINE_SPMM_LOOKUP(spmm_lookup_sum, SGNN_REDUCE_SUM)
}  // namespace sgnn

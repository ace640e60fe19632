// spmm_max.cu -- SpMM worker kernels for ReduceOp::max (types.hpp:116).
#include "spmm_inst.cuh"

namespace sgnn {
SGNN_DEFINE_SPMM_LOOKUP(spmm_lookup_max, SGNN_REDUCE_MAX, SGNN_NO_OCC_CONFIGS)
}  // namespace sgnn

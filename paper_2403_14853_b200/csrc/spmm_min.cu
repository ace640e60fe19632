// spmm_min.cu -- SpMM worker kernels for ReduceOp::min (types.hpp:116).
#include "spmm_inst.cuh"

namespace sgnn {
SGNN_DEFINE_SPMM_LOOKUP(spmm_lookup_min, SGNN_REDUCE_MIN, SGNN_NO_OCC_CONFIGS)
}  // namespace sgnn

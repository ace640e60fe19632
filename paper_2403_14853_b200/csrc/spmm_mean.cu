// spmm_mean.cu -- SpMM worker kernels for ReduceOp::mean (types.hpp:116): the
// Sum chain with the exact divide by the row's nonzero count applied where
// the row is stored (worker or fixup), kernels.hpp:60-63.
#include "spmm_inst.cuh"

namespace sgnn {
SGNN_DEFINE_SPMM_LOOKUP(spmm_lookup_mean, SGNN_REDUCE_MEAN, SGNN_SPMM_OCC_CONFIGS)
}  // namespace sgnn

// fused_mul_sum.cu -- FusedMM worker kernels, edge op MUL, ReduceOp::Sum
// (kernels.hpp:216-270).
#include "spmm_inst.cuh"

namespace sgnn {
SGNN_DEFINE_FUSED_LOOKUP(fused_lookup_mul_sum, SGNN_REDUCE_SUM, dev::OP_FUSED_MUL)
}  // namespace sgnn

// fused_mul_max.cu -- FusedMM worker kernels, edge op MUL, ReduceOp::Max
// (kernels.hpp:216-270).
#include "spmm_inst.cuh"

namespace sgnn {
SGNN_DEFINE_FUSED_LOOKUP(fused_lookup_mul_max, SGNN_REDUCE_MAX, dev::OP_FUSED_MUL)
}  // namespace sgnn

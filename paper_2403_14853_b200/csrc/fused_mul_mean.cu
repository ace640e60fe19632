// fused_mul_mean.cu -- FusedMM worker kernels, edge op MUL, ReduceOp::Mean
// (kernels.hpp:216-270).
#include "spmm_inst.cuh"

namespace sgnn {
SGNN_DEFINE_FUSED_LOOKUP(fused_lookup_mul_mean, SGNN_REDUCE_MEAN, dev::OP_FUSED_MUL)
}  // namespace sgnn

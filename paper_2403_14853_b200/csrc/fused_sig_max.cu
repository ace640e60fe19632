// fused_sig_max.cu -- FusedMM worker kernels, edge op SIGMOID, ReduceOp::Max
// (kernels.hpp:216-270).
#include "spmm_inst.cuh"

namespace sgnn {
SGNN_DEFINE_FUSED_LOOKUP(fused_lookup_sig_max, SGNN_REDUCE_MAX, dev::OP_FUSED_SIGMOID)
}  // namespace sgnn

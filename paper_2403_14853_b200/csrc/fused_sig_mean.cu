// fused_sig_mean.cu -- FusedMM worker kernels, edge op SIGMOID, ReduceOp::Mean
// (kernels.hpp:216-270).
#include "spmm_inst.cuh"

namespace sgnn {
SGNN_DEFINE_FUSED_LOOKUP(fused_lookup_sig_mean, SGNN_REDUCE_MEAN, dev::OP_FUSED_SIGMOID)
}  // namespace sgnn

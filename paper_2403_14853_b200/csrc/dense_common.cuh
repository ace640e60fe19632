// dense_common.cuh -- FP32 GEMMs of the GNN engine on the 5th-gen tensor
// cores: CUTLASS (vendored headers) sm100 "FastFP32" kernels, which split
// every fp32 operand into three bf16 terms and accumulate the significant
// products in fp32 (tcgen05.mma, TMEM accumulators, TMA).  Measured on the
// cfg5 shapes against cuBLAS pedantic SGEMM (scripts/probes/fp32emu*.cu):
// max |err| / sum|a*b| 7e-8 vs 2.4e-7 (more accurate), 4M x 128 x 128 in
// 1.73 vs 2.85 ms; the 128 x 128 weight gradients over 4M rows (split-K,
// deterministic reduction) 1.90 vs 2.35 ms.
#pragma once

#include "cutlass/cutlass.h"
#include "cute/tensor.hpp"
#include "cutlass/gemm/collective/collective_builder.hpp"
#include "cutlass/epilogue/collective/collective_builder.hpp"
#include "cutlass/gemm/device/gemm_universal_adapter.h"
#include "cutlass/gemm/kernel/gemm_universal.hpp"
#include "cutlass/gemm/kernel/tile_scheduler_params.h"
#include "cutlass/util/packed_stride.hpp"

namespace sgnn {
namespace dense {

using namespace cute;
using TileShape = Shape<_128, _128, _16>;
using ClusterShape = Shape<_1, _1, _1>;
using Tile2Sm = Shape<_256, _128, _16>;     // 256 x 128 tiles on SM pairs (cta_group::2)
using Cluster2Sm = Shape<_2, _1, _1>;
using LinComb = cutlass::epilogue::fusion::LinearCombination<float, float, float, float>;
using LinCombRelu = cutlass::epilogue::fusion::LinCombEltAct<cutlass::epilogue::thread::ReLu, float, float, float, float>;

// The kernel for given operand layouts and tile scheduler, spelled out at
// namespace scope in each translation unit (SGNN_DENSE_GEMM) -- nvcc's host
// pass rejects these builder chains as member aliases of a class template.
#define SGNN_DENSE_GEMM(NAME, LAYOUT_A, LAYOUT_B, SCHEDULER) \
    SGNN_DENSE_GEMM_CFG(NAME, LAYOUT_A, LAYOUT_B, SCHEDULER, sgnn::dense::TileShape, sgnn::dense::ClusterShape, \
                        cutlass::epilogue::TmaWarpSpecialized1Sm, cutlass::gemm::KernelTmaWarpSpecialized1SmFastFP32Sm100)
#define SGNN_DENSE_GEMM_CFG(NAME, LAYOUT_A, LAYOUT_B, SCHEDULER, TILE, CLUSTER, EPI_SCHED, MMA_SCHED)              \
    SGNN_DENSE_GEMM_FUSED(NAME, LAYOUT_A, LAYOUT_B, SCHEDULER, TILE, CLUSTER, EPI_SCHED, MMA_SCHED,               \
                          sgnn::dense::LinComb)
// (FUSION: the epilogue's per-element op, e.g. LinCombEltAct<ReLu, ...> to
// write relu(A B) directly)
#define SGNN_DENSE_GEMM_FUSED(NAME, LAYOUT_A, LAYOUT_B, SCHEDULER, TILE, CLUSTER, EPI_SCHED, MMA_SCHED, FUSION)    \
    using NAME##_Epilogue = typename cutlass::epilogue::collective::CollectiveBuilder<                          \
        cutlass::arch::Sm100, cutlass::arch::OpClassTensorOp, TILE, CLUSTER,                                      \
        cutlass::epilogue::collective::EpilogueTileAuto, float, float, float, cutlass::layout::RowMajor, 4, float, \
        cutlass::layout::RowMajor, 4, EPI_SCHED, FUSION>::CollectiveOp;                                           \
    using NAME##_Mainloop = typename cutlass::gemm::collective::CollectiveBuilder<                              \
        cutlass::arch::Sm100, cutlass::arch::OpClassTensorOp, float, LAYOUT_A, 4, float, LAYOUT_B, 4, float,      \
        TILE, CLUSTER,                                                                                            \
        cutlass::gemm::collective::StageCountAutoCarveout<static_cast<int>(                                       \
            sizeof(typename NAME##_Epilogue::SharedStorage))>,                                                    \
        MMA_SCHED>::CollectiveOp;                                                                                 \
    using NAME = cutlass::gemm::device::GemmUniversalAdapter<cutlass::gemm::kernel::GemmUniversal<                \
        cute::Shape<int, int, int, int>, NAME##_Mainloop, NAME##_Epilogue, SCHEDULER>>;

// C[m x n] (row-major) = A' B' + beta C with A' m x k, B' k x n in the
// kernel's layouts; splits > 1: deterministic split-K.  0 on success.
// ws == nullptr && ws_bytes == 0: only query -- *ws_needed gets the
// workspace size (return 1 when the kernel cannot take the shape).
template <class Gemm, bool SPLITK>
int run_gemm(int m, int n, int k, const float* a, const float* b, float* c, float beta, int splits, void* ws,
             size_t ws_bytes, cudaStream_t s, size_t* ws_needed = nullptr) {
    using Kernel = typename Gemm::GemmKernel;
    using SA = typename Kernel::StrideA;
    using SB = typename Kernel::StrideB;
    using SC = typename Kernel::StrideC;
    using SD = typename Kernel::StrideD;
    typename Gemm::Arguments args{cutlass::gemm::GemmUniversalMode::kGemm,
                                  {m, n, k, 1},
                                  {a, cutlass::make_cute_packed_stride(SA{}, {m, k, 1}), b,
                                   cutlass::make_cute_packed_stride(SB{}, {n, k, 1})},
                                  {{1.0f, beta}, c, cutlass::make_cute_packed_stride(SC{}, {m, n, 1}), c,
                                   cutlass::make_cute_packed_stride(SD{}, {m, n, 1})}};
    if constexpr (SPLITK) {
        args.scheduler.splits = splits;
        args.scheduler.reduction_mode = cutlass::gemm::kernel::detail::ReductionMode::Deterministic;
        args.scheduler.decomposition_mode = cutlass::gemm::kernel::detail::DecompositionMode::SplitK;
    }
    Gemm gemm;
    if (gemm.can_implement(args) != cutlass::Status::kSuccess) return 1;
    if (ws_needed) {
        *ws_needed = Gemm::get_workspace_size(args);
        if (!ws && !ws_bytes) return 0;
    }
    if (Gemm::get_workspace_size(args) > ws_bytes) return 2;
    if (gemm.initialize(args, ws, s) != cutlass::Status::kSuccess) return 3;
    if (gemm.run(s) != cutlass::Status::kSuccess) return 4;
    return 0;
}

}  // namespace dense
}  // namespace sgnn

#include "cutlass/cutlass.h"
#include "cute/tensor.hpp"
#include "cutlass/gemm/collective/collective_builder.hpp"
#include "cutlass/epilogue/collective/collective_builder.hpp"
#include "cutlass/gemm/device/gemm_universal_adapter.h"
#include "cutlass/gemm/kernel/gemm_universal.hpp"
#include "cutlass/gemm/kernel/tile_scheduler_params.h"
#include "cutlass/util/packed_stride.hpp"
using namespace cute;
using LayoutA = cutlass::layout::RowMajor;
using LayoutB = cutlass::layout::RowMajor;
using LayoutC = cutlass::layout::RowMajor;
using TileShape = Shape<_128, _128, _16>;
using ClusterShape = Shape<_1, _1, _1>;
using CollectiveEpilogue = typename cutlass::epilogue::collective::CollectiveBuilder<
    cutlass::arch::Sm100, cutlass::arch::OpClassTensorOp, TileShape, ClusterShape,
    cutlass::epilogue::collective::EpilogueTileAuto, float, float,
    float, LayoutC, 4, float, LayoutC, 4, cutlass::epilogue::TmaWarpSpecialized1Sm>::CollectiveOp;
using CollectiveMainloop = typename cutlass::gemm::collective::CollectiveBuilder<
    cutlass::arch::Sm100, cutlass::arch::OpClassTensorOp, float, LayoutA, 4, float, LayoutB, 4, float,
    TileShape, ClusterShape,
    cutlass::gemm::collective::StageCountAutoCarveout<static_cast<int>(sizeof(typename CollectiveEpilogue::SharedStorage))>,
    cutlass::gemm::KernelTmaWarpSpecialized1SmFastFP32Sm100>::CollectiveOp;
using GemmKernel = cutlass::gemm::kernel::GemmUniversal<Shape<int, int, int, int>, CollectiveMainloop, CollectiveEpilogue, void>;
using Gemm = cutlass::gemm::device::GemmUniversalAdapter<GemmKernel>;

extern "C" int emu_gemm(int m, int n, int k, const float* A, const float* B, float* C, float beta, void* ws, size_t ws_bytes, cudaStream_t s) {
  using StrideA = typename Gemm::GemmKernel::StrideA;
  using StrideB = typename Gemm::GemmKernel::StrideB;
  using StrideC = typename Gemm::GemmKernel::StrideC;
  using StrideD = typename Gemm::GemmKernel::StrideD;
  auto sa = cutlass::make_cute_packed_stride(StrideA{}, {m, k, 1});
  auto sb = cutlass::make_cute_packed_stride(StrideB{}, {n, k, 1});
  auto sc = cutlass::make_cute_packed_stride(StrideC{}, {m, n, 1});
  auto sd = cutlass::make_cute_packed_stride(StrideD{}, {m, n, 1});
  typename Gemm::Arguments args{cutlass::gemm::GemmUniversalMode::kGemm, {m, n, k, 1},
                                {A, sa, B, sb}, {{1.0f, beta}, C, sc, C, sd}};
  Gemm gemm;
  if (gemm.can_implement(args) != cutlass::Status::kSuccess) return 1;
  if (Gemm::get_workspace_size(args) > ws_bytes) return 2;
  if (gemm.initialize(args, ws, s) != cutlass::Status::kSuccess) return 3;
  if (gemm.run(s) != cutlass::Status::kSuccess) return 4;
  return 0;
}

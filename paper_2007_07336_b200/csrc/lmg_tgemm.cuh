// lmg_tgemm.cuh -- warp-specialised persistent TMA step GEMM (kernel in lmg_tgemm.cu).
#pragma once

#include <cuda_runtime.h>

#include "lmg_gemm.cuh"

namespace lmg {

struct TgPlan;
// builds the launch (tensor maps) if the TMA kernel applies to this step (64 x 64 tiles on the
// adjoint layout by default, no E_RESID / E_PGRAD) and every operand is describable; else false
bool tgemm_prepare(const StepArgs& a, bool adj, TgPlan** plan);
// launches a prepared plan and frees it
cudaError_t tgemm_launch(TgPlan* plan, bool adj, cudaStream_t st);
// true for the 16 x 32 small-batch tile (LMG_TGEMM=small), false for the 64 x 64 one
bool tgemm_small(const TgPlan* plan);

}  // namespace lmg

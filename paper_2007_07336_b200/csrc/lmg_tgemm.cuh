// lmg_tgemm.cuh -- warp-specialised persistent TMA step GEMM (kernel in lmg_tgemm.cu).
#pragma once

#include <cuda_runtime.h>

#include "lmg_gemm.cuh"

namespace lmg {

// 1 if the TMA kernel can run this launch (64 x 64 tiles, no E_RESID / E_PGRAD)
int tgemm_eligible(const StepArgs& a, bool adj);
// launches it; *launched = false (and cudaSuccess) if an operand cannot be described by a
// tensor map, so the caller falls back to step_gemm
cudaError_t tgemm_launch(const StepArgs& a, bool adj, cudaStream_t st, bool* launched);

}  // namespace lmg

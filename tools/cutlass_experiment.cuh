// cutlass_experiment.cuh -- EXPERIMENT, not in the product library (tools/tile_probe.cu group 3;
// build with -I <cutlass include>).  Measured on B200 (c2 forward step, 256 tasks): bitwise the
// production tiles; identity epilogue 32.4 TF/s (= step_gemm's 2-stage 32 x 32 tiles, 32.3; cuBLAS
// 33.5), tanh epilogue 27.3 vs 30.0: the mainloop keeps the FP64 pipe ~96% busy, so the FP64 tanh
// of the epilogue cannot overlap with DMMAs the way it does across step_gemm's 10 CTAs per SM.
//
// forward layer step on CUTLASS's SM80-class FP64 tensor-op mainloop (the
// structure cuBLAS itself runs for DGEMM on this GPU: cutlass_80_tensorop_d884gemm_64x128_16x3,
// DMMA pipe 94-96% busy under ncu) with this library's fused FAS epilogues, sm_100a.
//
// The mainloop is CUTLASS's threadblock MmaMultistage (64 x 128 x 16 CTA tile, four 32 x 64 warp
// tiles, 3-stage cp.async ring, DMMA.8x8x4), instantiated from the vendored CUTLASS headers inside
// this kernel.  Each output is one DMMA chain over the k4 steps in ascending order, exactly like
// step_gemm, so results are bitwise those of the other tiles.  The accumulator tile is staged in
// the (idle) operand ring and the epilogue walks it by column pairs with coalesced 16-byte loads
// of its operands, CH pairs at a time before any arithmetic: with 8 warps per SM a per-fragment
// epilogue leaves its global-load latency exposed (ncu on a hand-written kernel of this shape put
// 59% of the stall samples there; tools/gemmx_experiment.cuh).
//
// Layouts: A = states (M = B samples x K = q, row-major, lda), B(k, n) = W[n][k] (the weights
// are (out, in) row-major: a column-major K x N operand, ldb).  Fully tiled shapes only
// (M % 64 == N % 128 == K % 16 == 0).  Epilogues: every forward one except the residual (its
// canonical partials need 32-column tiles) and the parameter gradient (another layout).
#pragma once

#include <cutlass/arch/arch.h>
#include <cutlass/gemm/gemm.h>
#include <cutlass/gemm/threadblock/default_mma.h>
#include <cutlass/layout/matrix.h>

#include "../paper_2007_07336_b200/csrc/lmg_gemm.cuh"

namespace lmg {

struct CutlassFwd {
  static constexpr int BM = 64, BN = 128, BK = 16, NT = 128;
  using Mma = typename cutlass::gemm::threadblock::DefaultMma<
      double, cutlass::layout::RowMajor, 1, double, cutlass::layout::ColumnMajor, 1, double,
      cutlass::layout::RowMajor, cutlass::arch::OpClassTensorOp, cutlass::arch::Sm80,
      cutlass::gemm::GemmShape<BM, BN, BK>, cutlass::gemm::GemmShape<32, 64, BK>,
      cutlass::gemm::GemmShape<8, 8, 4>, 3, cutlass::arch::OpMultiplyAdd>::ThreadblockMma;
  static constexpr int CLD = BN + 4;  // staged accumulator tile row stride (doubles)
  static constexpr size_t SMEM_MMA = sizeof(typename Mma::SharedStorage);
  static constexpr size_t SMEM_C = (size_t)BM * CLD * sizeof(double);
  static constexpr size_t SMEM = SMEM_MMA > SMEM_C ? SMEM_MMA : SMEM_C;
};

__global__ void __launch_bounds__(CutlassFwd::NT, 2) step_gemm_cutlass(const StepArgs a) {
  using CF = CutlassFwd;
  using Mma = CF::Mma;
  constexpr int BM = CF::BM, BN = CF::BN, BK = CF::BK, CLD = CF::CLD;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto& ss = *reinterpret_cast<typename Mma::SharedStorage*>(smem_raw);
  double* cs = reinterpret_cast<double*>(smem_raw);

  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const int n0 = blockIdx.x * BN, m0 = blockIdx.y * BM;
  const int64_t t = blockIdx.z;

  typename Mma::IteratorA::Params pa(cutlass::layout::RowMajor(a.lda));
  typename Mma::IteratorB::Params pb(cutlass::layout::ColumnMajor(a.ldb));
  // the weights never depend on the previous launch, but CUTLASS's mainloop issues A and B stages
  // together: wait for the upstream grid before the prologue (programmatic dependent launch)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (!a.pdl_late) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  typename Mma::IteratorA it_a(pa, const_cast<double*>(a.A + t * a.A_ts), {a.M, a.K}, tid, {m0, 0});
  typename Mma::IteratorB it_b(pb, const_cast<double*>(a.Bm + t * a.B_ts), {a.K, a.N}, tid, {0, n0});
  Mma mma(ss, tid, warp, lane);
  typename Mma::FragmentC acc;
  acc.clear();
  mma(a.K / BK, acc, it_a, it_b, acc);
  cutlass::arch::cp_async_wait<0>();
  if (a.pdl_late) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  // accumulators -> staged tile: warp (warp % 2, warp / 2) owns rows 32*wm.., columns 64*wn..;
  // fragment element f: m8n8 tile i = f / 2 (m = i % 4, n = i / 4), lane (fr, fk) holds
  // C[fr][2 fk + f % 2] of it (CUTLASS's MmaTensorOp column-major tile order)
  __syncthreads();  // every warp is done with the operand ring
  {
    const int wm = warp % 2, wn = warp / 2, fr = lane >> 2, fk = lane & 3;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int m = i % 4, n = i / 4;
      const int row = wm * 32 + m * 8 + fr, col = wn * 64 + n * 8 + 2 * fk;
      *reinterpret_cast<double2*>(cs + row * CLD + col) = make_double2(acc[2 * i], acc[2 * i + 1]);
    }
  }
  __syncthreads();

  const int epi = a.epi;
  const double h = a.h, h2 = a.h2;
  const double* bias = a.bias ? a.bias + t * a.bias_ts : nullptr;
  const double* Xp = a.x ? a.x + t * a.x_ts : nullptr;
  const double* Sp = a.s ? a.s + t * a.s_ts : nullptr;
  const double* Yp = a.y ? a.y + t * a.y_ts : nullptr;
  const double* Pp = a.p ? a.p + t * a.p_ts : nullptr;
  double* Op = a.out + t * a.out_ts;
  double* O2p = a.out2 ? a.out2 + t * a.out2_ts : nullptr;
  const bool needX = epi != E_DERIV && epi != E_APPLY;
  const bool needY = epi == E_COARSE || epi == E_COARSE_R || epi == E_PROPOP;
  const bool needP = epi == E_COARSE || epi == E_COARSE_R;
  constexpr int PER = BM * BN / 2 / CF::NT, CH = 4;
#pragma unroll 1
  for (int c0 = 0; c0 < PER; c0 += CH) {
    double2 xv[CH], sv[CH], yv[CH], pv[CH], bv[CH];
    const double2 z = make_double2(0.0, 0.0);
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      const int p = tid + (c0 + u) * CF::NT;
      const int row = p / (BN / 2), col = 2 * (p % (BN / 2));
      const int64_t gi = (int64_t)(m0 + row) * a.ldc + n0 + col;
      xv[u] = needX ? *reinterpret_cast<const double2*>(Xp + gi) : z;
      sv[u] = (Sp && epi == E_PROP) ? *reinterpret_cast<const double2*>(Sp + gi) : z;
      yv[u] = needY ? *reinterpret_cast<const double2*>(Yp + gi) : z;
      pv[u] = needP ? *reinterpret_cast<const double2*>(Pp + gi) : z;
      bv[u] = bias ? *reinterpret_cast<const double2*>(bias + n0 + col) : z;
    }
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      const int p = tid + (c0 + u) * CF::NT;
      const int row = p / (BN / 2), col = 2 * (p % (BN / 2));
      const int64_t gi = (int64_t)(m0 + row) * a.ldc + n0 + col;
      const double2 accv = *reinterpret_cast<const double2*>(cs + row * CLD + col);
      double r[2], r2[2] = {0.0, 0.0};
#pragma unroll
      for (int e = 0; e < 2; ++e) {  // lmg_gemm.cuh epilogue<EPI>, element by element
        const double acc1 = e ? accv.y : accv.x;
        const double x1 = e ? xv[u].y : xv[u].x, s1 = e ? sv[u].y : sv[u].x;
        const double y1 = e ? yv[u].y : yv[u].x, p1 = e ? pv[u].y : pv[u].x;
        double pre = acc1;
        if (bias) pre = __dadd_rn(pre, e ? bv[u].y : bv[u].x);
        if (epi == E_DERIV) {
          r[e] = act_der(a.act, pre);
          continue;
        }
        const double v = act_fwd(a.act, pre);
        if (epi == E_APPLY) {
          r[e] = v;
          continue;
        }
        const double adv = __dadd_rn(x1, __dmul_rn(h, v));
        if (epi == E_PROP) {
          r[e] = __dadd_rn(Sp ? s1 : 0.0, adv);
          r2[e] = __dadd_rn(x1, __dmul_rn(h2, v));
        } else if (epi == E_COARSE) {
          r[e] = __dadd_rn(__dadd_rn(y1, -adv), __dadd_rn(p1, -y1));
          r2[e] = y1;
        } else if (epi == E_COARSE_R) {
          r[e] = __dadd_rn(__dadd_rn(y1, -adv), p1);
        } else if (epi == E_PROPOP) {
          r[e] = __dadd_rn(y1, -adv);
        } else {  // E_ADV
          r[e] = adv;
        }
      }
      *reinterpret_cast<double2*>(Op + gi) = make_double2(r[0], r[1]);
      if (O2p && (epi == E_PROP || epi == E_COARSE))
        *reinterpret_cast<double2*>(O2p + gi) = make_double2(r2[0], r2[1]);
    }
  }
}

}  // namespace lmg

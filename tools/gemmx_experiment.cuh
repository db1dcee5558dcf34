// gemmx_experiment.cuh -- EXPERIMENT, not in the product library (tools/tile_probe.cu group 3).
// Measured on B200 (c2 forward step, 256 tasks): bitwise the production tiles, but 25.2 TF/s with
// the tanh epilogue (28.0 identity) vs 30.0 (32.3) for step_gemm's 2-stage 32 x 32 tiles, and
// cuBLAS's own kernel of this shape at 33.5 (identity): the structure alone does not reproduce
// CUTLASS's scheduling (255 registers with spills here vs its 220).  Kept as the record of the
// attempt.
//
// big-warp-tile FP64 DMMA layer step (sm_100a): 64 x 128 CTA tiles of four
// 32 x 64 warp tiles, two CTAs per SM, k-interleaved shared memory so that ONE 128-bit shared
// load feeds a fragment for two consecutive k4 steps.
//
// Why: the 32 x 32 tiles of step_gemm need one 64-bit fragment load per DMMA and hide DMMA
// latency with many warps (10 CTAs/SM); with 32 x 64 warp tiles a warp issues 32 independent
// DMMAs per k4 step from 4 + 8 fragments, and with the k-interleaved layout those 12 fragments
// of two k4 steps arrive in 12 LDS.128 -- 0.19 shared loads per DMMA instead of 1.  This is the
// structure of the FP64 GEMM cuBLAS runs on this GPU (ncu: cutlass_80_tensorop_d884gemm_64x128_
// 16x3, 4 warps, 220 registers, 2 CTAs/SM, DMMA pipe 96%; profiles/r2_ncu_summary.json).
//
// Shared layout of a K-major operand tile (rows x 16 k): row stride XLD = 24 doubles (192 B: the
// two rows of a quarter-warp's 128-bit loads fall in opposite bank halves), and inside each group
// of 8 k the order [k0 k4 k1 k5 k2 k6 k3 k7], so lane (fr, fk) finds A[fr][8g+fk] and
// A[fr][8g+fk+4] in one 16-byte word.  Global -> shared copies are 8-byte cp.async (a 16-byte
// global pair is not adjacent after the permutation); each thread owns one k column and every
// 8th row of a tile, so it needs one source pointer per operand.
//
// Arithmetic: every output is one DMMA chain over k4 steps 0, 1, 2, ... in order -- bitwise the
// result of step_gemm's tiles -- and the fused epilogues are lmg_gemm.cuh's.
#pragma once

#include "../paper_2007_07336_b200/csrc/lmg_gemm.cuh"

namespace lmg {

struct TileX {
  static constexpr int BM = 64, BN = 128, BK = 16, WM = 2, WN = 2, STAGES = 3;
  static constexpr int NT = WM * WN * 32;       // 128 threads
  static constexpr int WTM = BM / WM, WTN = BN / WN;  // 32 x 64 warp tile
  static constexpr int MT = WTM / 8, NTF = WTN / 8;   // 4 x 8 m8n8 fragments
  static constexpr int XLD = BK + 8;            // row stride (doubles)
  static constexpr int A_SZ = BM * XLD, B_SZ = BN * XLD;
  static constexpr int STAGE = A_SZ + B_SZ;
  static constexpr size_t SMEM = (size_t)STAGES * STAGE * sizeof(double);
};

// position of k (0..15) inside a row of the interleaved layout
__host__ __device__ constexpr int xperm(int k) {
  return (k & 8) | ((k & 3) << 1) | ((k >> 2) & 1);
}

// one operand tile (ROWS x 16 k, K-major in global memory, row stride ld): thread t copies column
// k = t % 16 of rows t/16 + 8i
template <int ROWS>
struct XLoader {
  static constexpr int PER = ROWS * TileX::BK / TileX::NT;  // elements per thread
  const double* src;  // this thread's first element, k-tile 0
  int64_t row8;       // 8 rows, in doubles
  int soff;           // shared offset of the first element
  __device__ __forceinline__ void init(const double* base, int ld, int r0, int tid) {
    const int k = tid & 15, r = tid >> 4;
    src = base + (int64_t)(r0 + r) * ld + k;
    row8 = (int64_t)8 * ld;
    soff = pin(r * TileX::XLD + xperm(k));
  }
  __device__ __forceinline__ void load_next(double* sm) {
#pragma unroll
    for (int i = 0; i < PER; ++i) cp_async_full<1>(sm + soff + i * 8 * TileX::XLD, src + i * row8);
    src += TileX::BK;
  }
};

template <bool DB = true>  // DB: fragments double-buffered across k8 groups
__global__ void __launch_bounds__(TileX::NT, 2) step_gemm_x(const StepArgs a) {
  using X = TileX;
  constexpr int BM = X::BM, BN = X::BN, BK = X::BK, MT = X::MT, NTF = X::NTF, STAGES = X::STAGES;
  extern __shared__ __align__(16) double smem[];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / X::WN, wn = warp % X::WN;
  const int n0 = blockIdx.x * BN, m0 = blockIdx.y * BM;
  const int64_t t = blockIdx.z;
  const int KT = a.K / BK;

  XLoader<BM> la;
  XLoader<BN> lb;
  la.init(a.A + t * a.A_ts, a.lda, m0, tid);
  lb.init(a.Bm + t * a.B_ts, a.ldb, n0, tid);

  double acc[MT][NTF][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NTF; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // programmatic dependent launch as in step_gemm: the weight stages first (they never depend on
  // the previous launch), then wait, then the state stages
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s)
    if (s < KT) lb.load_next(smem + s * X::STAGE + X::A_SZ);
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (!a.pdl_late) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) la.load_next(smem + s * X::STAGE);
    cp_commit();
  }

  const int fr = lane >> 2, fk = lane & 3;
  const int a_off = pin((wm * X::WTM + fr) * X::XLD + 2 * fk);
  const int b_off = pin((wn * X::WTN + fr) * X::XLD + 2 * fk);
  if constexpr (!DB) {
    int sidx = 0;  // ring slot of k-tile kt (no division by STAGES)
    for (int kt = 0; kt < KT; ++kt) {
      cp_wait<STAGES - 2>();
      __syncthreads();
      {
        int nslot = sidx + STAGES - 1;
        if (nslot >= STAGES) nslot -= STAGES;
        if (kt + STAGES - 1 < KT) {
          double* base = smem + nslot * X::STAGE;
          la.load_next(base);
          lb.load_next(base + X::A_SZ);
        }
        cp_commit();
      }
      const double* As = smem + sidx * X::STAGE;
      const double* Bs = As + X::A_SZ;
#pragma unroll
      for (int g = 0; g < BK / 8; ++g) {
        double2 af[MT], bf[NTF];
#pragma unroll
        for (int i = 0; i < MT; ++i)
          af[i] = *reinterpret_cast<const double2*>(As + a_off + i * 8 * X::XLD + g * 8);
#pragma unroll
        for (int j = 0; j < NTF; ++j)
          bf[j] = *reinterpret_cast<const double2*>(Bs + b_off + j * 8 * X::XLD + g * 8);
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
          for (int j = 0; j < NTF; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i].x, bf[j].x);
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
          for (int j = 0; j < NTF; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i].y, bf[j].y);
      }
      if (++sidx == STAGES) sidx = 0;
    }
  } else {
  // fragments double-buffered across k8 groups: the next group's 12 LDS.128 are in flight while
  // this group's 64 DMMAs issue; at a k-tile's last group the next stage is waited for, the stage
  // after it is issued, and its first fragments are loaded (one CTA barrier per k-tile)
  double2 af[2][MT], bf[2][NTF];
  auto ldfrag = [&](int buf, const double* As, int g) {
    const double* Bs = As + X::A_SZ;
#pragma unroll
    for (int i = 0; i < MT; ++i)
      af[buf][i] = *reinterpret_cast<const double2*>(As + a_off + i * 8 * X::XLD + g * 8);
#pragma unroll
    for (int j = 0; j < NTF; ++j)
      bf[buf][j] = *reinterpret_cast<const double2*>(Bs + b_off + j * 8 * X::XLD + g * 8);
  };
  cp_wait<STAGES - 2>();  // stage 0
  __syncthreads();
  ldfrag(0, smem, 0);
  int cur = 0;
  for (int kt = 0; kt < KT; ++kt) {
    const double* As = smem + (kt % STAGES) * X::STAGE;
#pragma unroll
    for (int g = 0; g < BK / 8; ++g) {
      if (g + 1 < BK / 8) {
        ldfrag(cur ^ 1, As, g + 1);
      } else if (kt + 1 < KT) {
        cp_wait<0>();     // stage kt+1 landed (this thread's copies) ...
        __syncthreads();  // ... everyone's; and every warp is done with stage kt-1
        const int nk = kt + STAGES - 1;
        if (nk < KT) {
          double* base = smem + (nk % STAGES) * X::STAGE;
          la.load_next(base);
          lb.load_next(base + X::A_SZ);
        }
        cp_commit();
        ldfrag(cur ^ 1, smem + ((kt + 1) % STAGES) * X::STAGE, 0);
      }
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NTF; ++j)  // k4 step 2g
          dmma(acc[i][j][0], acc[i][j][1], af[cur][i].x, bf[cur][j].x);
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NTF; ++j)  // k4 step 2g + 1
          dmma(acc[i][j][0], acc[i][j][1], af[cur][i].y, bf[cur][j].y);
      cur ^= 1;
    }
  }
  }
  cp_wait<0>();
  if (a.pdl_late) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  // ---------------------------------------------------------------- epilogue through shared memory
  // With 8 warps per SM the register-fragment epilogue (64 outputs per thread, each behind its own
  // global loads of x / bias / s) left its load latency exposed -- ncu put 59% of the stall
  // samples there.  The accumulator tile is staged in the (now idle) ring, then all threads walk
  // it by column pairs: coalesced 16-byte loads of the epilogue operands, issued CH pairs at a
  // time before any arithmetic, then the same per-element operations as lmg_gemm.cuh's epilogue.
  constexpr int CLD = BN + 4;  // staged tile row stride (doubles)
  static_assert((size_t)BM * CLD * sizeof(double) <= X::SMEM, "staged tile fits the ring");
  __syncthreads();  // every warp is done with the ring
  {
    const int rl = wm * X::WTM + fr, cl = wn * X::WTN + 2 * fk;
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int j = 0; j < NTF; ++j)
        *reinterpret_cast<double2*>(smem + (rl + i * 8) * CLD + cl + j * 8) =
            make_double2(acc[i][j][0], acc[i][j][1]);
  }
  __syncthreads();
  const int epi = a.epi;
  const double h = a.h, h2 = a.h2;
  const double* bias = a.bias ? a.bias + t * a.bias_ts : nullptr;
  const double* Xp = a.x ? a.x + t * a.x_ts : nullptr;
  const double* Sp = a.s ? a.s + t * a.s_ts : nullptr;
  const double* Yp = a.y ? a.y + t * a.y_ts : nullptr;
  const double* Pp = a.p ? a.p + t * a.p_ts : nullptr;
  double* Op = a.out ? a.out + t * a.out_ts : nullptr;
  double* O2p = a.out2 ? a.out2 + t * a.out2_ts : nullptr;
  const bool needX = epi != E_DERIV && epi != E_APPLY;
  const bool needY = epi == E_COARSE || epi == E_COARSE_R || epi == E_PROPOP;
  constexpr int PAIRS = BM * BN / 2, PER = PAIRS / X::NT, CH = 8;
  static_assert(PER % CH == 0, "pairs per thread");
#pragma unroll 1
  for (int c0 = 0; c0 < PER; c0 += CH) {
    double2 xv[CH], sv[CH], yv[CH], pv[CH], bv[CH];
    int64_t gi[CH];
    int si[CH];
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      const int p = tid + (c0 + u) * X::NT;
      const int row = p / (BN / 2), col = 2 * (p % (BN / 2));
      si[u] = row * CLD + col;
      gi[u] = (int64_t)(m0 + row) * a.ldc + n0 + col;
      const double2 z = make_double2(0.0, 0.0);
      xv[u] = needX ? *reinterpret_cast<const double2*>(Xp + gi[u]) : z;
      sv[u] = (Sp && (epi == E_PROP)) ? *reinterpret_cast<const double2*>(Sp + gi[u]) : z;
      yv[u] = needY ? *reinterpret_cast<const double2*>(Yp + gi[u]) : z;
      pv[u] = (epi == E_COARSE || epi == E_COARSE_R) ? *reinterpret_cast<const double2*>(Pp + gi[u]) : z;
      bv[u] = bias ? *reinterpret_cast<const double2*>(bias + n0 + col) : z;
    }
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      const double2 accv = *reinterpret_cast<const double2*>(smem + si[u]);
      double r[2], r2[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const double acc1 = e ? accv.y : accv.x, b1 = e ? bv[u].y : bv[u].x;
        const double x1 = e ? xv[u].y : xv[u].x, s1 = e ? sv[u].y : sv[u].x;
        const double y1 = e ? yv[u].y : yv[u].x, p1 = e ? pv[u].y : pv[u].x;
        double pre = acc1;
        if (bias) pre = __dadd_rn(pre, b1);
        if (epi == E_DERIV) { r[e] = act_der(a.act, pre); continue; }
        const double v = act_fwd(a.act, pre);
        if (epi == E_APPLY) { r[e] = v; continue; }
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
      *reinterpret_cast<double2*>(Op + gi[u]) = make_double2(r[0], r[1]);
      if (O2p && (epi == E_PROP || epi == E_COARSE))
        *reinterpret_cast<double2*>(O2p + gi[u]) = make_double2(r2[0], r2[1]);
    }
  }
}

}  // namespace lmg

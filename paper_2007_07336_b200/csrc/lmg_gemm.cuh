// lmg_gemm.cuh -- FP64 tensor-core (DMMA, mma.sync.m8n8k4.f64) batched "layer step" GEMM with
// the FAS epilogues fused in.  sm_100a.
//
// Why DMMA and not tcgen05: the path must run in float64 (fp32 already floors the
// residual at 1e-6 vs tol 1e-9) and tcgen05.mma has no f64 kind.  On sm_100a the f64
// mma.sync lowers to DMMA.8x8x4 on the FP64 tensor pipe (64 FMA/clk/SM, ~37 TF/s at 1.965 GHz).
//
// One launch evaluates `ntasks` independent layer steps ("tasks"), e.g. every block's j-th
// F-relaxation step of a sweep.  Task t's operands are affine in t (base + t*stride), so a whole
// sweep step is described by a handful of pointers and strides -- no device task tables.
//
//   C[m][n] = sum_k A(m,k) * B(k,n)          (per task)
//   A K-major: A(m,k) = A[m*lda + k]        MN-major: A(m,k) = A[k*lda + m]
//   B K-major: B(k,n) = B[n*ldb + k]        MN-major: B(k,n) = B[k*ldb + n]
//   A_SCALE:   A(m,k) *= Ds(m,k)  (same layout as A) -- the adjoint's act'(pre) * lambda
//
// forward step   (m=b, n=i, k=k): A = U_{j-1} (B x q, K-major), B = W_j (q x q, K-major)
// adjoint step   (m=b, n=k, k=i): A = mu * D  (K-major, scaled), B = W_j (MN-major)
// parameter grad (m=i, n=k, k=b): A = lam * D (MN-major, scaled), B = U_j (MN-major)
//
// Pipeline: STAGES-deep cp.async ring (global -> smem, 16 B vectors when aligned), +4-double row
// padding so every m8n8k4 fragment load is bank-conflict free, fragments for k4-step kk+1 loaded
// while the DMMAs of kk issue.  The epilogue mode is switched once per CTA, outside the unrolled
// fragment loops (an in-loop switch blew the instruction cache: ncu 'no_instruction' stalls).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "lmg.h"

namespace lmg {

enum Epi {
  E_PROP = 0,      // out = s + (x + h*act(pre))                       network.py:100
  E_RESID = 1,     // r = (s + (x + h*act(pre))) - y; out=r; out2=s+(..); sum r^2  multigrid.py:124-127
  E_COARSE = 2,    // out = (y - (x + h*act(pre))) + (p - y); out2 = y multigrid.py:142, network.py:138
  E_COARSE_R = 3,  // out = (y - (x + h*act(pre))) + p                 multigrid.py:142
  E_PROPOP = 4,    // out = y - (x + h*act(pre))                       network.py:138
  E_DERIV = 5,     // out = act'(pre)                                  kernels.py:44-48
  E_PGRAD = 6,     // g = (acc*h)*scale; out2 = g; out = x - lr*g      training.py:218-236
  E_APPLY = 7,     // out = act(pre)                                   kernels.py:139-150
  E_ADV = 8        // out = x + h*act(pre)  (a halo value without its source row)
};

struct StepArgs {
  int M, N, K, ntasks;
  int epi, act;
  double h, lr, scale;
  const double* A; int64_t A_ts; int lda;
  const double* Ds; int64_t Ds_ts;
  const double* Bm; int64_t B_ts; int ldb;
  const double* bias; int64_t bias_ts;
  const double* x; int64_t x_ts;
  const double* s; int64_t s_ts;
  const double* y; int64_t y_ts;
  const double* p; int64_t p_ts;
  double* out; int64_t out_ts;
  double* out2; int64_t out2_ts;
  int ldc;
  double* part; int64_t part_slot0; int part_ld;
  int accum;  // E_PGRAD: add the gradient already in out2 (accumulate over batch slices)
  double h2;  // E_PROP with out2: out2 = x + h2*act(pre) (the coarse step's advance, same pre)
  int pdl_late;  // programmatic launch trigger after the mainloop (multi-wave grids), not at start
};

// FP64 tanh for the epilogues (~22 FP64-pipe operations instead of libdevice's ~37: the tanh
// shares the FP64 pipe with the DMMAs, and was ~11% of the c2 forward step).  Relative error of a
// few ulp (tests/test_gpu_parity.py pins it against numpy's tanh); NaN propagates, +-inf -> +-1.
//   tanh(x) = em1 / (em1 + 2),  em1 = e^(2x) - 1 = 2^m * T[j] * (1 + q) - 1
// with n = rint(x * 128/ln2) = 64 m + j, rh = x - n * ln2/128 (Cody-Waite, |rh| <= ln2/256),
// T[j] = 2^(j/64) (table as hi + lo), q = e^(2 rh) - 1 (degree-6 Taylor, error < 1e-19
// relative), em1 = sT (1 + q) - 1 with sT - 1 exact for m = 0 and the table's low part added
// (em1 cancels to ~1/3 of its terms for small negative x: the hi-only table gave 25 ulp there),
// and the quotient by a refined reciprocal (rcp.approx + two Newton steps + one correction).
static __device__ const double2 kTanhExp2[64] = {  // {hi, lo}: 2^(j/64) = hi + lo
    {0x1.0000000000000p+0, 0x0.0p+0},
    {0x1.02c9a3e778061p+0, -0x1.19083535b085dp-56},
    {0x1.059b0d3158574p+0, 0x1.d73e2a475b465p-55},
    {0x1.0874518759bc8p+0, 0x1.186be4bb284ffp-57},
    {0x1.0b5586cf9890fp+0, 0x1.8a62e4adc610bp-54},
    {0x1.0e3ec32d3d1a2p+0, 0x1.03a1727c57b53p-59},
    {0x1.11301d0125b51p+0, -0x1.6c51039449b3ap-54},
    {0x1.1429aaea92de0p+0, -0x1.32fbf9af1369ep-54},
    {0x1.172b83c7d517bp+0, -0x1.19041b9d78a76p-55},
    {0x1.1a35beb6fcb75p+0, 0x1.e5b4c7b4968e4p-55},
    {0x1.1d4873168b9aap+0, 0x1.e016e00a2643cp-54},
    {0x1.2063b88628cd6p+0, 0x1.dc775814a8495p-55},
    {0x1.2387a6e756238p+0, 0x1.9b07eb6c70573p-54},
    {0x1.26b4565e27cddp+0, 0x1.2bd339940e9d9p-55},
    {0x1.29e9df51fdee1p+0, 0x1.612e8afad1255p-55},
    {0x1.2d285a6e4030bp+0, 0x1.0024754db41d5p-54},
    {0x1.306fe0a31b715p+0, 0x1.6f46ad23182e4p-55},
    {0x1.33c08b26416ffp+0, 0x1.32721843659a6p-54},
    {0x1.371a7373aa9cbp+0, -0x1.63aeabf42eae2p-54},
    {0x1.3a7db34e59ff7p+0, -0x1.5e436d661f5e3p-56},
    {0x1.3dea64c123422p+0, 0x1.ada0911f09ebcp-55},
    {0x1.4160a21f72e2ap+0, -0x1.ef3691c309278p-58},
    {0x1.44e086061892dp+0, 0x1.89b7a04ef80d0p-59},
    {0x1.486a2b5c13cd0p+0, 0x1.3c1a3b69062f0p-56},
    {0x1.4bfdad5362a27p+0, 0x1.d4397afec42e2p-56},
    {0x1.4f9b2769d2ca7p+0, -0x1.4b309d25957e3p-54},
    {0x1.5342b569d4f82p+0, -0x1.07abe1db13cadp-55},
    {0x1.56f4736b527dap+0, 0x1.9bb2c011d93adp-54},
    {0x1.5ab07dd485429p+0, 0x1.6324c054647adp-54},
    {0x1.5e76f15ad2148p+0, 0x1.ba6f93080e65ep-54},
    {0x1.6247eb03a5585p+0, -0x1.383c17e40b497p-54},
    {0x1.6623882552225p+0, -0x1.bb60987591c34p-54},
    {0x1.6a09e667f3bcdp+0, -0x1.bdd3413b26456p-54},
    {0x1.6dfb23c651a2fp+0, -0x1.bbe3a683c88abp-57},
    {0x1.71f75e8ec5f74p+0, -0x1.16e4786887a99p-55},
    {0x1.75feb564267c9p+0, -0x1.0245957316dd3p-54},
    {0x1.7a11473eb0187p+0, -0x1.41577ee04992fp-55},
    {0x1.7e2f336cf4e62p+0, 0x1.05d02ba15797ep-56},
    {0x1.82589994cce13p+0, -0x1.d4c1dd41532d8p-54},
    {0x1.868d99b4492edp+0, -0x1.fc6f89bd4f6bap-54},
    {0x1.8ace5422aa0dbp+0, 0x1.6e9f156864b27p-54},
    {0x1.8f1ae99157736p+0, 0x1.5cc13a2e3976cp-55},
    {0x1.93737b0cdc5e5p+0, -0x1.75fc781b57ebcp-57},
    {0x1.97d829fde4e50p+0, -0x1.d185b7c1b85d1p-54},
    {0x1.9c49182a3f090p+0, 0x1.c7c46b071f2bep-56},
    {0x1.a0c667b5de565p+0, -0x1.359495d1cd533p-54},
    {0x1.a5503b23e255dp+0, -0x1.d2f6edb8d41e1p-54},
    {0x1.a9e6b5579fdbfp+0, 0x1.0fac90ef7fd31p-54},
    {0x1.ae89f995ad3adp+0, 0x1.7a1cd345dcc81p-54},
    {0x1.b33a2b84f15fbp+0, -0x1.2805e3084d708p-57},
    {0x1.b7f76f2fb5e47p+0, -0x1.5584f7e54ac3bp-56},
    {0x1.bcc1e904bc1d2p+0, 0x1.23dd07a2d9e84p-55},
    {0x1.c199bdd85529cp+0, 0x1.11065895048ddp-55},
    {0x1.c67f12e57d14bp+0, 0x1.2884dff483cadp-54},
    {0x1.cb720dcef9069p+0, 0x1.503cbd1e949dbp-56},
    {0x1.d072d4a07897cp+0, -0x1.cbc3743797a9cp-54},
    {0x1.d5818dcfba487p+0, 0x1.2ed02d75b3707p-55},
    {0x1.da9e603db3285p+0, 0x1.c2300696db532p-54},
    {0x1.dfc97337b9b5fp+0, -0x1.1a5cd4f184b5cp-54},
    {0x1.e502ee78b3ff6p+0, 0x1.39e8980a9cc8fp-55},
    {0x1.ea4afa2a490dap+0, -0x1.e9c23179c2893p-54},
    {0x1.efa1bee615a27p+0, 0x1.dc7f486a4b6b0p-54},
    {0x1.f50765b6e4540p+0, 0x1.9d3e12dd8a18bp-54},
    {0x1.fa7c1819e90d8p+0, 0x1.74853f3a5931ep-55}};

// TL: the table lookup (global __ldg here; the latency-bound warp sweep reads a shared-memory
// copy so the lookup is not an L2 round trip on every step of its serial chain)
template <class TL>
__device__ __forceinline__ double fast_tanh_impl(double x, TL tl) {
  x = x > 20.0 ? 20.0 : x;  // |tanh| rounds to 1 beyond 19.06; comparisons keep NaN
  x = x < -20.0 ? -20.0 : x;
  const double kMagic = 6755399441055744.0;  // 1.5 * 2^52: rint by addition
  const double k = fma(x, 0x1.71547652b82fep+7, kMagic);  // x * 128/ln2 + magic
  const double n = k - kMagic;
  const int ni = __double2loint(k);
  double rh = fma(-n, 0x1.62e42fefa2000p-8, x);   // x - n * (ln2/128)_hi (exact product)
  rh = fma(-n, 0x1.9ef35793c7673p-48, rh);        //   - n * (ln2/128)_lo
  double p = fma(rh, 0x1.6c16c16c16c17p-4, 0x1.1111111111111p-2);  // 4/45, 4/15
  p = fma(rh, p, 0x1.5555555555555p-1);  // 2/3
  p = fma(rh, p, 0x1.5555555555555p+0);  // 4/3
  p = fma(rh, p, 2.0);
  p = fma(rh, p, 2.0);
  const double q = rh * p;                // e^(2 rh) - 1
  const double sc = __hiloint2double((1023 + (ni >> 6)) << 20, 0);  // 2^m
  const double2 T = tl(ni & 63);
  const double sT = sc * T.x;  // exact
  // sT - 1 is exact when m = 0; the table's low part keeps em1 accurate where it cancels
  const double em1 = fma(sT, q, fma(sc, T.y, sT - 1.0));
  const double d = em1 + 2.0;
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  y = fma(y, fma(-d, y, 1.0), y);
  y = fma(y, fma(-d, y, 1.0), y);
  double t = em1 * y;
  t = fma(fma(-d, t, em1), y, t);
  return copysign(t, x);  // odd: keeps the sign of -0.0 (numpy's tanh(-0.0) = -0.0)
}

__device__ __forceinline__ double fast_tanh(double x) {
  return fast_tanh_impl(x, [](int i) { return __ldg(&kTanhExp2[i]); });
}

__device__ __forceinline__ double act_fwd(int a, double v) {
  if (a == LMG_ACT_TANH) return fast_tanh(v);
  if (a == LMG_ACT_RELU) return (v >= 0.0 || v != v) ? v : 0.0;  // np.maximum(pre, 0.0)
  return v;
}

__device__ __forceinline__ double act_der(int a, double v) {
  if (a == LMG_ACT_TANH) {
    double t = fast_tanh(v);
    return __dadd_rn(1.0, -__dmul_rn(t, t));  // 1.0 - t*t, no contraction
  }
  if (a == LMG_ACT_RELU) return v > 0.0 ? 1.0 : 0.0;
  return 1.0;
}

template <int VEC>
__device__ __forceinline__ void cp_async(double* dst, const double* src, bool ok) {
  unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  int sz = ok ? 8 * VEC : 0;
  if (VEC == 2)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(sz));
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(sz));
}
// unpredicated form for fully tiled shapes
template <int VEC>
__device__ __forceinline__ void cp_async_full(double* dst, const double* src) {
  unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  if (VEC == 2)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src));
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }

// keep a loop-invariant value in a register: ptxas otherwise rematerializes thread-index
// arithmetic inside the k-loop (measured: ~30 extra integer instructions per k-tile)
__device__ __forceinline__ int pin(int v) {
  int r;
  asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
  return r;
}
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// smem footprint (doubles) of one operand tile of T (M or N) x BK
template <bool KMAJ, int T, int BK>
struct TileShape {
  static constexpr int LD = KMAJ ? (BK + 4) : (T + 4);  // +4 doubles: conflict-free fragments
  static constexpr int SIZE = KMAJ ? T * (BK + 4) : BK * (T + 4);
};

template <bool KMAJ, int T, int BK, int VEC, int NT>
__device__ __forceinline__ void load_tile(double* sm, const double* g, int ld, int mn0, int mnlim,
                                          int k0, int klim, int tid) {
  using S = TileShape<KMAJ, T, BK>;
  if (KMAJ) {
    constexpr int PR = BK / VEC;
#pragma unroll
    for (int e = tid; e < T * PR; e += NT) {
      int r = e / PR, kk = (e % PR) * VEC;
      int gm = mn0 + r, gk = k0 + kk;
      bool ok = gm < mnlim && gk < klim;
      cp_async<VEC>(sm + r * S::LD + kk, ok ? g + (int64_t)gm * ld + gk : g, ok);
    }
  } else {
    constexpr int PR = T / VEC;
#pragma unroll
    for (int e = tid; e < BK * PR; e += NT) {
      int kk = e / PR, r = (e % PR) * VEC;
      int gm = mn0 + r, gk = k0 + kk;
      bool ok = gm < mnlim && gk < klim;
      cp_async<VEC>(sm + kk * S::LD + r, ok ? g + (int64_t)gk * ld + gm : g, ok);
    }
  }
}

// Per-thread precomputed global->smem copy plan for one operand tile: the k-loop only adds a
// constant pointer advance (no index math, no per-tile bounds checks unless K % BK != 0).
template <bool KMAJ, int T, int BK, int VEC, int NT>
struct Loader {
  using S = TileShape<KMAJ, T, BK>;
  static constexpr int PR = KMAJ ? BK / VEC : T / VEC;  // vectors per smem row
  static constexpr int NV = (KMAJ ? T : BK) * PR;        // vectors per tile
  static constexpr int IT = (NV + NT - 1) / NT;          // vectors per thread
  const double* g;
  int64_t kadv;  // pointer advance per k-tile
  int goff[IT], soff[IT], kin[IT];
  unsigned okmask;

  __device__ __forceinline__ void init(const double* base, int ld, int mn0, int mnlim, int tid) {
    g = base;
    kadv = KMAJ ? BK : (int64_t)BK * ld;
    okmask = 0;
#pragma unroll
    for (int i = 0; i < IT; ++i) {
      const int e = tid + i * NT;
      int r, kk;
      if (KMAJ) {
        r = e / PR;
        kk = (e % PR) * VEC;
      } else {
        kk = e / PR;
        r = (e % PR) * VEC;
      }
      const bool ok = (e < NV) && (mn0 + r < mnlim);
      goff[i] = KMAJ ? (mn0 + r) * ld + kk : kk * ld + mn0 + r;
      soff[i] = pin(KMAJ ? r * S::LD + kk : kk * S::LD + r);
      kin[i] = kk;
      okmask |= (ok ? 1u : 0u) << i;
    }
  }
  // copy k-tile `kt` (first k index k0) into sm; kfull: the whole tile lies inside K
  __device__ __forceinline__ void load(double* sm, int kt, int k0, int klim, bool kfull) const {
    const double* gt = g + kt * kadv;
#pragma unroll
    for (int i = 0; i < IT; ++i) {
      bool ok = (okmask >> i) & 1u;
      if (!kfull) ok = ok && (k0 + kin[i] < klim);
      if (IT * NT > NV && tid_out_of_range(i)) continue;
      cp_async<VEC>(sm + soff[i], ok ? gt + goff[i] : g, ok);
    }
  }
  __device__ __forceinline__ bool tid_out_of_range(int i) const {
    return (int)(threadIdx.x + i * NT) >= NV;
  }
  // the adjoint's act' scaling applied once per staged element, by the thread that copied it
  // (its cp.async data is visible to it after cp.async.wait_group; the CTA barrier that follows
  // publishes the product): sm[e] *= ds[e] over this thread's vectors of the stage.  Same
  // __dmul_rn as scaling each fragment at use -- bitwise -- but once per element per CTA instead
  // of once per warp that reads it (the per-fragment DMULs cost the adjoint ~25% of its DMMA
  // issue: tools/tile_probe.cu, 23.2 vs 31.9 TF/s unscaled).
  __device__ __forceinline__ void scale_own(double* sm, const double* ds) const {
#pragma unroll
    for (int i = 0; i < IT; ++i) {
      if (IT * NT > NV && tid_out_of_range(i)) continue;
      if (VEC == 2) {
        double2 v = *reinterpret_cast<const double2*>(sm + soff[i]);
        const double2 d = *reinterpret_cast<const double2*>(ds + soff[i]);
        v.x = __dmul_rn(v.x, d.x);
        v.y = __dmul_rn(v.y, d.y);
        *reinterpret_cast<double2*>(sm + soff[i]) = v;
      } else {
        sm[soff[i]] = __dmul_rn(sm[soff[i]], ds[soff[i]]);
      }
    }
  }
  // fully tiled shapes: running per-thread source pointers, advanced by one k-tile per call
  const double* cur[IT];
  __device__ __forceinline__ void init_full() {
#pragma unroll
    for (int i = 0; i < IT; ++i) cur[i] = g + goff[i];
  }
  __device__ __forceinline__ void load_next(double* sm) {
#pragma unroll
    for (int i = 0; i < IT; ++i) {
      if (IT * NT > NV && tid_out_of_range(i)) continue;
      cp_async_full<VEC>(sm + soff[i], cur[i]);
      cur[i] += kadv;
    }
  }
};

template <bool KMAJ, int T, int BK>
__device__ __forceinline__ double frag(const double* sm, int mn, int k) {
  using S = TileShape<KMAJ, T, BK>;
  return KMAJ ? sm[mn * S::LD + k] : sm[k * S::LD + mn];
}

template <int BM_, int BN_, int BK_, int WM_, int WN_, int STAGES_>
struct Tile {
  static constexpr int BM = BM_, BN = BN_, BK = BK_, WM = WM_, WN = WN_, STAGES = STAGES_;
  static constexpr bool RS = false;
};
// Register-staged scaled A (the adjoint layout, fully tiled, 2 stages): each thread loads its
// A and act' vectors of the NEXT k-tile into registers while the DMMAs of this one run, and
// stores their product into the A stage -- act' never touches shared memory and no pass over
// the staged tile is needed.  W keeps its cp.async stage.
template <int BM_, int BN_, int BK_, int WM_, int WN_>
struct TileR : Tile<BM_, BN_, BK_, WM_, WN_, 2> {
  static constexpr bool RS = true;
};
// the same staging with a deeper weight ring (persistent chain launches: the W stages run ahead
// of each item's dependency wait; A goes through registers one k-tile ahead)
template <int BM_, int BN_, int BK_, int WM_, int WN_, int STAGES_>
struct TileRW : Tile<BM_, BN_, BK_, WM_, WN_, STAGES_> {
  static constexpr bool RS = true;
};

template <class T, bool AK, bool BKM, bool ASC>
struct GemmCfg {
  static constexpr int BM = T::BM, BN = T::BN, BK = T::BK, WM = T::WM, WN = T::WN;
  static constexpr int STAGES = T::STAGES;
  static constexpr int NTHREADS = WM * WN * 32;
  static constexpr int WTM = BM / WM, WTN = BN / WN;  // warp tile
  static constexpr int MT = WTM / 8, NTF = WTN / 8;   // m8n8 fragments per warp
  static constexpr int A_SZ = TileShape<AK, BM, BK>::SIZE;
  static constexpr int B_SZ = TileShape<BKM, BN, BK>::SIZE;
  static constexpr bool RS = ASC && AK && T::RS;  // register-staged scaled A (TileR)
  static constexpr int B_OFF = A_SZ * ((ASC && !RS) ? 2 : 1);  // W's offset within a stage
  static constexpr int STAGE = B_OFF + B_SZ;
  static constexpr size_t SMEM = (size_t)STAGES * STAGE * sizeof(double);
};

// Per-task epilogue operands.
struct EpiPtrs {
  const double *bias, *X, *S, *Y, *P;
  double *O, *O2;
};

// E_PGRAD epilogue in two halves.  out (the weights, SGD in place) aliases x: loads and stores
// interleaved would keep each W load behind the previous store -- one HBM round trip per element
// (c5: 1.8 ms per gradient launch, 0.36 of HBM).  Every element is read and written by this
// thread only, so all loads are issued first.
template <int MT, int NTF>
__device__ __forceinline__ void pgrad_load(const StepArgs& a, const EpiPtrs& q, int mrow0, int ncol0,
                                           double (&xv)[MT][NTF][2], double (&gv)[MT][NTF][2]) {
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NTF; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int m = mrow0 + i * 8, n = ncol0 + j * 8 + e;
        const bool in = m < a.M && n < a.N;
        const int64_t idx = (int64_t)m * a.ldc + n;
        xv[i][j][e] = (in && a.lr != 0.0) ? q.X[idx] : 0.0;
        gv[i][j][e] = (in && a.accum && q.O2) ? q.O2[idx] : 0.0;
      }
}
template <int MT, int NTF>
__device__ __forceinline__ void pgrad_store(const StepArgs& a, const EpiPtrs& q,
                                            const double (&acc)[MT][NTF][2], int mrow0, int ncol0,
                                            const double (&xv)[MT][NTF][2],
                                            const double (&gv)[MT][NTF][2]) {
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NTF; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int m = mrow0 + i * 8, n = ncol0 + j * 8 + e;
        if (m >= a.M || n >= a.N) continue;
        const int64_t idx = (int64_t)m * a.ldc + n;
        double g = __dmul_rn(__dmul_rn(acc[i][j][e], a.h), a.scale);
        if (a.accum && q.O2) g = __dadd_rn(gv[i][j][e], g);
        if (q.O2) q.O2[idx] = g;
        if (a.lr != 0.0) q.O[idx] = __dadd_rn(xv[i][j][e], -__dmul_rn(a.lr, g));
      }
}

// Apply epilogue EPI to this thread's accumulators.  Returns per-fragment-row sums of r^2 for
// E_RESID in rowsq.
template <int EPI, int MT, int NTF>
__device__ __forceinline__ void epilogue(const StepArgs& a, const EpiPtrs& q, double (&acc)[MT][NTF][2],
                                         int mrow0, int ncol0, double (&rowsq)[MT]) {
  const int actk = a.act;
  const double h = a.h;
  const int ldc = a.ldc;
  if constexpr (EPI == E_PGRAD) {
    double xv[MT][NTF][2], gv[MT][NTF][2];
    pgrad_load(a, q, mrow0, ncol0, xv, gv);
    pgrad_store(a, q, acc, mrow0, ncol0, xv, gv);
    for (int i = 0; i < MT; ++i) rowsq[i] = 0.0;
    return;
  } else {
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    rowsq[i] = 0.0;
    const int m = mrow0 + i * 8;
    if (m >= a.M) continue;
#pragma unroll
    for (int j = 0; j < NTF; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int n = ncol0 + j * 8 + e;
        if (n >= a.N) continue;
        const int64_t idx = (int64_t)m * ldc + n;
        const double accv = acc[i][j][e];
        double pre = accv;
        if (q.bias) pre = __dadd_rn(pre, q.bias[n]);
        if (EPI == E_DERIV) {
          q.O[idx] = act_der(actk, pre);
          continue;
        }
        const double v = act_fwd(actk, pre);
        if (EPI == E_APPLY) {
          q.O[idx] = v;
          continue;
        }
        const double adv = __dadd_rn(q.X[idx], __dmul_rn(h, v));  // u + h*F(u)
        if (EPI == E_ADV) {
          q.O[idx] = adv;
        } else if (EPI == E_PROP) {
          q.O[idx] = __dadd_rn(q.S ? q.S[idx] : 0.0, adv);
          if (q.O2) q.O2[idx] = __dadd_rn(q.X[idx], __dmul_rn(a.h2, v));
        } else if (EPI == E_RESID) {
          const double prop = __dadd_rn(q.S ? q.S[idx] : 0.0, adv);
          double r = __dadd_rn(prop, -q.Y[idx]);
          if (q.O) q.O[idx] = r;
          if (q.O2) q.O2[idx] = prop;  // the propagated row, reused by the next F sweep
          rowsq[i] = fma(r, r, rowsq[i]);
        } else if (EPI == E_COARSE) {
          const double yv = q.Y[idx];
          q.O[idx] = __dadd_rn(__dadd_rn(yv, -adv), __dadd_rn(q.P[idx], -yv));
          if (q.O2) q.O2[idx] = yv;
        } else if (EPI == E_COARSE_R) {
          q.O[idx] = __dadd_rn(__dadd_rn(q.Y[idx], -adv), q.P[idx]);
        } else {  // E_PROPOP
          q.O[idx] = __dadd_rn(q.Y[idx], -adv);
        }
      }
    }
  }
  }
}

template <class T, bool AK, bool BKM, bool ASC, int VEC, bool FULL = false>
__global__ void __launch_bounds__(T::WM* T::WN * 32)
    step_gemm(const StepArgs a) {
  using C = GemmCfg<T, AK, BKM, ASC>;
  constexpr int BM = C::BM, BN = C::BN, BK = C::BK, WN = C::WN, STAGES = C::STAGES;
  extern __shared__ __align__(16) double smem[];
  __shared__ double red[WN][BM];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WN, wn = warp % WN;
  const int n0 = blockIdx.x * BN, m0 = blockIdx.y * BM;
  const int64_t t = blockIdx.z;

  const double* A = a.A + t * a.A_ts;
  const double* Ds = ASC ? a.Ds + t * a.Ds_ts : nullptr;
  const double* Bm = a.Bm + t * a.B_ts;

  double acc[C::MT][C::NTF][2];
#pragma unroll
  for (int i = 0; i < C::MT; ++i)
#pragma unroll
    for (int j = 0; j < C::NTF; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int KT = (a.K + BK - 1) / BK;
  const bool kfull_all = (a.K % BK) == 0;
  Loader<AK, BM, BK, VEC, C::NTHREADS> la;
  Loader<BKM, BN, BK, VEC, C::NTHREADS> lb;
  la.init(A, a.lda, m0, a.M, tid);
  lb.init(Bm, a.ldb, n0, a.N, tid);
  Loader<AK, BM, BK, VEC, C::NTHREADS> ld_;
  if (ASC) ld_.init(Ds, a.lda, m0, a.M, tid);
  if (FULL) {
    la.init_full();
    lb.init_full();
    if (ASC) ld_.init_full();
  }
  auto load_stage = [&](int s, int kt) {
    double* base = smem + s * C::STAGE;
    if (FULL) {  // loads are issued for kt = 0, 1, 2, ... in order
      la.load_next(base);
      if (ASC) ld_.load_next(base + C::A_SZ);
      lb.load_next(base + C::B_OFF);
      return;
    }
    const int k0 = kt * BK;
    const bool kfull = kfull_all || (k0 + BK <= a.K);
    la.load(base, kt, k0, a.K, kfull);
    if (ASC) ld_.load(base + C::A_SZ, kt, k0, a.K, kfull);
    lb.load(base + C::B_OFF, kt, k0, a.K, kfull);
  };

  // Programmatic dependent launch: when B is the weight stack (forward / adjoint layouts) its
  // first stages do not depend on the previous launch, so they are fetched before waiting for it
  // (griddepcontrol.wait is a no-op without PDL); everything produced upstream -- A, the scales,
  // every epilogue operand -- is read only after the wait, and every write happens after it, so
  // there is no WAR hazard either.  The trigger lets the NEXT step's prologue overlap this one's
  // tail; the parameter-gradient launch (it writes W) never triggers.
  if (AK) {
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
      if (s >= KT) break;
      double* base = smem + s * C::STAGE + C::B_OFF;
      if (FULL) {
        lb.load_next(base);
      } else {
        const int k0 = s * BK;
        lb.load(base, s, k0, a.K, kfull_all || (k0 + BK <= a.K));
      }
    }
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (a.epi != E_PGRAD && !a.pdl_late) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  const int wm0 = wm * C::WTM, wn0 = wn * C::WTN;
  const int fr = lane >> 2, fk = lane & 3;
  constexpr int LDA_ = TileShape<AK, BM, BK>::LD, LDB_ = TileShape<BKM, BN, BK>::LD;
  const int a_thr = pin(AK ? (wm0 + fr) * LDA_ + fk : fk * LDA_ + wm0 + fr);
  const int b_thr = pin(BKM ? (wn0 + fr) * LDB_ + fk : fk * LDB_ + wn0 + fr);
  // the DMMAs of one staged k-tile (fragments double-buffered across the k4 steps)
  auto compute = [&](const double* As, const double* Bs) {
    double af[2][C::MT], bf[2][C::NTF];
    // per-thread fragment offsets are loop invariant (a_thr / b_thr); only constants vary below
    auto ldfrag = [&](int buf, int kk) {
#pragma unroll
      for (int i = 0; i < C::MT; ++i) {
        const int o = a_thr + (AK ? i * 8 * LDA_ + kk : kk * LDA_ + i * 8);
        af[buf][i] = As[o];  // already scaled by act' (ASC: scale_own / register staging)
      }
#pragma unroll
      for (int j = 0; j < C::NTF; ++j) bf[buf][j] = Bs[b_thr + (BKM ? j * 8 * LDB_ + kk : kk * LDB_ + j * 8)];
    };
    ldfrag(0, 0);
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      const int cur = (kk >> 2) & 1;
      if (kk + 4 < BK) ldfrag(cur ^ 1, kk + 4);
#pragma unroll
      for (int i = 0; i < C::MT; ++i)
#pragma unroll
        for (int j = 0; j < C::NTF; ++j) dmma(acc[i][j][0], acc[i][j][1], af[cur][i], bf[cur][j]);
    }
  };

  if constexpr (C::RS) {
    static_assert(STAGES == 2 && FULL && VEC == 2, "register staging: 2 stages, fully tiled, 16-byte vectors");
    constexpr int IT = decltype(la)::IT;
    double2 ra[IT], rd[IT];
    auto ldg = [&] {  // this thread's A and act' vectors of the next k-tile
#pragma unroll
      for (int i = 0; i < IT; ++i) {
        if (IT * C::NTHREADS > decltype(la)::NV && la.tid_out_of_range(i)) continue;
        ra[i] = *reinterpret_cast<const double2*>(la.cur[i]);
        rd[i] = *reinterpret_cast<const double2*>(ld_.cur[i]);
        la.cur[i] += la.kadv;
        ld_.cur[i] += ld_.kadv;
      }
    };
    auto sts = [&](double* base) {  // their products into the A stage (same __dmul_rn: bitwise)
#pragma unroll
      for (int i = 0; i < IT; ++i) {
        if (IT * C::NTHREADS > decltype(la)::NV && la.tid_out_of_range(i)) continue;
        double2 v;
        v.x = __dmul_rn(ra[i].x, rd[i].x);
        v.y = __dmul_rn(ra[i].y, rd[i].y);
        *reinterpret_cast<double2*>(base + la.soff[i]) = v;
      }
    };
    ldg();
    sts(smem);
    cp_commit();  // group 0: the weight stage prefetched before griddepcontrol.wait
    if (KT > 1) ldg();
    for (int kt = 0; kt < KT; ++kt) {
      cp_wait<0>();
      __syncthreads();  // W stage kt landed and A stage kt stored; stage kt-1 fully consumed
      double* nxt = smem + ((kt + 1) & 1) * C::STAGE;
      if (kt + 1 < KT) lb.load_next(nxt + C::B_OFF);
      cp_commit();
      compute(smem + (kt & 1) * C::STAGE, smem + (kt & 1) * C::STAGE + C::B_OFF);
      if (kt + 1 < KT) {
        sts(nxt);
        if (kt + 2 < KT) ldg();
      }
    }
  } else {
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) {
      double* base = smem + s * C::STAGE;
      if (FULL) {
        la.load_next(base);
        if (ASC) ld_.load_next(base + C::A_SZ);
        if (!AK) lb.load_next(base + C::B_OFF);
      } else {
        const int k0 = s * BK;
        const bool kfull = kfull_all || (k0 + BK <= a.K);
        la.load(base, s, k0, a.K, kfull);
        if (ASC) ld_.load(base + C::A_SZ, s, k0, a.K, kfull);
        if (!AK) lb.load(base + C::B_OFF, s, k0, a.K, kfull);
      }
    }
    cp_commit();  // group 0 also carries the prefetched weight stages
  }
  for (int kt = 0; kt < KT; ++kt) {
    cp_wait<STAGES - 2>();
    if (ASC) {
      double* st0 = smem + (kt % STAGES) * C::STAGE;
      la.scale_own(st0, st0 + C::A_SZ);
    }
    __syncthreads();
    {
      int nk = kt + STAGES - 1;
      if (nk < KT) load_stage(nk % STAGES, nk);
      cp_commit();
    }
    compute(smem + (kt % STAGES) * C::STAGE, smem + (kt % STAGES) * C::STAGE + C::B_OFF);
  }
  }  // register staging / cp.async staging
  cp_wait<0>();
  // multi-wave grids trigger here: the dependent grid launches once every CTA has reached its
  // epilogue, i.e. while the last wave finishes, instead of parking on slots the grid still needs
  if (a.epi != E_PGRAD && a.pdl_late) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  // ---------------------------------------------------------------- fused epilogue
  EpiPtrs q;
  q.bias = a.bias ? a.bias + t * a.bias_ts : nullptr;
  q.X = a.x ? a.x + t * a.x_ts : nullptr;
  q.S = a.s ? a.s + t * a.s_ts : nullptr;
  q.Y = a.y ? a.y + t * a.y_ts : nullptr;
  q.P = a.p ? a.p + t * a.p_ts : nullptr;
  q.O = a.out ? a.out + t * a.out_ts : nullptr;
  q.O2 = a.out2 ? a.out2 + t * a.out2_ts : nullptr;
  const int mrow0 = m0 + wm0 + fr, ncol0 = n0 + wn0 + 2 * fk;
  double rowsq[C::MT];
  switch (a.epi) {
    case E_PROP: epilogue<E_PROP>(a, q, acc, mrow0, ncol0, rowsq); break;
    case E_RESID: epilogue<E_RESID>(a, q, acc, mrow0, ncol0, rowsq); break;
    case E_COARSE: epilogue<E_COARSE>(a, q, acc, mrow0, ncol0, rowsq); break;
    case E_COARSE_R: epilogue<E_COARSE_R>(a, q, acc, mrow0, ncol0, rowsq); break;
    case E_PROPOP: epilogue<E_PROPOP>(a, q, acc, mrow0, ncol0, rowsq); break;
    case E_DERIV: epilogue<E_DERIV>(a, q, acc, mrow0, ncol0, rowsq); break;
    case E_PGRAD:  // only the parameter-gradient layout (A MN-major) runs it (measured and not
      // kept: W loaded into registers before the mainloop, 1.23 vs 1.07 ms per c5 gradient
      // launch; W staged into shared memory by cp.async with the first stages, no change)
      if constexpr (!AK) epilogue<E_PGRAD>(a, q, acc, mrow0, ncol0, rowsq);
      break;
    case E_APPLY: epilogue<E_APPLY>(a, q, acc, mrow0, ncol0, rowsq); break;
    default: epilogue<E_ADV>(a, q, acc, mrow0, ncol0, rowsq); break;
  }
  if (a.epi == E_RESID && a.part) {
    // deterministic per-row partial sums: 4 lanes of a fragment row, then the WN warps
#pragma unroll
    for (int i = 0; i < C::MT; ++i) {
      rowsq[i] += __shfl_xor_sync(0xffffffffu, rowsq[i], 1);
      rowsq[i] += __shfl_xor_sync(0xffffffffu, rowsq[i], 2);
      if (fk == 0) red[wn][wm0 + i * 8 + fr] = rowsq[i];
    }
    __syncthreads();
    for (int r = tid; r < BM; r += C::NTHREADS) {
      const int m = m0 + r;
      if (m < a.M) {
        double sum = 0.0;
#pragma unroll
        for (int w = 0; w < WN; ++w) sum += red[w][r];
        const int64_t slot = a.part_slot0 + t * gridDim.x + blockIdx.x;
        a.part[slot * a.part_ld + m] = sum;
      }
    }
  }
}

}  // namespace lmg

// ------------------------------------------------------------------------------------------------
// Split-K layer step for inherently serial steps (coarsest exact solve, sequential_forward, the
// serial adjoint): one step's K range is split over the KS CTAs of a thread-block cluster
// (gridDim.z == cluster z == KS), each accumulates its slice with the same DMMA mainloop, then the
// partial tiles are summed through distributed shared memory in fixed rank order (deterministic)
// and the E_PROP / E_ADV epilogue is applied, each CTA finishing 1/KS of the tile.  Fully tiled
// shapes only (M % BM == N % BN == (K/KS) % BK == 0).
#include <cooperative_groups.h>

namespace lmg {

__device__ __forceinline__ double epi_point(int epi, int actk, double h, double pre, double xv,
                                            double sv) {
  const double v = act_fwd(actk, pre);
  const double adv = __dadd_rn(xv, __dmul_rn(h, v));
  return epi == E_ADV ? adv : __dadd_rn(sv, adv);
}

template <class T, bool AK, bool BKM, bool ASC>
__global__ void __launch_bounds__(T::WM* T::WN * 32)
    serial_gemm(const StepArgs a) {
  namespace cg = cooperative_groups;
  using C = GemmCfg<T, AK, BKM, ASC>;
  constexpr int BM = C::BM, BN = C::BN, BK = C::BK, WN = C::WN, STAGES = C::STAGES;
  extern __shared__ __align__(16) double smem[];
  cg::cluster_group cluster = cg::this_cluster();
  const int KS = gridDim.z, rank = blockIdx.z;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WN, wn = warp % WN;
  const int n0 = blockIdx.x * BN, m0 = blockIdx.y * BM;
  const int KT = a.K / BK / KS, kt0 = rank * KT;

  double acc[C::MT][C::NTF][2];
#pragma unroll
  for (int i = 0; i < C::MT; ++i)
#pragma unroll
    for (int j = 0; j < C::NTF; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  Loader<AK, BM, BK, 2, C::NTHREADS> la, ld_;
  Loader<BKM, BN, BK, 2, C::NTHREADS> lb;
  la.init(a.A, a.lda, m0, a.M, tid);
  lb.init(a.Bm, a.ldb, n0, a.N, tid);
  if (ASC) ld_.init(a.Ds, a.lda, m0, a.M, tid);
  la.init_full();
  lb.init_full();
  if (ASC) ld_.init_full();
#pragma unroll
  for (int i = 0; i < la.IT; ++i) la.cur[i] += kt0 * la.kadv;
#pragma unroll
  for (int i = 0; i < lb.IT; ++i) lb.cur[i] += kt0 * lb.kadv;
  if (ASC) {
#pragma unroll
    for (int i = 0; i < ld_.IT; ++i) ld_.cur[i] += kt0 * ld_.kadv;
  }
  auto load_stage = [&](int s) {
    double* base = smem + s * C::STAGE;
    la.load_next(base);
    if (ASC) ld_.load_next(base + C::A_SZ);
    lb.load_next(base + C::B_OFF);
  };
  // programmatic dependent launch (as step_gemm): the weight stages of this CTA's K slice do not
  // depend on the previous serial step, so they are fetched before griddepcontrol.wait; the state
  // (A), the scales and every epilogue operand are read, and everything is written, after it
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s)
    if (s < KT) lb.load_next(smem + s * C::STAGE + C::B_OFF);
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) {
      double* base = smem + s * C::STAGE;
      la.load_next(base);
      if (ASC) ld_.load_next(base + C::A_SZ);
    }
    cp_commit();  // group 0 also carries the prefetched weight stages
  }
  const int wm0 = wm * C::WTM, wn0 = wn * C::WTN;
  const int fr = lane >> 2, fk = lane & 3;
  constexpr int LDA_ = TileShape<AK, BM, BK>::LD, LDB_ = TileShape<BKM, BN, BK>::LD;
  const int a_thr = AK ? (wm0 + fr) * LDA_ + fk : fk * LDA_ + wm0 + fr;
  const int b_thr = BKM ? (wn0 + fr) * LDB_ + fk : fk * LDB_ + wn0 + fr;
  for (int kt = 0; kt < KT; ++kt) {
    cp_wait<STAGES - 2>();
    if (ASC) {
      double* st0 = smem + (kt % STAGES) * C::STAGE;
      la.scale_own(st0, st0 + C::A_SZ);
    }
    __syncthreads();
    if (kt + STAGES - 1 < KT) load_stage((kt + STAGES - 1) % STAGES);
    cp_commit();
    const double* As = smem + (kt % STAGES) * C::STAGE;
    const double* Bs = As + C::B_OFF;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[C::MT], bf[C::NTF];
#pragma unroll
      for (int i = 0; i < C::MT; ++i) {
        const int o = a_thr + (AK ? i * 8 * LDA_ + kk : kk * LDA_ + i * 8);
        af[i] = As[o];  // scaled in place (scale_own)
      }
#pragma unroll
      for (int j = 0; j < C::NTF; ++j) bf[j] = Bs[b_thr + (BKM ? j * 8 * LDB_ + kk : kk * LDB_ + j * 8)];
#pragma unroll
      for (int i = 0; i < C::MT; ++i)
#pragma unroll
        for (int j = 0; j < C::NTF; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_wait<0>();
  __syncthreads();
  // partial tile -> own smem [BM][BN]
  double* part = smem;
#pragma unroll
  for (int i = 0; i < C::MT; ++i)
#pragma unroll
    for (int j = 0; j < C::NTF; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e)
        part[(wm0 + i * 8 + fr) * BN + wn0 + j * 8 + 2 * fk + e] = acc[i][j][e];
  cluster.sync();
  // reduce a 1/KS share of the tile over the cluster in rank order, then the epilogue
  const int per = (BM * BN + KS - 1) / KS;
  const int e0 = rank * per, e1 = min(BM * BN, e0 + per);
  const double* X = a.x;
  const double* S = a.s;
  for (int e = e0 + tid; e < e1; e += C::NTHREADS) {
    double sum = 0.0;
    for (int r = 0; r < KS; ++r) sum += cluster.map_shared_rank(part, r)[e];
    const int m = m0 + e / BN, n = n0 + e % BN;
    const int64_t idx = (int64_t)m * a.ldc + n;
    double pre = sum;
    if (a.bias) pre = __dadd_rn(pre, a.bias[n]);
    a.out[idx] = epi_point(a.epi, a.act, a.h, pre, X[idx], S ? S[idx] : 0.0);
  }
  cluster.sync();
}

}  // namespace lmg

// lmg_conv.cuh -- 3x3, zero-pad-1, stride-1 convolution residual blocks (kernels.py:110-188) as
// implicit FP64 DMMA GEMMs on the reference's CHW raster layout, sm_100a.
//
// State rows are (B, q) with q = C*H*W, sample b's raster u[b][c][y][x] contiguous (CHW).  Weights
// are HWIO (k, k, C_in, C_out) flattened: W[((dy*3+dx)*C + ci)*C + co].  The reduction index is
// ordered tap-major, k = tap*C + ch (tap = dy*3 + dx), so a BK-wide k-tile (BK | C) has one tap.
//
//   FWD   (step E_PROP/E_RESID/...): m = (b, pix) [B*HW], n = co [C], k = (tap, ci) [9C]
//         A(m,k) = u[b][ci][y+dy-1][x+dx-1] (0 outside)      B(k,n) = W[k*C + n]  (MN-major)
//   ADJ   (transposed conv of gp = mu * act'):  m = (b, pix), n = ci, k = (tap, co)
//         A(m,k) = (mu*D)[b][co][y+1-dy][x+1-dx]               B(k,n) = W[(tap*C + n)*C + co]
//   PGRAD (weight gradient):  m = (tap, ci) [9C], n = co [C], k = (b, pix) [B*HW]
//         A(m,k) = u[b][ci][y+dy-1][x+dx-1]                     B(k,n) = (lam*D)[b][n][pix]
//
// Tiles never straddle samples (BM | HW for FWD/ADJ, BK | HW for PGRAD), so a CTA's output rows
// belong to one sample and the residual partial sums stay per sample.
#pragma once

#include "lmg_gemm.cuh"

namespace lmg {

enum ConvVariant { CV_FWD = 0, CV_ADJ = 1, CV_PGRAD = 2 };

// Logical padding: channels to Cp (a multiple of 32) and each sample's pixel range to HWp (a
// multiple of the M tile), with zero-filled loads and masked stores -- nothing is padded in
// memory, every k-tile has one tap and no tile straddles two samples.
struct ConvGeom {
  int C, Cp, H, W, HW, HWp;
  int64_t q;
};

template <int BM_, int BN_, int BK_, int WM_, int WN_, int STAGES_, bool SCALE_ONCE_ = false,
          bool RS_ = false, bool PRE_ = false>
struct ConvTile {
  // adjoint with a pre-scaled A operand (lambda * act' computed by a separate pass): one raster
  // tile per stage, no scaling in the kernel
  static constexpr bool PRE = PRE_;
  static constexpr int BM = BM_, BN = BN_, BK = BK_, WM = WM_, WN = WN_, STAGES = STAGES_;
  // adjoint: act' applied once per staged element by the thread that copied it (as step_gemm's
  // scale_own) instead of to every fragment at use
  static constexpr bool SCALE_ONCE = SCALE_ONCE_;
  // adjoint, register-staged (as step_gemm's TileR): each thread gathers its lambda and act'
  // elements of the NEXT k-tile into registers while this k-tile's DMMAs run and stores their
  // product into the A stage (act' never enters shared memory; 2 stages)
  static constexpr bool RS = RS_;
  static constexpr int NT = WM * WN * 32;
  static constexpr int LDA = BM + 4;  // A tiles are stored [k][m] (m contiguous)
  static constexpr int LDB_MN = BN + 4;
  static constexpr int LDB_K = BK + 4;
};

// Loads of the shifted raster tile A[kk][mm] for k-tile (tap, ch0) and pixel tile starting at
// pixel p0 of sample b: value x[b][ch0+kk][y+sy][x+sx] with (sy, sx) the tap's shift.  With NT a
// multiple of BM every element a thread loads has the same pixel mm = tid % BM, so its (y, x) are
// computed once per CTA (RasterPix) instead of two integer divisions per element per stage.
struct RasterPix {
  int y, x;
  bool in;  // pixel inside the image (pixel tiles are padded to HWp)
};

template <class T>
__device__ __forceinline__ RasterPix raster_pix(const ConvGeom& g, int p0, int tid) {
  static_assert(T::NT % T::BM == 0, "one pixel per thread");
  const int pix = p0 + tid % T::BM;
  return RasterPix{pix / g.W, pix % g.W, pix < g.HW};
}

template <class T>
__device__ __forceinline__ void conv_load_raster(double* sm, const double* x, const ConvGeom& g,
                                                 int b, const RasterPix& rp, int ch0, int sy, int sx,
                                                 int tid) {
  constexpr int NE = T::BK * T::BM;
  const double* xb = x + (int64_t)b * g.q;
  const int yy = rp.y + sy, xx = rp.x + sx;
  const bool pix_ok = rp.in && yy >= 0 && yy < g.H && xx >= 0 && xx < g.W;
  const int mm = tid % T::BM;
  const double* base = xb + yy * g.W + xx;
#pragma unroll
  for (int e = tid; e < NE; e += T::NT) {
    const int kk = e / T::BM;
    const bool ok = pix_ok && (ch0 + kk < g.C);
    const double* src = ok ? base + (int64_t)(ch0 + kk) * g.HW : x;
    cp_async<1>(sm + kk * T::LDA + mm, src, ok);
  }
}

// per-element variant (recomputes the pixel each stage): used by the adjoint, where keeping the
// hoisted coordinates live made ptxas spill (2.05 vs 1.95 ms per c3 sweep launch)
template <class T>
__device__ __forceinline__ void conv_load_raster_idx(double* sm, const double* x, const ConvGeom& g,
                                                     int b, int p0, int ch0, int sy, int sx, int tid) {
  constexpr int NE = T::BK * T::BM;
  const double* xb = x + (int64_t)b * g.q;
#pragma unroll
  for (int e = tid; e < NE; e += T::NT) {
    const int kk = e / T::BM, mm = e % T::BM;
    const int pix = p0 + mm;
    const int yy = pix / g.W + sy, xx = pix % g.W + sx;
    const bool ok = (pix < g.HW) && (ch0 + kk < g.C) && (yy >= 0) && (yy < g.H) && (xx >= 0) &&
                    (xx < g.W);
    const double* src = ok ? xb + (int64_t)(ch0 + kk) * g.HW + yy * g.W + xx : x;
    cp_async<1>(sm + kk * T::LDA + mm, src, ok);
  }
}

// PGRAD B tile: gp rows [kk = pixel][nn = co] from raster (lam or D) of sample b, pixels p0..,
// stored [k][n] (n contiguous).  Global reads are contiguous along pixels (k), so each thread
// copies single doubles.
template <class T>
__device__ __forceinline__ void conv_load_gp(double* sm, const double* x, const ConvGeom& g, int b,
                                             int p0, int n0, int tid) {
  constexpr int NE = T::BK * T::BN;
  const double* xb = x + (int64_t)b * g.q;
#pragma unroll
  for (int e = tid; e < NE; e += T::NT) {
    const int nn = e / T::BK, kk = e % T::BK;
    const bool ok = (n0 + nn) < g.C && (p0 + kk) < g.HW;
    const double* src = ok ? xb + (int64_t)(n0 + nn) * g.HW + p0 + kk : x;
    cp_async<1>(sm + kk * T::LDB_MN + nn, src, ok);
  }
}

template <class T, int V>
__global__ void __launch_bounds__(T::NT) conv_gemm(const StepArgs a, const ConvGeom g) {
  constexpr int BM = T::BM, BN = T::BN, BK = T::BK, WN = T::WN, STAGES = T::STAGES;
  constexpr int WTM = BM / T::WM, WTN = BN / WN, MT = WTM / 8, NTF = WTN / 8;
  constexpr bool ASC = (V != CV_FWD);
  // smem per stage: A [BK][BM+4] (+ scale tile for ADJ), B [BK][BN+4] (FWD, PGRAD) or
  // [BN][BK+4] (ADJ, K-major); PGRAD's B also needs a scale tile
  constexpr int A_SZ = BK * T::LDA;
  constexpr int B_SZ = (V == CV_ADJ) ? BN * T::LDB_K : BK * T::LDB_MN;
  constexpr bool RS = (V == CV_ADJ) && T::RS;
  constexpr bool PRE = (V == CV_ADJ) && T::PRE;
  static_assert(!RS || STAGES == 2, "register staging: 2 stages");
  constexpr int STAGE = A_SZ * ((V == CV_ADJ && !RS && !PRE) ? 2 : 1) + B_SZ * (V == CV_PGRAD ? 2 : 1);
  extern __shared__ __align__(16) double smem[];
  __shared__ double red[T::NT / 32];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WN, wn = warp % WN;
  const int n0 = blockIdx.x * BN, m0 = blockIdx.y * BM;
  const int64_t t = blockIdx.z;

  const double* A = a.A + t * a.A_ts;
  const double* Ds = ASC ? a.Ds + t * a.Ds_ts : nullptr;
  const double* Bm = a.Bm + t * a.B_ts;

  // FWD/ADJ: the CTA's pixels belong to sample b0
  const int b0 = (V == CV_PGRAD) ? 0 : m0 / g.HWp;
  const int p0 = (V == CV_PGRAD) ? 0 : m0 % g.HWp;

  double acc[MT][NTF][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NTF; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int KT = a.K / BK;  // host guarantees BK | K
  const RasterPix rpix = raster_pix<T>(g, p0, tid);
  auto load_stage = [&](int s, int kt) {
    double* base = smem + s * STAGE;
    const int k0 = kt * BK;
    if (V == CV_FWD || V == CV_ADJ) {
      const int tap = k0 / g.Cp, ch0 = k0 % g.Cp;
      const int dy = tap / 3, dx = tap % 3;
      const int sy = (V == CV_FWD) ? dy - 1 : 1 - dy, sx = (V == CV_FWD) ? dx - 1 : 1 - dx;
      if (V == CV_ADJ) {
        if (PRE) {  // A is lambda * act' already
          conv_load_raster_idx<T>(base, A, g, b0, p0, ch0, sy, sx, tid);
        } else if (!RS) {  // RS: the A stage is written from registers (rs_gather / rs_store)
          conv_load_raster_idx<T>(base, A, g, b0, p0, ch0, sy, sx, tid);
          conv_load_raster_idx<T>(base + A_SZ, Ds, g, b0, p0, ch0, sy, sx, tid);
        }
      } else {
        conv_load_raster<T>(base, A, g, b0, rpix, ch0, sy, sx, tid);
      }
      double* bs = base + A_SZ * ((V == CV_ADJ && !RS && !PRE) ? 2 : 1);
      // weight rows are contiguous: 16-byte vectors when C is even (pairs never straddle the
      // channel bound and stay 16B-aligned); the padded smem rows keep 16B alignment
      const bool vec = (g.C & 1) == 0 && (reinterpret_cast<uintptr_t>(Bm) & 15) == 0;
      if (V == CV_FWD) {  // B(k,n) = W[k*C + n]: rows k contiguous in n
        if (vec) {
#pragma unroll
          for (int e = tid; e < BK * BN / 2; e += T::NT) {
            const int kk = e / (BN / 2), nn = (e % (BN / 2)) * 2;
            const bool ok = (n0 + nn) < g.C && (ch0 + kk) < g.C;
            const double* src = Bm + ((int64_t)tap * g.C + ch0 + kk) * g.C + n0 + nn;
            cp_async<2>(bs + kk * T::LDB_MN + nn, ok ? src : Bm, ok);
          }
        } else {
#pragma unroll
          for (int e = tid; e < BK * BN; e += T::NT) {
            const int kk = e / BN, nn = e % BN;
            const bool ok = (n0 + nn) < g.C && (ch0 + kk) < g.C;
            const double* src = Bm + ((int64_t)tap * g.C + ch0 + kk) * g.C + n0 + nn;
            cp_async<1>(bs + kk * T::LDB_MN + nn, ok ? src : Bm, ok);
          }
        }
      } else {  // B(k,n) = W[(tap*C + n)*C + co], co = ch0 + kk: stored [n][k]
        if (vec) {
#pragma unroll
          for (int e = tid; e < BK * BN / 2; e += T::NT) {
            const int nn = e / (BK / 2), kk = (e % (BK / 2)) * 2;
            const bool ok = (n0 + nn) < g.C && (ch0 + kk) < g.C;
            const double* src = Bm + ((int64_t)tap * g.C + n0 + nn) * g.C + ch0 + kk;
            cp_async<2>(bs + nn * T::LDB_K + kk, ok ? src : Bm, ok);
          }
        } else {
#pragma unroll
          for (int e = tid; e < BK * BN; e += T::NT) {
            const int nn = e / BK, kk = e % BK;
            const bool ok = (n0 + nn) < g.C && (ch0 + kk) < g.C;
            const double* src = Bm + ((int64_t)tap * g.C + n0 + nn) * g.C + ch0 + kk;
            cp_async<1>(bs + nn * T::LDB_K + kk, ok ? src : Bm, ok);
          }
        }
      }
    } else {  // PGRAD: k-tile = pixels [pk, pk+BK) of sample kb; m rows = (tap, ci)
      const int kb = k0 / g.HWp, pk = k0 % g.HWp;
      // A[kk][mm]: m = tap*Cp + ci over the tile's rows; one tap per m-tile (BM | Cp)
      const int tap = m0 / g.Cp, ci0 = m0 % g.Cp;
      const int dy = tap / 3, dx = tap % 3;
      const double* xb = A + (int64_t)kb * g.q;
#pragma unroll
      for (int e = tid; e < BK * BM; e += T::NT) {
        const int mm = e / BK, kk = e % BK;
        const int pix = pk + kk;
        const int yy = pix / g.W + dy - 1, xx = pix % g.W + dx - 1;
        const bool ok = (pix < g.HW) && (ci0 + mm < g.C) && (yy >= 0) && (yy < g.H) && (xx >= 0) &&
                        (xx < g.W);
        const double* src = ok ? xb + (int64_t)(ci0 + mm) * g.HW + yy * g.W + xx : A;
        cp_async<1>(base + kk * T::LDA + mm, src, ok);
      }
      conv_load_gp<T>(base + A_SZ, Bm, g, kb, pk, n0, tid);
      conv_load_gp<T>(base + A_SZ + B_SZ, Ds, g, kb, pk, n0, tid);
    }
  };

  // register-staged adjoint A: this thread's elements e = tid + i*NT of a k-tile
  constexpr int EPT = (BK * BM + T::NT - 1) / T::NT;
  double ra[RS ? EPT : 1], rd[RS ? EPT : 1];
  auto rs_gather = [&](int kt) {
    const int k0 = kt * BK;
    const int tap = k0 / g.Cp, ch0 = k0 % g.Cp;
    const int sy = 1 - tap / 3, sx = 1 - tap % 3;
    const double* xb = A + (int64_t)b0 * g.q;
    const double* db = Ds + (int64_t)b0 * g.q;
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
      const int e = tid + i * T::NT;
      const int kk = e / BM, mm = e % BM;
      const int pix = p0 + mm;
      const int yy = pix / g.W + sy, xx = pix % g.W + sx;
      const bool ok = e < BK * BM && (pix < g.HW) && (ch0 + kk < g.C) && (yy >= 0) && (yy < g.H) &&
                      (xx >= 0) && (xx < g.W);
      const int64_t o = (int64_t)(ch0 + kk) * g.HW + yy * g.W + xx;
      ra[i] = ok ? xb[o] : 0.0;
      rd[i] = ok ? db[o] : 0.0;
    }
  };
  auto rs_store = [&](double* as) {
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
      const int e = tid + i * T::NT;
      if (e < BK * BM) as[(e / BM) * T::LDA + e % BM] = __dmul_rn(ra[i], rd[i]);
    }
  };
  if constexpr (RS) {
    rs_gather(0);
    rs_store(smem);
    load_stage(0, 0);  // the weight tile of k-tile 0
    cp_commit();
    if (KT > 1) rs_gather(1);
  } else {
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
      if (s < KT) load_stage(s, s);
      cp_commit();
    }
  }
  const int wm0 = wm * WTM, wn0 = wn * WTN;
  const int fr = lane >> 2, fk = lane & 3;
  for (int kt = 0; kt < KT; ++kt) {
    cp_wait<STAGES - 2>();
    if constexpr (V == CV_ADJ && T::SCALE_ONCE) {
      // this thread's own elements of stage kt (conv_load_raster_idx's e -> (kk, mm) mapping)
      double* as = smem + (kt % STAGES) * STAGE;
#pragma unroll
      for (int e = tid; e < BK * BM; e += T::NT) {
        const int o = (e / BM) * T::LDA + e % BM;
        as[o] = __dmul_rn(as[o], as[A_SZ + o]);
      }
    }
    __syncthreads();
    {
      const int nk = kt + STAGES - 1;
      if (nk < KT) load_stage(nk % STAGES, nk);
      cp_commit();
    }
    const double* As = smem + (kt % STAGES) * STAGE;
    const double* Asc = As + A_SZ;
    const double* Bs = As + A_SZ * ((V == CV_ADJ && !RS && !PRE) ? 2 : 1);
    const double* Bsc = Bs + B_SZ;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[MT], bf[NTF];
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        const int mm = wm0 + i * 8 + fr, k = kk + fk;
        af[i] = As[k * T::LDA + mm];
        if (V == CV_ADJ && !T::SCALE_ONCE && !RS && !PRE) af[i] = __dmul_rn(af[i], Asc[k * T::LDA + mm]);
      }
#pragma unroll
      for (int j = 0; j < NTF; ++j) {
        const int nn = wn0 + j * 8 + fr, k = kk + fk;
        if (V == CV_ADJ) {
          bf[j] = Bs[nn * T::LDB_K + k];
        } else {
          bf[j] = Bs[k * T::LDB_MN + nn];
          if (V == CV_PGRAD) bf[j] = __dmul_rn(bf[j], Bsc[k * T::LDB_MN + nn]);
        }
      }
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NTF; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    if constexpr (RS) {
      if (kt + 1 < KT) {  // stage kt+1's buffer was last read in iteration kt-1 (barrier passed)
        rs_store(smem + ((kt + 1) % STAGES) * STAGE);
        if (kt + 2 < KT) rs_gather(kt + 2);
      }
    }
  }
  cp_wait<0>();

  // ------------------------------------------------------------------ epilogue
  const int epi = a.epi, actk = a.act;
  const double h = a.h;
  const double* bias = a.bias ? a.bias + t * a.bias_ts : nullptr;
  const double* X = a.x ? a.x + t * a.x_ts : nullptr;
  const double* S = a.s ? a.s + t * a.s_ts : nullptr;
  const double* Y = a.y ? a.y + t * a.y_ts : nullptr;
  const double* P = a.p ? a.p + t * a.p_ts : nullptr;
  double* O = a.out ? a.out + t * a.out_ts : nullptr;
  double* O2 = a.out2 ? a.out2 + t * a.out2_ts : nullptr;
  double sq = 0.0;
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    const int m = m0 + wm0 + i * 8 + fr;
    if (m >= a.M) continue;
#pragma unroll
    for (int j = 0; j < NTF; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int n = n0 + wn0 + j * 8 + 2 * fk + e;
        if (n >= a.N) continue;
        const double accv = acc[i][j][e];
        if (V == CV_PGRAD) {  // gW[(tap*C + ci)*C + co] (HWIO); m = tap*Cp + ci
          const int tp = m / g.Cp, ci = m % g.Cp;
          if (ci >= g.C) continue;
          const int64_t idx = ((int64_t)tp * g.C + ci) * g.C + n;
          double gg = __dmul_rn(__dmul_rn(accv, h), a.scale);
          if (a.accum && O2) gg = __dadd_rn(O2[idx], gg);
          if (O2) O2[idx] = gg;
          if (a.lr != 0.0) O[idx] = __dadd_rn(X[idx], -__dmul_rn(a.lr, gg));
          continue;
        }
        // CHW raster index of (sample b0, channel n, pixel m - b0*HWp)
        const int pix = m - b0 * g.HWp;
        if (pix >= g.HW) continue;
        const int64_t idx = (int64_t)b0 * g.q + (int64_t)n * g.HW + pix;
        double pre = accv;
        if (bias) pre = __dadd_rn(pre, bias[n]);
        if (epi == E_DERIV) {
          O[idx] = act_der(actk, pre);
          continue;
        }
        const double v = act_fwd(actk, pre);
        if (epi == E_APPLY) {
          O[idx] = v;
          continue;
        }
        const double adv = __dadd_rn(X[idx], __dmul_rn(h, v));
        if (epi == E_ADV) {
          O[idx] = adv;
        } else if (epi == E_PROP) {
          O[idx] = __dadd_rn(S ? S[idx] : 0.0, adv);
          if (O2) O2[idx] = __dadd_rn(X[idx], __dmul_rn(a.h2, v));
        } else if (epi == E_RESID) {
          const double prop = __dadd_rn(S ? S[idx] : 0.0, adv);
          const double r = __dadd_rn(prop, -Y[idx]);
          if (O) O[idx] = r;
          if (O2) O2[idx] = prop;
          sq = fma(r, r, sq);
        } else if (epi == E_COARSE) {
          const double yv = Y[idx];
          O[idx] = __dadd_rn(__dadd_rn(yv, -adv), __dadd_rn(P[idx], -yv));
          if (O2) O2[idx] = yv;
        } else if (epi == E_COARSE_R) {
          O[idx] = __dadd_rn(__dadd_rn(Y[idx], -adv), P[idx]);
        } else {  // E_PROPOP
          O[idx] = __dadd_rn(Y[idx], -adv);
        }
      }
    }
  }
  if (V != CV_PGRAD && epi == E_RESID && a.part) {
    // one partial per CTA (its tile lies in sample b0), fixed-order reduction
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, off);
    if (lane == 0) red[warp] = sq;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int w = 0; w < T::NT / 32; ++w) s += red[w];
      const int mt_in_sample = p0 / BM;
      const int64_t slot = a.part_slot0 + t * ((int64_t)(g.HWp / BM) * gridDim.x) +
                           (int64_t)mt_in_sample * gridDim.x + blockIdx.x;
      a.part[slot * a.part_ld + b0] = s;
    }
  }
}

}  // namespace lmg

// lmg.cu -- C-ABI + stream-ordered orchestration of the layer-parallel FAS solver (sm_100a).
//
// Every reference numeric routine on the hot path maps onto launches of one FP64-DMMA step
// kernel (lmg_gemm.cuh) with a fused epilogue, plus a few HBM-bound elementwise kernels:
//
//   fused FCF sweep        multigrid.py:160-172   2c launches, each one step of every block
//   C-row residual (P)     multigrid.py:208       1 extra step of the same sweep
//   coarse source + inject multigrid.py:209-212   1 launch (E_COARSE) + row 0
//   coarsest solve         multigrid.py:214-215   n_coarse-1 single-task launches
//   correction             multigrid.py:227       1 elementwise launch
//   post-correction norm   multigrid.py:228       2 launches on rows {kc, kc+1} + reduction
//
// Residual rows that are algebraically zero (F rows after FCF; all but {kc, kc+1} after the
// correction) are exactly 0.0 in the reference because the same propagate_values recomputes
// them (multigrid.py:118-119); they are skipped here and contribute exactly 0.

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <type_traits>
#include <vector>

#include "lmg.h"
#include "lmg_chain.cuh"
#include "lmg_conv.cuh"
#include "lmg_sweep.cuh"
#include "lmg_tgemm.cuh"

namespace lmg {
std::atomic<int> g_canonical{0};  // lmg_set_canonical_order
bool canonical_order() { return g_canonical.load(std::memory_order_relaxed) != 0; }
}  // namespace lmg

using namespace lmg;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& m) {
  g_err = m;
  return code;
}

#define CUDA_TRY(x)                                                              \
  do {                                                                           \
    cudaError_t e_ = (x);                                                        \
    if (e_ != cudaSuccess)                                                       \
      return fail(LMG_ERR_CUDA, std::string(#x ": ") + cudaGetErrorString(e_)); \
  } while (0)

#define TRY(x)                  \
  do {                          \
    int r_ = (x);               \
    if (r_ != LMG_OK) return r_; \
  } while (0)

inline cudaStream_t S_(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ------------------------------------------------------------------------------------------
// elementwise kernels (HBM-bound; grid-stride, 2 doubles per thread-iteration where possible)
//
// Programmatic dependent launch: each elementwise kernel waits for its upstream grid first and
// then lets its own dependents launch, so in the latency-bound regime (a cycle of ~a dozen tiny
// launches, c1 / c6) the next launch overlaps this one instead of following its drain.  Waiting
// before triggering keeps the chain transitive: a dependent's pre-wait prologue (the step
// kernels' W prefetch) only ever overlaps a kernel whose own upstream work is complete.
// griddepcontrol.wait is a no-op for a kernel launched without the attribute.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__global__ void k_copy_rows(double* __restrict__ dst, int64_t dst_ts, const double* __restrict__ src,
                            int64_t src_ts, int64_t nrows, int64_t len) {
  pdl_enter();
  const int64_t total = nrows * len;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = e / len, i = e - r * len;
    dst[r * dst_ts + i] = src[r * src_ts + i];
  }
}

// out[t][e] = a[t][e] * d[t][e] for the rows of every task (the conv adjoint's lambda * act'
// operand, computed once instead of per gathered raster tile); len even, 16-byte aligned rows
__global__ void k_prescale(double* __restrict__ out, const double* __restrict__ a, int64_t a_ts,
                           const double* __restrict__ d, int64_t d_ts, int64_t ntasks, int64_t len) {
  pdl_enter();
  const int64_t half = len / 2, total = ntasks * half;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = e / half, i = 2 * (e - t * half);
    const double2 x = *reinterpret_cast<const double2*>(a + t * a_ts + i);
    const double2 y = *reinterpret_cast<const double2*>(d + t * d_ts + i);
    double2 r;
    r.x = __dmul_rn(x.x, y.x);
    r.y = __dmul_rn(x.y, y.y);
    *reinterpret_cast<double2*>(out + t * len + i) = r;
  }
}

// multigrid.py:227  states[::c] += solved - coarse_states   (coarse_states == states[::c] bitwise)
__global__ void k_correct(double* __restrict__ U, int64_t u_ts, const double* __restrict__ V,
                          int64_t v_ts, int64_t nrows, int64_t len) {
  pdl_enter();
  const int64_t total = nrows * len;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = e / len, i = e - r * len;
    double u = U[r * u_ts + i];
    U[r * u_ts + i] = __dadd_rn(u, __dadd_rn(V[r * v_ts + i], -u));
  }
}

__global__ void k_add(double* __restrict__ out, const double* __restrict__ a,
                      const double* __restrict__ b, int64_t len) {
  pdl_enter();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __dadd_rn(a[i], b[i]);
}

// row 0 of the coarse source: S_H[0] = U_H[0] + (f[0] - U[0])  (propagation_operator row 0 +
// residual row 0, multigrid.py:124,142); optionally V[0] = U[0] (the copy the recursion edits)
__global__ void k_row0_coarse(const double* __restrict__ U0, const double* __restrict__ S0,
                              double* __restrict__ SH0, double* __restrict__ V0, int64_t len) {
  pdl_enter();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len;
       i += (int64_t)gridDim.x * blockDim.x) {
    double u = U0[i];
    SH0[i] = __dadd_rn(u, __dadd_rn(S0[i], -u));
    if (V0) V0[i] = u;
  }
}

// residual row 0: r = f[0] - u[0] (multigrid.py:124) + per-sample partial sum of squares
__global__ void k_resid_row0(const double* __restrict__ S0, const double* __restrict__ U0,
                             double* __restrict__ R0, double* __restrict__ part, int64_t slot,
                             int B, int q) {
  pdl_enter();
  __shared__ double sh[256];
  const int b = blockIdx.x;
  double acc = 0.0;
  for (int i = threadIdx.x; i < q; i += blockDim.x) {
    int64_t idx = (int64_t)b * q + i;
    double r = U0 ? __dadd_rn(S0[idx], -U0[idx]) : S0[idx];
    if (R0) R0[idx] = r;
    acc = fma(r, r, acc);
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0 && part) part[slot * B + b] = sh[0];
}

// Residual of a non-first rank's row 0 (its source row finished with the halo, minus U[0]) summed
// exactly as the step GEMM's E_RESID epilogue sums that row on one GPU, where it is an interior
// row: per 32-column tile (TSmall/TTiny: two 16-column warps, lanes fk = 0..3 each holding
// columns 2fk + {0, 1} and 8 + 2fk + {0, 1} fma-accumulated in that order, then a shfl-xor 1 / 2
// tree, then the warps in order), tiles summed in order -- so the block partials, and the norms,
// are bitwise the single-GPU ones whatever the partition (a tree over the row differs in the last
// bit).  Dense systems (the partitioned path is dense-only).  One thread per sample.
__global__ void k_resid_row0_tiles(const double* __restrict__ S0, const double* __restrict__ U0,
                                   double* __restrict__ part, int B, int q) {
  pdl_enter();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const double* s = S0 + (int64_t)b * q;
  const double* u = U0 + (int64_t)b * q;
  double rs = 0.0;
  for (int t0 = 0; t0 < q; t0 += 32) {
    double tile = 0.0;
    for (int wn = 0; wn < 2; ++wn) {
      double v[4];
      for (int fk = 0; fk < 4; ++fk) {
        double acc = 0.0;
        for (int j = 0; j < 2; ++j)
          for (int e = 0; e < 2; ++e) {
            const int n = t0 + wn * 16 + 2 * fk + j * 8 + e;
            if (n < q) {
              const double r = __dadd_rn(s[n], -u[n]);
              acc = fma(r, r, acc);
            }
          }
        v[fk] = acc;
      }
      tile += (v[0] + v[1]) + (v[2] + v[3]);
    }
    rs += tile;
  }
  part[b] = rs;
}

// norms[b] = sqrt(sum over slots, in slot order) -- deterministic for any launch geometry.  One
// warp per sample: the lanes fetch a chunk of 256 slots at once into shared memory (one memory
// latency per chunk instead of a dependent load per slot), then lane 0 adds them in slot order.
constexpr int kNormChunk = 256;
__global__ void k_reduce_norms(const double* __restrict__ part, int64_t nslots, int B,
                               double* __restrict__ norms) {
  pdl_enter();
  __shared__ double buf[4][kNormChunk];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x * 4 + w;
  if (b >= B) return;  // whole warps
  double s = 0.0;
  for (int64_t k0 = 0; k0 < nslots; k0 += kNormChunk) {
    const int n = nslots - k0 < kNormChunk ? (int)(nslots - k0) : kNormChunk;
#pragma unroll
    for (int i = 0; i < kNormChunk / 32; ++i) {
      const int kk = lane + 32 * i;
      if (kk < n) buf[w][kk] = part[(k0 + kk) * B + b];
    }
    __syncwarp();
    if (lane == 0)
      for (int kk = 0; kk < n; ++kk) s += buf[w][kk];
    __syncwarp();
  }
  if (lane == 0) norms[b] = sqrt(s);
}

// bias gradient + SGD: gb_n[i] = (h * sum_b lam^{n+1}[b,i] D_n[b,i]) * scale ; b_n -= lr*gb_n
__global__ void k_bias_grads(const double* __restrict__ lam_top, int64_t lam_ts,
                             const double* __restrict__ D, int N, int B, int q, double h,
                             double scale, double lr, double* __restrict__ gb,
                             double* __restrict__ bias, int64_t b_stride, int accum = 0) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (int64_t)N * q) return;
  int n = (int)(e / q), i = (int)(e - (int64_t)n * q);
  const double* L = lam_top + (int64_t)n * lam_ts;
  const double* Dn = D + (int64_t)n * B * q;
  double s = 0.0;
  for (int b = 0; b < B; ++b) s += __dmul_rn(L[(int64_t)b * q + i], Dn[(int64_t)b * q + i]);
  double g = __dmul_rn(__dmul_rn(s, h), scale);
  if (accum && gb) g = __dadd_rn(gb[e], g);
  if (gb) gb[e] = g;
  if (lr != 0.0 && bias) {
    double* bp = bias + (int64_t)n * b_stride + i;
    *bp = __dadd_rn(*bp, -__dmul_rn(lr, g));
  }
}

// out = (s0 ? s0 : 0.0) + adv: finish a halo value received from the previous rank with this
// rank's own source row (network.py:100 `source[j] + (u + h*fv)`).
__global__ void k_halo_finish(const double* __restrict__ s0, const double* __restrict__ adv,
                              double* __restrict__ out, int64_t len) {
  pdl_enter();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __dadd_rn(s0 ? s0[i] : 0.0, adv[i]);
}

// device-side stopping test of the solve loop (multigrid.py:297-309 per sample): record this
// cycle's norms for the samples still running; keep looping (the enclosing conditional WHILE graph
// node) until some sample reaches tol or max_cycles -- the host then parks it and resumes
__global__ void k_cycle_book(const double* __restrict__ norms, int B, double tol,
                             const int* __restrict__ done, double* __restrict__ hist,
                             int* __restrict__ cyc, int max_cycles, cudaGraphConditionalHandle h) {
  __shared__ int any;
  if (threadIdx.x == 0) any = 0;
  __syncthreads();
  const int c = *cyc + 1;
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    if (done[b]) continue;
    hist[(int64_t)c * B + b] = norms[b];
    if (norms[b] <= tol) atomicOr(&any, 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    *cyc = c;
    cudaGraphSetConditional(h, (!any && c < max_cycles) ? 1u : 0u);
  }
}

// after a fused FCF sweep: U[0] = f[0] (c_relaxation, multigrid.py:157) and U[kc] = Cn[k], k >= 1
__global__ void k_fcf_commit(double* __restrict__ U, const double* __restrict__ src0,
                             const double* __restrict__ Cn, int nb, int c, int64_t BQ) {
  pdl_enter();
  const int64_t total = (int64_t)nb * BQ;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / BQ, i = e - r * BQ;
    if (r == 0 && !src0) continue;  // row 0 already finished from the incoming halo
    U[r * c * BQ + i] = r == 0 ? src0[i] : Cn[e];
  }
}

// k_fcf_commit + k_coarse_from_adv + k_row0_coarse in one pass (single GPU, first rank): the
// new C rows are committed and the coarse source assembled from them with the same operations
//   U[0] = f[0],  S_H[0] = U[0] + (f[0] - U[0]),  V[0] = U[0]
//   U[nc] = Cn[n], S_H[n] = (U[nc] - advH[n-1]) + (P[n] - U[nc]),  V[n] = U[nc]   (n >= 1)
__global__ void k_commit_coarse(double* __restrict__ U, const double* __restrict__ src0,
                                const double* __restrict__ Cn, const double* __restrict__ adv,
                                const double* __restrict__ P, double* __restrict__ SH,
                                double* __restrict__ V, int nb, int c, int64_t BQ) {
  pdl_enter();
  const int64_t total = (int64_t)nb * BQ;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / BQ, i = e - r * BQ;
    double y;
    if (r == 0) {
      y = src0[i];
      SH[i] = __dadd_rn(y, __dadd_rn(src0[i], -y));
    } else {
      y = Cn[e];
      SH[e] = __dadd_rn(__dadd_rn(y, -adv[e - BQ]), __dadd_rn(P[e], -y));
    }
    U[r * c * BQ + i] = y;
    if (V) V[e] = y;
  }
}

// coarse FAS source rows n >= 1 from the advance computed in the F sweep:
//   S_H[n] = (U[nc] - advH[n-1]) + (P[n] - U[nc]),  V[n] = U[nc]      (multigrid.py:142)
__global__ void k_coarse_from_adv(const double* __restrict__ Uc, int64_t u_ts,
                                  const double* __restrict__ adv, const double* __restrict__ P,
                                  double* __restrict__ SH, double* __restrict__ V, int64_t nrows,
                                  int64_t len) {
  pdl_enter();
  const int64_t total = nrows * len;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / len, i = e - r * len;
    const double y = Uc[r * u_ts + i];
    SH[e] = __dadd_rn(__dadd_rn(y, -adv[e]), __dadd_rn(P[e], -y));
    if (V) V[e] = y;
  }
}

// first coarse-source row of a non-first rank: S_H[0] = (U[0] - adv_in) + (P[0] - U[0]), where
// adv_in = U_prev + H*F(U_prev) came from the previous rank (multigrid.py:142, network.py:138)
__global__ void k_row0_coarse_halo(const double* __restrict__ U0, const double* __restrict__ adv,
                                   const double* __restrict__ P0, double* __restrict__ SH0,
                                   double* __restrict__ V0, int64_t len) {
  pdl_enter();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len;
       i += (int64_t)gridDim.x * blockDim.x) {
    double u = U0[i];
    SH0[i] = __dadd_rn(__dadd_rn(u, -adv[i]), __dadd_rn(P0[i], -u));
    if (V0) V0[i] = u;
  }
}

// C-row residual partials after the correction: block k, sample b:
//   r = (k == 0 && is_first) ? f[0] - U[0] : P[k] - U[kc]        (multigrid.py:124-127)
// one CTA per (k, b), fixed-order tree reduction -> cpart[k*B + b]
__global__ void k_cpart(const double* __restrict__ U, const double* __restrict__ P,
                        const double* __restrict__ S0, int is_first, int c, int B, int q,
                        double* __restrict__ cpart) {
  pdl_enter();
  __shared__ double sh[256];
  const int k = blockIdx.y, b = blockIdx.x;
  const int64_t BQ = (int64_t)B * q;
  const double* u = U + (int64_t)k * c * BQ + (int64_t)b * q;
  const double* p = (k == 0 && is_first) ? (S0 ? S0 + (int64_t)b * q : nullptr)
                                         : P + (int64_t)k * BQ + (int64_t)b * q;
  double acc = 0.0;
  for (int i = threadIdx.x; i < q; i += blockDim.x) {
    double r = __dadd_rn(p ? p[i] : 0.0, -u[i]);
    acc = fma(r, r, acc);
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) cpart[(int64_t)k * B + b] = sh[0];
}

// k_correct + k_cpart in one pass (the finest level of a single-GPU cycle): the correction
// U[kc] += V[k] - U[kc] (multigrid.py:227), then the C-row residual partial of the corrected row
// with k_cpart's summation order
__global__ void k_correct_cpart(double* __restrict__ U, const double* __restrict__ V,
                                const double* __restrict__ P, const double* __restrict__ S0,
                                int is_first, int c, int B, int q, double* __restrict__ cpart) {
  pdl_enter();
  __shared__ double sh[256];
  const int k = blockIdx.y, b = blockIdx.x;
  const int64_t BQ = (int64_t)B * q;
  double* u = U + (int64_t)k * c * BQ + (int64_t)b * q;
  const double* v = V + (int64_t)k * BQ + (int64_t)b * q;
  const double* p = (k == 0 && is_first) ? (S0 ? S0 + (int64_t)b * q : nullptr)
                                         : P + (int64_t)k * BQ + (int64_t)b * q;
  double acc = 0.0;
  for (int i = threadIdx.x; i < q; i += blockDim.x) {
    const double u0 = u[i];
    const double u1 = __dadd_rn(u0, __dadd_rn(v[i], -u0));
    u[i] = u1;
    double r = __dadd_rn(p ? p[i] : 0.0, -u1);
    acc = fma(r, r, acc);
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) cpart[(int64_t)k * B + b] = sh[0];
}

// block partials after the correction: block_part[k][b] = cpart[k][b] + sum_t fpart[k][t][b]
__global__ void k_combine_post(const double* __restrict__ cpart, const double* __restrict__ fpart,
                               int nb, int nt, int B, double* __restrict__ block_part) {
  pdl_enter();
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (int64_t)nb * B) return;
  int k = (int)(e / B), b = (int)(e - (int64_t)k * B);
  double s = cpart[e];
  for (int t = 0; t < nt; ++t) s += fpart[((int64_t)k * nt + t) * B + b];
  block_part[e] = s;
}

// block partials of a full residual: block k = sum over its c rows (row order), each row the sum
// of its tile partials; row 0 of the rank comes from r0part
__global__ void k_combine_full(const double* __restrict__ rpart, const double* __restrict__ r0part,
                               int nb, int c, int nt, int B, double* __restrict__ block_part) {
  pdl_enter();
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (int64_t)nb * B) return;
  int k = (int)(e / B), b = (int)(e - (int64_t)k * B);
  double s = 0.0;
  for (int j = k * c; j < (k + 1) * c; ++j) {
    if (j == 0) {
      s += r0part[b];
      continue;
    }
    double rs = 0.0;
    for (int t = 0; t < nt; ++t) rs += rpart[((int64_t)j * nt + t) * B + b];
    s += rs;
  }
  block_part[e] = s;
}

// conv bias gradient + SGD: gb_n[co] = (h * sum_{b,pix} lam^{n+1}[b][co][pix] D_n[b][co][pix])*scale
__global__ void k_conv_bias_grads(const double* __restrict__ lam_top, int64_t lam_ts,
                                  const double* __restrict__ D, int B, int C, int HW, double h,
                                  double scale, double lr, double* __restrict__ gb,
                                  double* __restrict__ bias, int64_t b_stride, int accum = 0) {
  __shared__ double sh[256];
  const int co = blockIdx.x, n = blockIdx.y;
  const int64_t q = (int64_t)C * HW;
  const double* L = lam_top + (int64_t)n * lam_ts;
  const double* Dn = D + (int64_t)n * B * q;
  double s = 0.0;
  for (int64_t e = threadIdx.x; e < (int64_t)B * HW; e += blockDim.x) {
    const int64_t b = e / HW, p = e - b * HW;
    const int64_t idx = b * q + (int64_t)co * HW + p;
    s += __dmul_rn(L[idx], Dn[idx]);
  }
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int k = blockDim.x / 2; k > 0; k >>= 1) {
    if (threadIdx.x < k) sh[threadIdx.x] += sh[threadIdx.x + k];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double g = __dmul_rn(__dmul_rn(sh[0], h), scale);
    if (accum && gb) g = __dadd_rn(gb[(int64_t)n * C + co], g);
    if (gb) gb[(int64_t)n * C + co] = g;
    if (lr != 0.0 && bias) {
      double* bp = bias + (int64_t)n * b_stride + co;
      *bp = __dadd_rn(*bp, -__dmul_rn(lr, g));
    }
  }
}

// SM count of the current device (148 on B200), queried once per device: grid sizing, the
// single-wave test for programmatic dependent launch, tile and split-K choices
int num_sms() {
  static std::mutex mu;
  static std::vector<std::pair<int, int>> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  for (auto& kv : cache)
    if (kv.first == dev) return kv.second;
  int n = 148;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n < 1) n = 148;
  cache.emplace_back(dev, n);
  return n;
}

int grid_for(int64_t total) {
  int64_t g = (total + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, (int64_t)num_sms() * 16));
}

// launch of an elementwise kernel (one that starts with pdl_enter): with the programmatic
// stream-serialization attribute when its grid fits one wave (multi-wave grids keep plain
// launches, as the step kernels do).  LMG_NO_PDL=1 disables.
template <class... KA, class... A>
void ew_launch(void (*kern)(KA...), dim3 grid, int block, cudaStream_t st, A... args) {
  static const bool pdl_on = getenv("LMG_NO_PDL") == nullptr && getenv("LMG_NO_PDL_ELEM") == nullptr;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(block, 1, 1);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  const int64_t blocks = (int64_t)grid.x * grid.y * grid.z;
  cfg.numAttrs = (pdl_on && blocks <= (int64_t)num_sms() * (2048 / block)) ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kern, static_cast<KA>(args)...);
}

// ------------------------------------------------------------------------------------------
// launch accounting: a counter of every kernel this library launches (bench "gpu_launches") and
// optional CUDA-event timing of each launch by class (bench roofline, measured over the timed
// region on the launching stream).

enum Cls {
  CLS_GEMM_FWD = 0,   // step GEMM, forward layout
  CLS_GEMM_ADJ = 1,   // step GEMM, adjoint layout
  CLS_GEMM_PG = 2,    // parameter-gradient GEMM
  CLS_ELEM = 3,       // elementwise / reductions
  CLS_SWEEP_FWD = 4,  // fused persistent sweep (lmg_sweep.cu), forward
  CLS_SWEEP_ADJ = 5,  // fused persistent sweep, adjoint
  CLS_SERIAL = 6,     // split-K cluster kernel: one serial layer step (coarsest solve, serial
                      // propagation) -- latency-bound, kept out of the relaxation classes 0/1
  CLS_N = 7
};

struct Rec {
  int cls;
  double flops, bytes;
  cudaEvent_t a, b;
};

std::atomic<unsigned long long> g_launches{0};
// launches issued by THIS host thread: a graph capture counts its own launches with it (several
// host threads -- one per batch-slice stream -- may launch concurrently)
thread_local unsigned long long t_launches = 0;
// per-kernel-variant launch counters (lmg_route_counts): which kernel each step actually ran on,
// so the parity tests can assert they exercised the routing the bench times
std::atomic<unsigned long long> g_route[LMG_ROUTE_N];
inline void route(int r) { g_route[r].fetch_add(1, std::memory_order_relaxed); }
bool g_timing = false;
std::vector<Rec> g_recs;
std::mutex g_rec_mu;  // several host threads (one per stream) may launch concurrently
std::vector<cudaEvent_t> g_pool;
size_t g_pool_used = 0;

cudaEvent_t pool_event() {
  if (g_pool_used == g_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    g_pool.push_back(e);
  }
  return g_pool[g_pool_used++];
}

template <class F>
int launch(int cls, double flops, double bytes, cudaStream_t st, F&& f) {
  Rec r{cls, flops, bytes, nullptr, nullptr};
  const bool timing = g_timing;
  if (timing) {
    std::lock_guard<std::mutex> lk(g_rec_mu);
    r.a = pool_event();
    r.b = pool_event();
  }
  if (timing) cudaEventRecord(r.a, st);
  f();
  CUDA_TRY(cudaGetLastError());
  if (timing) {
    cudaEventRecord(r.b, st);
    std::lock_guard<std::mutex> lk(g_rec_mu);
    g_recs.push_back(r);
  }
  ++g_launches;
  ++t_launches;
  return LMG_OK;
}

int copy_rows(double* dst, int64_t dst_ts, const double* src, int64_t src_ts, int64_t nrows,
              int64_t len, cudaStream_t st) {
  if (nrows <= 0 || len <= 0) return LMG_OK;
  return launch(CLS_ELEM, 0.0, 16.0 * nrows * len, st, [&] {
    ew_launch(k_copy_rows, dim3(grid_for(nrows * len)), 256, st, dst, dst_ts, src, src_ts, nrows, len);
  });
}

// ------------------------------------------------------------------------------------------
// step-GEMM dispatch

enum Layout { L_FWD = 0, L_ADJ = 1, L_PG = 2 };

// Tile configurations.  Every config accumulates each output over k in the same order (one
// DMMA chain, k ascending), so they are bitwise interchangeable; residual partial sums always
// use TSmall so norms are canonical.  Choice measured on B200 (tools/gemm_bench.py, profiles/):
// many warps per SMSP hide the DMMA latency better than big warp tiles.
//   sweep (256 tasks, 256x512x512):  TSmall 26.7 TF/s  TWide 25.8  64x64/32x32-warp 22.8
//   adjoint layout:                   TWide 25.1        TSmall 21.9
//   single-task serial step:          TSmall 18.9 us    TWide 24.3   64x64 47.9
using TSmall = Tile<32, 32, 16, 2, 2, 4>;  // 4 warps of 16x16, ~5 CTAs/SM
using TWide = Tile<32, 64, 16, 2, 4, 4>;   // 8 warps of 16x16
using TTiny = Tile<16, 32, 16, 1, 2, 4>;   // batches <= 16: 2 warps of 16x16, no wasted rows
// Multi-wave step launches (big batches) keep more CTAs resident rather than deeper rings: the
// other CTAs' mainloops hide a CTA's epilogue (the FP64 tanh) and its single-stage prefetch
// (tools/tile_probe.cu on the c2 forward step, 256 tasks x 256x512x512, E_PROP tanh: 4 stages /
// 5 CTAs per SM 27.5 TF/s, 3 / 7 29.0, 2 / 10 30.1; 64 tasks 26.4 -> 28.5).  Adjoint layout
// (act'-scaled A, MN-major W): scaling each fragment at use 23.2 TF/s (32x64), each staged
// element once 26.5-28.1 (32x64 / 32x128, 2 stages), the products staged from registers
// (TileR: act' never enters shared memory) at 64x128 30.6 (64 tasks 25.2 -> 29.3); unscaled 30.5.
using TFwd = Tile<32, 32, 16, 2, 2, 2>;
using TAdj = TileR<64, 128, 16, 2, 4>;
// adjoint residual steps (E_RESID: the canonical partials need 32-column tiles of two 16-column
// warps): register-staged 64 x 32 tiles, 26.0 TF/s vs 22.4 for TFwd's 32 x 32 (4 tile shapes
// measured, tools/tile_probe.cu); the partials are per row and tile, so bitwise the same
using TResA = TileR<64, 32, 16, 2, 2>;
using TTiny4 = Tile<16, 32, 16, 1, 4, 4>;  // batches <= 16, 4 warps of 16x8 (chain launches' tile)
// parameter gradients of a small batch (K = B <= 32: one or two k-tiles): deeper rings only cost
// occupancy (TWide's 4 stages left 3 CTAs/SM for a launch that streams W in and out)
using TPg = Tile<32, 64, 16, 2, 4, 2>;
static_assert(TTiny::BN == TSmall::BN && TTiny::WN == TSmall::WN, "canonical residual partials");
static_assert(TFwd::BN == TSmall::BN && TFwd::WN == TSmall::WN, "canonical residual partials");
static_assert(TResA::BN == TSmall::BN && TResA::WN == TSmall::WN, "canonical residual partials");

template <class T, bool AK, bool BKM, bool ASC, int VEC, bool FULL = false>
int launch_cfg(const StepArgs& a, cudaStream_t st) {
  using C = GemmCfg<T, AK, BKM, ASC>;
  constexpr int BM = C::BM, BN = C::BN;
  auto kern = step_gemm<T, AK, BKM, ASC, VEC, FULL>;
  static const cudaError_t attr =  // thread-safe one-time init
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
  if (attr != cudaSuccess) return fail(LMG_ERR_CUDA, cudaGetErrorString(attr));
  dim3 grid((a.N + BN - 1) / BN, (a.M + BM - 1) / BM, a.ntasks);
  const int cls = AK ? (BKM ? CLS_GEMM_FWD : CLS_GEMM_ADJ) : CLS_GEMM_PG;
  // algorithmic work: 2MNK per task + ~5 epilogue flops per output (2q^2+5q per F)
  const double flops = (double)a.ntasks * ((double)a.M * a.N * (2.0 * a.K + 5.0));
  const double bytes = 8.0 * a.ntasks * ((double)a.N * a.K + (double)a.M * a.K + 2.0 * a.M * a.N);
  // programmatic dependent launch only for single-wave grids (the small-batch steps): with more
  // waves, dependents launched at the last wave's start park in griddepcontrol.wait on SM slots
  // the primary still needs (c2 measured 1.58 s vs 1.08 s per step with PDL on every launch)
  static const bool pdl_on = getenv("LMG_NO_PDL") == nullptr;
  static const int per_sm = [] {
    int n = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, step_gemm<T, AK, BKM, ASC, VEC, FULL>,
                                                  C::NTHREADS, C::SMEM);
    return n;
  }();
  // multi-wave grids: opt-in (LMG_PDL_MULTI=1), with the trigger after the mainloop -- measured
  // within noise on c2 (1068 vs 1066-1125 ms per step)
  static const bool pdl_multi = getenv("LMG_PDL_MULTI") != nullptr;
  const bool single = (int64_t)grid.x * grid.y * grid.z <= (int64_t)per_sm * num_sms();
  const bool pdl = pdl_on && (single || pdl_multi);
  route((std::is_same<T, TTiny>::value || std::is_same<T, TTiny4>::value)
            ? (FULL ? LMG_ROUTE_STEP_TINY_FULL : LMG_ROUTE_STEP_TINY)
        : (std::is_same<T, TWide>::value || std::is_same<T, TAdj>::value || std::is_same<T, TPg>::value)
            ? (FULL ? LMG_ROUTE_STEP_WIDE_FULL : LMG_ROUTE_STEP_WIDE)
                                        : (FULL ? LMG_ROUTE_STEP_SMALL_FULL : LMG_ROUTE_STEP_SMALL));
  StepArgs al = a;  // the launched copy carries the trigger placement
  al.pdl_late = single ? 0 : 1;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = grid;
  lc.blockDim = dim3(C::NTHREADS, 1, 1);
  lc.dynamicSmemBytes = C::SMEM;
  lc.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = pdl ? 1 : 0;
  return launch(cls, flops, bytes, st, [&] { cudaLaunchKernelEx(&lc, kern, al); });
}

// residual partial slots are per TSmall n-tile
int n_tiles(int N) { return (N + TSmall::BN - 1) / TSmall::BN; }

bool aligned16(const void* p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

enum TileSel { SEL_AUTO = 0, SEL_SMALL = 1, SEL_WIDE = 2, SEL_TINY = 3 };
// Shapes measured and not kept (tools/gemm_bench.py, tools/sweep_bench.py): 32x32 BK 32 (26.6 vs
// 28.0 TF/s at c2), 64x32 8 warps (27.8); small batch 16x64 4 warps (= TTiny), 16x32 BK 32
// (-5%), 16x32 3 / 6 stages (+1% / -3% at c5).

int tile_override() {
  static int v = [] {
    const char* e = getenv("LMG_TILE");
    if (e && !strcmp(e, "small")) return (int)SEL_SMALL;
    if (e && !strcmp(e, "wide")) return (int)SEL_WIDE;
    if (e && !strcmp(e, "tiny")) return (int)SEL_TINY;
    return (int)SEL_AUTO;
  }();
  return v;
}

int64_t ctas_for(const StepArgs& a, int BM, int BN) {
  return (int64_t)a.ntasks * ((a.M + BM - 1) / BM) * ((a.N + BN - 1) / BN);
}

template <bool AK, bool BKM, bool ASC>
int choose_tile(const StepArgs& a) {
  if (a.epi == E_RESID) {
    // canonical partial-sum layout: one slot per 32-column CTA tile, two 16-column warps summed
    // in warp order -- TSmall and TTiny (same BN, WN and warp width) produce identical partials,
    // so small batches use the 16-row tile (c5: 0.76 -> ~0.4 ms initial residual)
    if (tile_override() == SEL_SMALL) return SEL_SMALL;
    return (AK && a.M <= 16) ? SEL_TINY : SEL_SMALL;
  }
  int o = tile_override();
  if (o != SEL_AUTO) return o;
  const bool adj = AK && !BKM;
  if (AK && a.M <= 16) return SEL_TINY;  // step launches with a small batch (M = B)
  // parameter gradients of a small batch (K = B <= 32): one k-tile per CTA, so the 32 x 32 grid
  // is launch/epilogue-bound; 32 x 64 tiles halve the CTAs (c5: 2.08 -> 1.85 ms per step)
  if (!AK && a.K <= 32) return SEL_WIDE;
  if (adj && ctas_for(a, TWide::BM, TWide::BN) >= 2 * num_sms()) return SEL_WIDE;
  return SEL_SMALL;
}

template <bool AK, bool BKM, bool ASC>
int launch_layout(const StepArgs& a, bool v2, cudaStream_t st) {
  if (!v2) return launch_cfg<TSmall, AK, BKM, ASC, 1>(a, st);
  auto full = [&](int BM, int BN, int BK) {
    return a.M % BM == 0 && a.N % BN == 0 && a.K % BK == 0 && !getenv("LMG_NO_FULL");
  };
  const int sel = choose_tile<AK, BKM, ASC>(a);
  if (sel == SEL_TINY) {
    // non-residual small-batch steps on the chain launches' 4-warp 16 x 32 tile (residual steps
    // keep TTiny's two 16-column warps: canonical partials)
    if (a.epi != E_RESID && full(TTiny4::BM, TTiny4::BN, TTiny4::BK))
      return launch_cfg<TTiny4, AK, BKM, ASC, 2, true>(a, st);
    if (full(TTiny::BM, TTiny::BN, TTiny::BK)) return launch_cfg<TTiny, AK, BKM, ASC, 2, true>(a, st);
    return launch_cfg<TTiny, AK, BKM, ASC, 2>(a, st);
  }
  if (sel == SEL_WIDE) {
    if (AK && !BKM && full(TAdj::BM, TAdj::BN, TAdj::BK)) return launch_cfg<TAdj, AK, BKM, ASC, 2, true>(a, st);
    if (!AK && full(TPg::BM, TPg::BN, TPg::BK)) return launch_cfg<TPg, AK, BKM, ASC, 2, true>(a, st);
    if (full(TWide::BM, TWide::BN, TWide::BK)) return launch_cfg<TWide, AK, BKM, ASC, 2, true>(a, st);
    return launch_cfg<TWide, AK, BKM, ASC, 2>(a, st);
  }
  if (AK && !BKM && ASC && full(TResA::BM, TResA::BN, TResA::BK))
    return launch_cfg<TResA, AK, BKM, ASC, 2, true>(a, st);
  if (full(TFwd::BM, TFwd::BN, TFwd::BK)) return launch_cfg<TFwd, AK, BKM, ASC, 2, true>(a, st);
  return launch_cfg<TSmall, AK, BKM, ASC, 2>(a, st);
}

// ---- split-K cluster kernel for serial single-task steps ----------------------------------------
template <class T, bool AK, bool BKM, bool ASC>
int launch_serial_cfg(const StepArgs& a, int KS, cudaStream_t st) {
  using C = GemmCfg<T, AK, BKM, ASC>;
  auto kern = serial_gemm<T, AK, BKM, ASC>;
  static const cudaError_t attr =
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
  if (attr != cudaSuccess) return fail(LMG_ERR_CUDA, cudaGetErrorString(attr));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.N / C::BN, a.M / C::BM, KS);
  cfg.blockDim = dim3(C::NTHREADS, 1, 1);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 1;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = KS;
  // serial steps are single-wave chains: programmatic dependent launch overlaps the next step's
  // launch and weight prefetch with this step's tail (LMG_NO_PDL=1 disables)
  static const bool pdl_on = getenv("LMG_NO_PDL") == nullptr;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_on ? 2 : 1;
  const int cls = CLS_SERIAL;
  const double flops = (double)a.M * a.N * (2.0 * a.K + 5.0);
  const double bytes = 8.0 * ((double)a.N * a.K + (double)a.M * a.K + 2.0 * a.M * a.N);
  route(LMG_ROUTE_SERIAL_SPLITK);
  return launch(cls, flops, bytes, st, [&] { cudaLaunchKernelEx(&cfg, kern, a); });
}

// returns LMG_OK after launching, or -1 if the step is not eligible (caller falls back)
int launch_serial(Layout L, const StepArgs& a, cudaStream_t st) {
  static const bool off = getenv("LMG_NO_SPLITK") != nullptr;
  if (off || canonical_order()) return -1;
  if (a.ntasks != 1 || (a.epi != E_PROP && a.epi != E_ADV) || L == L_PG) return -1;
  if (!aligned16(a.A) || !aligned16(a.Bm) || !aligned16(a.Ds) || (a.lda | a.ldb | a.K | a.N) & 1)
    return -1;
  const bool tiny = a.M <= 16;
  const int BM = tiny ? TTiny::BM : TSmall::BM, BN = tiny ? TTiny::BN : TSmall::BN, BK = 16;
  if (a.M % BM || a.N % BN || a.K % BK) return -1;
  const int64_t base = (int64_t)(a.N / BN) * (a.M / BM);
  int KS = 1;
  while (KS < 8 && base * KS * 2 <= 4 * num_sms() && (a.K / BK) % (KS * 2) == 0) KS *= 2;
  // LMG_SPLITK_KS (measurement knob): 2, 4 or 8; c2 measured 1,001 / 977 (default: 4) / 981 ms
  static const int ks_force = [] {
    const char* e = getenv("LMG_SPLITK_KS");
    return e ? atoi(e) : 0;
  }();
  if (ks_force >= 2 && ks_force <= 8 && (a.K / BK) % ks_force == 0) KS = ks_force;
  if (KS == 1) return -1;
  const bool adj = (L == L_ADJ);
  if (tiny)
    return adj ? launch_serial_cfg<TTiny, true, false, true>(a, KS, st)
               : launch_serial_cfg<TTiny, true, true, false>(a, KS, st);
  return adj ? launch_serial_cfg<TSmall, true, false, true>(a, KS, st)
             : launch_serial_cfg<TSmall, true, true, false>(a, KS, st);
}

int launch_step(Layout L, const StepArgs& a, cudaStream_t st) {
  if (a.ntasks <= 0 || a.M <= 0 || a.N <= 0) return LMG_OK;
  if (a.ntasks > 65535) return fail(LMG_ERR_CONFIGURATION, "too many tasks in one launch");
  bool v2 = (a.lda % 2 == 0) && (a.ldb % 2 == 0) && aligned16(a.A) && aligned16(a.Bm) &&
            aligned16(a.Ds) && (a.A_ts % 2 == 0) && (a.B_ts % 2 == 0) && (a.Ds_ts % 2 == 0);
  if (L == L_FWD) v2 = v2 && (a.K % 2 == 0);
  if (L == L_ADJ) v2 = v2 && (a.K % 2 == 0) && (a.N % 2 == 0);
  if (L == L_PG) v2 = v2 && (a.M % 2 == 0) && (a.N % 2 == 0);
  TgPlan* plan = nullptr;
  if (L != L_PG && v2 && tgemm_prepare(a, L == L_ADJ, &plan)) {
    // big-batch steps: the warp-specialised TMA kernel (lmg_tgemm.cu), bitwise the same math
    const int cls = L == L_FWD ? CLS_GEMM_FWD : CLS_GEMM_ADJ;
    const double flops = (double)a.ntasks * ((double)a.M * a.N * (2.0 * a.K + 5.0));
    const double bytes = 8.0 * a.ntasks * ((double)a.N * a.K + (double)a.M * a.K + 2.0 * a.M * a.N);
    cudaError_t e = cudaSuccess;
    route(tgemm_small(plan) ? LMG_ROUTE_TGEMM_SMALL : LMG_ROUTE_TGEMM_BIG);
    TRY(launch(cls, flops, bytes, st, [&] { e = tgemm_launch(plan, L == L_ADJ, st); }));
    if (e != cudaSuccess) return fail(LMG_ERR_CUDA, std::string("tgemm: ") + cudaGetErrorString(e));
    return LMG_OK;
  }
  switch (L) {
    case L_FWD: return launch_layout<true, true, false>(a, v2, st);
    case L_ADJ: return launch_layout<true, false, true>(a, v2, st);
    case L_PG: return launch_layout<false, false, true>(a, v2, st);
  }
  return fail(LMG_ERR_CONFIGURATION, "bad layout");
}

// ------------------------------------------------------------------------------------------
// systems

bool is_adjoint(const lmg_system& s) { return s.kind == LMG_DENSE_ADJOINT || s.kind == LMG_CONV_ADJOINT; }
bool is_conv(const lmg_system& s) { return s.kind == LMG_CONV || s.kind == LMG_CONV_ADJOINT; }

// ---- conv2d (lmg_conv.cuh) -------------------------------------------------------------------
using CT = ConvTile<32, 64, 16, 2, 2, 4>;  // 32 pixels x 64 channels, warp 16x32
// the adjoint stages two raster tiles (lambda and act'): 4 stages left it at 2 CTAs/SM (ncu:
// DMMA pipe 44%, 2.41 ms per c3 sweep launch); 3 stages fit 3 CTAs/SM
using CTA = ConvTile<32, 64, 16, 2, 2, 3>;

ConvGeom geom_of(const lmg_system& S) {
  ConvGeom g;
  g.C = S.channels;
  g.Cp = (g.C + 31) / 32 * 32;
  g.H = S.height;
  g.W = S.px_width;
  g.HW = g.H * g.W;
  g.HWp = (g.HW + CT::BM - 1) / CT::BM * CT::BM;
  g.q = (int64_t)g.C * g.HW;
  return g;
}

template <int V, class T>
int launch_conv_t(const StepArgs& a, const ConvGeom& g, cudaStream_t st) {
  static_assert(T::BM == CT::BM && T::BN == CT::BN, "geometry padding assumes CT's tile");
  constexpr int A_SZ = T::BK * T::LDA;
  constexpr int B_SZ = (V == CV_ADJ) ? T::BN * T::LDB_K : T::BK * T::LDB_MN;
  constexpr int STAGE = A_SZ * ((V == CV_ADJ && !T::RS && !T::PRE) ? 2 : 1) + B_SZ * (V == CV_PGRAD ? 2 : 1);
  constexpr size_t SMEM = (size_t)T::STAGES * STAGE * sizeof(double);
  auto kern = conv_gemm<T, V>;
  static const cudaError_t attr =
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
  if (attr != cudaSuccess) return fail(LMG_ERR_CUDA, cudaGetErrorString(attr));
  if (a.ntasks > 65535) return fail(LMG_ERR_CONFIGURATION, "too many tasks in one launch");
  dim3 grid((a.N + T::BN - 1) / T::BN, (a.M + T::BM - 1) / T::BM, a.ntasks);
  const int cls = V == CV_FWD ? CLS_GEMM_FWD : (V == CV_ADJ ? CLS_GEMM_ADJ : CLS_GEMM_PG);
  // algorithmic: 2 * 9 C^2 per pixel per sample (zero padding counted as work, kernels.py:135)
  const double flops = (double)a.ntasks * 2.0 * 9.0 * g.C * g.C * (double)g.HW *
                       (V == CV_PGRAD ? (double)(a.K / g.HWp) : (double)(a.M / g.HWp));
  route(V == CV_FWD ? LMG_ROUTE_CONV_FWD : V == CV_ADJ ? LMG_ROUTE_CONV_ADJ : LMG_ROUTE_CONV_PGRAD);
  return launch(cls, flops, 0.0, st, [&] { kern<<<grid, T::NT, SMEM, st>>>(a, g); });
}

// LMG_CONV_CFG=f,a,s (measurement knob): forward stages f in {2,3,4}, adjoint stages a in {2,3},
// adjoint act' scaling s: 0 per fragment, 1 once per staged element, 2 register-staged (2 stages);
// same tile shape (so the residual partials, and every result, are bitwise the same)
int conv_cfg(int i) {
  static const int3 v = [] {
    const char* e = getenv("LMG_CONV_CFG");
    int f = 4, ad = 3, sc = 0;
    if (e) sscanf(e, "%d,%d,%d", &f, &ad, &sc);
    return make_int3(f, ad, sc);
  }();
  return i == 0 ? v.x : i == 1 ? v.y : v.z;
}

// per-(device, stream) device scratch, grown outside stream capture only (nullptr when a capture
// would need a new or bigger buffer: callers fall back to a path without it)
double* stream_scratch(cudaStream_t st, size_t bytes) {
  struct Buf { int dev; cudaStream_t st; double* p; size_t n; };
  static std::mutex mu;
  static std::vector<Buf> bufs;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  Buf* b = nullptr;
  for (auto& x : bufs)
    if (x.dev == dev && x.st == st) b = &x;
  if (b && b->n >= bytes) return b->p;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  if (cs != cudaStreamCaptureStatusNone) return nullptr;
  if (b) {
    cudaStreamSynchronize(st);  // the old buffer may still be in use by this stream
    cudaFree(b->p);
    b->p = nullptr;
    b->n = 0;
  } else {
    bufs.push_back(Buf{dev, st, nullptr, 0});
    b = &bufs.back();
  }
  if (cudaMalloc(&b->p, bytes) != cudaSuccess) {
    cudaGetLastError();
    b->p = nullptr;
    return nullptr;
  }
  b->n = bytes;
  return b->p;
}

template <int V>
int launch_conv(const StepArgs& a, const ConvGeom& g, cudaStream_t st) {
  if (V == CV_FWD) {
    const int f = conv_cfg(0);
    if (f == 2) return launch_conv_t<V, ConvTile<32, 64, 16, 2, 2, 2>>(a, g, st);
    if (f == 3) return launch_conv_t<V, ConvTile<32, 64, 16, 2, 2, 3>>(a, g, st);
    return launch_conv_t<V, CT>(a, g, st);
  }
  if (V == CV_ADJ) {
    const int ad = conv_cfg(1), sc = conv_cfg(2);
    // default: lambda * act' computed once per element by k_prescale into a stream scratch, then
    // the adjoint conv stages one raster tile per k-step (c3 launch: 1.91 ms with the scaling in
    // the kernel -- two gathered raster tiles per stage -- vs 1.62 + 0.13 ms; tools/conv_probe.py).
    // Same __dmul_rn products: bitwise.
    static const bool no_pre = getenv("LMG_CONV_NO_PRESCALE") != nullptr;
    if (sc == 0 && !no_pre) {
      const int64_t len = (int64_t)(a.M / g.HWp) * g.q;  // B samples x q per task
      const bool ok = (len % 2 == 0) && (a.A_ts % 2 == 0) && (a.Ds_ts % 2 == 0) &&
                      aligned16(a.A) && aligned16(a.Ds);
      double* scr = ok ? stream_scratch(st, (size_t)a.ntasks * len * sizeof(double)) : nullptr;
      if (scr) {
        TRY(launch(CLS_ELEM, 0.0, 24.0 * a.ntasks * len, st, [&] {
          ew_launch(k_prescale, dim3(grid_for(a.ntasks * len / 2)), 256, st, scr, a.A, a.A_ts, a.Ds, a.Ds_ts,
                                                                    a.ntasks, len);
        }));
        StepArgs p = a;
        p.A = scr;
        p.A_ts = len;
        p.Ds = nullptr;
        return launch_conv_t<V, ConvTile<32, 64, 16, 2, 2, 3, false, false, true>>(p, g, st);
      }
    }
    if (sc == 2) return launch_conv_t<V, ConvTile<32, 64, 16, 2, 2, 2, false, true>>(a, g, st);
    // 9: the pre-scaled kernel alone on the UNSCALED operand (wrong results: a speed bound only)
    if (sc == 9) return launch_conv_t<V, ConvTile<32, 64, 16, 2, 2, 3, false, false, true>>(a, g, st);
    if (sc == 8) return launch_conv_t<V, ConvTile<32, 64, 16, 2, 2, 4, false, false, true>>(a, g, st);
    if (ad == 2 && sc) return launch_conv_t<V, ConvTile<32, 64, 16, 2, 2, 2, true>>(a, g, st);
    if (ad == 2) return launch_conv_t<V, ConvTile<32, 64, 16, 2, 2, 2>>(a, g, st);
    if (sc) return launch_conv_t<V, ConvTile<32, 64, 16, 2, 2, 3, true>>(a, g, st);
    return launch_conv_t<V, CTA>(a, g, st);
  }
  return launch_conv_t<V, CT>(a, g, st);
}

// residual partial slots per state row (one per CTA tile of a row, canonical per tile config)
int row_slots(const lmg_system& S) {
  if (!is_conv(S)) return (S.width + TSmall::BN - 1) / TSmall::BN;
  const ConvGeom g = geom_of(S);
  return (g.HWp / CT::BM) * ((g.C + CT::BN - 1) / CT::BN);
}

int check_sys(const lmg_system* s, int B) {
  if (!s) return fail(LMG_ERR_CONFIGURATION, "null system");
  if (s->num_layers < 1) return fail(LMG_ERR_CONFIGURATION, "a system needs at least one block");
  if (s->width < 1 || B < 1) return fail(LMG_ERR_DIMENSION, "width and batch must be >= 1");
  if (s->kind < LMG_DENSE || s->kind > LMG_CONV_ADJOINT)
    return fail(LMG_ERR_CONFIGURATION, "unknown system kind");
  if (is_conv(*s)) {
    if (s->channels < 1 || s->height < 1 || s->px_width < 1 ||
        (int64_t)s->channels * s->height * s->px_width != s->width)
      return fail(LMG_ERR_DIMENSION, "conv2d geometry does not match the state width");
  }
  if (s->act < 0 || s->act > 2) return fail(LMG_ERR_CONFIGURATION, "unknown activation");
  if (!s->W) return fail(LMG_ERR_CONFIGURATION, "null weights");
  if (is_adjoint(*s) && !s->D) return fail(LMG_ERR_CONFIGURATION, "adjoint system without D");
  if (!(std::isfinite(s->step)) || s->step < 0.0)
    return fail(LMG_ERR_CONFIGURATION, "step_size must be finite and >= 0");
  return LMG_OK;
}

lmg_system coarsen(const lmg_system& s, int c) {
  lmg_system r = s;
  r.num_layers = s.num_layers / c;
  r.step = s.step * c;  // multigrid.py:101 fine.step_size * coarsening, level by level
  r.w_stride = s.w_stride * c;
  r.b_stride = s.b_stride * c;
  r.d_stride = s.d_stride * c;
  return r;
}

// One launch of the layer step on `ntasks` blocks blk0, blk0+blk_step, ...: task t reads its input
// state at x + t*x_ts and writes according to `epi`.
struct Fam {
  int ntasks = 0, blk0 = 0, blk_step = 1;
  const double* x = nullptr; int64_t x_ts = 0;
  const double* s = nullptr; int64_t s_ts = 0;
  const double* y = nullptr; int64_t y_ts = 0;
  const double* p = nullptr; int64_t p_ts = 0;
  double* out = nullptr; int64_t out_ts = 0;
  double* out2 = nullptr; int64_t out2_ts = 0;
  double* part = nullptr; int64_t slot0 = 0;
  bool serial = false;  // an inherently serial single-task step: split-K cluster kernel
  double h2 = 0.0;      // E_PROP + out2: coarse-step advance from the same pre-activation
};

// the StepArgs of one dense layer-step launch (family() below launches it)
StepArgs dense_step_args(const lmg_system& S, int B, int epi, const Fam& f) {
  const int q = S.width;
  StepArgs a{};
  a.M = B; a.N = q; a.K = q; a.ntasks = f.ntasks;
  a.epi = epi; a.h = S.step; a.lr = 0.0; a.scale = 1.0;
  a.A = f.x; a.A_ts = f.x_ts; a.lda = q;
  a.Bm = S.W + (int64_t)f.blk0 * S.w_stride; a.B_ts = (int64_t)f.blk_step * S.w_stride; a.ldb = q;
  a.x = f.x; a.x_ts = f.x_ts;
  a.s = f.s; a.s_ts = f.s_ts;
  a.out = f.out; a.out_ts = f.out_ts;
  a.out2 = f.out2; a.out2_ts = f.out2_ts;
  a.ldc = q;
  a.h2 = f.h2;
  if (is_adjoint(S)) {
    a.act = LMG_ACT_IDENTITY;
    a.Ds = S.D + (int64_t)f.blk0 * S.d_stride; a.Ds_ts = (int64_t)f.blk_step * S.d_stride;
  } else {
    a.act = S.act;
    a.bias = S.b ? S.b + (int64_t)f.blk0 * S.b_stride : nullptr;
    a.bias_ts = (int64_t)f.blk_step * S.b_stride;
  }
  return a;
}

// ---- persistent chain launches (lmg_chain.cuh) ----------------------------------------------
// A sweep whose step s of task t continues the chain of step s-1 of task t (F sweeps, the C and
// P steps) runs as ONE cooperative persistent launch with per-(step, task) completion counters
// instead of one launch per step -- bitwise the same arithmetic.  Used for batches of at most
// 16 (the HBM-bound regime, where per-step launch ramps and tails cost most); LMG_NO_CHAIN=1
// disables, LMG_CHAIN_ALL=1 extends it to every fully tiled batch.

struct ChainBuf {
  int dev;
  cudaStream_t st;
  unsigned* flags;
  size_t n;
};
std::mutex g_chain_mu;
std::vector<ChainBuf> g_chain_bufs;

// per-(device, stream) completion counters: launches on one stream are ordered, concurrent
// streams get their own.  Allocated outside stream capture only (the first cycle of every solve
// runs eagerly); a capture that would need a new or bigger buffer falls back to per-step launches
unsigned* chain_flags(cudaStream_t st, size_t n) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_chain_mu);
  for (auto& b : g_chain_bufs)
    if (b.dev == dev && b.st == st) {
      if (b.n >= n) return b.flags;
      cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
      cudaStreamIsCapturing(st, &cs);
      if (cs != cudaStreamCaptureStatusNone) return nullptr;
      cudaStreamSynchronize(st);  // the old buffer may still be in use by this stream
      cudaFree(b.flags);
      b.flags = nullptr;
      b.n = 0;
      if (cudaMalloc(&b.flags, n * sizeof(unsigned)) != cudaSuccess) return nullptr;
      b.n = n;
      return b.flags;
    }
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  if (cs != cudaStreamCaptureStatusNone) return nullptr;
  unsigned* f = nullptr;
  if (cudaMalloc(&f, n * sizeof(unsigned)) != cudaSuccess) return nullptr;
  g_chain_bufs.push_back(ChainBuf{dev, st, f, n});
  return f;
}

template <class T, bool BKM, bool ASC>
int launch_chain_cfg(const ChainArgs& ca, cudaStream_t st) {
  using C = GemmCfg<T, true, BKM, ASC>;
  auto kern = chain_gemm<T, true, BKM, ASC>;
  static const cudaError_t attr =
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
  if (attr != cudaSuccess) return fail(LMG_ERR_CUDA, cudaGetErrorString(attr));
  static const int per_sm = [] {
    int n = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, chain_gemm<T, true, BKM, ASC>, C::NTHREADS, C::SMEM);
    return n;
  }();
  if (per_sm < 1) return -1;
  const int grid = (int)std::min<int64_t>(ca.total, (int64_t)per_sm * num_sms());
  CUDA_TRY(cudaMemsetAsync(ca.flags, 0, (size_t)ca.nsteps * ca.max_tasks * sizeof(unsigned), st));
  double flops = 0.0, bytes = 0.0;
  for (int s = 0; s < ca.nsteps; ++s) {
    const double nt = ca.st[s].ntasks;
    flops += nt * ((double)ca.a.M * ca.a.N * (2.0 * ca.a.K + 5.0));
    bytes += 8.0 * nt * ((double)ca.a.N * ca.a.K + (double)ca.a.M * ca.a.K + 2.0 * ca.a.M * ca.a.N);
  }
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(grid, 1, 1);
  lc.blockDim = dim3(C::NTHREADS, 1, 1);
  lc.dynamicSmemBytes = C::SMEM;
  lc.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;  // every CTA resident: the counters cannot deadlock
  at[0].val.cooperative = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  route(LMG_ROUTE_CHAIN);
  return launch(ASC ? CLS_GEMM_ADJ : CLS_GEMM_FWD, flops, bytes, st,
                [&] { cudaLaunchKernelEx(&lc, kern, ca); });
}

bool chain_disabled() {
  static const bool v = getenv("LMG_NO_CHAIN") != nullptr;
  return v;
}
bool chain_all() {
  static const bool v = getenv("LMG_CHAIN_ALL") != nullptr;
  return v;
}

// one chain launch of the steps `fams` (step s of task t reads what step s-1 of task t wrote);
// war_last: the last step overwrites the row step 0 of the next task reads.  -1: not eligible
int chain_steps(const lmg_system& S, int B, const Fam* fams, int nsteps, bool war_last, cudaStream_t st) {
  if (chain_disabled() || is_conv(S) || nsteps < 2 || nsteps > kChainMaxSteps) return -1;
  if (B > 16 && !chain_all()) return -1;
  const bool tiny = B <= 16;
  const int BM = tiny ? TTiny::BM : TSmall::BM, BN = tiny ? TTiny::BN : TSmall::BN, BK = 16;
  const int q = S.width;
  if (B % BM || q % BN || q % BK || (q & 1)) return -1;
  const bool adj = is_adjoint(S);
  ChainArgs ca{};
  ca.a = dense_step_args(S, B, E_PROP, fams[0]);
  ca.nsteps = nsteps;
  ca.ntn = q / BN;
  ca.tiles = ca.ntn * (B / BM);
  ca.war_last = war_last ? 1 : 0;
  int total = 0, max_tasks = 0;
  for (int s = 0; s < nsteps; ++s) {
    const StepArgs a = dense_step_args(S, B, E_PROP, fams[s]);
    if (a.ntasks <= 0 || a.B_ts != ca.a.B_ts || a.bias_ts != ca.a.bias_ts || a.Ds_ts != ca.a.Ds_ts)
      return -1;
    if (a.s && ca.a.s && a.s_ts != ca.a.s_ts) return -1;
    if (a.s && !ca.a.s) { ca.a.s_ts = a.s_ts; }
    if (a.out2) {
      if (ca.a.out2 && a.out2_ts != ca.a.out2_ts) return -1;
      ca.a.out2 = a.out2;
      ca.a.out2_ts = a.out2_ts;
    }
    if (!aligned16(a.A) || !aligned16(a.Bm) || !aligned16(a.Ds) || !aligned16(a.out) ||
        (a.A_ts | a.B_ts | a.Ds_ts) & 1)
      return -1;
    ChainStep& cs = ca.st[s];
    cs.A = a.A; cs.A_ts = a.A_ts;
    cs.Ds = a.Ds;
    cs.Bm = a.Bm;
    cs.bias = a.bias;
    cs.s = a.s;
    cs.out = a.out; cs.out_ts = a.out_ts;
    cs.out2 = a.out2; cs.h2 = a.h2;
    cs.ntasks = a.ntasks;
    cs.item0 = total;
    total += a.ntasks * ca.tiles;
    max_tasks = std::max(max_tasks, a.ntasks);
  }
  // the WAR guard compares against step 0's tasks; the other steps never have more tasks
  for (int s = 1; s < nsteps; ++s)
    if (fams[s].ntasks > fams[0].ntasks && war_last) return -1;
  ca.total = total;
  ca.max_tasks = max_tasks;
  ca.flags = chain_flags(st, (size_t)nsteps * max_tasks);
  if (!ca.flags) return -1;
  if (tiny) {
    // Chain tiles: 16 x 32 with 4 warps of 16 x 8 (the default, 1) -- twice the warps of the
    // per-step kernel's TTiny at the same shared memory per CTA, which hides the per-k-tile
    // barrier and the W stream's latency better: c5 relaxation class 0.71 -> 0.78 of HBM, step
    // 20.6 -> 19.8 ms.  Measured alternatives (LMG_CHAIN_TILE, c5 class fraction of HBM):
    // 0 = TTiny 2 warps 0.71, 2 = 16x64 4 warps 0.77, 3 / 4 = TTiny 3 / 6 stages 0.68 / 0.64,
    // 5 = 16x64 8 warps 0.78, 6 = 16x128 8 warps 0.72, 7 = 16x32 4 warps 5 stages 0.77,
    // 8 = 16x64 8 warps 3 stages 0.73.
    static const int v = [] {
      const char* e = getenv("LMG_CHAIN_TILE");
      return e ? atoi(e) : 1;
    }();
    auto retile = [&](int bn) {  // item geometry for a BN-column tile
      if (q % bn) return false;
      ca.ntn = q / bn;
      ca.tiles = ca.ntn * (B / 16);
      int tot = 0;
      for (int s = 0; s < nsteps; ++s) {
        ca.st[s].item0 = tot;
        tot += ca.st[s].ntasks * ca.tiles;
      }
      ca.total = tot;
      return true;
    };
    auto go = [&](auto tile) -> int {
      using T = decltype(tile);
      if (!retile(T::BN)) return -1;
      return adj ? launch_chain_cfg<T, false, true>(ca, st) : launch_chain_cfg<T, true, false>(ca, st);
    };
    switch (v) {
      case 0: return go(TTiny{});
      case 2: return go(Tile<16, 64, 16, 1, 4, 4>{});
      case 3: return go(Tile<16, 32, 16, 1, 2, 3>{});
      case 4: return go(Tile<16, 32, 16, 1, 2, 6>{});
      case 5: return go(Tile<16, 64, 16, 1, 8, 4>{});
      case 6: return go(Tile<16, 128, 16, 1, 8, 4>{});
      case 7: return go(Tile<16, 32, 16, 1, 4, 5>{});
      case 8: return go(Tile<16, 64, 16, 1, 8, 3>{});
      case 9: return go(Tile<16, 32, 16, 1, 4, 4>{});  // the adjoint with act' staged in smem
      default:
        // (the adjoint at 3 stages -- 7 CTAs/SM instead of 5 -- measured the same as 4; the
        // register-staged act' keeps 4 stages at 7 CTAs/SM)
        if (adj) return go(TileRW<16, 32, 16, 1, 4, 4>{});
        return go(Tile<16, 32, 16, 1, 4, 4>{});
    }
  }
  // batches > 16 (opt-in, LMG_CHAIN_ALL=1): forward sweeps on TFwd; the adjoint keeps its
  // register-staged 64 x 128 step launches
  if (adj) return -1;
  return launch_chain_cfg<TFwd, true, false>(ca, st);
}

int family(const lmg_system& S, int B, int epi, const Fam& f, cudaStream_t st) {
  if (f.ntasks <= 0) return LMG_OK;
  const int q = S.width;
  StepArgs a{};
  a.M = B; a.N = q; a.K = q; a.ntasks = f.ntasks;
  a.epi = epi; a.h = S.step; a.lr = 0.0; a.scale = 1.0;
  a.A = f.x; a.A_ts = f.x_ts; a.lda = q;
  a.Bm = S.W + (int64_t)f.blk0 * S.w_stride; a.B_ts = (int64_t)f.blk_step * S.w_stride; a.ldb = q;
  a.x = f.x; a.x_ts = f.x_ts;
  a.s = f.s; a.s_ts = f.s_ts;
  a.y = f.y; a.y_ts = f.y_ts;
  a.p = f.p; a.p_ts = f.p_ts;
  a.out = f.out; a.out_ts = f.out_ts;
  a.out2 = f.out2; a.out2_ts = f.out2_ts;
  a.ldc = q;
  a.part = f.part; a.part_slot0 = f.slot0; a.part_ld = B;
  a.h2 = f.h2;
  if (is_conv(S)) {
    const ConvGeom g = geom_of(S);
    a.M = B * g.HWp; a.N = g.C; a.K = 9 * g.Cp;
    if (is_adjoint(S)) {
      a.act = LMG_ACT_IDENTITY;
      a.bias = nullptr;
      a.Ds = S.D + (int64_t)f.blk0 * S.d_stride; a.Ds_ts = (int64_t)f.blk_step * S.d_stride;
      return launch_conv<CV_ADJ>(a, g, st);
    }
    a.act = S.act;
    a.bias = S.b ? S.b + (int64_t)f.blk0 * S.b_stride : nullptr;
    a.bias_ts = (int64_t)f.blk_step * S.b_stride;
    return launch_conv<CV_FWD>(a, g, st);
  }
  if (is_adjoint(S)) {
    a.act = LMG_ACT_IDENTITY;
    a.bias = nullptr;
    a.Ds = S.D + (int64_t)f.blk0 * S.d_stride; a.Ds_ts = (int64_t)f.blk_step * S.d_stride;
    if (f.serial) {
      const int r = launch_serial(L_ADJ, a, st);
      if (r >= 0) return r;
    }
    return launch_step(L_ADJ, a, st);
  }
  a.act = S.act;
  a.bias = S.b ? S.b + (int64_t)f.blk0 * S.b_stride : nullptr;
  a.bias_ts = (int64_t)f.blk_step * S.b_stride;
  if (f.serial) {
    const int r = launch_serial(L_FWD, a, st);
    if (r >= 0) return r;
  }
  return launch_step(L_FWD, a, st);
}

// source row pointer for row j (NULL = zero row)
inline const double* src_row(const double* src, int mode, int64_t BQ, int j) {
  if (!src) return nullptr;
  if (mode == LMG_SRC_HEAD) return j == 0 ? src : nullptr;
  return src + (int64_t)j * BQ;
}
// source family pointer for rows j0, j0+step, ... (all >= 1 in head mode -> NULL)
inline const double* src_fam(const double* src, int mode, int64_t BQ, int j0) {
  if (!src || mode == LMG_SRC_HEAD) return nullptr;
  return src + (int64_t)j0 * BQ;
}

// ------------------------------------------------------------------------------------------
// fused persistent sweeps (lmg_sweep.cu): one launch per relaxation sweep / serial solve, state
// kept on chip, W streamed by TMA.  Used where the launch-per-step path is latency- or HBM-bound
// (small batches); bitwise identical to it.  LMG_NO_SWEEP=1 disables, LMG_SWEEP_MAXB sets the
// largest batch routed to the fused FCF sweep.

unsigned long long* g_sweep_trace = nullptr;  // lmg_debug_sweep_trace

// Instantiated cycle graphs, reused across solves: a training step reissues the same solves on
// the same buffers every step, and capturing + instantiating ~100 launches per solve cost
// milliseconds of host time (visible at small batches).  The key holds every parameter the
// captured launches depend on.
struct CycleKey {
  lmg_system fine;
  int nlevels, c, B, src_mode;
  const void *states, *src, *work, *trace;
};
struct CycleGraph {
  CycleKey key;
  cudaGraphExec_t exec;
  unsigned long long launches, used;
  int in_use;  // solves currently replaying it (concurrent batch slices): never evicted then
};
std::mutex g_graph_mu;
std::vector<CycleGraph> g_graphs;
unsigned long long g_graph_clock = 0;
constexpr size_t kGraphCacheSize = 16;
constexpr size_t kSpecMaxBytes = size_t(16) << 20;  // speculative cycles up to 16 MB of states

bool sweep_disabled() {
  static const bool v = getenv("LMG_NO_SWEEP") != nullptr;
  return v;
}
int sweep_max_batch() {
  static const int v = [] {
    const char* e = getenv("LMG_SWEEP_MAXB");
    return e ? atoi(e) : 64;
  }();
  return v;
}

bool sweep_basic_ok(const lmg_system& S) {
  if (sweep_disabled() || is_conv(S)) return false;
  if (!aligned16(S.W) || (S.width & 1) || (S.w_stride & 1)) return false;
  if (is_adjoint(S) && (!aligned16(S.D) || (S.d_stride & 1))) return false;
  if (!is_adjoint(S) && S.b && ((S.b_stride & 1) || !aligned16(S.b))) return false;
  return true;
}

SweepArgs sweep_args(const lmg_system& S, int B, int mode, int c, const double* src, int src_mode,
                     double* U) {
  SweepArgs a{};
  a.mode = mode;
  a.B = B; a.q = S.width; a.n = S.num_layers; a.c = c;
  a.adj = is_adjoint(S) ? 1 : 0;
  a.act = a.adj ? LMG_ACT_IDENTITY : S.act;
  a.h = S.step;
  a.W = S.W; a.w_stride = S.w_stride;
  a.bias = a.adj ? nullptr : S.b; a.b_stride = S.b_stride;
  a.D = a.adj ? S.D : nullptr; a.d_stride = S.d_stride;
  a.src = src; a.src_head = src_mode == LMG_SRC_HEAD;
  a.U = U;
  a.trace = g_sweep_trace;
  a.is_first = 1;
  return a;
}

// co-resident clusters of a sweep configuration, cached per (q, adjoint, cfg)
int sweep_clusters(int q, int adj, int cfg) {
  static std::mutex mu;
  static std::vector<std::pair<int64_t, int>> cache;
  const int64_t key = ((int64_t)q << 8) | (adj << 4) | cfg;
  std::lock_guard<std::mutex> lk(mu);
  for (auto& kv : cache)
    if (kv.first == key) return kv.second;
  const int n = sweep_max_clusters(q, adj, cfg);
  cache.emplace_back(key, n);
  return n;
}

// algorithmic work of one sweep launch: `steps` layer steps over the whole batch, `written`
// state rows stored to HBM (2q^2+5q flops per F-evaluation; W read once per step)
int run_sweep(const SweepArgs& a, const SweepShape& sh, double steps, double written, cudaStream_t st) {
  const double q = a.q, B = a.B, row = 8.0 * B * q;
  const double flops = steps * B * (2.0 * q * q + 5.0 * q);
  double bytes = steps * 8.0 * q * q + written * row + (double)sh.grid.z * row;
  if (a.src && !a.src_head) bytes += steps * row;
  if (a.adj) bytes += steps * row;
  cudaError_t e = cudaSuccess;
  route(a.mode == SW_SEQ ? LMG_ROUTE_SWEEP_SEQ : LMG_ROUTE_SWEEP_FCF);
  if (sh.cfg == SWEEP_CFG_WARP) route(LMG_ROUTE_WSWEEP);
  TRY(launch(a.adj ? CLS_SWEEP_ADJ : CLS_SWEEP_FWD, flops, bytes, st, [&] { e = sweep_launch(a, sh, st); }));
  if (e != cudaSuccess) return fail(LMG_ERR_CUDA, std::string("sweep launch: ") + cudaGetErrorString(e));
  return LMG_OK;
}

// serial forward substitution as one persistent launch (one chain per 16-sample tile); -1 when
// not eligible.  Only when all chains fit in one wave (otherwise the per-step path is faster).
int seq_sweep(const lmg_system& S, int B, const double* src, int mode, double* U, cudaStream_t st,
              double* corrU = nullptr, int64_t corr_ts = 0, bool* corrected = nullptr) {
  if (S.num_layers < 2 || !sweep_basic_ok(S) || !aligned16(src) || !aligned16(U)) return -1;
  SweepArgs a = sweep_args(S, B, SW_SEQ, 1, src, mode, U);
  SweepShape sh;
  if (sweep_shape(a, &sh) < 0) return -1;
  // one wave of clusters only (cudaOccupancyMaxActiveClusters: at q = 512 on B200, 7 clusters of
  // 16 CTAs or 15 of 8): beyond that the split-K per-step path measured faster (B = 256, 64
  // steps: 12.4 vs 18.7 us per step with 8-CTA clusters in two waves)
  // wider CTAs (smaller clusters) until every batch tile's chain is resident at once.  The
  // 128-column / 4-CTA shape (cfg 2) also fits B = 256 in one wave but measured no faster than
  // the split-K path under graph replay (c2: 1076 vs 1071 ms per step), so it is opt-in
  // (LMG_SWEEP_CFG=2)
  for (int cfg : {0}) {
    if ((int)sh.grid.y <= sweep_clusters(S.width, a.adj, sh.cfg)) break;
    SweepShape alt;
    if (sweep_shape(a, &alt, cfg) == 0 && alt.cfg == cfg) sh = alt;
  }
  if ((int)sh.grid.y > sweep_clusters(S.width, a.adj, sh.cfg)) return -1;
  const int64_t BQ = (int64_t)B * S.width;
  if (sh.cfg == SWEEP_CFG_WARP) {
    a.write_row0 = 1;  // the warp sweep stores states[0] itself (one launch fewer per solve)
    if (corrU && corrected) {  // ... and applies the parent level's correction row by row
      a.corrU = corrU;
      a.corr_ts = corr_ts;
      *corrected = true;
    }
  } else
    TRY(copy_rows(U, 0, src, 0, 1, BQ, st));  // states[0] = source[0]
  return run_sweep(a, sh, S.num_layers - 1, S.num_layers - 1, st);
}

// FCF relaxation + P steps of a whole level as one persistent launch (lmg_sweep.cu SW_FCF), then
// the commit of the new C rows; -1 when not eligible.  Same outputs as local_fcf_a + local_fcf_b
// on a single GPU (is_first, no next rank).
int fcf_sweep(const lmg_system& S, int B, int c, double* U, const double* src, int mode, double* P,
              double* advH, double* Cn, const double* Q, cudaStream_t st, double* SH = nullptr,
              double* Vc = nullptr) {
  if (!Cn || !P || !src || B > sweep_max_batch() || !sweep_basic_ok(S)) return -1;
  if (!aligned16(src) || !aligned16(U) || !aligned16(Q) || !aligned16(P) || !aligned16(advH) ||
      !aligned16(Cn))
    return -1;
  const int nb = S.num_layers / c;
  SweepArgs a = sweep_args(S, B, SW_FCF, c, src, mode, U);
  a.h2 = S.step * c;
  a.Q = Q; a.Cn = Cn; a.P = P; a.advH = advH;
  SweepShape sh;
  if (sweep_shape(a, &sh) < 0) return -1;
  // latency-bound levels only: when every chain of the level is resident at once (one wave of
  // clusters).  With more chains than that the per-step launches keep all SMs streaming W and
  // measured faster (c5 fine level: 64 chains x 8 CTAs).  LMG_SWEEP_ALL=1 lifts the limit.
  static const bool all = getenv("LMG_SWEEP_ALL") != nullptr;
  if (!all && (int)(sh.grid.y * sh.grid.z) > sweep_clusters(S.width, a.adj, sh.cfg)) return -1;
  double steps = (c - 1) + (nb > 1 ? 1 : 0), written = steps;
  for (int k = 1; k < nb; ++k) {
    const int r0 = (k - 1) * c + (Q ? 1 : 0);
    const int tail = (k < nb - 1) ? 1 : 0;
    steps += k * c + c - 1 + tail - r0;
    written += c + tail;
  }
  if (advH) written += nb;
  const int64_t BQ = (int64_t)B * S.width;
  // (a last-CTA-done commit inside the warp sweep instead of this launch measured much slower:
  // one CTA then does the whole level's commit -- c7 3.70 vs 2.46 ms per step)
  TRY(run_sweep(a, sh, steps, written, st));
  if (SH && advH)  // the commit and the level's coarse FAS source in one pass
    return launch(CLS_ELEM, 0.0, 48.0 * nb * BQ, st, [&] {
      ew_launch(k_commit_coarse, dim3(grid_for((int64_t)nb * BQ)), 256, st, U, src, Cn, advH, P, SH,
                Vc, nb, c, BQ);
    });
  return launch(CLS_ELEM, 0.0, 16.0 * nb * BQ, st, [&] {
    ew_launch(k_fcf_commit, dim3(grid_for((int64_t)nb * BQ)), 256, st, U, src, Cn, nb, c, BQ);
  });
}

// Layer-partitioned FCF as fused sweeps (one rank's run of blocks).  part 0: every chain that
// needs no halo -- blocks 1..nb-1, block 0 on the first rank, and with has_next the halo chain
// whose last row (the next rank's C row, no source) lands in U[L] -- then the C-row commit;
// part 1 (after the halo exchange and lmg_halo_finish of U[0]): block 0 of a non-first rank, and
// adv_out = advH[nb-1] for the next rank's coarse source.  Same layer steps on the same operands
// as local_fcf_a + local_fcf_b.
SweepArgs local_fused_args(const lmg_system& S, int B, int c, double* U, const double* src, int mode,
                           bool is_first, bool has_next, const double* Q, double* P, double* advH,
                           double* Cn, int part) {
  const int nb = S.num_layers / c;
  SweepArgs a = sweep_args(S, B, SW_FCF, c, src, mode, U);
  a.h2 = S.step * c;
  a.Q = Q; a.Cn = Cn; a.P = P; a.advH = advH;
  a.is_first = is_first ? 1 : 0;
  a.has_next = has_next ? 1 : 0;
  a.halo = U + (int64_t)S.num_layers * B * S.width;
  if (part == 0) {
    a.k0 = is_first ? 0 : 1;
    a.nchains = nb + (has_next ? 1 : 0) - a.k0;
  } else {
    a.k0 = 0;
    a.nchains = is_first ? 0 : 1;
  }
  return a;
}

bool local_fused_ok(const lmg_system& S, int B, int c, bool is_first, bool has_next) {
  if (B > sweep_max_batch() || !sweep_basic_ok(S) || S.num_layers % c) return false;
  SweepArgs a = local_fused_args(S, B, c, nullptr, nullptr, LMG_SRC_HEAD, is_first, has_next,
                                 nullptr, nullptr, nullptr, nullptr, 0);
  if (a.nchains <= 0) a.nchains = 1;
  SweepShape sh;
  if (sweep_shape(a, &sh) < 0) return false;
  static const bool all = getenv("LMG_SWEEP_ALL") != nullptr;
  return all || (int)(sh.grid.y * sh.grid.z) <= sweep_clusters(S.width, a.adj, sh.cfg);
}

int local_fcf_fused(const lmg_system& S, int B, int c, double* U, const double* src, int mode,
                    bool is_first, bool has_next, const double* Q, double* P, double* advH,
                    double* Cn, int part, double* adv_out, cudaStream_t st) {
  const int nb = S.num_layers / c;
  const int64_t BQ = (int64_t)B * S.width;
  if (!aligned16(src) || !aligned16(U) || !aligned16(Q) || !aligned16(P) || !aligned16(advH) ||
      !aligned16(Cn) || !P || !Cn || (is_first && !src))
    return fail(LMG_ERR_CONFIGURATION, "fused FCF: missing or misaligned buffers");
  SweepArgs a = local_fused_args(S, B, c, U, src, mode, is_first, has_next, Q, P, advH, Cn, part);
  if (a.nchains > 0) {
    SweepShape sh;
    if (sweep_shape(a, &sh) < 0) return fail(LMG_ERR_CONFIGURATION, "fused FCF not available");
    double steps = 0.0, written = 0.0;
    for (int k = a.k0; k < a.k0 + a.nchains; ++k) {
      const bool p_step = k < nb - 1 || has_next;
      if (k == 0) {
        steps += (c - 1) + (p_step ? 1 : 0);
        written += (c - 1) + (p_step ? 1 : 0);
        continue;
      }
      const int r0 = (k - 1) * c + (Q ? 1 : 0);
      const int last = k == nb ? nb * c : k * c + c - 1 + (p_step ? 1 : 0);
      steps += last - r0;
      written += k == nb ? 1 : c + (p_step ? 1 : 0);
    }
    if (advH) written += a.nchains;
    TRY(run_sweep(a, sh, steps, written, st));
  }
  if (part == 0 && nb > 0) {  // U[0] = f[0] on the first rank; U[kc] = Cn[k], k = 1..nb-1
    TRY(launch(CLS_ELEM, 0.0, 16.0 * nb * BQ, st, [&] {
      ew_launch(k_fcf_commit, dim3(grid_for((int64_t)nb * BQ)), 256, st, U, is_first ? src : nullptr, Cn, nb, c, BQ);
    }));
  }
  if (part == 1 && has_next && adv_out && advH)
    TRY(copy_rows(adv_out, 0, advH + (int64_t)(nb - 1) * BQ, 0, 1, BQ, st));
  return LMG_OK;
}

// ------------------------------------------------------------------------------------------
// reference routines

int seq_forward(const lmg_system& S, int B, const double* src, int mode, double* U, cudaStream_t st,
                double* corrU = nullptr, int64_t corr_ts = 0, bool* corrected = nullptr) {
  {
    const int r = seq_sweep(S, B, src, mode, U, st, corrU, corr_ts, corrected);
    if (r >= 0) return r;
  }
  const int64_t BQ = (int64_t)B * S.width;
  TRY(copy_rows(U, 0, src, 0, 1, BQ, st));  // states[0] = source[0]
  for (int j = 1; j < S.num_layers; ++j) {
    Fam f;
    f.ntasks = 1; f.blk0 = j - 1;
    f.x = U + (int64_t)(j - 1) * BQ;
    f.s = src_row(src, mode, BQ, j);
    f.out = U + (int64_t)j * BQ;
    f.serial = true;
    TRY(family(S, B, E_PROP, f, st));
  }
  return LMG_OK;
}

// F-sweep step i (1..c-1) of every block k: row kc+i from row kc+i-1
int f_step(const lmg_system& S, int B, int c, double* U, const double* src, int mode, int i,
           int k_first, cudaStream_t st, double* advH = nullptr) {
  const int64_t BQ = (int64_t)B * S.width;
  const int nb = S.num_layers / c;
  Fam f;
  f.ntasks = nb - k_first; f.blk0 = k_first * c + i - 1; f.blk_step = c;
  f.x = U + (int64_t)(k_first * c + i - 1) * BQ; f.x_ts = c * BQ;
  f.s = src_fam(src, mode, BQ, k_first * c + i); f.s_ts = c * BQ;
  f.out = U + (int64_t)(k_first * c + i) * BQ; f.out_ts = c * BQ;
  if (advH && i == 1) {  // rows kc: U[kc] + H*act(W_kc U[kc] + b_kc), H = c*h (coarse step)
    f.out2 = advH; f.out2_ts = BQ;
    f.h2 = S.step * c;
  }
  return family(S, B, E_PROP, f, st);
}

int f_relax(const lmg_system& S, int B, int c, double* U, const double* src, int mode, cudaStream_t st) {
  for (int i = 1; i < c; ++i) TRY(f_step(S, B, c, U, src, mode, i, 0, st));
  return LMG_OK;
}

// C-sweep: rows kc (k >= 1) from rows kc-1 (pre-sweep values), states[0] = source[0]
int c_step(const lmg_system& S, int B, int c, double* U, const double* src, int mode,
           double* out, int64_t out_ts, cudaStream_t st) {
  const int64_t BQ = (int64_t)B * S.width;
  const int nb = S.num_layers / c;
  Fam f;
  f.ntasks = nb - 1; f.blk0 = c - 1; f.blk_step = c;
  f.x = U + (int64_t)(c - 1) * BQ; f.x_ts = c * BQ;
  f.s = src_fam(src, mode, BQ, c); f.s_ts = c * BQ;
  f.out = out; f.out_ts = out_ts;
  return family(S, B, E_PROP, f, st);
}

int c_relax(const lmg_system& S, int B, int c, double* U, const double* src, int mode, cudaStream_t st) {
  const int64_t BQ = (int64_t)B * S.width;
  TRY(c_step(S, B, c, U, src, mode, U + (int64_t)c * BQ, c * BQ, st));
  return copy_rows(U, 0, src, 0, 1, BQ, st);
}

// ---- partition-aware ("local") level operations -----------------------------------------
// A rank holds L = nb*c consecutive states of a level: U has L rows (+1 outgoing halo slot when
// has_next), src is the head (row 0 only) or dense rows (+1 zero row when has_next), P has nb+1
// rows (P[0] incoming from the previous rank, P[nb] outgoing).  The single-GPU solve is the
// special case is_first = 1, has_next = 0.  Every arithmetic step is the same kernel on the same
// operands whatever the partition, so states are bitwise identical for any number of ranks.

// FCF part A -- launches s = 0..c-2: first F sweep (block k's rows from its old C row), then the
// C step of every block k >= 1 from the first-sweep F row kc-1 (and, with has_next, the outgoing
// value U[L] = 0 + (U[L-1] + h F(U[L-1])) for the next rank's first C row).  Each C row's old value
// is consumed at s = 0, before the C step overwrites it at s = c-1; without has_next the last
// block's first sweep is dead in the reference (overwritten, never read) and is skipped.
int local_fcf_a(const lmg_system& S, int B, int c, double* U, const double* src, int mode,
                bool is_first, bool has_next, const double* Q, cudaStream_t st) {
  const int64_t BQ = (int64_t)B * S.width;
  const int nb = S.num_layers / c;
  const int K1 = nb - 1 + (has_next ? 1 : 0);
  int s0 = 0;
  if (Q && c > 1) {
    // rows kc+1 = propagate(U[kc]) were produced by the previous cycle's residual (Q) from the
    // same, unchanged U[kc]: reuse instead of recomputing (bitwise identical).  For c > 2 the row
    // is only the next F step's input, so that step reads Q directly; with c = 2 the C step
    // reads row kc+1 from U, so it is copied there.
    if (c == 2) TRY(copy_rows(U + BQ, c * BQ, Q, BQ, K1, BQ, st));
    s0 = 1;
  }
  // steps s0..c-1 of every block's chain: F rows s+1 from s, the last one (s = c-1) the C step
  // writing row (k+1)c -- which block k+1's step 0 reads (old value) when s0 = 0
  Fam fams[kChainMaxSteps];
  int nf = 0;
  for (int s = s0; s < c; ++s) {
    Fam f;
    f.ntasks = K1; f.blk0 = s; f.blk_step = c;
    f.x = U + (int64_t)s * BQ; f.x_ts = c * BQ;
    if (s == 1 && Q) {  // row kc+1 lives in Q (contiguous rows)
      f.x = Q; f.x_ts = BQ;
    }
    f.s = src_fam(src, mode, BQ, s + 1); f.s_ts = c * BQ;
    f.out = U + (int64_t)(s + 1) * BQ; f.out_ts = c * BQ;
    if (nf < kChainMaxSteps) fams[nf] = f;
    ++nf;
  }
  const int rc = nf <= kChainMaxSteps ? chain_steps(S, B, fams, nf, s0 == 0, st) : -1;
  if (rc < 0) {
    for (int i = 0; i < nf; ++i) TRY(family(S, B, E_PROP, fams[i], st));
  } else if (rc != LMG_OK) {
    return rc;
  }
  if (is_first) TRY(copy_rows(U, 0, src, 0, 1, BQ, st));  // states[0] = source[0]
  return LMG_OK;
}

// FCF part B -- second F sweep of every block, then P[k] = propagate(U[kc-1]) for k = 1..nb-1
// (+ outgoing P[nb] with has_next): the propagated value of every C row, so the C-row residual is
// R[kc] = P[k] - U[kc] both before (multigrid.py:208) and after (multigrid.py:228) the correction,
// which only moves C rows.  With has_next, adv_out = U[(nb-1)c] + H F_H(U[(nb-1)c]) on the coarse
// system: the next rank's first coarse-source row needs it (network.py:138).
int local_fcf_b(const lmg_system& S, int B, int c, double* U, const double* src, int mode,
                double* P, bool has_next, double* adv_out, cudaStream_t st,
                double* advH = nullptr) {
  const int64_t BQ = (int64_t)B * S.width;
  const int nb = S.num_layers / c;
  const int K1 = nb - 1 + (has_next ? 1 : 0);
  // second F sweep; its first step also emits advH[k] = U[kc] + H F_H(U[kc]) for the coarse
  // source (same weights W_kc and pre-activation as row kc+1, only the step differs); then the
  // P step continues every block's chain from its last F row.  One chain launch when eligible.
  Fam fams[kChainMaxSteps];
  int nf = 0;
  for (int i = 1; i < c && nf < kChainMaxSteps; ++i) {
    Fam f;
    f.ntasks = nb; f.blk0 = i - 1; f.blk_step = c;
    f.x = U + (int64_t)(i - 1) * BQ; f.x_ts = c * BQ;
    f.s = src_fam(src, mode, BQ, i); f.s_ts = c * BQ;
    f.out = U + (int64_t)i * BQ; f.out_ts = c * BQ;
    if (advH && i == 1) {
      f.out2 = advH; f.out2_ts = BQ;
      f.h2 = S.step * c;
    }
    fams[nf++] = f;
  }
  const bool chain_p = P && K1 > 0 && nf < kChainMaxSteps;
  if (chain_p) {
    Fam f;
    f.ntasks = K1; f.blk0 = c - 1; f.blk_step = c;
    f.x = U + (int64_t)(c - 1) * BQ; f.x_ts = c * BQ;
    f.s = src_fam(src, mode, BQ, c); f.s_ts = c * BQ;
    f.out = P + BQ; f.out_ts = BQ;
    fams[nf++] = f;
  }
  int rc = (nf == c - (chain_p ? 0 : 1) && c - 1 + (chain_p ? 1 : 0) <= kChainMaxSteps)
               ? chain_steps(S, B, fams, nf, false, st) : -1;
  if (rc != LMG_OK && rc >= 0) return rc;
  const bool chained = rc == LMG_OK;
  if (!chained)
    for (int i = 1; i < c; ++i) TRY(f_step(S, B, c, U, src, mode, i, 0, st, advH));
  if (has_next && adv_out && advH) {
    TRY(copy_rows(adv_out, 0, advH + (int64_t)(nb - 1) * BQ, 0, 1, BQ, st));
    adv_out = nullptr;  // done
  }
  if (P && !(chained && chain_p)) {
    Fam f;
    f.ntasks = K1; f.blk0 = c - 1; f.blk_step = c;
    f.x = U + (int64_t)(c - 1) * BQ; f.x_ts = c * BQ;
    f.s = src_fam(src, mode, BQ, c); f.s_ts = c * BQ;
    f.out = P + BQ; f.out_ts = BQ;
    TRY(family(S, B, E_PROP, f, st));
  }
  if (has_next && adv_out) {
    const lmg_system Sc = coarsen(S, c);
    Fam f;
    f.ntasks = 1; f.blk0 = nb - 1;
    f.x = U + (int64_t)(nb - 1) * c * BQ;
    f.out = adv_out;
    TRY(family(Sc, B, E_ADV, f, st));
  }
  return LMG_OK;
}

// plain FCF on a whole level (multigrid.py:160-172)
int fcf(const lmg_system& S, int B, int c, double* U, const double* src, int mode, double* P,
        cudaStream_t st) {
  TRY(local_fcf_a(S, B, c, U, src, mode, true, false, nullptr, st));
  return local_fcf_b(S, B, c, U, src, mode, P, false, nullptr, st);
}

// coarse FAS source S_H = L_H(U_H) + R_H (multigrid.py:209-212), fused with the injection copy
// V = U[::c] the recursion edits.  Row 0: S_H[0] = U[0] + (f[0] - U[0]) on the first rank, else
// (U[0] - adv_in) + (P[0] - U[0]) with the previous rank's adv.
int local_coarse_source(const lmg_system& S, int B, int c, const double* U, const double* src,
                        int mode, const double* P, const double* adv_in, bool is_first, double* SH,
                        double* V, cudaStream_t st, const double* advH = nullptr) {
  const int64_t BQ = (int64_t)B * S.width;
  const int nb = S.num_layers / c;
  const lmg_system Sc = coarsen(S, c);
  if (advH) {  // S_H[n] = (U[nc] - advH[n-1]) + (P[n] - U[nc]); V[n] = U[nc]: elementwise
    if (nb > 1)
      TRY(launch(CLS_ELEM, 0.0, 40.0 * (nb - 1) * BQ, st, [&] {
        ew_launch(k_coarse_from_adv, dim3(grid_for((int64_t)(nb - 1) * BQ)), 256, st, 
            U + (int64_t)c * BQ, c * BQ, advH, P + BQ, SH + BQ, V ? V + BQ : nullptr, nb - 1, BQ);
      }));
    if (is_first)
      return launch(CLS_ELEM, 0.0, 24.0 * BQ, st, [&] {
        ew_launch(k_row0_coarse, dim3(grid_for(BQ)), 256, st, U, src, SH, V, BQ);
      });
    return launch(CLS_ELEM, 0.0, 32.0 * BQ, st, [&] {
      ew_launch(k_row0_coarse_halo, dim3(grid_for(BQ)), 256, st, U, adv_in, P, SH, V, BQ);
    });
  }
  Fam f;
  f.ntasks = nb - 1; f.blk0 = 0; f.blk_step = 1;  // coarse block n-1 == fine block (n-1)c
  f.x = U; f.x_ts = c * BQ;
  f.y = U + (int64_t)c * BQ; f.y_ts = c * BQ;
  f.p = P + BQ; f.p_ts = BQ;
  f.out = SH + BQ; f.out_ts = BQ;
  f.out2 = V ? V + BQ : nullptr; f.out2_ts = BQ;
  TRY(family(Sc, B, E_COARSE, f, st));
  if (is_first) {
    TRY(launch(CLS_ELEM, 0.0, 24.0 * BQ, st, [&] {
      ew_launch(k_row0_coarse, dim3(grid_for(BQ)), 256, st, U, src, SH, V, BQ);
    }));
  } else {
    TRY(launch(CLS_ELEM, 0.0, 32.0 * BQ, st, [&] {
      ew_launch(k_row0_coarse_halo, dim3(grid_for(BQ)), 256, st, U, adv_in, P, SH, V, BQ);
    }));
  }
  return LMG_OK;
}

int local_correct(int nb, int B, int q, int c, double* U, const double* V, cudaStream_t st) {
  const int64_t BQ = (int64_t)B * q;
  return launch(CLS_ELEM, 0.0, 24.0 * nb * BQ, st, [&] {
    ew_launch(k_correct, dim3(grid_for((int64_t)nb * BQ)), 256, st, U, c * BQ, V, BQ, nb, BQ);
  });
}

// partial-sum scratch of the local residuals (doubles)
size_t local_part_doubles(int L, int B, int q) {
  const size_t nt = (size_t)((q + TSmall::BN - 1) / TSmall::BN);
  return (size_t)L * nt * B + 2 * (size_t)L * B + 2 * (size_t)B + (size_t)B * q + 64;
}

// residual after the correction (multigrid.py:228): C rows elementwise from P, rows kc+1 by
// the step GEMM, everything else exactly zero.  Writes canonical per-block partials nb x B.
int local_residual_post(const lmg_system& S, int B, int c, const double* U, const double* src,
                        int mode, const double* P, bool is_first, double* block_part, double* work,
                        double* Q, cudaStream_t st, const double* Vcorr = nullptr) {
  const int q = S.width;
  const int64_t BQ = (int64_t)B * q;
  const int nb = S.num_layers / c;
  const int nt = row_slots(S);
  double* fpart = work;
  double* cpart = work + (size_t)nb * nt * B;
  static const bool no_wresid = getenv("LMG_NO_WRESID") != nullptr;
  if (Vcorr && is_first && (q == 16 || q == 32) && !is_conv(S) && !no_wresid && sweep_basic_ok(S)) {
    // narrow networks: correction, C-row partials, kc+1 residual rows and block partials in one
    // warp launch (same sums in the same order)
    ResidArgs ra{};
    ra.B = B; ra.q = q; ra.nb = nb; ra.c = c;
    ra.adj = is_adjoint(S) ? 1 : 0;
    ra.act = S.act; ra.is_first = 1; ra.h = S.step;
    ra.W = S.W; ra.w_stride = S.w_stride;
    ra.bias = ra.adj ? nullptr : S.b; ra.b_stride = S.b_stride;
    ra.D = ra.adj ? S.D : nullptr; ra.d_stride = S.d_stride;
    ra.src = src; ra.src_head = mode == LMG_SRC_HEAD;
    ra.U = const_cast<double*>(U); ra.V = Vcorr; ra.P = P; ra.Q = Q; ra.block_part = block_part;
    const double flops = (double)nb * B * (2.0 * q * q + 5.0 * q);
    cudaError_t e = cudaSuccess;
    route(LMG_ROUTE_WSWEEP);
    TRY(launch(ra.adj ? CLS_SWEEP_ADJ : CLS_SWEEP_FWD, flops, 8.0 * nb * (q * q + 6.0 * B * q), st,
               [&] { e = wresid_launch(ra, st); }));
    if (e != cudaSuccess) return fail(LMG_ERR_CUDA, std::string("wresid launch: ") + cudaGetErrorString(e));
    return LMG_OK;
  }
  if (Vcorr)  // the correction U[kc] += V - U[kc] fused in (U is then written)
    TRY(launch(CLS_ELEM, 0.0, 32.0 * nb * BQ, st, [&] {
      ew_launch(k_correct_cpart, dim3(B, nb), 256, st, const_cast<double*>(U), Vcorr, P, src,
                is_first ? 1 : 0, c, B, q, cpart);
    }));
  else
    TRY(launch(CLS_ELEM, 0.0, 16.0 * nb * BQ, st, [&] {
      ew_launch(k_cpart, dim3(dim3(B, nb)), 256, st, U, P, src, is_first ? 1 : 0, c, B, q, cpart);
    }));
  Fam f;  // rows kc+1, k = 0..nb-1
  f.ntasks = nb; f.blk0 = 0; f.blk_step = c;
  f.x = U; f.x_ts = c * BQ;
  f.s = src_fam(src, mode, BQ, 1); f.s_ts = c * BQ;
  f.y = U + BQ; f.y_ts = c * BQ;
  f.out2 = Q; f.out2_ts = BQ;
  f.part = fpart; f.slot0 = 0;
  TRY(family(S, B, E_RESID, f, st));
  return launch(CLS_ELEM, 0.0, 0.0, st, [&] {
    ew_launch(k_combine_post, dim3((int)(((int64_t)nb * B + 255) / 256)), 256, st, cpart, fpart, nb, nt, B,
                                                                          block_part);
  });
}

// full residual, part a: rows 1..L-1 (+ the outgoing adv of row L with has_next)
int local_residual_full_a(const lmg_system& S, int B, const double* U, const double* src, int mode,
                          bool has_next, double* adv_out, double* work, cudaStream_t st) {
  const int64_t BQ = (int64_t)B * S.width;
  const int L = S.num_layers;
  Fam f;
  f.ntasks = L - 1; f.blk0 = 0; f.blk_step = 1;
  f.x = U; f.x_ts = BQ;
  f.s = src_fam(src, mode, BQ, 1); f.s_ts = BQ;
  f.y = U + BQ; f.y_ts = BQ;
  f.part = work; f.slot0 = row_slots(S);  // row j's tiles at slot j*nt
  TRY(family(S, B, E_RESID, f, st));
  if (has_next && adv_out) {
    Fam g;
    g.ntasks = 1; g.blk0 = L - 1;
    g.x = U + (int64_t)(L - 1) * BQ;
    g.out = adv_out;
    TRY(family(S, B, E_ADV, g, st));
  }
  return LMG_OK;
}

// full residual, part b: row 0 (f[0] - U[0] on the first rank, (f[0] + adv_in) - U[0] elsewhere)
// and the canonical block partials
int local_residual_full_b(const lmg_system& S, int B, int c, const double* U, const double* src,
                          int mode, const double* adv_in, bool is_first, double* block_part,
                          double* work, cudaStream_t st) {
  const int q = S.width;
  const int64_t BQ = (int64_t)B * q;
  const int L = S.num_layers;
  const int nb = L / c;
  const int nt = row_slots(S);
  double* rpart = work;
  double* r0part = work + (size_t)L * nt * B;
  double* tmp = r0part + 2 * (size_t)B;  // one (B, q) row: f[0] + adv_in
  const double* s0 = src;
  if (!is_first) {
    double* row = reinterpret_cast<double*>(tmp);
    TRY(launch(CLS_ELEM, 0.0, 24.0 * BQ, st, [&] {
      ew_launch(k_halo_finish, dim3(grid_for(BQ)), 256, st, src, adv_in, row, BQ);
    }));
    s0 = row;
  }
  if (is_first || is_conv(S)) {
    // the system's row 0: reduced as the single-GPU solve reduces it (residual_full)
    TRY(launch(CLS_ELEM, 0.0, 16.0 * BQ, st, [&] {
      ew_launch(k_resid_row0, dim3(B), 256, st, s0, U, nullptr, r0part, 0, B, q);
    }));
  } else {
    // an interior row of the whole system: the E_RESID tile order (bitwise the one-GPU norm)
    TRY(launch(CLS_ELEM, 0.0, 16.0 * BQ, st, [&] {
      ew_launch(k_resid_row0_tiles, dim3((B + 127) / 128), 128, st, s0, U, r0part, B, q);
    }));
  }
  return launch(CLS_ELEM, 0.0, 0.0, st, [&] {
    ew_launch(k_combine_full, dim3((int)(((int64_t)nb * B + 255) / 256)), 256, st, rpart, r0part, nb, c, nt, B,
                                                                          block_part);
  });
}

// full residual (all rows) -> optional R, per-sample partials from slot 0
int residual_full(const lmg_system& S, int B, const double* U, const double* src, int mode,
                  double* R, double* part, cudaStream_t st, int64_t* nslots) {
  const int q = S.width;
  const int64_t BQ = (int64_t)B * q;
  const int n = S.num_layers;
  TRY(launch(CLS_ELEM, 0.0, 0.0, st, [&] { ew_launch(k_resid_row0, dim3(B), 256, st, src, U, R, part, 0, B, q); }));
  Fam f;
  f.ntasks = n - 1; f.blk0 = 0; f.blk_step = 1;
  f.x = U; f.x_ts = BQ;
  f.s = src_fam(src, mode, BQ, 1); f.s_ts = BQ;
  f.y = U + BQ; f.y_ts = BQ;
  f.out = R ? R + BQ : nullptr; f.out_ts = BQ;
  f.part = part; f.slot0 = 1;
  TRY(family(S, B, E_RESID, f, st));
  *nslots = 1 + (int64_t)(n - 1) * row_slots(S);
  return LMG_OK;
}

int reduce_norms(const double* part, int64_t nslots, int B, double* norms, cudaStream_t st) {
  TRY(launch(CLS_ELEM, 0.0, 0.0, st, [&] { ew_launch(k_reduce_norms, dim3((B + 3) / 4), 128, st, part, nslots, B, norms); }));
  return LMG_OK;
}

// ------------------------------------------------------------------------------------------
// hierarchy + workspace

int levels_for(int n, int c, int threshold, std::vector<int>* sizes) {
  if (c < 2) return fail(LMG_ERR_CONFIGURATION, "coarsening factor must be an integer >= 2, got " + std::to_string(c));
  if (threshold <= 0) threshold = std::max(1, n / c);
  sizes->clear();
  sizes->push_back(n);
  while (sizes->back() > threshold) {
    if (sizes->back() % c != 0)
      return fail(LMG_ERR_CONFIGURATION, "cannot coarsen " + std::to_string(sizes->back()) +
                                             " layers by factor " + std::to_string(c));
    sizes->push_back(sizes->back() / c);
  }
  return LMG_OK;
}

struct Workspace {
  std::vector<double*> P, SH, V;  // per relaxed level l: P[l]; per coarse level l+1: SH, V
  std::vector<double*> advH;      // per relaxed level: U[kc] + H F_H(U[kc]) from the F sweep
  std::vector<double*> Cn;        // per relaxed level: new C rows of the fused sweep
  double* part = nullptr;         // residual partial-sum scratch
  double* block_part = nullptr;   // canonical per-block partials (N/c x B)
  double* Q = nullptr;            // finest level: propagate(U[kc]) rows from the last residual
  double* norms = nullptr;
  size_t bytes = 0;
};

size_t part_slots(int n, int q) { return 1 + (size_t)n * (size_t)n_tiles(q); }

int layout_ws(const lmg_system& fine, int nlevels, int c, int B, char* base, Workspace* ws) {
  const int64_t BQ = (int64_t)B * fine.width;
  size_t off = 0;
  auto take = [&](size_t doubles) {
    double* p = base ? reinterpret_cast<double*>(base + off) : nullptr;
    off += ((doubles * sizeof(double) + 255) / 256) * 256;
    return p;
  };
  ws->P.assign(nlevels, nullptr);
  ws->SH.assign(nlevels, nullptr);
  ws->V.assign(nlevels, nullptr);
  ws->advH.assign(nlevels, nullptr);
  ws->Cn.assign(nlevels, nullptr);
  int n = fine.num_layers;
  for (int l = 0; l + 1 < nlevels; ++l) {
    int nb = n / c;
    ws->P[l] = take((size_t)(nb + 1) * BQ);
    ws->advH[l] = take((size_t)nb * BQ);
    ws->Cn[l] = B <= sweep_max_batch() ? take((size_t)nb * BQ) : nullptr;
    ws->SH[l + 1] = take((size_t)nb * BQ);
    ws->V[l + 1] = take((size_t)nb * BQ);
    n = nb;
  }
  ws->part = take(local_part_doubles(fine.num_layers, B, fine.width));
  ws->block_part = take((size_t)(fine.num_layers / c + 1) * B);
  ws->Q = take((size_t)(fine.num_layers / c + 1) * BQ);
  ws->norms = take((size_t)B);
  ws->bytes = off;
  return LMG_OK;
}

int norms_from_blocks(const double* block_part, int nblocks, int B, double* norms, cudaStream_t st) {
  return launch(CLS_ELEM, 0.0, 0.0, st, [&] {
    ew_launch(k_reduce_norms, dim3((B + 3) / 4), 128, st, block_part, nblocks, B, norms);
  });
}

// residual norms of a whole level from the initial iterate (multigrid.py:293), canonical order
int full_norms(const lmg_system& S, int B, int c, const double* U, const double* src, int mode,
               const Workspace& ws, double* norms, cudaStream_t st) {
  if (S.num_layers % c) c = S.num_layers;  // single-level hierarchy of indivisible depth: 1 block
  TRY(local_residual_full_a(S, B, U, src, mode, false, nullptr, ws.part, st));
  TRY(local_residual_full_b(S, B, c, U, src, mode, nullptr, true, ws.block_part, ws.part, st));
  return norms_from_blocks(ws.block_part, S.num_layers / c, B, norms, st);
}

// multigrid.py:175-228 on one GPU.  `want_norm` only at the finest level: the recursive call's
// return value is discarded by the reference (multigrid.py:218-226).
int cycle(const lmg_system& S, int nlevels, int l, int c, int B, double* U, const double* src,
          int mode, const Workspace& ws, bool want_norm, double* norms, cudaStream_t st,
          bool q_valid = false) {
  if (l == nlevels - 1) {  // single-level hierarchy: exact solve
    TRY(seq_forward(S, B, src, mode, U, st));
    if (want_norm) TRY(full_norms(S, B, c, U, src, mode, ws, norms, st));
    return LMG_OK;
  }
  const int nb = S.num_layers / c;
  double* P = ws.P[l];
  const double* Qs = (l == 0 && q_valid) ? ws.Q : nullptr;
  const lmg_system Sc = coarsen(S, c);
  const bool coarsest = (l + 1 == nlevels - 1);
  double* SH = ws.SH[l + 1];
  double* V = ws.V[l + 1];
  const int rs = fcf_sweep(S, B, c, U, src, mode, P, ws.advH[l], ws.Cn[l], Qs, st, SH,
                           coarsest ? nullptr : V);
  if (rs < 0) {
    TRY(local_fcf_a(S, B, c, U, src, mode, true, false, Qs, st));
    TRY(local_fcf_b(S, B, c, U, src, mode, P, false, nullptr, st, ws.advH[l]));
  } else if (rs != LMG_OK) {
    return rs;
  }
  if (rs < 0)  // (the fused sweep assembled the coarse source with its commit)
    TRY(local_coarse_source(S, B, c, U, src, mode, P, nullptr, true, SH, coarsest ? nullptr : V, st,
                            ws.advH[l]));
  bool corrected = false;  // the warp serial sweep applies this level's correction itself
  if (coarsest)
    TRY(seq_forward(Sc, B, SH, LMG_SRC_DENSE, V, st, want_norm ? nullptr : U,
                    (int64_t)c * B * S.width, &corrected));
  else
    TRY(cycle(Sc, nlevels, l + 1, c, B, V, SH, LMG_SRC_DENSE, ws, false, nullptr, st));
  if (!want_norm && !corrected) TRY(local_correct(nb, B, S.width, c, U, V, st));
  if (want_norm) {  // correction fused into the C-row residual partials
    TRY(local_residual_post(S, B, c, U, src, mode, P, true, ws.block_part, ws.part,
                            l == 0 ? ws.Q : nullptr, st, V));
    TRY(norms_from_blocks(ws.block_part, nb, B, norms, st));
  }
  return LMG_OK;
}

int check_levels(const lmg_system& fine, int nlevels, int c) {
  if (c < 2) return fail(LMG_ERR_CONFIGURATION, "coarsening factor must be an integer >= 2");
  if (nlevels < 1) return fail(LMG_ERR_CONFIGURATION, "need at least one level");
  int n = fine.num_layers;
  for (int l = 0; l + 1 < nlevels; ++l) {
    if (n % c) return fail(LMG_ERR_CONFIGURATION, "cannot coarsen " + std::to_string(n) + " layers by factor " + std::to_string(c));
    n /= c;
  }
  return LMG_OK;
}

}  // namespace

// ============================================================================================
// C-ABI

extern "C" {

int lmg_abi_version(void) { return 1; }

unsigned long long lmg_launch_count(void) { return g_launches.load(); }

int lmg_set_canonical_order(int on) {
  const int prev = lmg::g_canonical.exchange(on ? 1 : 0);
  return prev;
}

int lmg_route_counts(unsigned long long* out, int n) {
  if (!out || n < 0) return fail(LMG_ERR_CONFIGURATION, "route counts: bad buffer");
  for (int i = 0; i < n && i < LMG_ROUTE_N; ++i) out[i] = g_route[i].load();
  return LMG_ROUTE_N;
}

int lmg_timing_enable(int on) {
  std::lock_guard<std::mutex> lk(g_rec_mu);
  g_timing = on != 0;
  g_recs.clear();
  g_pool_used = 0;
  return LMG_OK;
}

int lmg_timing_read(int cls, double* ms_total, double* flops_total, double* bytes_total,
                    unsigned long long* launches) {
  double ms = 0.0, fl = 0.0, by = 0.0;
  unsigned long long n = 0;
  for (const Rec& r : g_recs) {
    if (cls >= 0 && r.cls != cls) continue;
    CUDA_TRY(cudaEventSynchronize(r.b));
    float t = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&t, r.a, r.b));
    ms += t;
    fl += r.flops;
    by += r.bytes;
    ++n;
  }
  if (ms_total) *ms_total = ms;
  if (flops_total) *flops_total = fl;
  if (bytes_total) *bytes_total = by;
  if (launches) *launches = n;
  return LMG_OK;
}

const char* lmg_last_error(void) { return g_err.c_str(); }

// debug instrumentation: device buffer (>= 4 * steps u64) receiving per-step globaltimer stamps
// (step start, state ready, mainloop done, epilogue done) of chain 0 / CTA 0 of every fused sweep
int lmg_debug_sweep_clusters(int q, int adj, int cfg) { return sweep_max_clusters(q, adj, cfg); }

int lmg_debug_sweep_trace(unsigned long long* dev_buf) {
  g_sweep_trace = dev_buf;
  return LMG_OK;
}

int lmg_propagate(const lmg_system* sys, int B, const double* u_start, const double* src,
                  int src_mode, int start, int stop, double* out, void* stream) {
  TRY(check_sys(sys, B));
  if (start < 1 || stop < start || stop - 1 > sys->num_layers)
    return fail(LMG_ERR_DIMENSION, "propagate range out of bounds");
  const int64_t BQ = (int64_t)B * sys->width;
  for (int j = start; j < stop; ++j) {
    Fam f;
    f.ntasks = 1; f.blk0 = j - 1;
    f.x = j == start ? u_start : out + (int64_t)(j - 1 - start) * BQ;
    f.s = src_row(src, src_mode, BQ, j);
    f.out = out + (int64_t)(j - start) * BQ;
    f.serial = true;
    TRY(family(*sys, B, E_PROP, f, S_(stream)));
  }
  return LMG_OK;
}

int lmg_sequential_forward(const lmg_system* sys, int B, const double* src, int src_mode,
                           double* states, void* stream) {
  TRY(check_sys(sys, B));
  return seq_forward(*sys, B, src, src_mode, states, S_(stream));
}

int lmg_propagation_operator(const lmg_system* sys, int B, const double* states, double* out,
                             void* stream) {
  TRY(check_sys(sys, B));
  const int64_t BQ = (int64_t)B * sys->width;
  TRY(copy_rows(out, 0, states, 0, 1, BQ, S_(stream)));
  Fam f;
  f.ntasks = sys->num_layers - 1;
  f.x = states; f.x_ts = BQ;
  f.y = states + BQ; f.y_ts = BQ;
  f.out = out + BQ; f.out_ts = BQ;
  return family(*sys, B, E_PROPOP, f, S_(stream));
}

size_t lmg_residual_workspace(const lmg_system* sys, int B) {
  if (!sys) return 0;
  return (part_slots(sys->num_layers, sys->width) * (size_t)B) * sizeof(double) + 256;
}

int lmg_compute_residual(const lmg_system* sys, int B, const double* states, const double* src,
                         int src_mode, double* out, double* norms, void* work, void* stream) {
  TRY(check_sys(sys, B));
  if (norms && !work) return fail(LMG_ERR_CONFIGURATION, "norms requested without workspace");
  int64_t nslots = 0;
  double* part = norms ? reinterpret_cast<double*>(work) : nullptr;
  TRY(residual_full(*sys, B, states, src, src_mode, out, part, S_(stream), &nslots));
  if (norms) TRY(reduce_norms(part, nslots, B, norms, S_(stream)));
  return LMG_OK;
}

int lmg_restrict(const double* fine, int n, int B, int q, int c, double* out, void* stream) {
  if (c < 1 || n % c) return fail(LMG_ERR_DIMENSION, "cannot restrict " + std::to_string(n) + " rows by factor " + std::to_string(c));
  const int64_t BQ = (int64_t)B * q;
  return copy_rows(out, BQ, fine, c * BQ, n / c, BQ, S_(stream));
}

int lmg_assemble_coarse_source(const lmg_system* coarse, int B, const double* UH,
                               const double* RH, double* out, void* stream) {
  TRY(check_sys(coarse, B));
  const int64_t BQ = (int64_t)B * coarse->width;
  // row 0: propagation_operator row 0 (U_H[0]) plus the residual row 0
  TRY(launch(CLS_ELEM, 0.0, 0.0, S_(stream), [&] { ew_launch(k_add, dim3(grid_for(BQ)), 256, S_(stream), out, UH, RH, BQ); }));
  Fam f;
  f.ntasks = coarse->num_layers - 1;
  f.x = UH; f.x_ts = BQ;
  f.y = UH + BQ; f.y_ts = BQ;
  f.p = RH + BQ; f.p_ts = BQ;
  f.out = out + BQ; f.out_ts = BQ;
  return family(*coarse, B, E_COARSE_R, f, S_(stream));
}

int lmg_f_relax(const lmg_system* sys, int B, int c, double* states, const double* src,
                int src_mode, void* stream) {
  TRY(check_sys(sys, B));
  TRY(check_levels(*sys, 2, c));
  return f_relax(*sys, B, c, states, src, src_mode, S_(stream));
}

int lmg_c_relax(const lmg_system* sys, int B, int c, double* states, const double* src,
                int src_mode, void* stream) {
  TRY(check_sys(sys, B));
  TRY(check_levels(*sys, 2, c));
  return c_relax(*sys, B, c, states, src, src_mode, S_(stream));
}

int lmg_fcf_relax(const lmg_system* sys, int B, int c, double* states, const double* src,
                  int src_mode, void* stream) {
  TRY(check_sys(sys, B));
  TRY(check_levels(*sys, 2, c));
  return fcf(*sys, B, c, states, src, src_mode, nullptr, S_(stream));
}

int lmg_num_levels(int n, int c, int threshold, int* levels_out) {
  std::vector<int> sizes;
  TRY(levels_for(n, c, threshold, &sizes));
  if (levels_out) *levels_out = (int)sizes.size();
  return LMG_OK;
}

size_t lmg_solver_workspace(const lmg_system* fine, int nlevels, int c, int B) {
  if (!fine || nlevels < 1 || c < 2) return 0;
  Workspace ws;
  layout_ws(*fine, nlevels, c, B, nullptr, &ws);
  return ws.bytes;
}

int lmg_mg_cycle(const lmg_system* fine, int nlevels, int c, int B, double* states,
                 const double* src, int src_mode, double* norms, void* work, size_t work_bytes,
                 void* stream) {
  TRY(check_sys(fine, B));
  TRY(check_levels(*fine, nlevels, c));
  Workspace ws;
  layout_ws(*fine, nlevels, c, B, reinterpret_cast<char*>(work), &ws);
  if (work_bytes < ws.bytes) return fail(LMG_ERR_CONFIGURATION, "workspace too small");
  return cycle(*fine, nlevels, 0, c, B, states, src, src_mode, ws, norms != nullptr,
               norms ? norms : ws.norms, S_(stream));
}

int solve_on(const lmg_system* fine, int nlevels, int c, int B, double* states,
             const double* src, int src_mode, int use_initial, double tol, int max_cycles,
             double* hist_host, int32_t* cycles_host, int32_t* converged_host, void* work,
             size_t work_bytes, cudaStream_t st);

int lmg_solve(const lmg_system* fine, int nlevels, int c, int B, double* states,
              const double* src, int src_mode, int use_initial, double tol, int max_cycles,
              double* hist_host, int32_t* cycles_host, int32_t* converged_host, void* work,
              size_t work_bytes, void* stream) {
  cudaStream_t st = S_(stream);
  if (st != nullptr && st != cudaStreamLegacy)
    return solve_on(fine, nlevels, c, B, states, src, src_mode, use_initial, tol, max_cycles,
                    hist_host, cycles_host, converged_host, work, work_bytes, st);
  // graphs cannot be captured on the legacy default stream: run on a private stream of this
  // thread, ordered after / before the caller's stream by events
  static thread_local cudaStream_t own = nullptr;
  static thread_local cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  if (!own) {
    CUDA_TRY(cudaStreamCreateWithFlags(&own, cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(&ev_in, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&ev_out, cudaEventDisableTiming));
  }
  CUDA_TRY(cudaEventRecord(ev_in, st));
  CUDA_TRY(cudaStreamWaitEvent(own, ev_in, 0));
  int rc = solve_on(fine, nlevels, c, B, states, src, src_mode, use_initial, tol, max_cycles,
                    hist_host, cycles_host, converged_host, work, work_bytes, own);
  CUDA_TRY(cudaEventRecord(ev_out, own));
  CUDA_TRY(cudaStreamWaitEvent(st, ev_out, 0));
  return rc;
}

// The current device's default stream-ordered pool keeps freed memory for reuse (release
// threshold = unlimited), once per device.
void keep_pool_memory() {
  static std::mutex mu;
  static std::vector<int> done;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  std::lock_guard<std::mutex> lk(mu);
  if (std::find(done.begin(), done.end(), dev) != done.end()) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done.push_back(dev);
}

int solve_on(const lmg_system* fine, int nlevels, int c, int B, double* states,
             const double* src, int src_mode, int use_initial, double tol, int max_cycles,
             double* hist_host, int32_t* cycles_host, int32_t* converged_host, void* work,
             size_t work_bytes, cudaStream_t st) {
  TRY(check_sys(fine, B));
  if (!(std::isfinite(tol) && tol > 0))
    return fail(LMG_ERR_CONFIGURATION, "tolerance must be a finite positive number");
  if (max_cycles < 1) return fail(LMG_ERR_CONFIGURATION, "max_cycles must be >= 1");
  TRY(check_levels(*fine, nlevels, c));
  Workspace ws;
  layout_ws(*fine, nlevels, c, B, reinterpret_cast<char*>(work), &ws);
  if (work_bytes < ws.bytes) return fail(LMG_ERR_CONFIGURATION, "workspace too small");
  const int n = fine->num_layers, q = fine->width;
  const int64_t BQ = (int64_t)B * q;

  if (!use_initial) TRY(copy_rows(states, BQ, src, 0, n, BQ, st));  // initial_guess: tile(f[0])
  TRY(full_norms(*fine, B, c, states, src, src_mode, ws, ws.norms, st));

  std::vector<double> nrm(B);
  CUDA_TRY(cudaMemcpyAsync(nrm.data(), ws.norms, B * sizeof(double), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  std::vector<int> done(B, 0);
  int ndone = 0;
  for (int b = 0; b < B; ++b) {
    hist_host[b] = nrm[b];
    cycles_host[b] = 0;
    if (nrm[b] <= tol) { done[b] = 1; ++ndone; }
  }
  // samples that stop while others continue are parked here (multigrid.py:297 per sample).
  // Stream-ordered allocations from the device's default pool, which keeps freed memory
  // (keep_pool_memory): with the default release threshold of 0 every synchronize returned the
  // parked blocks to the OS and the next park re-mapped them -- c2 backward solves that park
  // ~100 samples ran 0.7-3.9 s instead of 0.54 s.  The guard frees them on every exit path.
  keep_pool_memory();
  struct Parked {
    std::vector<std::pair<int, double*>> v;
    cudaStream_t st;
    ~Parked() {
      for (auto& pb : v) cudaFreeAsync(pb.second, st);
    }
  } parked_guard{{}, st};
  auto& parked = parked_guard.v;
  auto park = [&](int b) -> int {
    double* buf = nullptr;
    CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&buf), (size_t)n * q * sizeof(double), st));
    parked.emplace_back(b, buf);
    TRY(copy_rows(buf, q, states + (int64_t)b * q, BQ, n, q, st));
    return LMG_OK;
  };
  auto park_from = [&](int b, const double* from) -> int {  // sample b of a (n, B, q) buffer
    double* buf = nullptr;
    CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&buf), (size_t)n * q * sizeof(double), st));
    parked.emplace_back(b, buf);
    TRY(copy_rows(buf, q, from + (int64_t)b * q, BQ, n, q, st));
    return LMG_OK;
  };
  for (int b = 0; b < B && ndone < B; ++b)
    if (done[b]) TRY(park(b));

  // Cycles 2.. issue an identical launch sequence: capture it once as a CUDA graph and replay
  // it (one host call per cycle instead of ~100 launches).  Not under per-launch timing.
  const bool use_graph = !g_timing && !getenv("LMG_NO_GRAPH");
  cudaGraphExec_t gexec = nullptr;  // owned by the cycle-graph cache (g_graphs)
  unsigned long long graph_launches = 0;
  struct InUse {  // releases this solve's hold on its cached graph
    cudaGraphExec_t* g;
    ~InUse() {
      if (!*g) return;
      std::lock_guard<std::mutex> lk(g_graph_mu);
      for (auto& e : g_graphs)
        if (e.exec == *g) --e.in_use;
    }
  } in_use_guard{&gexec};
  // Device-side loop (opt-in, LMG_DEVLOOP=1): cycles 2.. run inside a conditional WHILE graph
  // node whose body is one cycle + k_cycle_book; the loop leaves the device only when some sample
  // converges (to park it) or at max_cycles.  Correct (GPU tests pass with it), but measured
  // SLOWER on this driver (580.159): c1 3.14 vs 2.15 ms, c5 26.5 vs 25.6 ms, c2 1.20 vs 1.08 s per
  // step -- kernels in a conditional body pay ~17 us each -- so the per-cycle host test stays.
  const bool dev_loop = use_graph && getenv("LMG_DEVLOOP") != nullptr;
  cudaGraphExec_t dexec = nullptr;
  struct GraphGuard2 {
    cudaGraphExec_t* g;
    ~GraphGuard2() {
      if (*g) cudaGraphExecDestroy(*g);
    }
  } guard2{&dexec};
  unsigned long long iter_launches = 0;
  int* done_d = nullptr;
  int* cyc_d = nullptr;
  double* hist_d = nullptr;
  struct DevFree {
    int** a; int** b; double** c; cudaStream_t st;
    ~DevFree() {
      if (*a) cudaFreeAsync(*a, st);
      if (*b) cudaFreeAsync(*b, st);
      if (*c) cudaFreeAsync(*c, st);
    }
  } devfree{&done_d, &cyc_d, &hist_d, st};
  int cyc = 0;
  // one FAS cycle at the finest level: the cached cycle graph from the second cycle on
  auto issue_cycle = [&](bool first) -> int {
      if (use_graph && !first) {
        if (!gexec) {
          CycleKey key;
          std::memset(&key, 0, sizeof(key));
          key.fine = *fine;
          key.nlevels = nlevels; key.c = c; key.B = B; key.src_mode = src_mode;
          key.states = states; key.src = src; key.work = work; key.trace = g_sweep_trace;
          {
            std::lock_guard<std::mutex> lk(g_graph_mu);
            for (auto& e : g_graphs)
              if (!std::memcmp(&e.key, &key, sizeof(key))) {
                gexec = e.exec;
                graph_launches = e.launches;
                e.used = ++g_graph_clock;
                ++e.in_use;
                break;
              }
          }
          if (!gexec) {
            cudaGraph_t graph;
            const unsigned long long n0 = t_launches;
            CUDA_TRY(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
            int rc = cycle(*fine, nlevels, 0, c, B, states, src, src_mode, ws, true, ws.norms, st, true);
            cudaError_t ce = cudaStreamEndCapture(st, &graph);
            if (rc != LMG_OK) return rc;
            if (ce != cudaSuccess) return fail(LMG_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
            graph_launches = t_launches - n0;
            ce = cudaGraphInstantiate(&gexec, graph, 0);
            cudaGraphDestroy(graph);
            if (ce != cudaSuccess) return fail(LMG_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(ce));
            g_launches -= graph_launches;  // counted per replay below
            std::lock_guard<std::mutex> lk(g_graph_mu);
            if (g_graphs.size() >= kGraphCacheSize) {  // evict the least recently used idle entry
              size_t lru = g_graphs.size();
              for (size_t i = 0; i < g_graphs.size(); ++i)
                if (g_graphs[i].in_use == 0 && (lru == g_graphs.size() || g_graphs[i].used < g_graphs[lru].used))
                  lru = i;
              if (lru < g_graphs.size()) {
                cudaGraphExecDestroy(g_graphs[lru].exec);
                g_graphs.erase(g_graphs.begin() + lru);
              }
            }
            g_graphs.push_back(CycleGraph{key, gexec, graph_launches, ++g_graph_clock, 1});
          }
        }
        CUDA_TRY(cudaGraphLaunch(gexec, st));
        g_launches += graph_launches;
      } else {
        TRY(cycle(*fine, nlevels, 0, c, B, states, src, src_mode, ws, true, ws.norms, st, !first));
      }
    return LMG_OK;
  };

  // Speculative cycles (small states): the host's stopping test after cycle k (read-back, test,
  // next graph launch: ~20 us of idle GPU per cycle at c6/c7) overlaps cycle k+1, already queued.
  // Before each speculative cycle the states are snapshotted (state after cycle k); samples found
  // converged at k are parked from the snapshot, and when the solve stops after k the snapshot is
  // copied back -- so results, histories and cycle counts are exactly the unspeculated ones.  The
  // price is one discarded cycle per solve plus a state copy per cycle, hence small states only.
  // Measured SLOWER on B200 (c7 3.08 vs 2.86 ms, c6 1.85 vs 1.62 ms per training step,
  // profiles/r2_spec_ab.txt): the discarded cycle costs more than the host turnaround it hides,
  // which is small once the cycle is graph-replayed -- so it is opt-in (LMG_SPEC=1).
  static const bool spec_on = getenv("LMG_SPEC") != nullptr;
  const size_t state_bytes = (size_t)n * BQ * sizeof(double);
  if (use_graph && !dev_loop && spec_on && state_bytes <= kSpecMaxBytes && ndone < B && max_cycles > 1) {
    double* snap = nullptr;
    CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&snap), state_bytes, st));
    struct SnapFree {
      double** p; cudaStream_t st;
      ~SnapFree() { if (*p) cudaFreeAsync(*p, st); }
    } snap_guard{&snap, st};
    static thread_local double* hn = nullptr;  // pinned norms of two cycles in flight
    static thread_local int hn_cap = 0;
    static thread_local cudaEvent_t ev[2] = {nullptr, nullptr};
    if (hn_cap < 2 * B) {
      if (hn) cudaFreeHost(hn);
      hn = nullptr;
      hn_cap = 0;
      CUDA_TRY(cudaMallocHost(reinterpret_cast<void**>(&hn), 2 * (size_t)B * sizeof(double)));
      hn_cap = 2 * B;
    }
    for (auto& e : ev)
      if (!e) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    int issued = 0;
    auto issue = [&]() -> int {  // cycle issued + 1, its norms into slot (issued + 1) & 1
      if (issued > 0) TRY(copy_rows(snap, BQ, states, BQ, n, BQ, st));  // state after `issued`
      TRY(issue_cycle(issued == 0));
      ++issued;
      CUDA_TRY(cudaMemcpyAsync(hn + (size_t)(issued & 1) * B, ws.norms, B * sizeof(double),
                               cudaMemcpyDeviceToHost, st));
      CUDA_TRY(cudaEventRecord(ev[issued & 1], st));
      return LMG_OK;
    };
    TRY(issue());
    for (;;) {
      const int k = cyc + 1;  // the cycle evaluated now
      const bool more = k < max_cycles;
      if (more) TRY(issue());  // cycle k + 1, speculatively
      CUDA_TRY(cudaEventSynchronize(ev[k & 1]));
      const double* nk = hn + (size_t)(k & 1) * B;
      cyc = k;
      int newly = 0;
      for (int b = 0; b < B; ++b) {
        if (done[b]) continue;
        hist_host[(int64_t)cyc * B + b] = nk[b];
        cycles_host[b] = cyc;
        if (nk[b] <= tol) { done[b] = 1; ++newly; }
      }
      ndone += newly;
      if (ndone == B || !more) {
        if (more) TRY(copy_rows(states, BQ, snap, BQ, n, BQ, st));  // undo cycle k + 1
        break;
      }
      if (newly)
        for (int b = 0; b < B; ++b)
          if (done[b] && std::none_of(parked.begin(), parked.end(), [&](auto& pb) { return pb.first == b; }))
            TRY(park_from(b, snap));
    }
  }
  std::vector<int> done_i(B);
  std::vector<double> hrows;
  while (ndone < B && cyc < max_cycles) {
    if (dev_loop && cyc > 0) {
      if (!dexec) {
        CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&done_d), B * sizeof(int), st));
        CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&cyc_d), sizeof(int), st));
        CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&hist_d),
                                 (size_t)(max_cycles + 1) * B * sizeof(double), st));
        cudaGraph_t g;
        CUDA_TRY(cudaGraphCreate(&g, 0));
        cudaGraphConditionalHandle hnd;
        CUDA_TRY(cudaGraphConditionalHandleCreate(&hnd, g, 1, cudaGraphCondAssignDefault));
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = hnd;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t node;
        CUDA_TRY(cudaGraphAddNode(&node, g, nullptr, 0, &cp));
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        const unsigned long long n0 = t_launches;
        CUDA_TRY(cudaStreamBeginCaptureToGraph(st, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
        int rc = cycle(*fine, nlevels, 0, c, B, states, src, src_mode, ws, true, ws.norms, st, true);
        if (rc == LMG_OK)
          rc = launch(CLS_ELEM, 0.0, 0.0, st, [&] {
            k_cycle_book<<<1, 256, 0, st>>>(ws.norms, B, tol, done_d, hist_d, cyc_d, max_cycles, hnd);
          });
        cudaGraph_t body_out = nullptr;
        cudaError_t ce = cudaStreamEndCapture(st, &body_out);
        if (rc != LMG_OK) {
          cudaGraphDestroy(g);
          return rc;
        }
        if (ce != cudaSuccess) {
          cudaGraphDestroy(g);
          return fail(LMG_ERR_CUDA, std::string("loop capture: ") + cudaGetErrorString(ce));
        }
        iter_launches = t_launches - n0;
        g_launches -= iter_launches;  // counted per executed iteration below
        ce = cudaGraphInstantiate(&dexec, g, 0);
        cudaGraphDestroy(g);
        if (ce != cudaSuccess) return fail(LMG_ERR_CUDA, std::string("loop instantiate: ") + cudaGetErrorString(ce));
      }
      for (int b = 0; b < B; ++b) done_i[b] = done[b];
      CUDA_TRY(cudaMemcpyAsync(done_d, done_i.data(), B * sizeof(int), cudaMemcpyHostToDevice, st));
      CUDA_TRY(cudaMemcpyAsync(cyc_d, &cyc, sizeof(int), cudaMemcpyHostToDevice, st));
      CUDA_TRY(cudaGraphLaunch(dexec, st));
      int newcyc = cyc;
      CUDA_TRY(cudaMemcpyAsync(&newcyc, cyc_d, sizeof(int), cudaMemcpyDeviceToHost, st));
      CUDA_TRY(cudaStreamSynchronize(st));
      hrows.resize((size_t)(newcyc - cyc) * B);
      CUDA_TRY(cudaMemcpyAsync(hrows.data(), hist_d + (int64_t)(cyc + 1) * B,
                               hrows.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
      CUDA_TRY(cudaStreamSynchronize(st));
      g_launches += iter_launches * (unsigned long long)(newcyc - cyc);
      int newly = 0;
      for (int cc = cyc + 1; cc <= newcyc; ++cc)
        for (int b = 0; b < B; ++b) {
          if (done[b]) continue;
          const double nv = hrows[(size_t)(cc - cyc - 1) * B + b];
          hist_host[(int64_t)cc * B + b] = nv;
          cycles_host[b] = cc;
          if (cc == newcyc && nv <= tol) { done[b] = 1; ++newly; }
        }
      cyc = newcyc;
      ndone += newly;
      if (newly && ndone < B)
        for (int b = 0; b < B; ++b)
          if (done[b] && std::none_of(parked.begin(), parked.end(), [&](auto& pb) { return pb.first == b; }))
            TRY(park(b));
      continue;
    }
    TRY(issue_cycle(cyc == 0));
    ++cyc;
    CUDA_TRY(cudaMemcpyAsync(nrm.data(), ws.norms, B * sizeof(double), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    int newly = 0;
    for (int b = 0; b < B; ++b) {
      if (done[b]) continue;
      hist_host[(int64_t)cyc * B + b] = nrm[b];
      cycles_host[b] = cyc;
      if (nrm[b] <= tol) { done[b] = 1; ++newly; }
    }
    ndone += newly;
    if (newly && ndone < B)
      for (int b = 0; b < B; ++b)
        if (done[b] && std::none_of(parked.begin(), parked.end(), [&](auto& pb) { return pb.first == b; }))
          TRY(park(b));
  }
  for (auto& pb : parked) TRY(copy_rows(states + (int64_t)pb.first * q, BQ, pb.second, q, n, q, st));
  for (int b = 0; b < B; ++b) converged_host[b] = done[b];
  CUDA_TRY(cudaStreamSynchronize(st));
  return LMG_OK;
}

int lmg_act_deriv(const lmg_system* fine, int B, const double* states, double* D, void* stream) {
  TRY(check_sys(fine, B));
  if (is_adjoint(*fine)) return fail(LMG_ERR_CONFIGURATION, "act_deriv needs a forward system");
  const int64_t BQ = (int64_t)B * fine->width;
  Fam f;
  f.ntasks = fine->num_layers;
  f.x = states; f.x_ts = BQ;
  f.out = D; f.out_ts = BQ;
  return family(*fine, B, E_DERIV, f, S_(stream));
}

int lmg_param_grads(const lmg_system* fine, int B, const double* states, const double* lam,
                    const double* D, double scale, double lr, double* gW, double* gb,
                    void* stream) {
  return lmg_param_grads_ex(fine, B, states, lam, D, scale, lr, gW, gb, 0, stream);
}

int lmg_param_grads_ex(const lmg_system* fine, int B, const double* states, const double* lam,
                       const double* D, double scale, double lr, double* gW, double* gb,
                       int accumulate, void* stream) {
  TRY(check_sys(fine, B));
  if (accumulate && (!gW || !gb))
    return fail(LMG_ERR_CONFIGURATION, "accumulating gradients needs gW and gb buffers");
  if (is_adjoint(*fine)) return fail(LMG_ERR_CONFIGURATION, "param_grads needs the forward system");
  if (!gW && lr == 0.0 && !gb) return LMG_OK;
  const int N = fine->num_layers, q = fine->width;
  const int64_t BQ = (int64_t)B * q;
  cudaStream_t st = S_(stream);
  if (is_conv(*fine)) {
    // gW[tap][ci][co] = h*scale*sum_{b,pix} (lam*D)[b][co][pix] u[b][ci][pix + shift(tap)]
    const ConvGeom g = geom_of(*fine);
    StepArgs a{};
    a.M = 9 * g.Cp; a.N = g.C; a.K = B * g.HWp; a.ntasks = N;
    a.epi = E_PGRAD; a.act = LMG_ACT_IDENTITY; a.h = fine->step; a.lr = lr; a.scale = scale;
    a.A = states; a.A_ts = BQ;
    a.Bm = lam + (int64_t)(N - 1) * BQ; a.B_ts = -BQ;  // lambda^{n+1} = lam[N-1-n]
    a.Ds = D; a.Ds_ts = BQ;
    a.x = fine->W; a.x_ts = fine->w_stride;
    a.out = const_cast<double*>(fine->W); a.out_ts = fine->w_stride;
    a.out2 = gW; a.out2_ts = 9LL * g.C * g.C;
    a.accum = accumulate;
    TRY(launch_conv<CV_PGRAD>(a, g, st));
    return launch(CLS_ELEM, 0.0, 0.0, st, [&] {
      k_conv_bias_grads<<<dim3(g.C, N), 256, 0, st>>>(lam + (int64_t)(N - 1) * BQ, -BQ, D, B, g.C,
                                                     g.HW, fine->step, scale, lr, gb,
                                                     const_cast<double*>(fine->b), fine->b_stride,
                                                     accumulate);
    });
  }
  StepArgs a{};
  a.M = q; a.N = q; a.K = B; a.ntasks = N;
  a.epi = E_PGRAD; a.act = LMG_ACT_IDENTITY; a.h = fine->step; a.lr = lr; a.scale = scale;
  a.A = lam + (int64_t)(N - 1) * BQ; a.A_ts = -BQ; a.lda = q;  // lambda^{n+1} = lam[N-1-n]
  a.Ds = D; a.Ds_ts = BQ;
  a.Bm = states; a.B_ts = BQ; a.ldb = q;
  a.x = fine->W; a.x_ts = fine->w_stride;
  a.out = const_cast<double*>(fine->W); a.out_ts = fine->w_stride;
  a.out2 = gW; a.out2_ts = (int64_t)q * q;
  a.ldc = q;
  a.accum = accumulate;
  TRY(launch_step(L_PG, a, st));
  const int64_t tot = (int64_t)N * q;
  TRY(launch(CLS_ELEM, 0.0, 0.0, st, [&] { k_bias_grads<<<(int)((tot + 255) / 256), 256, 0, st>>>(lam + (int64_t)(N - 1) * BQ, -BQ, D, N, B, q,
                                                         fine->step, scale, lr, gb,
                                                         const_cast<double*>(fine->b), fine->b_stride,
                                                         accumulate); }));
  return LMG_OK;
}

int lmg_apply_block(const lmg_system* sys, int B, int j, const double* X, double* Y, void* stream) {
  TRY(check_sys(sys, B));
  if (is_adjoint(*sys)) return fail(LMG_ERR_CONFIGURATION, "apply_block needs a forward system");
  if (j < 0 || j >= sys->num_layers) return fail(LMG_ERR_DIMENSION, "block index out of range");
  Fam f;
  f.ntasks = 1; f.blk0 = j;
  f.x = X; f.out = Y;
  return family(*sys, B, E_APPLY, f, S_(stream));
}

int lmg_vjp_block(const lmg_system* sys, int B, int j, const double* X, const double* G, double* gX,
                  double* gW, double* gb, double* work, void* stream) {
  TRY(check_sys(sys, B));
  if (is_adjoint(*sys)) return fail(LMG_ERR_CONFIGURATION, "vjp_block needs a forward system");
  if (j < 0 || j >= sys->num_layers) return fail(LMG_ERR_DIMENSION, "block index out of range");
  cudaStream_t st = S_(stream);
  Fam f;  // work = act'(pre(X))
  f.ntasks = 1; f.blk0 = j;
  f.x = X; f.out = work;
  TRY(family(*sys, B, E_DERIV, f, st));
  lmg_system one = *sys;
  one.num_layers = 1;
  one.W = sys->W + (int64_t)j * sys->w_stride;
  one.b = sys->b ? sys->b + (int64_t)j * sys->b_stride : nullptr;
  one.w_stride = one.b_stride = 0;
  if (gX) {  // gX = J^T (G * act'): the adjoint block on its own
    lmg_system adj = one;
    adj.kind = is_conv(*sys) ? LMG_CONV_ADJOINT : LMG_DENSE_ADJOINT;
    adj.D = work;
    adj.d_stride = 0;
    adj.b = nullptr;
    Fam g;
    g.ntasks = 1; g.blk0 = 0;
    g.x = G; g.out = gX;
    TRY(family(adj, B, E_APPLY, g, st));
  }
  if (gW || gb) {
    one.step = 1.0;
    TRY(lmg_param_grads(&one, B, X, G, work, 1.0, 0.0, gW, gb, stream));
  }
  return LMG_OK;
}

// ---- partition-aware level operations (include/lmg.h "layer-partitioned" section) ----------

int lmg_local_fcf_a(const lmg_system* sys, int B, int c, double* U, const double* src,
                    int src_mode, int is_first, int has_next, const double* Q, void* stream) {
  TRY(check_sys(sys, B));
  TRY(check_levels(*sys, 2, c));
  return local_fcf_a(*sys, B, c, U, src, src_mode, is_first != 0, has_next != 0, Q, S_(stream));
}

int lmg_local_fcf_b(const lmg_system* sys, int B, int c, double* U, const double* src,
                    int src_mode, double* P, int has_next, double* adv_out, double* advH,
                    void* stream) {
  TRY(check_sys(sys, B));
  TRY(check_levels(*sys, 2, c));
  return local_fcf_b(*sys, B, c, U, src, src_mode, P, has_next != 0, adv_out, S_(stream), advH);
}

int lmg_local_fcf_fused_ok(const lmg_system* sys, int B, int c, int is_first, int has_next) {
  if (check_sys(sys, B) != LMG_OK || check_levels(*sys, 2, c) != LMG_OK) return 0;
  return local_fused_ok(*sys, B, c, is_first != 0, has_next != 0) ? 1 : 0;
}

int lmg_local_fcf_fused(const lmg_system* sys, int B, int c, double* U, const double* src,
                        int src_mode, int is_first, int has_next, const double* Q, double* P,
                        double* advH, double* Cn, int part, double* adv_out, void* stream) {
  TRY(check_sys(sys, B));
  TRY(check_levels(*sys, 2, c));
  if (part != 0 && part != 1) return fail(LMG_ERR_CONFIGURATION, "part must be 0 or 1");
  return local_fcf_fused(*sys, B, c, U, src, src_mode, is_first != 0, has_next != 0, Q, P, advH, Cn,
                         part, adv_out, S_(stream));
}

int lmg_halo_finish(const double* s0, const double* adv_in, double* out, int64_t len, void* stream) {
  cudaStream_t st = S_(stream);
  return launch(CLS_ELEM, 0.0, 24.0 * len, st, [&] {
    ew_launch(k_halo_finish, dim3(grid_for(len)), 256, st, s0, adv_in, out, len);
  });
}

int lmg_local_coarse_source(const lmg_system* sys, int B, int c, const double* U,
                            const double* src, int src_mode, const double* P,
                            const double* adv_in, int is_first, double* SH, double* V,
                            const double* advH, void* stream) {
  TRY(check_sys(sys, B));
  TRY(check_levels(*sys, 2, c));
  if (!is_first && !adv_in) return fail(LMG_ERR_PROTOCOL, "non-first rank needs the previous rank's adv row");
  return local_coarse_source(*sys, B, c, U, src, src_mode, P, adv_in, is_first != 0, SH, V,
                             S_(stream), advH);
}

int lmg_local_correct(int n_blocks, int B, int q, int c, double* U, const double* V, void* stream) {
  return local_correct(n_blocks, B, q, c, U, V, S_(stream));
}

size_t lmg_local_workspace(int L, int B, int q) {
  return local_part_doubles(L, B, q) * sizeof(double);
}

int lmg_local_residual_post(const lmg_system* sys, int B, int c, const double* U,
                            const double* src, int src_mode, const double* P, int is_first,
                            double* block_part, void* work, double* Q, void* stream) {
  TRY(check_sys(sys, B));
  TRY(check_levels(*sys, 2, c));
  return local_residual_post(*sys, B, c, U, src, src_mode, P, is_first != 0, block_part,
                             reinterpret_cast<double*>(work), Q, S_(stream));
}

int lmg_local_residual_full_a(const lmg_system* sys, int B, const double* U, const double* src,
                              int src_mode, int has_next, double* adv_out, void* work,
                              void* stream) {
  TRY(check_sys(sys, B));
  return local_residual_full_a(*sys, B, U, src, src_mode, has_next != 0, adv_out,
                               reinterpret_cast<double*>(work), S_(stream));
}

int lmg_local_residual_full_b(const lmg_system* sys, int B, int c, const double* U,
                              const double* src, int src_mode, const double* adv_in, int is_first,
                              double* block_part, void* work, void* stream) {
  TRY(check_sys(sys, B));
  if (sys->num_layers % c) return fail(LMG_ERR_CONFIGURATION, "rank's layers are not whole blocks");
  if (!is_first && !adv_in) return fail(LMG_ERR_PROTOCOL, "non-first rank needs the previous rank's adv row");
  return local_residual_full_b(*sys, B, c, U, src, src_mode, adv_in, is_first != 0, block_part,
                               reinterpret_cast<double*>(work), S_(stream));
}

int lmg_norms_from_blocks(const double* block_part, int nblocks, int B, double* norms,
                          void* stream) {
  return norms_from_blocks(block_part, nblocks, B, norms, S_(stream));
}

int lmg_dense_apply(const double* W, const double* b, int act, int M, int q_out, int q_in,
                    const double* X, double* Y, void* stream) {
  if (M < 1 || q_out < 1 || q_in < 1) return fail(LMG_ERR_DIMENSION, "empty transform");
  if (act < 0 || act > 2) return fail(LMG_ERR_CONFIGURATION, "unknown activation");
  StepArgs a{};
  a.M = M; a.N = q_out; a.K = q_in; a.ntasks = 1;
  a.epi = E_APPLY; a.act = act; a.h = 1.0; a.scale = 1.0;
  a.A = X; a.lda = q_in;
  a.Bm = W; a.ldb = q_in;
  a.bias = b;
  a.out = Y; a.ldc = q_out;
  return launch_step(L_FWD, a, S_(stream));
}

int lmg_dense_vjp(const double* W, const double* b, int act, int M, int q_out, int q_in,
                  const double* X, const double* G, double* gX, double* gW, double* gb,
                  double* work, void* stream) {
  if (M < 1 || q_out < 1 || q_in < 1) return fail(LMG_ERR_DIMENSION, "empty transform");
  if (act < 0 || act > 2) return fail(LMG_ERR_CONFIGURATION, "unknown activation");
  cudaStream_t st = S_(stream);
  // work <- act'(X W^T + b)
  StepArgs d{};
  d.M = M; d.N = q_out; d.K = q_in; d.ntasks = 1;
  d.epi = E_DERIV; d.act = act; d.h = 1.0; d.scale = 1.0;
  d.A = X; d.lda = q_in; d.Bm = W; d.ldb = q_in; d.bias = b;
  d.out = work; d.ldc = q_out;
  TRY(launch_step(L_FWD, d, st));
  if (gX) {  // gX = (G * D) W    (m=row, n=input feature, k=output feature)
    StepArgs a{};
    a.M = M; a.N = q_in; a.K = q_out; a.ntasks = 1;
    a.epi = E_APPLY; a.act = LMG_ACT_IDENTITY; a.h = 1.0; a.scale = 1.0;
    a.A = G; a.lda = q_out; a.Ds = work;
    a.Bm = W; a.ldb = q_in;
    a.out = gX; a.ldc = q_in;
    TRY(launch_step(L_ADJ, a, st));
  }
  if (gW) {  // gW = sum_m (G*D)_m (x) x_m
    StepArgs a{};
    a.M = q_out; a.N = q_in; a.K = M; a.ntasks = 1;
    a.epi = E_PGRAD; a.act = LMG_ACT_IDENTITY; a.h = 1.0; a.scale = 1.0; a.lr = 0.0;
    a.A = G; a.lda = q_out; a.Ds = work;
    a.Bm = X; a.ldb = q_in;
    a.out2 = gW; a.ldc = q_in;
    TRY(launch_step(L_PG, a, st));
  }
  if (gb) {
    TRY(launch(CLS_ELEM, 0.0, 0.0, st, [&] { k_bias_grads<<<(q_out + 255) / 256, 256, 0, st>>>(G, 0, work, 1, M, q_out, 1.0, 1.0, 0.0, gb,
                                                       nullptr, 0); }));
  }
  return LMG_OK;
}

int lmg_l2_norms(const double* x, int n, int B, int q, double* norms, void* work, void* stream) {
  if (n < 1 || B < 1 || q < 1) return fail(LMG_ERR_DIMENSION, "empty array");
  cudaStream_t st = S_(stream);
  double* part = reinterpret_cast<double*>(work);
  const int64_t BQ = (int64_t)B * q;
  for (int j = 0; j < n; ++j) {  // one slot per row: sum_b of row j (zero source minus -x)
    TRY(launch(CLS_ELEM, 0.0, 0.0, st, [&] { ew_launch(k_resid_row0, dim3(B), 256, st, x + j * BQ, nullptr, nullptr, part, j, B, q); }));
  }
  return reduce_norms(part, n, B, norms, st);
}

}  // extern "C"

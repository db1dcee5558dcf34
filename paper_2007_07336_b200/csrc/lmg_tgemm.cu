// lmg_tgemm.cu -- warp-specialised persistent FP64 DMMA layer-step GEMM with TMA staging (sm_100a).
//
// The big-batch counterpart of lmg_gemm.cuh's step_gemm (same StepArgs, same task model, same
// fused epilogues, same k-ascending DMMA chain per output -> bitwise identical results):
//   * persistent CTAs (2 per SM) walk the 64 x 64 output tiles of all tasks, task-major so the
//     CTAs working on one layer's W at a time share it in L2;
//   * a producer warp streams the operands with 2D tensor-map TMA into an ST-deep mbarrier ring
//     that runs ahead across tile boundaries (no __syncthreads in the mainloop, no cp.async
//     address arithmetic on the DMMA warps);
//   * 8 DMMA warps own 32 x 16 sub-tiles (8 independent m8n8k4 chains each) and run the fused
//     epilogue straight from registers while the producer already fills the next tile's stages.
// Operand boxes have 32-byte rows, so the 16 lanes of each half-warp of an m8n8k4 fragment load
// read 128 contiguous bytes (64-bit shared loads are served per half-warp; a 128B-swizzled
// 16-k slab measured 2-way conflicted): A = states and D = act' (K-major, {4 k, 64 rows} boxes),
// forward W (K-major, same), adjoint W^T (MN-major W[k][n], {4 n, 16 k} boxes).
//
// A slot is released one stage late (after the next stage's DMMAs issue): ptxas hoists the
// mbarrier arrive above the stage's DMMAs, and the slot's refill is an async-proxy (TMA) write.
#include <cuda.h>

#include <cstdlib>
#include <cstring>

#include "lmg.h"
#include "lmg_async.cuh"
#include "lmg_gemm.cuh"
#include "lmg_tgemm.cuh"

namespace lmg {
namespace {

constexpr int TBM = 64, TBN = 64, TBK = 16;

template <bool ADJ>
struct TG {
  static constexpr int A_SZ = TBM * TBK;  // doubles per operand slab (8 KB)
  static constexpr int B_SZ = TBN * TBK;
  static constexpr int D_SZ = ADJ ? TBM * TBK : 0;
  static constexpr int STAGE = A_SZ + B_SZ + D_SZ;
  static constexpr int ST = ADJ ? 4 : 6;
  static constexpr int NW = 8;  // DMMA warps: 2 (m) x 4 (n) of 32 x 16
  static constexpr int NT = (NW + 1) * 32;
  static constexpr size_t SMEM = (size_t)STAGE * 8 * ST + 2 * ST * 8 + 1024;
  static_assert((A_SZ * 8) % 128 == 0 && (STAGE * 8) % 128 == 0, "TMA destinations 128B-aligned");
};

struct alignas(64) TgParams {
  CUtensorMap amap, bmap, dmap;
  StepArgs a;
  int64_t a_row0, a_rowts;  // A rows of task t: a_row0 + t*a_rowts + m
  int64_t b_row0, b_rowts;  // W rows of task t: b_row0 + t*b_rowts + (n forward | k adjoint)
  int64_t d_row0, d_rowts;
  int mtiles, ntiles, ntiles_total;
};

// K-major slab of four {4 k, 64 rows} boxes: element (row, k) at box k/4
__device__ __forceinline__ int kmaj(int row, int k) { return (k >> 2) * 256 + row * 4 + (k & 3); }

template <bool ADJ, int EPI>
__device__ __forceinline__ void run_epi(const StepArgs& a, const EpiPtrs& q, double (&acc)[4][2][2],
                                        int mrow0, int ncol0) {
  double rowsq[4];
  epilogue<EPI>(a, q, acc, mrow0, ncol0, rowsq);
}

template <bool ADJ>
__global__ void __launch_bounds__(TG<ADJ>::NT, 2) tgemm_kernel(const __grid_constant__ TgParams p) {
  using C = TG<ADJ>;
  const StepArgs& a = p.a;
  extern __shared__ __align__(1024) unsigned char smraw[];
  const uint32_t pad = (1024u - (s_u32(smraw) & 1023u)) & 1023u;
  double* ring = reinterpret_cast<double*>(smraw + pad);
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + C::ST * C::STAGE);
  uint64_t* empty = full + C::ST;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int KT = a.K / TBK;
  const int per_task = p.mtiles * p.ntiles;

  if (tid == 0) {
    for (int i = 0; i < C::ST; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], C::NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == C::NW) {
    // ------------------------------------------------------------------------ producer warp
    if (lane == 0) {
      int g = 0;
      for (int tile = blockIdx.x; tile < p.ntiles_total; tile += gridDim.x) {
        const int t = tile / per_task, r = tile - t * per_task;
        const int mt = r / p.ntiles, nt = r - mt * p.ntiles;
        const int arow = (int)(p.a_row0 + (int64_t)t * p.a_rowts) + mt * TBM;
        const int brow = (int)(p.b_row0 + (int64_t)t * p.b_rowts);
        const int drow = ADJ ? (int)(p.d_row0 + (int64_t)t * p.d_rowts) + mt * TBM : 0;
        for (int kt = 0; kt < KT; ++kt, ++g) {
          const int stg = g % C::ST;
          mbar_wait(&empty[stg], ((uint32_t)(g / C::ST) & 1u) ^ 1u);
          mbar_expect_tx(&full[stg], (uint32_t)(C::STAGE * 8));
          double* dst = ring + stg * C::STAGE;
#pragma unroll
          for (int b = 0; b < TBK / 4; ++b) tma_2d(dst + b * 256, &p.amap, kt * TBK + 4 * b, arow, &full[stg]);
          if (ADJ) {
#pragma unroll
            for (int b = 0; b < TBN / 4; ++b)  // {4 n, 16 k}: W[k][n]
              tma_2d(dst + C::A_SZ + b * 64, &p.bmap, nt * TBN + 4 * b, brow + kt * TBK, &full[stg]);
#pragma unroll
            for (int b = 0; b < TBK / 4; ++b)
              tma_2d(dst + C::A_SZ + C::B_SZ + b * 256, &p.dmap, kt * TBK + 4 * b, drow, &full[stg]);
          } else {
#pragma unroll
            for (int b = 0; b < TBK / 4; ++b)
              tma_2d(dst + C::A_SZ + b * 256, &p.bmap, kt * TBK + 4 * b, brow + nt * TBN, &full[stg]);
          }
        }
      }
    }
    return;
  }

  // ------------------------------------------------------------------------ DMMA warps
  const int fr = lane >> 2, fk = lane & 3;
  const int wm = warp >> 2, wn = warp & 3;  // 32-row x 16-column sub-tile
  int g = 0, prev = -1;
  for (int tile = blockIdx.x; tile < p.ntiles_total; tile += gridDim.x) {
    const int t = tile / per_task, r = tile - t * per_task;
    const int mt = r / p.ntiles, nt = r - mt * p.ntiles;
    double acc[4][2][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    for (int kt = 0; kt < KT; ++kt, ++g) {
      const int stg = g % C::ST;
      mbar_wait(&full[stg], (uint32_t)(g / C::ST) & 1u);
      const double* As = ring + stg * C::STAGE;
      const double* Bs = As + C::A_SZ;
      const double* Ds = Bs + C::B_SZ;
#pragma unroll
      for (int kk = 0; kk < TBK; kk += 4) {
        double af[4], bf[2];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int o = kmaj(wm * 32 + i * 8 + fr, kk + fk);
          af[i] = As[o];
          if (ADJ) af[i] = __dmul_rn(af[i], Ds[o]);
        }
#pragma unroll
        for (int j = 0; j < 2; ++j)
          bf[j] = ADJ ? Bs[((wn * 16 + j * 8 + fr) >> 2) * 64 + (kk + fk) * 4 + (fr & 3)]
                      : Bs[kmaj(wn * 16 + j * 8 + fr, kk + fk)];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 2; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      }
      __syncwarp();
      if (lane == 0 && prev >= 0) mbar_arrive(&empty[prev]);
      prev = stg;
    }

    // fused epilogue (lmg_gemm.cuh), straight from the accumulators
    EpiPtrs q;
    q.bias = a.bias ? a.bias + (int64_t)t * a.bias_ts : nullptr;
    q.X = a.x ? a.x + (int64_t)t * a.x_ts : nullptr;
    q.S = a.s ? a.s + (int64_t)t * a.s_ts : nullptr;
    q.Y = a.y ? a.y + (int64_t)t * a.y_ts : nullptr;
    q.P = a.p ? a.p + (int64_t)t * a.p_ts : nullptr;
    q.O = a.out ? a.out + (int64_t)t * a.out_ts : nullptr;
    q.O2 = a.out2 ? a.out2 + (int64_t)t * a.out2_ts : nullptr;
    const int mrow0 = mt * TBM + wm * 32 + fr, ncol0 = nt * TBN + wn * 16 + 2 * fk;
    switch (a.epi) {
      case E_PROP: run_epi<ADJ, E_PROP>(a, q, acc, mrow0, ncol0); break;
      case E_COARSE: run_epi<ADJ, E_COARSE>(a, q, acc, mrow0, ncol0); break;
      case E_COARSE_R: run_epi<ADJ, E_COARSE_R>(a, q, acc, mrow0, ncol0); break;
      case E_PROPOP: run_epi<ADJ, E_PROPOP>(a, q, acc, mrow0, ncol0); break;
      case E_DERIV: run_epi<ADJ, E_DERIV>(a, q, acc, mrow0, ncol0); break;
      case E_APPLY: run_epi<ADJ, E_APPLY>(a, q, acc, mrow0, ncol0); break;
      default: run_epi<ADJ, E_ADV>(a, q, acc, mrow0, ncol0); break;
    }
  }
}

typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                 const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                 const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                 CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encoder() {
  static EncodeTiled fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &qr) != cudaSuccess ||
        qr != cudaDriverEntryPointSuccess)
      return (EncodeTiled) nullptr;
    return (EncodeTiled)f;
  }();
  return fn;
}

// 2D map [rows][ld] over every task's operand (base + t*ts, `rows` rows each); returns false if
// the operand cannot be described (strides not whole rows, misalignment)
bool make_map(CUtensorMap* map, int64_t* row0, int64_t* rowts, const double* ptr, int64_t ts,
              int ntasks, int rows, int ld, int box0, int box1, bool swizzle) {
  if (!ptr || ld <= 0 || ts % ld != 0) return false;
  const double* lo = ts < 0 ? ptr + (int64_t)(ntasks - 1) * ts : ptr;
  const double* hi = (ts < 0 ? ptr : ptr + (int64_t)(ntasks - 1) * ts) + (int64_t)rows * ld;
  if ((reinterpret_cast<uintptr_t>(lo) & 15) || (ld * 8) % 16) return false;
  const int64_t total = (hi - lo) / ld;
  if (total >= (int64_t)1 << 31) return false;
  *row0 = (ptr - lo) / ld;
  *rowts = ts / ld;
  cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)total};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
  cuuint32_t box[2] = {(cuuint32_t)box0, (cuuint32_t)box1}, estr[2] = {1, 1};
  return encoder()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(lo), dims, strides, box,
                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <bool ADJ>
cudaError_t launch_t(TgParams& prm, cudaStream_t st) {
  using C = TG<ADJ>;
  auto kern = tgemm_kernel<ADJ>;
  static cudaError_t attr = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)C::SMEM);
  if (attr != cudaSuccess) return attr;
  static int sms = [] {
    int dev = 0, n = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  const int grid = prm.ntiles_total < 2 * sms ? prm.ntiles_total : 2 * sms;
  kern<<<grid, C::NT, C::SMEM, st>>>(prm);
  return cudaGetLastError();
}

}  // namespace

// Routing (measured on B200, tools/gemm_bench.py, 256 tasks x 256x512x512): the adjoint layout
// runs 27.4 TF/s here vs 26.3 in step_gemm; the forward 26.9 vs 28.0 (step_gemm's 5 CTAs/SM hide
// the FP64 tanh epilogue better than 2 persistent CTAs), so forward steps stay on step_gemm unless
// LMG_TGEMM=all.
int tgemm_eligible(const StepArgs& a, bool adj) {
  static const bool off = getenv("LMG_NO_TGEMM") != nullptr;
  static const bool all = [] {
    const char* e = getenv("LMG_TGEMM");
    return e && !strcmp(e, "all");
  }();
  if (off || !encoder() || (!adj && !all)) return 0;
  if (a.epi == E_RESID || a.epi == E_PGRAD) return 0;
  if (a.M % TBM || a.N % TBN || a.K % TBK || a.M <= 0 || a.ntasks <= 0) return 0;
  if ((int64_t)a.ntasks * (a.M / TBM) * (a.N / TBN) >= ((int64_t)1 << 31)) return 0;
  if (adj && !a.Ds) return 0;
  return 1;
}

cudaError_t tgemm_launch(const StepArgs& a, bool adj, cudaStream_t st, bool* launched) {
  *launched = false;
  TgParams prm;
  prm.a = a;
  prm.mtiles = a.M / TBM;
  prm.ntiles = a.N / TBN;
  prm.ntiles_total = a.ntasks * prm.mtiles * prm.ntiles;
  // A: rows m of task t (K-major, lda); W: forward rows n (K-major, ldb), adjoint rows k (ldb)
  if (!make_map(&prm.amap, &prm.a_row0, &prm.a_rowts, a.A, a.A_ts, a.ntasks, a.M, a.lda, 4, TBM, false))
    return cudaSuccess;
  if (!make_map(&prm.bmap, &prm.b_row0, &prm.b_rowts, a.Bm, a.B_ts, a.ntasks, adj ? a.K : a.N, a.ldb,
                4, adj ? TBK : TBN, false))
    return cudaSuccess;
  if (adj && !make_map(&prm.dmap, &prm.d_row0, &prm.d_rowts, a.Ds, a.Ds_ts, a.ntasks, a.M, a.lda, 4,
                       TBM, false))
    return cudaSuccess;
  if (!adj) {
    prm.d_row0 = prm.d_rowts = 0;
    prm.dmap = prm.amap;
  }
  *launched = true;
  return adj ? launch_t<true>(prm, st) : launch_t<false>(prm, st);
}

}  // namespace lmg

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

constexpr int TBK = 16;

// BM x BN output tile per CTA, WM x WN DMMA warps (warp tile (BM/WM) x (BN/WN)), ST ring stages,
// MINB CTAs per SM.  Big: 64 x 64, 8 warps of 32 x 16, persistent (2/SM).  Small batch (M <= 16,
// HBM/latency-bound): 16 x 32, 4 warps of 16 x 8, 8 CTAs/SM so one wave covers a c5 sweep step.
template <bool ADJ_, int BM_, int BN_, int WM_, int WN_, int ST_, int MINB_>
struct TG {
  static constexpr bool ADJ = ADJ_;
  static constexpr int BM = BM_, BN = BN_, WM = WM_, WN = WN_, ST = ST_, MINB = MINB_;
  static constexpr int MT = BM / WM / 8, NTF = BN / WN / 8;
  static constexpr int A_SZ = BM * TBK;  // doubles per operand slab
  static constexpr int B_SZ = BN * TBK;
  static constexpr int D_SZ = ADJ ? BM * TBK : 0;
  static constexpr int STAGE = A_SZ + B_SZ + D_SZ;
  static constexpr int NW = WM * WN;
  static constexpr int NT = (NW + 1) * 32;
  static constexpr size_t SMEM = (size_t)STAGE * 8 * ST + 2 * ST * 8 + 1024;
  static_assert((A_SZ * 8) % 128 == 0 && (STAGE * 8) % 128 == 0, "TMA destinations 128B-aligned");
};
using TBig = TG<false, 64, 64, 2, 4, 6, 2>;
using TBigA = TG<true, 64, 64, 2, 4, 4, 2>;
using TSm = TG<false, 16, 32, 1, 4, 4, 8>;
using TSmA = TG<true, 16, 32, 1, 4, 3, 8>;

struct alignas(64) TgParams {
  CUtensorMap amap, bmap, dmap;
  StepArgs a;
  int64_t a_row0, a_rowts;  // A rows of task t: a_row0 + t*a_rowts + m
  int64_t b_row0, b_rowts;  // W rows of task t: b_row0 + t*b_rowts + (n forward | k adjoint)
  int64_t d_row0, d_rowts;
  int mtiles, ntiles, ntiles_total;
};

// K-major slab of four {4 k, ROWS rows} boxes: element (row, k) at box k/4
template <int ROWS>
__device__ __forceinline__ int kmaj(int row, int k) { return (k >> 2) * (ROWS * 4) + row * 4 + (k & 3); }

template <int EPI, int MT, int NTF>
__device__ __forceinline__ void run_epi(const StepArgs& a, const EpiPtrs& q, double (&acc)[MT][NTF][2],
                                        int mrow0, int ncol0) {
  double rowsq[MT];
  epilogue<EPI>(a, q, acc, mrow0, ncol0, rowsq);
}

template <class C>
__global__ void __launch_bounds__(C::NT, C::MINB) tgemm_kernel(const __grid_constant__ TgParams p) {
  constexpr bool ADJ = C::ADJ;
  constexpr int BM = C::BM, BN = C::BN, MT = C::MT, NTF = C::NTF;
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
        const int arow = (int)(p.a_row0 + (int64_t)t * p.a_rowts) + mt * BM;
        const int brow = (int)(p.b_row0 + (int64_t)t * p.b_rowts);
        const int drow = ADJ ? (int)(p.d_row0 + (int64_t)t * p.d_rowts) + mt * BM : 0;
        for (int kt = 0; kt < KT; ++kt, ++g) {
          const int stg = g % C::ST;
          mbar_wait(&empty[stg], ((uint32_t)(g / C::ST) & 1u) ^ 1u);
          mbar_expect_tx(&full[stg], (uint32_t)(C::STAGE * 8));
          double* dst = ring + stg * C::STAGE;
#pragma unroll
          for (int b = 0; b < TBK / 4; ++b) tma_2d(dst + b * BM * 4, &p.amap, kt * TBK + 4 * b, arow, &full[stg]);
          if (ADJ) {
#pragma unroll
            for (int b = 0; b < BN / 4; ++b)  // {4 n, 16 k}: W[k][n]
              tma_2d(dst + C::A_SZ + b * 64, &p.bmap, nt * BN + 4 * b, brow + kt * TBK, &full[stg]);
#pragma unroll
            for (int b = 0; b < TBK / 4; ++b)
              tma_2d(dst + C::A_SZ + C::B_SZ + b * BM * 4, &p.dmap, kt * TBK + 4 * b, drow, &full[stg]);
          } else {
#pragma unroll
            for (int b = 0; b < TBK / 4; ++b)
              tma_2d(dst + C::A_SZ + b * BN * 4, &p.bmap, kt * TBK + 4 * b, brow + nt * BN, &full[stg]);
          }
        }
      }
    }
    return;
  }

  // ------------------------------------------------------------------------ DMMA warps
  const int fr = lane >> 2, fk = lane & 3;
  const int wm = warp / C::WN, wn = warp % C::WN;  // (BM/WM) x (BN/WN) sub-tile
  constexpr int WTM = BM / C::WM, WTN = BN / C::WN;
  int g = 0, prev = -1;
  for (int tile = blockIdx.x; tile < p.ntiles_total; tile += gridDim.x) {
    const int t = tile / per_task, r = tile - t * per_task;
    const int mt = r / p.ntiles, nt = r - mt * p.ntiles;
    double acc[MT][NTF][2];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int j = 0; j < NTF; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    for (int kt = 0; kt < KT; ++kt, ++g) {
      const int stg = g % C::ST;
      mbar_wait(&full[stg], (uint32_t)(g / C::ST) & 1u);
      const double* As = ring + stg * C::STAGE;
      const double* Bs = As + C::A_SZ;
      const double* Ds = Bs + C::B_SZ;
#pragma unroll
      for (int kk = 0; kk < TBK; kk += 4) {
        double af[MT], bf[NTF];
#pragma unroll
        for (int i = 0; i < MT; ++i) {
          const int o = kmaj<BM>(wm * WTM + i * 8 + fr, kk + fk);
          af[i] = As[o];
          if (ADJ) af[i] = __dmul_rn(af[i], Ds[o]);
        }
#pragma unroll
        for (int j = 0; j < NTF; ++j)
          bf[j] = ADJ ? Bs[((wn * WTN + j * 8 + fr) >> 2) * 64 + (kk + fk) * 4 + (fr & 3)]
                      : Bs[kmaj<BN>(wn * WTN + j * 8 + fr, kk + fk)];
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
          for (int j = 0; j < NTF; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
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
    const int mrow0 = mt * BM + wm * WTM + fr, ncol0 = nt * BN + wn * WTN + 2 * fk;
    switch (a.epi) {
      case E_PROP: run_epi<E_PROP>(a, q, acc, mrow0, ncol0); break;
      case E_COARSE: run_epi<E_COARSE>(a, q, acc, mrow0, ncol0); break;
      case E_COARSE_R: run_epi<E_COARSE_R>(a, q, acc, mrow0, ncol0); break;
      case E_PROPOP: run_epi<E_PROPOP>(a, q, acc, mrow0, ncol0); break;
      case E_DERIV: run_epi<E_DERIV>(a, q, acc, mrow0, ncol0); break;
      case E_APPLY: run_epi<E_APPLY>(a, q, acc, mrow0, ncol0); break;
      default: run_epi<E_ADV>(a, q, acc, mrow0, ncol0); break;
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

template <class C>
cudaError_t launch_t(TgParams& prm, cudaStream_t st) {
  auto kern = tgemm_kernel<C>;
  static cudaError_t attr = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)C::SMEM);
  if (attr != cudaSuccess) return attr;
  static int sms = [] {
    int dev = 0, n = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  const int slots = C::MINB * sms;
  const int grid = prm.ntiles_total < slots ? prm.ntiles_total : slots;
  kern<<<grid, C::NT, C::SMEM, st>>>(prm);
  return cudaGetLastError();
}

}  // namespace

// Routing (measured on B200, opt-in since round 2): big batches (M % 64 == 0; 256 tasks x
// 256x512x512).  Round 1 routed the adjoint layout here (27.4 TF/s vs 26.3 in step_gemm with the
// act' scaling applied per fragment); once step_gemm scaled each staged element once and ran
// 2-stage 32 x 128 tiles (lmg.cu TAdj) the whole c2 step was faster there (1018-1024 vs
// 1037-1050 ms; scaling once per element here too -- a slab pass behind a named barrier plus a
// proxy fence -- measured slower than the per-fragment DMULs).  LMG_TGEMM=adj routes big adjoint
// steps here, =all also the forward steps.  The 16 x 32 small-batch variant (M = 16, the c5
// regime) is bitwise too but measured slower than step_gemm's 16-row tiles (c5 fine-level step
// 3.40 vs 3.76 TB/s): LMG_TGEMM=small.
namespace {
int tile_kind(const StepArgs& a, bool adj) {  // 0: none, 1: big, 2: small
  static const bool off = getenv("LMG_NO_TGEMM") != nullptr;
  static const int mode = [] {  // 0 default (off), 1 all, 2 small, 3 adjoint
    const char* e = getenv("LMG_TGEMM");
    return !e ? 0 : !strcmp(e, "all") ? 1 : !strcmp(e, "small") ? 2 : !strcmp(e, "adj") ? 3 : 0;
  }();
  if (off || mode == 0 || !encoder()) return 0;
  if (a.epi == E_RESID || a.epi == E_PGRAD || a.M <= 0 || a.ntasks <= 0 || a.K % TBK) return 0;
  if (adj && !a.Ds) return 0;
  if (mode == 2 && a.M == 16 && a.N % 32 == 0) return 2;
  if (a.M % 64 == 0 && a.N % 64 == 0 && ((adj && mode == 3) || mode == 1)) return 1;
  return 0;
}
}  // namespace

struct TgPlan {
  TgParams prm;
  int kind = 0;
};

bool tgemm_prepare(const StepArgs& a, bool adj, TgPlan** plan) {
  *plan = nullptr;
  const int kind = tile_kind(a, adj);
  if (!kind) return false;
  const int BM = kind == 1 ? 64 : 16, BN = kind == 1 ? 64 : 32;
  if ((int64_t)a.ntasks * (a.M / BM) * (a.N / BN) >= ((int64_t)1 << 31)) return false;
  TgPlan* pl = new TgPlan;
  TgParams& prm = pl->prm;
  prm.a = a;
  prm.mtiles = a.M / BM;
  prm.ntiles = a.N / BN;
  prm.ntiles_total = a.ntasks * prm.mtiles * prm.ntiles;
  // A: rows m of task t (K-major, lda); W: forward rows n (K-major, ldb), adjoint rows k (ldb)
  bool ok = make_map(&prm.amap, &prm.a_row0, &prm.a_rowts, a.A, a.A_ts, a.ntasks, a.M, a.lda, 4, BM, false) &&
            make_map(&prm.bmap, &prm.b_row0, &prm.b_rowts, a.Bm, a.B_ts, a.ntasks, adj ? a.K : a.N, a.ldb,
                     4, adj ? TBK : BN, false);
  if (ok && adj)
    ok = make_map(&prm.dmap, &prm.d_row0, &prm.d_rowts, a.Ds, a.Ds_ts, a.ntasks, a.M, a.lda, 4, BM, false);
  if (!ok) {
    delete pl;
    return false;
  }
  if (!adj) {
    prm.d_row0 = prm.d_rowts = 0;
    prm.dmap = prm.amap;
  }
  pl->kind = kind;
  *plan = pl;
  return true;
}

bool tgemm_small(const TgPlan* plan) { return plan->kind == 2; }

cudaError_t tgemm_launch(TgPlan* plan, bool adj, cudaStream_t st) {
  TgParams& prm = plan->prm;
  cudaError_t e;
  if (plan->kind == 1)
    e = adj ? launch_t<TBigA>(prm, st) : launch_t<TBig>(prm, st);
  else
    e = adj ? launch_t<TSmA>(prm, st) : launch_t<TSm>(prm, st);
  delete plan;
  return e;
}

}  // namespace lmg

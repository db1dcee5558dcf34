// lmg_sweep.cu -- persistent fused relaxation sweep (sm_100a).  See lmg_sweep.cuh.
//
// Grid: (CS, batch tiles, chains); cluster (CS, 1, 1).  CTA r of a cluster owns output columns
// [r*NC, (r+1)*NC) of every step of its chain.  Per CTA:
//   warps 0..NW-1  consumers: DMMA m8n8k4 mainloop (A = the full 16-row state from smem,
//                  B = the streamed W slice), fused E_PROP epilogue, DSMEM all-gather of the new
//                  state slice into every CTA's next A buffer, one cluster barrier per step
//   warp NW        producer: 2D tensor-map TMA loads of the W slice into an ST-deep ring
//                  guarded by full/empty mbarriers; it runs ahead across step boundaries
// Shared memory (1024-aligned): ring (ST stages) | A[2][16][q+4] (double-buffered state, +4
// padding: conflict-free fragments) | xs[16][NC] (adjoint) | mbarriers.
// W stage layouts (both give the minimum two wavefronts per m8n8k4 B-fragment load):
//   forward  W[n][k] (K-major): BK/16 boxes of {16 k, NC rows}, 128B rows, SWIZZLE_128B
//   adjoint  W[k][n] (MN-major): NC/8 boxes of {8 n, BK rows}, 64B rows, no swizzle
//
// Step s of a chain produces layer row j = r0 + 1 + s from row j-1 with block j-1:
//   o = s_j + (u + h*act(W_{j-1} u + b_{j-1}))               forward  (network.py:100)
//   o = s_j + (m + h*(W_{j-1}^T (D_{j-1} * m)))               adjoint  (training.py:216-224)
// SW_FCF chain k (block k of the level, nb = n/c blocks):
//   k = 0:  start at f[0] (the C row of block 0 after c_relaxation, multigrid.py:157); rows
//           1..c-1 -> U (second F sweep), row c -> P[1] (if nb > 1)
//   k >= 1: start at the OLD C row U[(k-1)c] (or Q[k-1] = its first step, already computed);
//           rows (k-1)c+1..kc-1 are block k-1's first F sweep (transient: only feed the C step),
//           row kc is the C step -> Cn[k], rows kc+1..kc+c-1 -> U (second F sweep), row (k+1)c
//           -> P[k+1] (if k < nb-1).  advH[k] = U[kc] + h2*act(pre) at row kc+1.
//   That is exactly multigrid.py:160-172 (F, C, F) plus the C-row propagation of :208: the same
//   layer steps on the same operands, regrouped by chain.  C rows go to Cn (not U) because chain
//   k+1 reads the old U[kc]; the caller commits Cn -> U[kc] and f[0] -> U[0] afterwards.
// SW_SEQ (one chain per batch tile): start at f[0], rows 1..n-1 -> U.
#include <cooperative_groups.h>
#include <cuda.h>

#include <cstdlib>

#include "lmg.h"
#include "lmg_gemm.cuh"
#include "lmg_sweep.cuh"
#include "lmg_async.cuh"

namespace lmg {
namespace {

namespace cg = cooperative_groups;

constexpr int SW_BM = 16;  // batch rows per chain tile (two m8 fragments)
constexpr int SMEM_MAX = 232448;

template <int NC_, int KS_, int ST_, bool ADJ_, int BK_ = 32>
struct SwCfg {
  static constexpr int NC = NC_, KS = KS_, BK = BK_, ST = ST_;
  static constexpr bool ADJ = ADJ_;
  static constexpr int MT = SW_BM / 8;
  static constexpr int NFG = NC / 8;        // 8-column fragment groups (one per warp, per k-split)
  static constexpr int NW = NFG * KS;       // consumer warps; warp = ks * NFG + fg
  static constexpr int NT = (NW + 1) * 32;  // + producer warp
  static constexpr int LDS_ = NC + 4;       // padded row of one state slice: conflict-free A frags
  static constexpr int SL = SW_BM * LDS_;   // doubles per slice (16 rows x NC columns of one rank)
  static constexpr int STAGE = NC * BK;     // doubles, dense (TMA boxes)
  static constexpr int BOXES = ADJ ? NC / 8 : BK / 16;  // fewer, wider boxes: TMA issue-bound
                                                       // (32B-row boxes measured slower here)
  static constexpr int BOX = STAGE / BOXES;
  static_assert((STAGE * 8) % 1024 == 0, "stages must keep the 1024B swizzle alignment");
  static_assert(BK % (4 * KS) == 0, "k-split must divide the stage");
  static size_t smem(int q) {
    const int cs = q / NC;
    return sizeof(double) * ((size_t)ST * STAGE + 2 * (size_t)cs * SL + 2 * (size_t)NFG * 32 * 4 * (KS - 1) +
                             (ADJ ? (size_t)SW_BM * NC : 0)) +
           (2 * ST + 2) * sizeof(uint64_t) + 1024;  // + alignment slack
  }
};

// kernel parameter block: the sweep plus the W tensor map (a 2D view [rows][q] of the weight
// stack; block j's first row is row_off + j*row_stride)
struct alignas(64) SweepParams {
  CUtensorMap wmap;
  SweepArgs a;
  int64_t row_off, row_stride;
};

struct Chain {
  int r0, nsteps;
  const double* start;
};

__device__ __forceinline__ Chain chain_of(const SweepArgs& a, int k, int64_t BQ) {
  Chain ch;
  if (a.mode == SW_SEQ) {
    ch.r0 = 0;
    ch.nsteps = a.n - 1;
    ch.start = a.src;
    return ch;
  }
  const int c = a.c, nb = a.n / c;
  const bool p_last = a.has_next || nb > 1;  // block nb-1 / chain k < nb-1 has a P step
  if (k == 0) {
    ch.r0 = 0;
    ch.start = a.is_first ? a.src : a.U;  // f[0], or U[0] finished from the incoming halo
    ch.nsteps = (c - 1) + (p_last ? 1 : 0);
    return ch;
  }
  if (a.Q) {
    ch.r0 = (k - 1) * c + 1;
    ch.start = a.Q + (int64_t)(k - 1) * BQ;
  } else {
    ch.r0 = (k - 1) * c;
    ch.start = a.U + (int64_t)ch.r0 * BQ;
  }
  const int lastrow = k == nb ? nb * c  // halo chain: up to the next rank's C row
                              : k * c + c - 1 + ((k < nb - 1 || a.has_next) ? 1 : 0);
  ch.nsteps = lastrow - ch.r0;
  return ch;
}

// destination of row j in chain k (SW_FCF) or row j (SW_SEQ); nullptr = transient row
__device__ __forceinline__ double* dest_of(const SweepArgs& a, int k, int j, int64_t BQ) {
  if (a.mode == SW_SEQ) return a.U + (int64_t)j * BQ;
  const int c = a.c;
  if (j < k * c) return nullptr;
  if (j == k * c) return k == a.n / c ? a.halo : a.Cn + (int64_t)k * BQ;  // k >= 1 here
  if (j < (k + 1) * c) return a.U + (int64_t)j * BQ;
  return a.P + (int64_t)(k + 1) * BQ;
}

// remote (or own) 16-byte store completing on the destination CTA's mbarrier
__device__ __forceinline__ void st_async2(uint32_t dst, double a, double b, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(dst),
               "d"(a), "d"(b), "r"(bar)
               : "memory");
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void consumers_sync(int n) {
  asm volatile("bar.sync 1, %0;" ::"r"(n) : "memory");
}

// State layout in shared memory: A[buf][rank][16][NC+4] -- the 16 x q state of one batch tile as
// CS column slices, each padded; rank r's slice is written by CTA r and pushed to the others.
template <class C>
__global__ void __launch_bounds__(C::NT, 1) sweep_kernel(const __grid_constant__ SweepParams p) {
  constexpr int NC = C::NC, KS = C::KS, BK = C::BK, ST = C::ST, MT = C::MT, NW = C::NW;
  constexpr int NFG = C::NFG, SL = C::SL, LDS_ = C::LDS_;
  constexpr bool ADJ = C::ADJ;
  const SweepArgs& a = p.a;
  extern __shared__ __align__(1024) unsigned char smraw[];
  double* ring = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  const int q = a.q;
  cg::cluster_group cl = cg::this_cluster();
  const int CS = (int)cl.num_blocks();
  const int rank = (int)cl.block_rank();
  double* Ab = ring + ST * C::STAGE;             // [2][CS][SL]
  double* red = Ab + 2 * CS * SL;                // [2][NFG][32][4] k-split partials (by step parity)
  double* xs = red + 2 * NFG * 32 * 4 * (KS - 1);  // [16][NC] adjoint: own slice, unscaled
  uint64_t* full = reinterpret_cast<uint64_t*>(xs + (ADJ ? SW_BM * NC : 0));
  uint64_t* empty = full + ST;
  uint64_t* sready = empty + ST;                 // [2]: peer slices of A[buf] have landed

  const int n0 = rank * NC;
  const int k = a.k0 + (int)blockIdx.z;
  const int m0 = blockIdx.y * SW_BM;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t BQ = (int64_t)a.B * q;
  const Chain ch = chain_of(a, k, BQ);
  const int KT = q / BK;
  if (ch.nsteps <= 0) return;  // uniform over the cluster

  if (tid == 0) {
    for (int i = 0; i < ST; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], NW);
    }
    mbar_init(&sready[0], 1);
    mbar_init(&sready[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == NW) {
    // ------------------------------------------------------------------ producer warp
    cluster_arrive();  // startup: peers' barriers are initialised before any push lands
    cluster_wait();
    if (lane == 0) {
      int g = 0;
      for (int s = 0; s < ch.nsteps; ++s) {
        const int row = (int)(p.row_off + (int64_t)(ch.r0 + s) * p.row_stride);  // block r0+s
        for (int kt = 0; kt < KT; ++kt, ++g) {
          const int stg = g % ST;
          mbar_wait(&empty[stg], ((uint32_t)(g / ST) & 1u) ^ 1u);
          mbar_expect_tx(&full[stg], (uint32_t)(C::STAGE * 8));
          double* dst = ring + stg * C::STAGE;
#pragma unroll
          for (int b = 0; b < C::BOXES; ++b) {
            if (ADJ)  // {8 n, BK k} at (n0 + 8b, k rows kt*BK..)
              tma_2d(dst + b * C::BOX, &p.wmap, n0 + 8 * b, row + kt * BK, &full[stg]);
            else      // {16 k, NC n} at (k kt*BK + 16b, n rows n0..)
              tma_2d(dst + b * C::BOX, &p.wmap, kt * BK + 16 * b, row + n0, &full[stg]);
          }
        }
      }
    }
    __syncwarp();
    cluster_arrive();  // exit: no CTA leaves while a peer may still push into it
    cluster_wait();
    return;
  }

  // -------------------------------------------------------------------- consumer warps
  const int NCT = NW * 32;
  {  // start state: A[0] = rows m0..m0+15 of the chain's start row (zero beyond the batch)
    const double* Dst = ADJ ? a.D + (int64_t)ch.r0 * a.d_stride : nullptr;
    const int h2 = q / 2;
    for (int e = tid; e < SW_BM * h2; e += NCT) {
      const int m = e / h2, n = (e - m * h2) * 2;
      double2 v = make_double2(0.0, 0.0);
      if (m0 + m < a.B) v = *reinterpret_cast<const double2*>(ch.start + (int64_t)(m0 + m) * q + n);
      if (ADJ) {
        if (n >= n0 && n < n0 + NC) *reinterpret_cast<double2*>(xs + m * NC + n - n0) = v;
        if (m0 + m < a.B) {
          const double2 d = *reinterpret_cast<const double2*>(Dst + (int64_t)(m0 + m) * q + n);
          v.x = __dmul_rn(v.x, d.x);
          v.y = __dmul_rn(v.y, d.y);
        }
      }
      *reinterpret_cast<double2*>(Ab + (n / NC) * SL + m * LDS_ + (n % NC)) = v;
    }
  }
  consumers_sync(NCT);
  cluster_arrive();  // startup (pairs with the producer's)
  cluster_wait();

  const int fr = lane >> 2, fk = lane & 3;
  const int fg = warp % NFG, ks = warp / NFG;
  const int nl = fg * 8 + 2 * fk;  // this lane's output columns (nl, nl+1) within the slice
  // this warp's k4 chunks of a stage: kk = 4*KS*i + 4*ks; the ks part is folded into per-thread
  // offsets so the chunk loop is fully unrolled.  B fragment: forward W[n = 8fg+fr][k] in
  // 128B-swizzled rows (16B chunk ^= row & 7; the kk bits and 2ks are disjoint), adjoint W[k][n]
  // in box fg, 64B rows.
  const int t_sw = ((fk >> 1) ^ fr) ^ (2 * ks);
  const int b_thr = ADJ ? fg * C::BOX + (fk + 4 * ks) * 8 + fr : (fg * 8 + fr) * 16 + (fk & 1);
  const int a_thr = fr * LDS_ + fk + 4 * ks;
  const uint32_t bytes_in = (uint32_t)(SW_BM * q * 8);  // one full 16 x q state per step
  // cluster addresses of A[buf][rank] (this CTA's slice) and sready[buf] in every CTA
  const uint32_t slice_a = s_u32(Ab + rank * SL);
  const uint32_t sready_a = s_u32(&sready[0]);
  int g = 0, prev_stg = -1;
  for (int s = 0; s < ch.nsteps; ++s) {
    const int cur = s & 1;
    const int j = ch.r0 + 1 + s;  // row produced
    const bool last = (s + 1 == ch.nsteps);
    if (tid == 0 && !last) mbar_expect_tx(&sready[cur ^ 1], bytes_in);
    // epilogue operands, fetched now so their latency hides behind the mainloop
    double bia[2] = {0.0, 0.0}, src[MT][2], dn[MT][2];
    const double* srow = (a.src && (!a.src_head || j == 0)) ? a.src + (int64_t)j * BQ : nullptr;
    const double* brow = (!ADJ && a.bias) ? a.bias + (int64_t)(j - 1) * a.b_stride : nullptr;
    const double* drow = (ADJ && !last) ? a.D + (int64_t)j * a.d_stride : nullptr;
    {
      if (brow) {
        const double2 v = *reinterpret_cast<const double2*>(brow + n0 + nl);
        bia[0] = v.x;
        bia[1] = v.y;
      }
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        const int m = m0 + i * 8 + fr;
        src[i][0] = src[i][1] = dn[i][0] = dn[i][1] = 0.0;
        if (m < a.B && srow) {
          const double2 v = *reinterpret_cast<const double2*>(srow + (int64_t)m * q + n0 + nl);
          src[i][0] = v.x;
          src[i][1] = v.y;
        }
        if (m < a.B && drow) {
          const double2 v = *reinterpret_cast<const double2*>(drow + (int64_t)m * q + n0 + nl);
          dn[i][0] = v.x;
          dn[i][1] = v.y;
        }
      }
    }
    const bool tr = a.trace && tid == 0 && blockIdx.z == 0 && rank == 0 && blockIdx.y == 0;
    if (tr) a.trace[4 * s] = gtimer();
    if (s > 0) mbar_wait(&sready[cur], (uint32_t)((s - 1) >> 1) & 1u);
    if (tr) a.trace[4 * s + 1] = gtimer();

    double acc[MT][2];
#pragma unroll
    for (int i = 0; i < MT; ++i) acc[i][0] = acc[i][1] = 0.0;
    const double* Acur = Ab + cur * CS * SL;
    for (int kt = 0; kt < KT; ++kt, ++g) {
      const int stg = g % ST;
      mbar_wait(&full[stg], (uint32_t)(g / ST) & 1u);
      const double* Bs = ring + stg * C::STAGE + b_thr;
      // stage kt covers k in [kt*BK, kt*BK+BK): slice (kt*BK)/NC, columns (kt*BK)%NC ..
      const double* Ak = Acur + ((kt * BK) / NC) * SL + ((kt * BK) % NC) + a_thr;
#pragma unroll
      for (int kk = 0; kk < BK; kk += 4 * KS) {
        double af[MT];
#pragma unroll
        for (int i = 0; i < MT; ++i) af[i] = Ak[i * 8 * LDS_ + kk];
        const double bf = ADJ ? Bs[kk * 8] : Bs[(kk >> 4) * C::BOX + ((((kk & 15) >> 1) ^ t_sw) << 1)];
#pragma unroll
        for (int i = 0; i < MT; ++i) dmma(acc[i][0], acc[i][1], af[i], bf);
      }
      // Release the PREVIOUS stage's slot, not this one: the slot's next fill is an async-proxy
      // (TMA) write, and ptxas hoists the arrive above this stage's DMMAs, i.e. possibly before
      // this stage's LDS have returned (observed: stale W boxes under load).  The previous
      // stage's LDS results were consumed by DMMAs issued before this stage's, so its reads are
      // complete.  (A fence.proxy.async per stage also works but costs ~1 us per step.)
      __syncwarp();
      if (lane == 0 && prev_stg >= 0) mbar_arrive(&empty[prev_stg]);
      prev_stg = stg;
    }

    if (tr) a.trace[4 * s + 2] = gtimer();
    // k-split partials (KS = 2): the two warps of a pair swap halves through smem and each
    // finishes one m-fragment, summing in fixed order (ks = 0 part + ks = 1 part)
    int i_lo = 0, i_hi = MT;
    if (KS > 1) {
      // double-buffered by step parity: step s+1's hand-over cannot overwrite the slots the
      // partner warp reads at step s even without the all-gather's ordering (which racecheck
      // cannot see through the st.async / mbarrier chain)
      double* r = red + ((cur * NFG + fg) * 32 + lane) * 4;
      // the fragment this warp hands over: 1 (ks 0) or 0 (ks 1)
      r[2 * ks] = ks == 0 ? acc[MT - 1][0] : acc[0][0];
      r[2 * ks + 1] = ks == 0 ? acc[MT - 1][1] : acc[0][1];
      asm volatile("bar.sync %0, 64;" ::"r"(1 + fg) : "memory");
      const double p0 = r[2 * (1 - ks)], p1 = r[2 * (1 - ks) + 1];
      if (ks == 0) {  // fragment 0: own (ks 0) + partner (ks 1)
        acc[0][0] = acc[0][0] + p0;
        acc[0][1] = acc[0][1] + p1;
      } else {        // fragment 1: partner (ks 0) + own (ks 1)
        acc[MT - 1][0] = p0 + acc[MT - 1][0];
        acc[MT - 1][1] = p1 + acc[MT - 1][1];
      }
      i_lo = ks;
      i_hi = ks + 1;
    }

    // ---------------------------------------------------------------- fused E_PROP epilogue
    double* drow_out = dest_of(a, k, j, BQ);
    double* adv_out = (a.mode == SW_FCF && a.advH && j == k * a.c + 1) ? a.advH + (int64_t)k * BQ
                                                                      : nullptr;
    const double* own = Acur + rank * SL;
    const uint32_t nxt_off = (uint32_t)(((cur ^ 1) * CS * SL) * 8);
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      if (i < i_lo || i >= i_hi) continue;
      const int ml = i * 8 + fr;
      const int m = m0 + ml;
      double o[2], nx[2], ad[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        double pre = acc[i][e];
        if (brow) pre = __dadd_rn(pre, bia[e]);
        const double v = ADJ ? pre : act_fwd(a.act, pre);
        const double x = ADJ ? xs[ml * NC + nl + e] : own[ml * LDS_ + nl + e];
        const double adv = __dadd_rn(x, __dmul_rn(a.h, v));
        o[e] = __dadd_rn(srow ? src[i][e] : 0.0, adv);
        ad[e] = adv_out ? __dadd_rn(x, __dmul_rn(a.h2, v)) : 0.0;
        nx[e] = ADJ ? __dmul_rn(o[e], dn[i][e]) : o[e];
        if (ADJ) xs[ml * NC + nl + e] = o[e];
      }
      if (!last) {  // all-gather: this pair of the new state into A[cur^1] of every CTA
        const uint32_t off = nxt_off + (uint32_t)((ml * LDS_ + nl) * 8);
        for (int r = 0; r < CS; ++r) {
          const int dr = rank + r < CS ? rank + r : rank + r - CS;
          st_async2(mapa(slice_a + off, dr), nx[0], nx[1], mapa(sready_a + 8 * (cur ^ 1), dr));
        }
      }
      if (m < a.B) {
        if (drow_out)
          *reinterpret_cast<double2*>(drow_out + (int64_t)m * q + n0 + nl) = make_double2(o[0], o[1]);
        if (adv_out)
          *reinterpret_cast<double2*>(adv_out + (int64_t)m * q + n0 + nl) = make_double2(ad[0], ad[1]);
      }
    }
    if (tr) a.trace[4 * s + 3] = gtimer();
  }
  __syncwarp();
  cluster_arrive();  // exit
  cluster_wait();
}

// NC = 64: cluster q/64, 8 consumer warps (bitwise the per-step kernel: one k-ascending chain);
// NC = 32: cluster q/32, 8 consumer warps as two k-split halves (2 warps per SMSP)
using Cfg64F = SwCfg<64, 1, 5, false>;
// (9 ring stages for the 32-column shapes measured: forward unchanged, adjoint 1.30 -> 1.79 ms
// per c5 step -- its act' rows leave no room)
using Cfg32F = SwCfg<32, 2, 7, false>;
using Cfg64A = SwCfg<64, 1, 5, true>;
using Cfg32A = SwCfg<32, 2, 7, true>;
// 128 columns per CTA (cluster q/128, 16 DMMA warps, 16-k stages): for serial solves of many
// batch tiles -- at q = 512 only 15 eight-CTA clusters are co-resident, so B = 256 (16 tiles)
// needs the 4-CTA clusters to stay in one wave
using Cfg128F = SwCfg<128, 1, 5, false, 16>;
using Cfg128A = SwCfg<128, 1, 4, true, 16>;
// 16 columns per CTA, 16-k stages: narrow networks (q = 16 -- BASELINE.md 3.4's survey shape, the
// latency-bound regime), one CTA per chain
using Cfg16F = SwCfg<16, 1, 6, false, 16>;
using Cfg16A = SwCfg<16, 1, 6, true, 16>;

// ------------------------------------------------------------------------------------------
// Warp-level FMA sweep (cfg WSWEEP): narrow networks, q <= 32 -- a layer step is a q x q matvec
// per sample (a few hundred flops), far too small for tensor-core tiles and a cluster
// all-gather per step (north_star: "warp-level FMA paths otherwise").  One CTA per (chain,
// group of up to WPB samples), one warp per sample; lane i holds state column i in a register
// for all of the chain's steps.  The serial chain is latency-bound, so nothing the step needs
// may be a global round trip: every operand of step s -- W block, bias row, source and act'
// rows of the CTA's samples -- streams through a per-CTA cp.async ring WST-1 steps ahead, and
// the tanh table sits in shared memory.  W rows are padded to KM+1 doubles so both the forward
// (lane i reads row i) and the adjoint (lane n reads column n) fragments are conflict-free.
// The step: pre_i = sum_k W[i][k] x_k as ONE k-ascending FMA chain (x_k broadcast by shuffles)
// -- bitwise what one DMMA m8n8k4 chain computes (tools/dmma_fma_probe.cu: 0 mismatches in 4M
// outputs), so this path is bitwise the per-step and cluster paths -- then the E_PROP epilogue
// with the reference's rounding.  Same chains, destinations and transient rows as sweep_kernel.
constexpr int WST = 4;
constexpr int WPB_MAX = 8;
// samples (warps) per CTA: 1, 2, 4 or 8 (a compile-time copy split per CTA size)
__host__ __device__ inline int wsweep_wpb(int B) { return B >= 5 ? 8 : B >= 3 ? 4 : B; }

// one ring stage: W block (forward stored transposed, so both directions read [k][lane]), bias
// row, the CTA's source rows and act' rows
template <int KM>
struct WStage {
  static constexpr int W = 0, BIAS = KM * KM, SRC = BIAS + KM, D = SRC + WPB_MAX * KM;
  static constexpr int SIZE = D + WPB_MAX * KM;  // doubles
};

// V (measurement knob LMG_WSWEEP_V, 1 or 3): 1 = the next stage's copies issued after the
// matvec; 3 = a quarter into its FMA chain (they fill its dependency stalls).  Measured and
// dropped: 0 = before the matvec (the LDGSTS then queue ahead of its LDS), 2 = the state broadcast
// through shared memory (LDS.128 pairs) instead of 64-bit shuffles (profiles/r2_wsweep_*)
template <int KM, bool ADJ, int V = 1, int NW = WPB_MAX>
__global__ void __launch_bounds__(32 * NW) wsweep_kernel(const SweepArgs a) {
  using SG = WStage<KM>;
  constexpr int QQ = KM * KM;
  extern __shared__ double wsm[];  // [64] double2 tanh table | [WST][SG::SIZE] ring
  double2* tab = reinterpret_cast<double2*>(wsm);
  double* ring = wsm + 128;
  const int k = a.k0 + (int)blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int nw = NW;  // warps = samples per CTA
  const int b0 = (int)blockIdx.x * nw;
  const int b = b0 + warp;  // this warp's sample
  const int64_t BQ = (int64_t)a.B * KM;
  const Chain ch = chain_of(a, k, BQ);
  if (ch.nsteps <= 0) return;  // uniform over the CTA
  const bool on = b < a.B && lane < KM;  // warps beyond the batch still load and synchronise
  const int li = lane & (KM - 1);
  constexpr int nthr = 32 * NW;
  const int tid = (int)threadIdx.x;
  const int nwb = min(nw, a.B - b0) * KM;  // source / act' elements of this CTA's live samples
  const bool dense_src = a.src && !a.src_head;
  const bool has_b = !ADJ && a.bias;
  const bool tanh_act = !ADJ && a.act == LMG_ACT_TANH;
  if (tanh_act)
    for (int i = tid; i < 64; i += nthr) tab[i] = kTanhExp2[i];
  // programmatic dependent launch: everything below may read upstream results (source rows
  // written by the previous launch); dependents may launch once this grid is running
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  // operand streams of step s (row j = r0 + 1 + s, block j - 1), advanced once per loaded stage
  const double* wl = a.W + (int64_t)ch.r0 * a.w_stride;
  const double* bl = has_b ? a.bias + (int64_t)ch.r0 * a.b_stride : nullptr;
  const double* sl = dense_src ? a.src + (int64_t)(ch.r0 + 1) * BQ + (int64_t)b0 * KM : nullptr;
  const double* dl = ADJ ? a.D + (int64_t)(ch.r0 + 1) * a.d_stride + (int64_t)b0 * KM : nullptr;
  int loaded = 0;
  auto load_next = [&]() {  // everything step `loaded` reads -> slot loaded % WST
    if (loaded < ch.nsteps) {
      double* dst = ring + (loaded % WST) * SG::SIZE;
#pragma unroll
      for (int i = 0; i < (QQ + nthr - 1) / nthr; ++i) {  // straight-line copies (compile-time)
        const int e = tid + i * nthr;
        if (QQ % nthr == 0 || e < QQ) {
          const int r = e / KM, cc = e % KM;  // W[r][cc]
          cp_async<1>(dst + SG::W + (ADJ ? e : cc * KM + r), wl + e, true);
        }
      }
      if (has_b && tid < KM) cp_async<1>(dst + SG::BIAS + tid, bl + tid, true);
#pragma unroll
      for (int i = 0; i < (NW * KM + nthr - 1) / nthr; ++i) {
        const int e = tid + i * nthr;
        if (e < nwb) {
          if (dense_src) cp_async<1>(dst + SG::SRC + e, sl + e, true);
          if (ADJ && loaded + 1 < ch.nsteps)  // act' of row j scales the next step's operand
            cp_async<1>(dst + SG::D + e, dl + e, true);
        }
      }
      wl += a.w_stride;
      if (has_b) bl += a.b_stride;
      if (dense_src) sl += BQ;
      if (ADJ) dl += a.d_stride;
    }
    ++loaded;
    cp_commit();
  };
#pragma unroll
  for (int s = 0; s < WST - 1; ++s) load_next();

  // x: the state (unscaled); xa: the A operand (adjoint: D_row * m)
  double x = 0.0, xa = 0.0;
  if (on) {
    x = ch.start[(int64_t)b * KM + lane];
    xa = ADJ ? __dmul_rn(x, a.D[(int64_t)ch.r0 * a.d_stride + (int64_t)b * KM + lane]) : x;
    if (a.write_row0) a.U[(int64_t)b * KM + lane] = x;  // states[0] = source[0]
    if (a.corrU) {  // row 0's coarse-grid correction
      double* cu = a.corrU + (int64_t)b * KM + lane;
      const double u = *cu;
      *cu = __dadd_rn(u, __dadd_rn(x, -u));
    }
  }
  const bool tr = a.trace && blockIdx.x == 0 && blockIdx.y == 0 && tid == 0;
  // destinations (dest_of) without per-step divisions: SW_SEQ and the U rows of a chain advance by
  // one row per step; the C row, the P row and the advH row are fixed per chain
  const int64_t bq = (int64_t)b * KM;
  const bool fcf = a.mode == SW_FCF;
  const int kc = fcf ? k * a.c : 0;
  const int krow_end = fcf ? kc + a.c : 0;  // rows kc+1 .. kc+c-1 -> U, row (k+1)c -> P
  double* const cptr = fcf ? ((k == a.n / a.c) ? a.halo : a.Cn + (int64_t)k * BQ) + bq : nullptr;
  double* const pptr = fcf ? a.P + (int64_t)(k + 1) * BQ + bq : nullptr;
  double* const aptr = (fcf && a.advH) ? a.advH + (int64_t)k * BQ + bq : nullptr;
  double* urow = a.U + (int64_t)(ch.r0 + 1) * BQ + bq;
  for (int s = 0; s < ch.nsteps; ++s, urow += BQ) {
    const int j = ch.r0 + 1 + s;  // row produced, with block j-1
    const bool last = s + 1 == ch.nsteps;
    if (tr) a.trace[4 * s] = clock64();
    cp_wait<WST - 2>();  // this thread's copies of stage s landed
    __syncthreads();     // ... and everyone's; every warp is done with slot (s-1) % WST
    if (tr) a.trace[4 * s + 1] = clock64();
    // SW_SEQ correction of this step's row: its old value is loaded now, used after the epilogue
    // (a load consumed in the same step would stall the warp's in-order issue for its latency)
    double* cu = (a.corrU && on) ? a.corrU + (int64_t)j * a.corr_ts + bq + lane : nullptr;
    const double cu_old = cu ? *cu : 0.0;
    const double* st = ring + (s % WST) * SG::SIZE;
    const double bia = has_b ? st[SG::BIAS + li] : 0.0;
    const double sv = dense_src ? st[SG::SRC + warp * KM + li] : 0.0;
    const double dn = (ADJ && !last) ? st[SG::D + warp * KM + li] : 0.0;
    double acc = 0.0;
#pragma unroll
    for (int kk = 0; kk < KM; ++kk) {
      const double xk = __shfl_sync(0xffffffffu, xa, kk);
      acc = fma(st[SG::W + kk * KM + li], xk, acc);
      if (V == 3 && kk == KM / 4) load_next();  // copies issued in the FMA chain's stalls
    }
    if (V == 1) load_next();
    if (tr) a.trace[4 * s + 2] = clock64();
    double pre = acc;
    if (has_b) pre = __dadd_rn(pre, bia);
    double v = pre;
    if (!ADJ) v = tanh_act ? fast_tanh_impl(pre, [&](int i) { return tab[i]; }) : act_fwd(a.act, pre);
    const double adv = __dadd_rn(x, __dmul_rn(a.h, v));
    const double o = __dadd_rn(dense_src ? sv : 0.0, adv);
    if (on) {
      double* out = !fcf ? urow : j < kc ? nullptr : j == kc ? cptr : j < krow_end ? urow : pptr;
      if (out) out[lane] = o;
      if (aptr && j == kc + 1) aptr[lane] = __dadd_rn(x, __dmul_rn(a.h2, v));
      if (cu) *cu = __dadd_rn(cu_old, __dadd_rn(o, -cu_old));  // SW_SEQ: k_correct of row j
    }
    x = o;
    xa = ADJ ? __dmul_rn(o, dn) : o;
    if (tr) a.trace[4 * s + 3] = clock64();
  }
}

template <int KM, bool ADJ, int NW>
__global__ void __launch_bounds__(32 * NW) wresid_kernel(const ResidArgs a) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = (int)blockIdx.x * NW + warp, k = (int)blockIdx.y;
  if (b >= a.B) return;  // no block-wide synchronisation below
  const int q = KM;
  const int64_t BQ = (int64_t)a.B * q, bq = (int64_t)b * q;
  const bool on = lane < q;
  const int li = lane & (KM - 1);
  const int kc = k * a.c;
  // 1. correction + C-row partial: k_correct_cpart (one 256-thread tree; lanes >= q hold 0.0)
  double* urow = a.U + (int64_t)kc * BQ + bq;
  double u1 = 0.0, rc = 0.0;
  if (on) {
    const double u0 = urow[lane];
    u1 = __dadd_rn(u0, __dadd_rn(a.V[(int64_t)k * BQ + bq + lane], -u0));
    urow[lane] = u1;
    const double* p = (k == 0 && a.is_first) ? (a.src ? a.src + bq : nullptr) : a.P + (int64_t)k * BQ + bq;
    const double r = __dadd_rn(p ? p[lane] : 0.0, -u1);
    rc = fma(r, r, 0.0);
  }
#pragma unroll
  for (int s2 = 16; s2 >= 1; s2 >>= 1) rc += __shfl_down_sync(0xffffffffu, rc, s2);
  const double cpart = __shfl_sync(0xffffffffu, rc, 0);
  // 2. row kc+1 = one layer step from the corrected U[kc] with block kc (E_RESID)
  const double xa = ADJ ? __dmul_rn(u1, on ? a.D[(int64_t)kc * a.d_stride + bq + lane] : 0.0) : u1;
  const double* Wb = a.W + (int64_t)kc * a.w_stride;
  double acc = 0.0;
#pragma unroll
  for (int kk = 0; kk < KM; ++kk) {
    const double xk = __shfl_sync(0xffffffffu, xa, kk);
    acc = fma(ADJ ? Wb[kk * q + li] : Wb[li * q + kk], xk, acc);
  }
  double pre = acc;
  if (!ADJ && a.bias) pre = __dadd_rn(pre, a.bias[(int64_t)kc * a.b_stride + li]);
  const double v = ADJ ? pre : act_fwd(a.act, pre);
  const double adv = __dadd_rn(u1, __dmul_rn(a.h, v));
  const double sv = (a.src && !a.src_head && on) ? a.src[(int64_t)(kc + 1) * BQ + bq + lane] : 0.0;
  const double prop = __dadd_rn(sv, adv);
  double r = 0.0;
  if (on) {
    r = __dadd_rn(prop, -urow[BQ + lane]);
    if (a.Q) a.Q[(int64_t)k * BQ + bq + lane] = prop;
  }
  // E_RESID row partial: per 16-column warp of the 32-column tile, lane fk accumulates columns
  // 2fk, 2fk+1, 8+2fk, 9+2fk (fma, in that order), then a shfl-xor 1 / 2 tree, then the warps
  // in order from 0.0
  const int g = (lane >> 2) & 1, fk = lane & 3;  // lanes 0..7: (warp g, lane fk)
  double vsum = 0.0;
#pragma unroll
  for (int jj = 0; jj < 2; ++jj)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int n = 16 * g + 8 * jj + 2 * fk + e;
      const double rn = __shfl_sync(0xffffffffu, r, n & 31);
      if (n < q && lane < 8) vsum = fma(rn, rn, vsum);
    }
  vsum += __shfl_xor_sync(0xffffffffu, vsum, 1);
  vsum += __shfl_xor_sync(0xffffffffu, vsum, 2);
  const double w0 = __shfl_sync(0xffffffffu, vsum, 0), w1 = __shfl_sync(0xffffffffu, vsum, 4);
  double fpart = 0.0;
  fpart += w0;
  fpart += w1;
  // 3. block partial (k_combine_post: cpart, then the tile partials)
  if (lane == 0) {
    double s3 = cpart;
    s3 += fpart;
    a.block_part[(int64_t)k * a.B + b] = s3;
  }
}

template <int KM, bool ADJ>
cudaError_t wresid_launch_t(const ResidArgs& a, cudaStream_t st) {
  const int nw = wsweep_wpb(a.B);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((a.B + nw - 1) / nw, a.nb, 1);
  cfg.blockDim = dim3(32 * nw, 1, 1);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = getenv("LMG_NO_PDL") ? 0 : 1;
  switch (nw) {
    case 1: return cudaLaunchKernelEx(&cfg, wresid_kernel<KM, ADJ, 1>, a);
    case 2: return cudaLaunchKernelEx(&cfg, wresid_kernel<KM, ADJ, 2>, a);
    case 4: return cudaLaunchKernelEx(&cfg, wresid_kernel<KM, ADJ, 4>, a);
    default: return cudaLaunchKernelEx(&cfg, wresid_kernel<KM, ADJ, 8>, a);
  }
}

template <int KM>
size_t wsweep_smem() { return sizeof(double) * (128 + (size_t)WST * WStage<KM>::SIZE); }

// default 3 at q 16, 1 at q 32 (tools/_r2_ws_ab*.sh, profiles/r2_wsweep_variants.txt: serial
// propagation at 4096 x 16 B 1: 2.77 (1) vs 3.05 / 3.08 ms (0 / 2), then 2.77 (3) vs 3.04 (1)
// after the epilogue rework; at q 32 variant 3 slowed the c1 step 1.59 -> 2.23 ms)
int wsweep_variant(int q) {
  static const int v = [] {
    const char* e = getenv("LMG_WSWEEP_V");
    return e ? atoi(e) : -1;
  }();
  return v >= 0 ? v : (q <= 16 ? 3 : 1);
}



bool wsweep_enabled() {
  static const bool off = getenv("LMG_NO_WSWEEP") != nullptr;
  return !off;
}

template <int KM, bool ADJ, int V = 1, int NW = WPB_MAX>
cudaError_t wsweep_attr() {
  static const cudaError_t e = cudaFuncSetAttribute(
      wsweep_kernel<KM, ADJ, V, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsweep_smem<KM>());
  return e;
}

template <int KM, bool ADJ>
int wsweep_occupancy() {
  int per = 0;
  if (wsweep_attr<KM, ADJ>() != cudaSuccess) return 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, wsweep_kernel<KM, ADJ>, 32 * WPB_MAX,
                                                    wsweep_smem<KM>()) != cudaSuccess)
    return 0;
  return per;
}

template <int KM, bool ADJ, int V, int NW>
cudaError_t wlaunch_v(const SweepArgs& a, const SweepShape& s, cudaStream_t st) {
  const cudaError_t e = wsweep_attr<KM, ADJ, V, NW>();
  if (e != cudaSuccess) return e;
  static const bool pdl_on = getenv("LMG_NO_PDL") == nullptr;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(s.grid.y, s.grid.z, 1);
  cfg.blockDim = dim3(s.nthreads, 1, 1);
  cfg.dynamicSmemBytes = s.smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_on ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, wsweep_kernel<KM, ADJ, V, NW>, a);
}

template <int KM, bool ADJ>
cudaError_t wlaunch(const SweepArgs& a, const SweepShape& s, cudaStream_t st) {
  auto by_nw = [&](auto vtag) {
    constexpr int V = decltype(vtag)::value;
    switch (s.nthreads / 32) {
      case 1: return wlaunch_v<KM, ADJ, V, 1>(a, s, st);
      case 2: return wlaunch_v<KM, ADJ, V, 2>(a, s, st);
      case 4: return wlaunch_v<KM, ADJ, V, 4>(a, s, st);
      default: return wlaunch_v<KM, ADJ, V, 8>(a, s, st);
    }
  };
  return wsweep_variant(KM) == 3 ? by_nw(std::integral_constant<int, 3>{})
                                 : by_nw(std::integral_constant<int, 1>{});
}

cudaError_t wsweep_launch(const SweepArgs& a, const SweepShape& s, cudaStream_t st) {
  if (a.q <= 16) return a.adj ? wlaunch<16, true>(a, s, st) : wlaunch<16, false>(a, s, st);
  return a.adj ? wlaunch<32, true>(a, s, st) : wlaunch<32, false>(a, s, st);
}

// run f with the configuration tag of (cfg, adjoint)
template <class F>
auto with_cfg(int cfg, bool adj, F&& f) {
  switch (cfg) {
    case 0: return adj ? f(Cfg64A{}) : f(Cfg64F{});
    case 1: return adj ? f(Cfg32A{}) : f(Cfg32F{});
    case 3: return adj ? f(Cfg16A{}) : f(Cfg16F{});
    default: return adj ? f(Cfg128A{}) : f(Cfg128F{});
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

template <class C>
bool fits(int q) {
  return q % C::NC == 0 && q / C::NC <= 16 && q % C::BK == 0 && C::smem(q) <= (size_t)SMEM_MAX &&
         encoder() != nullptr;
}

// W of the level as a 2D tensor [rows][q]: blocks j = 0..n-1 at a.W + j*w_stride
template <class C>
cudaError_t make_params(const SweepArgs& a, SweepParams* p) {
  EncodeTiled enc = encoder();
  if (!enc) return cudaErrorNotSupported;
  const int64_t q = a.q;
  const int64_t span = (int64_t)(a.n - 1) * a.w_stride;  // may be negative (adjoint)
  const double* base = span < 0 ? a.W + span : a.W;
  p->a = a;
  p->row_stride = a.w_stride / q;
  p->row_off = (a.W - base) / q;
  const cuuint64_t rows = (cuuint64_t)((span < 0 ? -span : span) / q + q);
  cuuint64_t dims[2] = {(cuuint64_t)q, rows};
  cuuint64_t strides[1] = {(cuuint64_t)q * 8};
  cuuint32_t box[2], estr[2] = {1, 1};
  if (C::ADJ) {
    box[0] = 8;
    box[1] = C::BK;
  } else {
    box[0] = 16;
    box[1] = C::NC;
  }
  CUresult r = enc(&p->wmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims,
                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   C::ADJ ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <class C>
cudaError_t launch_c(const SweepArgs& a, const SweepShape& s, cudaStream_t st) {
  auto kern = sweep_kernel<C>;
  static cudaError_t attr = [&] {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_MAX);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    return e;
  }();
  if (attr != cudaSuccess) return attr;
  SweepParams prm;
  cudaError_t e = make_params<C>(a, &prm);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = s.grid;
  cfg.blockDim = dim3(C::NT, 1, 1);
  cfg.dynamicSmemBytes = s.smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = s.cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, prm);
}

}  // namespace

// 0: 64 columns per CTA (cluster q/64, one k-ascending chain: bitwise the per-step kernel),
// 1: 32 columns per CTA (cluster q/32, k split over two warps).  Measured on B200 (c5 shapes,
// tools/sweep_bench.py): many independent chains (FCF) -> 0 (more clusters resident, 63 vs 98
// SM-us per layer step); a single serial chain -> 1 (twice the SMs on the critical path).
int sweep_config(int q, int B, int adj, int nchains) {
  (void)B;
  static const int forced_env = [] {
    const char* e = getenv("LMG_SWEEP_CFG");
    return e ? atoi(e) : -1;
  }();
  // narrow networks: the warp-level FMA sweep (one k-ascending chain per output, like cfg 0)
  if ((q == 16 || q == 32) && wsweep_enabled() && (forced_env < 0 || forced_env == SWEEP_CFG_WARP))
    return SWEEP_CFG_WARP;
  const bool ok64 = adj ? fits<Cfg64A>(q) : fits<Cfg64F>(q);
  if (canonical_order()) return ok64 ? 0 : -1;  // one k-ascending chain or the per-step path
  const int forced = forced_env;
  const bool ok32 = adj ? fits<Cfg32A>(q) : fits<Cfg32F>(q);
  if (forced == 0 && ok64) return 0;
  if (forced == 1 && ok32) return 1;
  if (forced == 2 && (adj ? fits<Cfg128A>(q) : fits<Cfg128F>(q))) return 2;
  if (nchains > 16 && ok64) return 0;
  if (!ok32 && !ok64)  // q not a multiple of 32: the 16-column shape
    return (adj ? fits<Cfg16A>(q) : fits<Cfg16F>(q)) ? 3 : -1;
  return ok32 ? 1 : (ok64 ? 0 : -1);
}

int sweep_shape(const SweepArgs& a, SweepShape* s, int forced_cfg) {
  const int nchains = a.mode == SW_SEQ ? 1 : (a.nchains > 0 ? a.nchains : a.n / a.c);
  const int mt = (a.B + SW_BM - 1) / SW_BM;
  int cfg = sweep_config(a.q, a.B, a.adj, nchains);
  if (forced_cfg == SWEEP_CFG_WARP) {
    if (a.q != 16 && a.q != 32) return -1;
    cfg = SWEEP_CFG_WARP;
  } else if (cfg == SWEEP_CFG_WARP && forced_cfg >= 0) {
    cfg = -1;  // a cluster configuration was asked for: the generic selection below
  }
  if (cfg == SWEEP_CFG_WARP) {
    const int wpb = wsweep_wpb(a.B);
    s->cfg = cfg;
    s->cs = 1;
    // one warp per sample (always-8-warp CTAs that only share the copies measured slower for
    // one-sample chains: profiles/r2_wsweep_knobs.txt)
    s->nthreads = 32 * wpb;
    s->smem = a.q <= 16 ? wsweep_smem<16>() : wsweep_smem<32>();
    s->grid = dim3(1, (a.B + wpb - 1) / wpb, nchains);
    return 0;
  }
  if (forced_cfg >= 0) {
    const bool ok = with_cfg(forced_cfg, a.adj, [&](auto c) { return fits<decltype(c)>(a.q); });
    if (ok) cfg = forced_cfg;
    else if (forced_cfg == 2) return -1;
  }
  if (cfg < 0) return -1;
  s->cfg = cfg;
  with_cfg(cfg, a.adj, [&](auto c) {
    using C = decltype(c);
    s->cs = a.q / C::NC;
    s->nthreads = C::NT;
    s->smem = C::smem(a.q);
    return 0;
  });
  s->grid = dim3(s->cs, mt, nchains);
  return 0;
}

cudaError_t wresid_launch(const ResidArgs& a, cudaStream_t st) {
  if (a.q == 16) return a.adj ? wresid_launch_t<16, true>(a, st) : wresid_launch_t<16, false>(a, st);
  if (a.q == 32) return a.adj ? wresid_launch_t<32, true>(a, st) : wresid_launch_t<32, false>(a, st);
  return cudaErrorInvalidValue;
}

cudaError_t sweep_launch(const SweepArgs& a, const SweepShape& s, cudaStream_t st) {
  if (s.cfg == SWEEP_CFG_WARP) return wsweep_launch(a, s, st);
  return with_cfg(s.cfg, a.adj, [&](auto c) { return launch_c<decltype(c)>(a, s, st); });
}

// how many clusters of a configuration can be co-resident (cudaOccupancyMaxActiveClusters)
int sweep_max_clusters(int q, int adj, int cfg) {
  if (cfg == SWEEP_CFG_WARP) {
    // independent CTAs, no co-residency needed: allow a few waves of 8-warp CTAs (each CTA runs
    // a whole chain, so a second wave costs one more chain's latency, still far below per-step
    // launches)
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int per = q <= 16 ? (adj ? wsweep_occupancy<16, true>() : wsweep_occupancy<16, false>())
                            : (adj ? wsweep_occupancy<32, true>() : wsweep_occupancy<32, false>());
    return 4 * per * sms;
  }
  SweepArgs a{};
  a.mode = SW_SEQ; a.B = 16; a.q = q; a.n = 2; a.adj = adj;
  SweepShape sh;
  if (sweep_shape(a, &sh, cfg) < 0 || sh.cfg != cfg) return -1;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(sh.cs, 64, 1);
  lc.blockDim = dim3(sh.nthreads, 1, 1);
  lc.dynamicSmemBytes = sh.smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = sh.cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  int n = -1;
  const cudaError_t e = with_cfg(cfg, adj, [&](auto c) {
    auto k = sweep_kernel<decltype(c)>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_MAX);
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    return cudaOccupancyMaxActiveClusters(&n, k, &lc);
  });
  return e == cudaSuccess ? n : -(int)e;
}

}  // namespace lmg


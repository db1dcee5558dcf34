// lmg_chain.cuh -- persistent "chain" launch of a whole relaxation sweep (sm_100a).
//
// A relaxation sweep of a level is a sequence of layer steps in which step s of block (task) t
// reads the row step s-1 of the SAME task wrote (F sweep: row kc+s from row kc+s-1; the C step
// and the P step continue the same chain: row (k+1)c / P[k+1] from row kc+c-1).  The launch-per-
// step path runs one grid per step; here ONE persistent cooperative grid walks every (step,
// task, output tile) item of the sweep in step-major order and replaces the grid boundary by a
// per-(step, task) completion counter: an item waits only for the tiles of its own task's
// previous step, and fetches its weight tiles (which never depend on the state) before waiting.
// So the weight stream -- the HBM roofline of small batches -- never drains between steps, and
// there is no per-step launch ramp / tail.  (An L2 prefetch of the next item's first weight
// k-tiles, issued late in the current item, measured slower at every depth: c5 step 20.7 ms
// without, 20.8-25.2 ms with 4-32 k-tiles.)
//
// Arithmetic is the per-step kernel's (step_gemm, E_PROP): the same tile shape, the same
// k-ascending DMMA chain per output and the same epilogue, so results are bitwise identical to
// the launch-per-step path.
//
// Ordering: the producer's stores, __syncthreads, then one thread's fence + relaxed atomic
// (release); the consumer's ld.acquire spin in one thread, then __syncthreads before any thread
// reads (the CUTLASS semaphore pattern).  Items are assigned to CTAs round-robin in increasing
// order and every CTA is co-resident (cooperative launch), so the smallest unfinished item always
// has its dependencies done: no deadlock.
#pragma once

#include "lmg_gemm.cuh"

namespace lmg {

constexpr int kChainMaxSteps = 33;

struct ChainStep {       // the per-step operands; shape, strides and epilogue are shared
  const double* A;       // input rows of task 0 (also the epilogue's x)
  int64_t A_ts;
  const double* Ds;      // adjoint: act' scales of task 0
  const double* Bm;      // weights of task 0
  const double* bias;    // bias of task 0 (forward)
  const double* s;       // source rows of task 0 (NULL: zero)
  double* out;           // output rows of task 0
  int64_t out_ts;
  double* out2;          // optional second output (x + h2 * act(pre)), stride out2_ts
  double h2;
  int ntasks;
  int item0;             // first item index of this step
};

struct ChainArgs {
  StepArgs a;            // M, N, K, act, h, lda, ldb, ldc, B_ts, bias_ts, Ds_ts, s_ts, out2_ts
  int nsteps, total, max_tasks;
  int ntn, tiles;        // n tiles per task, tiles per task (m x n)
  int war_last;          // the last step of task t overwrites the row step 0 of task t+1 reads
  unsigned* flags;       // [nsteps][max_tasks] completed tiles, zeroed before the launch
  ChainStep st[kChainMaxSteps];
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// spin until *f >= n: relaxed polls, then ONE acquire fence (an ld.acquire per poll invalidates
// the SM's L1 every iteration -- ncu showed the CCTL.IVALL of the polls among the top stalls)
__device__ __forceinline__ void wait_count(const unsigned* f, unsigned n) {
  if (ld_relaxed(f) < n) {
    do {
      __nanosleep(32);
    } while (ld_relaxed(f) < n);
  }
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

template <class T, bool AK, bool BKM, bool ASC>
__global__ void __launch_bounds__(T::WM* T::WN * 32)
    chain_gemm(const __grid_constant__ ChainArgs ca) {
  using C = GemmCfg<T, AK, BKM, ASC>;
  constexpr int BM = C::BM, BN = C::BN, BK = C::BK, WN = C::WN, STAGES = C::STAGES;
  static_assert(AK, "chain launches are forward / adjoint layer steps");
  extern __shared__ __align__(16) double smem[];

  const StepArgs& a = ca.a;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WN, wn = warp % WN;
  const int KT = a.K / BK;  // fully tiled shapes only
  const int wm0 = wm * C::WTM, wn0 = wn * C::WTN;
  const int fr = lane >> 2, fk = lane & 3;
  constexpr int LDA_ = TileShape<AK, BM, BK>::LD, LDB_ = TileShape<BKM, BN, BK>::LD;
  const int a_thr = pin(AK ? (wm0 + fr) * LDA_ + fk : fk * LDA_ + wm0 + fr);
  const int b_thr = pin(BKM ? (wn0 + fr) * LDB_ + fk : fk * LDB_ + wn0 + fr);

  int s = 0;
  for (int item = blockIdx.x; item < ca.total; item += gridDim.x) {
    while (s + 1 < ca.nsteps && item >= ca.st[s + 1].item0) ++s;
    const ChainStep& cs = ca.st[s];
    const int r = item - cs.item0;
    const int t = r / ca.tiles, tile = r % ca.tiles;
    const int n0 = (tile % ca.ntn) * BN, m0 = (tile / ca.ntn) * BM;
    const double* A = cs.A + t * cs.A_ts;
    const double* Ds = ASC ? cs.Ds + t * a.Ds_ts : nullptr;
    const double* Bm = cs.Bm + t * a.B_ts;

    double acc[C::MT][C::NTF][2];
#pragma unroll
    for (int i = 0; i < C::MT; ++i)
#pragma unroll
      for (int j = 0; j < C::NTF; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    Loader<AK, BM, BK, 2, C::NTHREADS> la;
    Loader<BKM, BN, BK, 2, C::NTHREADS> lb;
    Loader<AK, BM, BK, 2, C::NTHREADS> ld_;
    la.init(A, a.lda, m0, a.M, tid);
    lb.init(Bm, a.ldb, n0, a.N, tid);
    if (ASC) ld_.init(Ds, a.lda, m0, a.M, tid);
    la.init_full();
    lb.init_full();
    if (ASC) ld_.init_full();

    __syncthreads();  // every warp is done with the previous item's stages
    // weight stages first: they do not depend on the previous step
#pragma unroll
    for (int st = 0; st < STAGES - 1; ++st)
      if (st < KT) lb.load_next(smem + st * C::STAGE + C::B_OFF);
    // wait for this task's previous step (all its tiles), and for the WAR guard
    if (tid == 0) {
      if (s > 0) wait_count(ca.flags + (int64_t)(s - 1) * ca.max_tasks + t, (unsigned)ca.tiles);
      // WAR guard: step 0 of task t+1 has read its input row (the one this step overwrites)
      if (ca.war_last && s == ca.nsteps - 1 && t + 1 < ca.st[0].ntasks)
        wait_count(ca.flags + t + 1, (unsigned)ca.tiles);
    }
    __syncthreads();
    // the epilogue's x (this tile's columns of the input row) and bias, fetched now so their
    // latency hides under the mainloop instead of stalling the epilogue (ncu: the epilogue's
    // dependent DADDs were ~10% of the stall samples)
    const int mrow0 = m0 + wm0 + fr, ncol0 = n0 + wn0 + 2 * fk;
    const double* bias = cs.bias ? cs.bias + t * a.bias_ts : nullptr;
    double xv[C::MT][C::NTF][2], bv[C::NTF][2];
#pragma unroll
    for (int j = 0; j < C::NTF; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) bv[j][e] = bias ? bias[ncol0 + j * 8 + e] : 0.0;
#pragma unroll
    for (int i = 0; i < C::MT; ++i)
#pragma unroll
      for (int j = 0; j < C::NTF; ++j) {
        const double2 x2 = *reinterpret_cast<const double2*>(A + (int64_t)(mrow0 + i * 8) * a.ldc + ncol0 + j * 8);
        xv[i][j][0] = x2.x;
        xv[i][j][1] = x2.y;
      }
    // register-staged act' scaling (C::RS, the adjoint): each thread's lambda and act' vectors of
    // the next k-tile are loaded into registers during this k-tile's DMMAs and their product is
    // stored into the next stage's A area -- act' never occupies shared memory (the staged act'
    // tile had cost the adjoint chain 2 of the forward's 7 CTAs per SM)
    constexpr int RIT = decltype(la)::IT;
    double2 ra[C::RS ? RIT : 1], rd[C::RS ? RIT : 1];
    auto rs_ldg = [&] {
#pragma unroll
      for (int i = 0; i < RIT; ++i) {
        if (RIT * C::NTHREADS > decltype(la)::NV && la.tid_out_of_range(i)) continue;
        ra[i] = *reinterpret_cast<const double2*>(la.cur[i]);
        rd[i] = *reinterpret_cast<const double2*>(ld_.cur[i]);
        la.cur[i] += la.kadv;
        ld_.cur[i] += ld_.kadv;
      }
    };
    auto rs_sts = [&](double* base) {
#pragma unroll
      for (int i = 0; i < RIT; ++i) {
        if (RIT * C::NTHREADS > decltype(la)::NV && la.tid_out_of_range(i)) continue;
        *reinterpret_cast<double2*>(base + la.soff[i]) =
            make_double2(__dmul_rn(ra[i].x, rd[i].x), __dmul_rn(ra[i].y, rd[i].y));
      }
    };
    if constexpr (C::RS) {
      rs_ldg();
      rs_sts(smem);  // A of stage 0
#pragma unroll
      for (int st = 0; st < STAGES - 1; ++st) cp_commit();  // the prefetched weight stages
      if (KT > 1) rs_ldg();
    } else {
#pragma unroll
      for (int st = 0; st < STAGES - 1; ++st) {
        if (st < KT) {
          double* base = smem + st * C::STAGE;
          la.load_next(base);
          if (ASC) ld_.load_next(base + C::A_SZ);
        }
        cp_commit();  // group 0 also carries the prefetched weight stages
      }
    }
    for (int kt = 0; kt < KT; ++kt) {
      cp_wait<STAGES - 2>();
      if (ASC && !C::RS) {
        double* st0 = smem + (kt % STAGES) * C::STAGE;
        la.scale_own(st0, st0 + C::A_SZ);
      }
      __syncthreads();
      {
        const int nk = kt + STAGES - 1;
        if (nk < KT) {
          double* base = smem + (nk % STAGES) * C::STAGE;
          if (!C::RS) {
            la.load_next(base);
            if (ASC) ld_.load_next(base + C::A_SZ);
          }
          lb.load_next(base + C::B_OFF);
        }
        cp_commit();
      }
      const double* As = smem + (kt % STAGES) * C::STAGE;
      const double* Bs = As + C::B_OFF;
      double af[2][C::MT], bf[2][C::NTF];
      auto ldfrag = [&](int buf, int kk) {
#pragma unroll
        for (int i = 0; i < C::MT; ++i) {
          const int o = a_thr + (AK ? i * 8 * LDA_ + kk : kk * LDA_ + i * 8);
          af[buf][i] = As[o];  // scaled in place (scale_own)
        }
#pragma unroll
        for (int j = 0; j < C::NTF; ++j)
          bf[buf][j] = Bs[b_thr + (BKM ? j * 8 * LDB_ + kk : kk * LDB_ + j * 8)];
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
      if constexpr (C::RS) {
        // stage kt+1's A area was last read at k-tile kt+1-STAGES (every warp passed this
        // k-tile's barrier since); it is published by the next k-tile's barrier
        if (kt + 1 < KT) {
          rs_sts(smem + ((kt + 1) % STAGES) * C::STAGE);
          if (kt + 2 < KT) rs_ldg();
        }
      }
    }
    cp_wait<0>();

    // E_PROP (lmg_gemm.cuh epilogue, same operations in the same order): out = s + (x + h*act(pre)),
    // out2 = x + h2*act(pre).  Fully tiled: every (m, n) is in range.
    {
      const double* S = cs.s ? cs.s + t * a.s_ts : nullptr;
      double* O = cs.out + t * cs.out_ts;
      double* O2 = cs.out2 ? cs.out2 + t * a.out2_ts : nullptr;
      const double h = a.h, h2 = cs.h2;
#pragma unroll
      for (int i = 0; i < C::MT; ++i)
#pragma unroll
        for (int j = 0; j < C::NTF; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int64_t idx = (int64_t)(mrow0 + i * 8) * a.ldc + ncol0 + j * 8 + e;
            double pre = acc[i][j][e];
            if (bias) pre = __dadd_rn(pre, bv[j][e]);
            const double v = act_fwd(a.act, pre);
            const double x = xv[i][j][e];
            const double adv = __dadd_rn(x, __dmul_rn(h, v));
            O[idx] = __dadd_rn(S ? S[idx] : 0.0, adv);
            if (O2) O2[idx] = __dadd_rn(x, __dmul_rn(h2, v));
          }
    }

    __syncthreads();  // every thread's stores issued before the completion is published
    if (tid == 0) {
      __threadfence();
      atomicAdd(ca.flags + (int64_t)s * ca.max_tasks + t, 1u);
    }
  }
}

}  // namespace lmg

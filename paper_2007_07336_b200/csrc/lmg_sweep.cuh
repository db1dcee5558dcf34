// lmg_sweep.cuh -- persistent fused relaxation sweep: interface (kernel in lmg_sweep.cu).
//
// One launch runs a whole relaxation sweep of a level (or a whole serial propagation): every
// thread-block cluster owns one chain of consecutive layer steps -- one block of the level at
// one 16-row batch tile -- and keeps that chain's state in shared memory for all of its steps.
// Only the weights stream from HBM (TMA bulk copies into an mbarrier ring, run ahead across
// step boundaries because W does not depend on the state); the state never round-trips through
// HBM between steps.  After each step the CTAs of the cluster exchange their column slices of
// the new state through distributed shared memory (all-gather) and meet at one cluster barrier.
//
// Same arithmetic as the per-step kernel (lmg_gemm.cuh step_gemm, E_PROP): each output is one
// DMMA m8n8k4 chain over k ascending, then pre + bias, act, u + h*act, s + (...) with the same
// rounding, so results are bitwise identical to the launch-per-step path.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace lmg {

// Canonical summation order (lmg_set_canonical_order): every layer step is one k-ascending DMMA
// (or, bitwise the same, FMA) chain per output -- the 64-column sweep configuration or the warp
// FMA sweep only, no split-K serial steps -- so the
// results are bitwise independent of batch size, partition and routing (defined in lmg.cu).
bool canonical_order();

enum SweepMode {
  SW_FCF = 0,  // FCF relaxation + the P step of every block (multigrid.py:160-172, :208)
  SW_SEQ = 1   // serial forward substitution rows 1..n-1 (network.py:111-123)
};

struct SweepArgs {
  int mode;
  int B, q;      // batch, width
  int n;         // layers at this level
  int c;         // SW_FCF: coarsening factor (blocks of c layers, nb = n / c)
  int adj;       // adjoint layout: G(m) = W^T (D * m), identity act, no bias
  int act;
  double h, h2;  // step; h2 = coarse step of the advH output (SW_FCF)
  const double* W; int64_t w_stride;  // block j at W + j*w_stride (doubles, may be negative)
  const double* bias; int64_t b_stride;
  const double* D; int64_t d_stride;  // adjoint: block j's act' scale, (B, q)
  const double* src; int src_head;    // source rows (n, B, q), or only row 0 when src_head
  const double* Q;                    // SW_FCF: optional start rows (k-1)c+1 = Q[k-1]
  double* U;                          // states (n, B, q): F rows written, C rows read
  double* Cn;                         // SW_FCF: new C rows kc, k >= 1 (Cn + k*BQ)
  double* P;                          // SW_FCF: P[k+1] = propagate(U[(k+1)c-1]) (P + (k+1)*BQ)
  double* advH;                       // SW_FCF: advH[k] = U[kc] + h2*F(U[kc]), nullable
  unsigned long long* trace;          // debug: per-step globaltimer stamps of chain 0, rank 0
  // layer-partitioned FCF (a rank's run of blocks): chains k0 .. k0+gridDim.z-1; chain 0 starts
  // at U[0] (already finished from the previous rank's halo) unless is_first; with has_next,
  // chain nb is the halo chain -- block nb-1's first F rows, then row nb*c (the next rank's
  // incoming C row, source row nb*c = the zero row) -> halo -- and block nb-1 gets its P step
  int k0, is_first, has_next;
  double* halo;
  int nchains;  // chains in this launch (0: all nb of the level)
  int write_row0;  // SW_SEQ, warp FMA sweep: also store U[0] = src[0] (the solve's first row)
  // warp FMA sweep only, SW_SEQ: the parent level's coarse-grid correction of each produced row
  // j, corrU[j*corr_ts] += row - corrU[j*corr_ts] (k_correct, same arithmetic)
  double* corrU; int64_t corr_ts;
};

// warp-level FMA sweep for narrow networks (q <= 32; lmg_sweep.cu wsweep_kernel): no clusters,
// grid (1, batch groups of 8 samples, chains)
constexpr int SWEEP_CFG_WARP = 4;
// Post-correction residual of a narrow level (q 16 / 32) in one launch (lmg_sweep.cu
// wresid_kernel): the correction U[kc] += V[k] - U[kc] with its C-row residual partial
// (k_correct_cpart), the kc+1 residual rows as one warp FMA step each (E_RESID, propagated rows
// -> Q) and the per-block partials (k_combine_post) -- every sum in the order those kernels use,
// so the block partials, and the norms, are bitwise theirs.
struct ResidArgs {
  int B, q, nb, c, adj, act, is_first;
  double h;
  const double* W; int64_t w_stride;
  const double* bias; int64_t b_stride;
  const double* D; int64_t d_stride;
  const double* src; int src_head;  // level source (head: only row 0)
  double* U;
  const double* V;  // coarse-grid solution rows (the correction)
  const double* P;  // propagated C rows
  double* Q;        // optional: propagated rows kc+1
  double* block_part;
};
cudaError_t wresid_launch(const ResidArgs& a, cudaStream_t st);

// configuration the launcher would use for (q, B, adj), or -1 if the fused sweep cannot run it
int sweep_config(int q, int B, int adj, int nclusters_hint);
// dynamic shared memory, cluster size and grid of a config
struct SweepShape {
  int cfg, cs, nthreads;
  size_t smem;
  dim3 grid;
};
// forced_cfg >= 0 picks a configuration (0: 64 columns per CTA, 1: 32) instead of the default
int sweep_shape(const SweepArgs& a, SweepShape* s, int forced_cfg = -1);
cudaError_t sweep_launch(const SweepArgs& a, const SweepShape& s, cudaStream_t st);
int sweep_max_clusters(int q, int adj, int cfg);

}  // namespace lmg

/* lmg.h -- C-ABI of the B200 (sm_100a) layer-parallel FAS solver.
 *
 * Drop-in boundary for the hot path of the reference package `layermg`
 * (/root/reference/pkg/src/layermg).  The reference's seam is Python; each entry
 * point below replaces one reference function, cited as file:line.  The Python mirror of the
 * reference API (paper_2007_07336_b200/) binds these with ctypes; INTEGRATION.md shows the
 * binding a layermg maintainer would add.
 *
 * Conventions
 *  - every array is float64 in DEVICE memory, caller-owned; the library never frees it.
 *  - a stack of layer states is (n, B, q) row-major: state row j of sample b at
 *    ptr[(j*B + b)*q]; B is the batch (the reference is B = 1), q the state width.
 *  - sources come in two modes: LMG_SRC_DENSE (n, B, q) or LMG_SRC_HEAD, where only row 0
 *    (B, q) is stored and rows 1.. are zero (network.py:80-85).
 *  - all work is stream-ordered on `stream` (a cudaStream_t, NULL = legacy default stream);
 *    functions that return host data synchronise that stream.
 *  - return value: LMG_OK or an error class mirroring errors.py:4-21; lmg_last_error() gives
 *    the message (thread-local).
 */
#ifndef LMG_H
#define LMG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  LMG_OK = 0,
  LMG_ERR_DIMENSION = 1,     /* errors.py:4  DimensionError     */
  LMG_ERR_CONFIGURATION = 2, /* errors.py:8  ConfigurationError */
  LMG_ERR_PROTOCOL = 3,      /* errors.py:12 ProtocolError      */
  LMG_ERR_CUDA = 4
};

enum { LMG_ACT_RELU = 0, LMG_ACT_TANH = 1, LMG_ACT_IDENTITY = 2 }; /* kernels.py:24-28 */
enum { LMG_SRC_DENSE = 0, LMG_SRC_HEAD = 1 };

/* kind of a system's blocks */
enum {
  LMG_DENSE = 0,         /* F(u) = act(W u + b), W (q, q) row-major (kernels.py:146-147)   */
  LMG_DENSE_ADJOINT = 1, /* G(m) = W^T (D * m): the reversed linear adjoint recursion of
                            training.py:216-224; D = act'(pre) at the forward states       */
  LMG_CONV = 2,          /* 3x3 pad-1 conv on CHW rasters, HWIO weights (kernels.py:130-136) */
  LMG_CONV_ADJOINT = 3
};

/* One level's view of the residual blocks: the reference's `system` duck type
 * (network.py:13-15; MgLevel multigrid.py:45-58).  Block j's parameters live at
 * W + j*w_stride and b + j*b_stride (strides in doubles, may be negative), so coarse levels are
 * strided views of the fine arrays -- they alias like multigrid.py:83-85, no copies. */
typedef struct lmg_system {
  int32_t num_layers; /* n: states / blocks at this level                          */
  int32_t width;      /* q                                                         */
  int32_t kind;       /* LMG_DENSE ...                                             */
  int32_t act;        /* LMG_ACT_*                                                 */
  double step;        /* h of this level (multigrid.py:101: h_{l+1} = h_l * c)     */
  const double* W;
  int64_t w_stride;
  const double* b; /* NULL for the adjoint kinds                                */
  int64_t b_stride;
  const double* D; /* adjoint kinds: block j scale at D + j*d_stride, (B, q)     */
  int64_t d_stride;
  int32_t channels, height, px_width; /* conv geometry (q = channels*height*px_width) */
  int32_t reserved;
} lmg_system;

int lmg_abi_version(void);
const char* lmg_last_error(void);

/* Instrumentation (not part of the reference API): number of kernels this library has launched,
 * and optional CUDA-event timing of every launch by class (0 forward step GEMM, 1 adjoint step
 * GEMM, 2 parameter-gradient GEMM, 3 elementwise/reduction, 4/5 fused forward/adjoint sweep,
 * 6 split-K serial step (coarsest solve / serial propagation); -1 = all).  lmg_timing_enable(1)
 * clears the records; lmg_timing_read synchronises on the recorded events. */
unsigned long long lmg_launch_count(void);
int lmg_timing_enable(int on);
int lmg_timing_read(int cls, double* ms_total, double* flops_total, double* bytes_total,
                    unsigned long long* launches);
/* Instrumentation: launches per kernel variant since load, written to out[0..n) in this order;
 * returns the number of variants (LMG_ROUTE_N).  Lets tests assert which kernels a call ran. */
enum {
  LMG_ROUTE_STEP_SMALL = 0,      /* step_gemm 32x32 tile, predicated loads            */
  LMG_ROUTE_STEP_SMALL_FULL = 1, /* step_gemm 32x32 tile, fully tiled shape            */
  LMG_ROUTE_STEP_WIDE = 2,       /* step_gemm 32x64                                    */
  LMG_ROUTE_STEP_WIDE_FULL = 3,
  LMG_ROUTE_STEP_TINY = 4,       /* step_gemm 16x32 (batches <= 16)                    */
  LMG_ROUTE_STEP_TINY_FULL = 5,
  LMG_ROUTE_TGEMM_BIG = 6,       /* warp-specialised TMA step GEMM, 64x64 tiles        */
  LMG_ROUTE_TGEMM_SMALL = 7,     /* same, 16x32 tiles                                  */
  LMG_ROUTE_SERIAL_SPLITK = 8,   /* split-K cluster kernel for serial single-task steps */
  LMG_ROUTE_SWEEP_FCF = 9,       /* fused persistent FCF sweep of a level               */
  LMG_ROUTE_SWEEP_SEQ = 10,      /* fused persistent serial solve                       */
  LMG_ROUTE_CONV_FWD = 11,       /* implicit-GEMM conv2d, forward step                  */
  LMG_ROUTE_CONV_ADJ = 12,       /* conv2d adjoint step                                 */
  LMG_ROUTE_CONV_PGRAD = 13,     /* conv2d parameter gradients                          */
  LMG_ROUTE_CHAIN = 14,          /* persistent chain launch of a whole relaxation sweep  */
  LMG_ROUTE_WSWEEP = 15,         /* warp-level FMA sweep (q 16/32, FCF or serial) or the fused narrow residual */
  LMG_ROUTE_N = 16
};
int lmg_route_counts(unsigned long long* out, int n);
/* Canonical summation order on (1) / off (0, default); returns the previous setting.  On: every
 * layer step is one k-ascending DMMA chain per output (64-column fused sweeps only, no split-K
 * serial steps), so states are bitwise independent of batch size, routing and layer partition
 * -- used by the CLI `scale` checksum (reference cli.py:243-263).  Off: the fastest routing,
 * equal to the canonical results within the parity tolerance. */
int lmg_set_canonical_order(int on);
/* Debug: device buffer (>= 4 u64 per step, or NULL to stop) receiving per-step %globaltimer
 * stamps (step start, state ready, mainloop done, epilogue done) of chain 0 / CTA 0 of every
 * fused persistent sweep launch.  Classes 4/5 of lmg_timing_read are those launches. */
int lmg_debug_sweep_trace(unsigned long long* dev_buf);
/* Debug: co-resident clusters of a fused-sweep configuration (cfg 0: 64 columns per CTA,
 * 1: 32) at width q, from cudaOccupancyMaxActiveClusters; negative on error. */
int lmg_debug_sweep_clusters(int q, int adj, int cfg);

/* network.py:88-102 propagate_values: out[j-start] = src[j] + (u + h*F_{j-1}(u)), j in
 * [start, stop), from u_start (B, q) = u^{start-1}.  out is (stop-start, B, q). */
int lmg_propagate(const lmg_system* sys, int B, const double* u_start, const double* src,
                  int src_mode, int start, int stop, double* out, void* stream);

/* network.py:111-123 sequential_forward: states (n, B, q) <- forward substitution. */
int lmg_sequential_forward(const lmg_system* sys, int B, const double* src, int src_mode,
                           double* states, void* stream);

/* network.py:126-139 propagation_operator. */
int lmg_propagation_operator(const lmg_system* sys, int B, const double* states, double* out,
                             void* stream);

/* multigrid.py:115-128 compute_residual (+ kernels.py:191-194 l2_norm per sample).
 * out (n,B,q) may be NULL; norms (B, device) may be NULL.  `work` needs
 * lmg_residual_workspace() bytes when norms != NULL. */
size_t lmg_residual_workspace(const lmg_system* sys, int B);
int lmg_compute_residual(const lmg_system* sys, int B, const double* states, const double* src,
                         int src_mode, double* out, double* norms, void* work, void* stream);

/* multigrid.py:105-112 restrict_states (injection): out (n/c, B, q) <- fine[::c]. */
int lmg_restrict(const double* fine, int n, int B, int q, int c, double* out, void* stream);

/* multigrid.py:131-142 assemble_coarse_source: out = L_H(U_H) + R_H. */
int lmg_assemble_coarse_source(const lmg_system* coarse, int B, const double* UH,
                               const double* RH, double* out, void* stream);

/* parallel.py:143-168 / multigrid.py:145-151 F-sweep, parallel.py:171-241 / multigrid.py:154-157
 * C-sweep, multigrid.py:160-172 FCF.  In place on states (n, B, q). */
int lmg_f_relax(const lmg_system* sys, int B, int c, double* states, const double* src,
                int src_mode, void* stream);
int lmg_c_relax(const lmg_system* sys, int B, int c, double* states, const double* src,
                int src_mode, void* stream);
int lmg_fcf_relax(const lmg_system* sys, int B, int c, double* states, const double* src,
                  int src_mode, void* stream);

/* multigrid.py:76-102 build_hierarchy: number of levels for (n, c, threshold<=0 -> n//c). */
int lmg_num_levels(int n, int c, int threshold, int* levels_out);

/* multigrid.py:175-228 mg_cycle (level 0 of an `nlevels` hierarchy built from `fine`), in place;
 * norms (B, device) receives the per-sample residual norm after the cycle. */
size_t lmg_solver_workspace(const lmg_system* fine, int nlevels, int c, int B);
int lmg_mg_cycle(const lmg_system* fine, int nlevels, int c, int B, double* states,
                 const double* src, int src_mode, double* norms, void* work, size_t work_bytes,
                 void* stream);

/* multigrid.py:263-311 solve, per sample.  states (n,B,q) holds the initial iterate when
 * use_initial != 0, else is overwritten with initial_guess (multigrid.py:257-260); on return it
 * holds each sample's states as of the cycle where that sample met tol (or max_cycles).
 * hist_host ((max_cycles+1) x B, host) receives residual_norms; cycles_host / converged_host
 * (B, host) the CycleReport fields.  Synchronises `stream` once per cycle (the stopping test). */
int lmg_solve(const lmg_system* fine, int nlevels, int c, int B, double* states,
              const double* src, int src_mode, int use_initial, double tol, int max_cycles,
              double* hist_host, int32_t* cycles_host, int32_t* converged_host, void* work,
              size_t work_bytes, void* stream);

/* training.py:216-224 support: D[n] = act'(W_n u^n + b_n) for every layer (n, B, q). */
int lmg_act_deriv(const lmg_system* fine, int B, const double* states, double* D, void* stream);

/* training.py:218,223,174-177,230-236: for every layer n,
 *   gW_n = scale * h * sum_b (lam^{n+1}_b * D_n,b) (x) u^n_b,   gb_n = scale * h * sum_b (...)
 * lam is the adjoint stack (n, B, q) in the reversed order the adjoint system produces it
 * (lam[m] = lambda^{N-m}); gW (n,q,q) / gb (n,q) may be NULL; when lr != 0 the SGD step
 * W -= lr*gW, b -= lr*gb is applied in the same pass (fine->W/b must then be writable). */
int lmg_param_grads(const lmg_system* fine, int B, const double* states, const double* lam,
                    const double* D, double scale, double lr, double* gW, double* gb,
                    void* stream);
/* Same, for one slice of a batch: with accumulate != 0 the slice's gradients are ADDED to gW / gb
 * (which then must be given), and the SGD step (lr != 0) uses the accumulated gradient -- the
 * reference's Gradients.accumulate + sgd_update over batch slices (training.py:174-177,287-288). */
int lmg_param_grads_ex(const lmg_system* fine, int B, const double* states, const double* lam,
                       const double* D, double scale, double lr, double* gW, double* gb,
                       int accumulate, void* stream);

/* ---- layer-partitioned level operations -------------------------------------------
 * A rank owns L = nb*c consecutive states of a level (nb whole blocks of the reference's
 * BlockPartition, parallel.py:61-79).  U has L rows plus, when has_next, one outgoing halo row
 * U[L]; a dense src has the matching rows (+ a zero row L); P has nb+1 rows (P[0] incoming,
 * P[nb] outgoing).  Halo values travel WITHOUT their source row ("adv" = u + h F(u)); the receiver
 * finishes them with lmg_halo_finish.  Per cycle and cross edge: U[L] after fcf_a (the
 * reference's one BoundaryMessage per edge per C-sweep, parallel.py:183-216), then P[nb] and
 * adv_out after fcf_b.  Single GPU == is_first = 1, has_next = 0.  States are bitwise identical
 * for every partition; norms too, since partials are per block and summed in global block order.
 */
/* Q (optional, nb rows): propagate(U[kc]) from the previous cycle's lmg_local_residual_post; when
 * given, the first F-sweep step is a copy instead of a launch (bitwise identical). */
int lmg_local_fcf_a(const lmg_system* sys, int B, int c, double* U, const double* src,
                    int src_mode, int is_first, int has_next, const double* Q, void* stream);
/* advH (optional, nb rows): receives U[kc] + H F_H(U[kc]) (H = c h) from the second sweep's first
 * step -- the same pre-activation -- so lmg_local_coarse_source needs no GEMM of its own. */
int lmg_local_fcf_b(const lmg_system* sys, int B, int c, double* U, const double* src,
                    int src_mode, double* P, int has_next, double* adv_out, double* advH,
                    void* stream);
/* Layer-partitioned FCF (the rank's run of blocks) as fused persistent sweeps: part 0 runs every
 * chain that needs no halo -- with has_next its halo chain writes the next rank's incoming C row
 * (no source) to states[L] -- and commits the new C rows; part 1, after the exchange and
 * lmg_halo_finish of states[0], runs block 0 of a non-first rank and copies advH[nb-1] to adv_out.
 * Same outputs as lmg_local_fcf_a/_b (parallel.py:143-241).  Cn: nb*(B,q) scratch.
 * lmg_local_fcf_fused_ok returns 1 when this path applies (small batch, one wave of clusters). */
int lmg_local_fcf_fused_ok(const lmg_system* sys, int B, int c, int is_first, int has_next);
int lmg_local_fcf_fused(const lmg_system* sys, int B, int c, double* states, const double* src,
                        int src_mode, int is_first, int has_next, const double* Q, double* P,
                        double* advH, double* Cn, int part, double* adv_out, void* stream);
int lmg_halo_finish(const double* s0, const double* adv_in, double* out, int64_t len, void* stream);
int lmg_local_coarse_source(const lmg_system* sys, int B, int c, const double* U,
                            const double* src, int src_mode, const double* P,
                            const double* adv_in, int is_first, double* SH, double* V,
                            const double* advH, void* stream);
int lmg_local_correct(int n_blocks, int B, int q, int c, double* U, const double* V, void* stream);
size_t lmg_local_workspace(int L, int B, int q);
int lmg_local_residual_post(const lmg_system* sys, int B, int c, const double* U,
                            const double* src, int src_mode, const double* P, int is_first,
                            double* block_part, void* work, double* Q, void* stream);
int lmg_local_residual_full_a(const lmg_system* sys, int B, const double* U, const double* src,
                              int src_mode, int has_next, double* adv_out, void* work,
                              void* stream);
int lmg_local_residual_full_b(const lmg_system* sys, int B, int c, const double* U,
                              const double* src, int src_mode, const double* adv_in, int is_first,
                              double* block_part, void* work, void* stream);
int lmg_norms_from_blocks(const double* block_part, int nblocks, int B, double* norms,
                          void* stream);

/* kernels.py:139-150 / 153-188 for block j of a system (dense or conv2d): Y = act(F_j(X)), and
 * the VJP: gX = J_j^T G, batch-summed gW / gb (HWIO for conv).  `work` needs B*q doubles. */
int lmg_apply_block(const lmg_system* sys, int B, int j, const double* X, double* Y, void* stream);
int lmg_vjp_block(const lmg_system* sys, int B, int j, const double* X, const double* G, double* gX,
                  double* gW, double* gb, double* work, void* stream);

/* kernels.py:139-150 apply_transform (dense) for a batch: Y (M, q_out) = act(X W^T + b),
 * X (M, q_in), W (q_out, q_in) row-major, b (q_out) or NULL. */
int lmg_dense_apply(const double* W, const double* b, int act, int M, int q_out, int q_in,
                    const double* X, double* Y, void* stream);

/* kernels.py:153-169 transform_vjp (dense), batch-summed parameter gradients:
 *   gp = G * act'(X W^T + b) ;  gX (M, q_in) = gp W ;  gW (q_out, q_in) = sum_m gp_m (x) x_m ;
 *   gb (q_out) = sum_m gp_m.   Any of gX / gW / gb may be NULL.  `work` needs M*q_out doubles. */
int lmg_dense_vjp(const double* W, const double* b, int act, int M, int q_out, int q_in,
                  const double* X, const double* G, double* gX, double* gW, double* gb,
                  double* work, void* stream);

/* kernels.py:191-194 l2_norm per sample of an (n, B, q) stack: norms (B, device). `work` needs
 * lmg_residual_workspace() bytes of a system with this n and q. */
int lmg_l2_norms(const double* x, int n, int B, int q, double* norms, void* work, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* LMG_H */

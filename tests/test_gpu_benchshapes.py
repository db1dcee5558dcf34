"""Oracle parity at the shapes the bench times (VERDICT r1 "next" #1).

Every case runs the bench's own hot path -- `DeviceTrainer.step` (FAS forward to tol, FAS adjoint
to tol, block gradients with the SGD step fused in, split=1 as bench.py) -- and checks it against
the CPU oracle (`oracle/fas.py`, pinned bitwise to the live reference by tests/golden/) on the
same seeded inputs:

  c5_full      BASELINE configs[4] point exactly as benched: 1024 x 512, B 16, cf 16,
               levels [1024, 64, 4] -- 16-row TTiny step tiles, the fused FCF sweeps on the coarse
               level, the fused serial solve at the coarsest level.
  c2_full_2cyc BASELINE configs[1] exactly as benched (1024 x 512, B 256, cf 4, [1024,256,64]),
               early-stopped at 2 FAS cycles forward and adjoint (the reference's own training
               semantics, mg_cycles=2, training.py:245) so the oracle finishes: fully tiled 32x32
               step_gemm, the TMA tgemm adjoint (B % 64 == 0), split-K coarsest solves.
  c2_depth64   the c2 shape at depth 64 ([64,16,4]) solved to tol 1e-9 (same kernels, full
               convergence, cycle counts compared).
  c4_depth32   the c4 width (q 1024) at depth 32 ([32, 8]), B 128.
  c6_full / c7_full / c1_full  the narrow bench shapes (q 16 at depth 1024 and 4096, q 32): the
               warp-level FMA sweeps for every relaxed level and serial solve.
  c3_depth32   the c3 conv geometry (64 channels, 32 x 32 rasters, relu) at depth 32 ([32,8,2]), B 2:
               implicit-GEMM conv kernels at C = 64 (unpadded tiles, the 3-stage adjoint ring).

Checked per case (reference lines: multigrid.py:263-311 solve, training.py:194-236 adjoint and
SGD, kernels.py:130-150 F): forward states <= 1e-12 relative to max|U|; every per-cycle FAS
residual norm within 1e-9 relative (+1e-12 sqrt(Nq) absolute); identical cycle counts for
forward and adjoint; adjoint states <= 1e-11 relative; updated theta within 1e-10 of the oracle
SGD step relative to max|lr g|; loss within 1e-10 relative.  Each case also asserts it ran the
kernel variants named above (lmg_route_counts).
"""

import numpy as np
import pytest

from _golden import fas

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2007_07336_b200 as P  # noqa: E402
from paper_2007_07336_b200 import _lib  # noqa: E402

LR = 0.1
CASES = {  # name: (N, q, B, c, threshold, max_cycles, kernel variants that must run)
    "c5_full": (1024, 512, 16, 16, 4, 50, ("step_tiny_full", "sweep_fcf", "sweep_seq")),
    "c2_full_2cyc": (1024, 512, 256, 4, 64, 2, ("step_small_full", "step_wide_full", "serial_splitk")),
    "c2_depth64": (64, 512, 256, 4, 4, 50, ("step_small_full", "step_wide_full", "serial_splitk")),
    "c4_depth32": (32, 1024, 128, 4, 8, 50, ("step_small_full", "step_wide_full")),
    # bench c6: BASELINE configs[4]'s shortest-critical-path point (q 16, one sample, cf 16)
    "c6_full": (1024, 16, 1, 16, 4, 50, ("sweep_fcf", "sweep_seq", "wsweep")),
    # bench c7: the deep narrow network (4096 x 16, cf 16, [4096, 256, 16]) -- warp FMA sweeps
    "c7_full": (4096, 16, 1, 16, 16, 50, ("sweep_fcf", "sweep_seq", "wsweep")),
    # bench c1: the reference demo's shape (q 32: the 32-column warp FMA sweeps)
    "c1_full": (64, 32, 64, 4, 16, 50, ("wsweep",)),
}


def band_ok(h_gpu, h_ref, N, q):
    return len(h_gpu) == len(h_ref) and all(
        abs(x - y) <= 1e-9 * abs(y) + 1e-12 * np.sqrt(N * q) for x, y in zip(h_gpu, h_ref))


def fast_block_grads(level, U, mu, D, scale):
    """fas.block_grads with the batch sum as one GEMM (the per-sample outer-product loop is
    minutes at B = 256); same quantity, different summation order (well inside 1e-10)."""
    N, h = level.n, level.step
    gW = np.empty((N,) + level.W.shape[1:])
    gb = np.empty((N, level.W.shape[1]))
    for n in range(N):
        gp = h * (mu[N - 1 - n] * D[n])
        gW[n] = (gp.T @ U[n]) * scale
        gb[n] = gp.sum(axis=0) * scale
    return gW, gb


def oracle_step(onet, X, labels, c, thr, max_cycles, lr):
    """The oracle's training step: FAS forward, FAS adjoint on the reversed linear system, block
    gradients (batch mean) and SGD; returns everything the GPU step is compared on."""
    B = X.shape[0]
    src = onet.source(X)
    U, fh, fconv = fas.solve(fas.build_levels(onet.blocks, c, thr), c, src, 1e-9, max_cycles)
    final, logits = fas.adjoint_head(onet, U)
    loss, dl = fas.loss_and_dlogits(logits, labels)
    gfin, _ = fas.g_final_from(onet, final, dl)
    D = fas.derivs(onet.blocks, U)
    adj = fas.adjoint_level(onet.blocks, D)
    s = np.zeros_like(U)
    s[0] = gfin
    mu, ah, aconv = fas.solve(fas.build_levels(adj, c, thr), c, s, 1e-9, max_cycles)
    gW, gb = fast_block_grads(onet.blocks, U, mu, D, 1.0 / B)
    return dict(U=U, fh=fh, mu=mu, ah=ah, loss=loss, W=onet.blocks.W - lr * gW,
                b=onet.blocks.b - lr * gb)


def _rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def _check(name, tr, d, W0, X, labels, ref, N, q, B, routes_before, want_routes):
    res = tr.step(torch.from_numpy(X).cuda(), torch.from_numpy(labels).cuda())
    U, lam, _ = tr._buffers(B, torch.device("cuda", 0))
    routes = _lib.route_counts()
    ran = {k: routes[k] - routes_before[k] for k in routes}
    for k in want_routes:
        assert ran[k] > 0, f"{name}: kernel variant {k} never ran ({ran})"
    e_u = _rel(U.cpu().numpy(), ref["U"])
    e_mu = _rel(lam.cpu().numpy(), ref["mu"])
    gW_sc = np.max(np.abs(d.stack.W.cpu().numpy() - ref["W"]))
    dW = np.max(np.abs(ref["W"] - W0))  # max |lr * g|
    for b in range(B):
        fc, ac = int(res.fwd_cycles[b]), int(res.adj_cycles[b])
        assert fc == len(ref["fh"][b]) - 1, (name, b, fc, ref["fh"][b])
        assert ac == len(ref["ah"][b]) - 1, (name, b, ac, ref["ah"][b])
        assert band_ok(res.fwd_hist[: fc + 1, b], ref["fh"][b], N, q), (name, b)
        assert band_ok(res.adj_hist[: ac + 1, b], ref["ah"][b], N, q), (name, b)
    print(f"{name}: |dU| {e_u:.1e} |dmu| {e_mu:.1e} |dW| {gW_sc / dW:.1e} of |lr g| cycles "
          f"{int(res.fwd_cycles.max())}+{int(res.adj_cycles.max())} routes "
          f"{ {k: v for k, v in ran.items() if v} }")
    assert e_u <= 1e-12, e_u
    assert e_mu <= 1e-11, e_mu
    assert gW_sc <= 1e-10 * dW + 1e-15, (gW_sc, dW)
    np.testing.assert_allclose(res.loss.cpu().numpy(), ref["loss"], rtol=1e-10)


@pytest.mark.parametrize("name", list(CASES))
def test_dense_step_matches_oracle_at_bench_shape(name):
    N, q, B, c, thr, mc, want = CASES[name]
    seed = [0, N, q]  # bench.py's seeding
    a = fas.random_network_arrays(N, q, seed)
    onet = fas.net_from_arrays(a)
    X = P.random_batch(q, seed, B)
    labels = np.arange(B) % 10
    ref = oracle_step(onet, X, labels, c, thr, mc, LR)
    d = P.device_network(N, q, seed, device="cuda:0")
    assert d.stack.W.cpu().numpy().tobytes() == a["W"].tobytes()
    tr = P.DeviceTrainer(d, coarsening=c, threshold=thr, tol=1e-9, max_cycles=mc, adjoint="fas",
                         learning_rate=LR)
    _check(name, tr, d, a["W"], X, labels, ref, N, q, B, _lib.route_counts(), want)


def test_conv_step_matches_oracle_at_c3_geometry():
    from paper_2007_07336_b200.synthetic import conv_device_network, conv_network_arrays

    N, C, side, B, c, thr = 32, 64, 32, 2, 4, 2
    seed = [0, N, C]  # bench.py's c3 seeding
    a = conv_network_arrays(N, C, side, seed, input_dim=64)
    fine = fas.ConvLevel(a["Wc"], a["b"], a["activation"], a["step"], side, side)
    onet = fas.Net(a["Wo"], a["bo"], "tanh", fine, a["Wr"], a["br"], "identity")
    X = P.random_batch(64, [0, N, C * side * side], B)
    labels = np.arange(B) % 10
    src = onet.source(X)
    U, fh, _ = fas.solve(fas.build_levels(fine, c, thr), c, src, 1e-9, 50)
    final, logits = fas.adjoint_head(onet, U)
    loss, dl = fas.loss_and_dlogits(logits, labels)
    gfin, _ = fas.g_final_from(onet, final, dl)
    D = fas.derivs(fine, U)
    s = np.zeros_like(U)
    s[0] = gfin
    mu, ah, _ = fas.solve(fas.build_levels(fas.adjoint_level(fine, D), c, thr), c, s, 1e-9, 50)
    gWc, gbc = fas.block_grads(fine, U, mu, D, 1.0 / B)

    d = conv_device_network(N, C, side, seed, device="cuda:0", input_dim=64)
    before = _lib.route_counts()
    tr = P.DeviceTrainer(d, coarsening=c, threshold=thr, tol=1e-9, max_cycles=50, adjoint="fas",
                         learning_rate=LR)
    res = tr.step(torch.from_numpy(X).cuda(), torch.from_numpy(labels).cuda())
    ran = {k: v - before[k] for k, v in _lib.route_counts().items()}
    for k in ("conv_fwd", "conv_adj", "conv_pgrad"):
        assert ran[k] > 0, (k, ran)
    assert int(res.fwd_cycles.max()) >= 3, "the c3-shaped case must exercise several FAS cycles"
    Ug, lam, _ = tr._buffers(B, torch.device("cuda", 0))
    q = C * side * side
    for b in range(B):
        fc, ac = int(res.fwd_cycles[b]), int(res.adj_cycles[b])
        assert fc == len(fh[b]) - 1 and ac == len(ah[b]) - 1, (b, fc, ac, fh[b], ah[b])
        assert band_ok(res.fwd_hist[: fc + 1, b], fh[b], N, q)
        assert band_ok(res.adj_hist[: ac + 1, b], ah[b], N, q)
    e_u, e_mu = _rel(Ug.cpu().numpy(), U), _rel(lam.cpu().numpy(), mu)
    # device conv weights are HWIO per block, like the reference's conv2d_params
    Wc_new = d.stack.W.cpu().numpy().reshape(a["Wc"].shape)
    want = a["Wc"] - LR * gWc
    gsc = np.max(np.abs(LR * gWc))
    e_w = np.max(np.abs(Wc_new - want))
    print(f"c3_depth32: |dU| {e_u:.1e} |dmu| {e_mu:.1e} |dW| {e_w / gsc:.1e} of |lr g| cycles "
          f"{int(res.fwd_cycles.max())}+{int(res.adj_cycles.max())}")
    assert e_u <= 1e-12 and e_mu <= 1e-11, (e_u, e_mu)
    assert e_w <= 1e-10 * gsc + 1e-15, (e_w, gsc)
    np.testing.assert_allclose(d.stack.b.cpu().numpy(), a["b"] - LR * gbc, rtol=0,
                               atol=1e-10 * np.max(np.abs(LR * gbc)) + 1e-15)
    np.testing.assert_allclose(res.loss.cpu().numpy(), loss, rtol=1e-10)

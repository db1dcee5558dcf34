"""GPU parity: the CUDA path (through the C-ABI) against the reference's golden vectors and the
CPU oracle.  Tolerances (FP64 GEMM summation order differs from OpenBLAS dgemv):
  states        <= 1e-12 max-abs
  history       |d norm_k| <= 1e-9 * norm_k + 1e-12 * sqrt(N q); identical cycles_used
  gradients     <= 1e-10 relative (1e-12 absolute floor)
Rows the reference produces as exact zeros must be exact zeros here too.
"""

import numpy as np
import pytest

from _golden import SOLVE_CASES, fas, histories, load, oracle_net

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2007_07336_b200 as P  # noqa: E402
from paper_2007_07336_b200 import _lib  # noqa: E402

DENSE_CASES = [c for c in SOLVE_CASES if not c.startswith("conv")]
CONV_CASES = [c for c in SOLVE_CASES if c.startswith("conv")]


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def gpu_net(g):
    """Our ResidualNetwork from a golden case's parameters."""
    act = str(g["activation"])
    if str(g["kind"]) == "conv2d":
        blocks = [P.conv2d_params(g["Wc"][i], g["b"][i], act, int(g["height"]), int(g["width"]))
                  for i in range(len(g["Wc"]))]
    else:
        blocks = [P.dense_params(g["W"][i], g["b"][i], act) for i in range(len(g["W"]))]
    return P.ResidualNetwork(P.dense_params(g["Wo"], g["bo"], str(g["open_act"])), blocks,
                             P.dense_params(g["Wr"], g["br"], str(g["read_act"])), float(g["step"]))


def band(a, b, N, q):
    return abs(a - b) <= 1e-9 * abs(b) + 1e-12 * np.sqrt(N * q)


def test_kat_one_cycle_and_sweeps():
    g = load("kat_n8_c4_q2")
    net = gpu_net(g)
    hier = P.build_hierarchy(net, 4)
    st = g["initial"].copy()
    norm = P.mg_cycle(hier, st, g["source"])
    assert np.max(np.abs(st - g["after"])) <= 1e-14
    assert abs(norm - float(g["norm"])) <= 1e-14
    part = P.make_partition(8, 4, 1)
    for name, fn in (("f_relaxed", P.f_relaxation), ("c_relaxed", P.c_relaxation),
                     ("fcf_relaxed", P.fcf_relaxation)):
        s = g["initial"].copy()
        fn(net, s, g["source"], part)
        assert np.max(np.abs(s - g[name])) <= 1e-14, name
    r0 = P.compute_residual(net, g["initial"], g["source"])
    assert np.max(np.abs(r0 - g["resid0"])) <= 1e-14
    assert np.max(np.abs(P.propagation_operator(net, g["after"]) - g["propop"])) <= 1e-14


@pytest.mark.parametrize("case", SOLVE_CASES)
def test_batched_solve_matches_reference(case):
    g = load(case)
    net = gpu_net(g)
    hier = P.build_hierarchy(net, int(g["c"]), int(g["threshold"]))
    assert [lv.num_layers for lv in hier.levels] == list(g["levels"])
    src = np.stack([np.asarray(P.source_from_input(net, x)) for x in g["samples"]], axis=1)
    states, rep = P.solve(hier, src, float(g["tol"]), int(g["max_cycles"]))
    N, B, q = states.shape
    assert np.max(np.abs(states - g["states"])) <= 1e-12
    for b, rh in enumerate(histories(g)):
        h = rep[b].residual_norms
        assert len(h) == len(rh), (b, h, rh)
        assert all(band(x, y, N, q) for x, y in zip(h, rh)), (h, rh)
        assert rep[b].converged == bool(g["converged"][b])
    # converged solves also agree with serial propagation (SPEC acceptance 2)
    seq = P.sequential_forward(net, src)
    assert np.max(np.abs(seq - g["seq"])) <= 1e-12


@pytest.mark.parametrize("case", ["c1_64x32_cf4", "ml3_64x8_cf4"])
def test_single_sample_api_matches_reference(case):
    g = load(case)
    net = gpu_net(g)
    hier = P.build_hierarchy(net, int(g["c"]), int(g["threshold"]))
    f = P.source_from_input(net, g["samples"][0])
    states, rep = P.solve(hier, f, float(g["tol"]), int(g["max_cycles"]))
    assert isinstance(states, np.ndarray) and states.shape == g["states"][:, 0].shape
    assert np.max(np.abs(states - g["states"][:, 0])) <= 1e-12
    assert rep.cycles_used == int(g["cycles"][0]) and rep.converged


def test_cycle_pieces_against_oracle():
    g = load("ml3_64x8_cf4")
    net, onet = gpu_net(g), oracle_net(g)
    rng = np.random.default_rng(0)
    N, q = g["W"].shape[:2]
    U = rng.normal(size=(N, 3, q))
    S = rng.normal(size=(N, 3, q))
    lev = onet.blocks
    assert np.max(np.abs(P.compute_residual(net, U, S) - fas.compute_residual(lev, U, S))) <= 1e-13
    assert np.max(np.abs(P.propagation_operator(net, U) - fas.propagation_operator(lev, U))) <= 1e-13
    assert np.max(np.abs(P.sequential_forward(net, S) - fas.sequential_forward(lev, S))) <= 1e-10
    assert np.array_equal(P.restrict_states(U, 4), fas.restrict_states(U, 4))
    hier = P.build_hierarchy(net, 4, 4)
    coarse = hier.levels[1]
    Uc, Rc = U[::4].copy(), S[::4].copy()
    got = P.assemble_coarse_source(Uc, Rc, coarse)
    want = fas.assemble_coarse_source(Uc, Rc, lev.coarsen(4))
    assert np.max(np.abs(got - want)) <= 1e-13
    # one full 3-level cycle from a random iterate
    a, b = U.copy(), U.copy()
    n1 = P.mg_cycle(hier, a, S)
    n2 = fas.mg_cycle(fas.build_levels(lev, 4, 4), 4, b, S)
    assert np.max(np.abs(a - b)) <= 1e-11
    assert np.all(np.abs(n1 - n2) <= 1e-9 * n2 + 1e-12 * np.sqrt(N * q))


def test_relaxation_exactness_rows_are_exact_zeros():
    """multigrid.py:145-157: after F (C) relaxation the F (C) residual rows are exactly zero --
    bitwise on the GPU too, since the same kernel recomputes them (test_multigrid.py:279-297)."""
    net = P.random_network(64, 24, [5, 64, 24])
    f = np.asarray(P.source_from_input(net, P.random_sample(24, 5)))
    part = P.make_partition(64, 4, 1)
    s = np.asarray(P.initial_guess(net, f)) + np.random.default_rng(1).normal(size=(64, 24))
    P.f_relaxation(net, s, f, part)
    r = P.compute_residual(net, s, f)
    fmask = np.arange(64) % 4 != 0
    assert np.all(r[fmask] == 0.0)
    P.c_relaxation(net, s, f, part)
    r = P.compute_residual(net, s, f)
    assert np.all(r[~fmask] == 0.0)


@pytest.mark.parametrize("case", SOLVE_CASES)
def test_gradients_match_reference(case):
    g = load(case)
    net = gpu_net(g)
    for b in range(len(g["samples"])):
        loss, gr = P.loss_and_grad(net, g["states"][:, b], g["samples"][b], int(g["labels"][b]))
        assert abs(loss - g["loss"][b]) <= 1e-12 * max(1.0, abs(g["loss"][b]))
        gW = np.stack([w for w, _ in gr.blocks])
        gb = np.stack([x for _, x in gr.blocks])
        for got, want in ((gW, g["gW"][b]), (gb, g["gb"][b]), (gr.opening[0], g["gWo"][b]),
                          (gr.opening[1], g["gbo"][b]), (gr.readout[0], g["gWr"][b]),
                          (gr.readout[1], g["gbr"][b])):
            scale = max(np.max(np.abs(want)), 1e-300)
            assert np.max(np.abs(got - want)) <= 1e-10 * scale + 1e-14


@pytest.mark.parametrize("case", ["c1_64x32_cf4", "ml3_64x8_cf4", "relu_128x24_cf8_3lvl",
                                  "conv_relu_d16_c4x8x8"])
def test_fas_adjoint_batch_matches_reference_grads(case):
    """The FAS adjoint (no reference implementation) converges to the reference's gradients;
    its residual history matches the oracle's FAS adjoint."""
    g = load(case)
    net = gpu_net(g)
    dnet = P.DeviceNet.from_network(net)
    U = dev(g["states"])
    X = dev(g["samples"])
    labels = dev(g["labels"])
    B = X.shape[0]
    r = P.backward(dnet, U, X, labels, adjoint="fas", coarsening=int(g["c"]),
                   threshold=int(g["threshold"]), tol=1e-12, max_cycles=60, scale=1.0)
    assert all(r.converged)
    gW = r.gW.cpu().numpy()
    want = (g["gW"] if "gW" in g else g["gW"]).sum(axis=0)
    assert np.max(np.abs(gW - want)) <= 1e-9 * np.max(np.abs(want))
    np.testing.assert_allclose(r.loss.cpu().numpy(), g["loss"], rtol=1e-12)
    # oracle FAS adjoint history
    onet = oracle_net(g)
    final, logits = fas.adjoint_head(onet, g["states"])
    _, dl = fas.loss_and_dlogits(logits, g["labels"])
    gfin, _ = fas.g_final_from(onet, final, dl)
    D = fas.derivs(onet.blocks, g["states"])
    adj = fas.adjoint_level(onet.blocks, D)
    src = np.zeros_like(g["states"])
    src[0] = gfin
    levels = fas.build_levels(adj, int(g["c"]), int(g["threshold"]))
    _, ohist, _ = fas.solve(levels, int(g["c"]), src, 1e-12, 60)
    N, q = g["states"].shape[0], g["states"].shape[2]
    for b in range(B):
        h = r.hist[: r.cycles[b] + 1, b]
        assert len(h) == len(ohist[b])
        assert all(band(x, y, N, q) for x, y in zip(h, ohist[b]))


def test_device_network_is_bitwise_the_references():
    net = P.random_network(64, 32, [0, 64, 32])
    d = P.device_network(64, 32, [0, 64, 32])
    assert d.stack.W.cpu().numpy().tobytes() == np.stack([b.weights for b in net.blocks]).tobytes()
    assert d.stack.b.cpu().numpy().tobytes() == np.stack([b.bias for b in net.blocks]).tobytes()


def test_trainer_step_matches_oracle_sgd():
    """One DeviceTrainer step (FAS forward to tol, FAS adjoint, fused SGD) equals the oracle's
    solve + sequential adjoint + batch-mean SGD within tolerance."""
    N, q, B, lr = 64, 32, 4, 0.1
    a = fas.random_network_arrays(N, q, [0, N, q])
    X = fas.random_sample(q, [0, N, q])[None].repeat(B, 0) + np.arange(B)[:, None] * 0.1
    labels = np.arange(B) % 10
    d = P.device_network(N, q, [0, N, q])
    tr = P.DeviceTrainer(d, coarsening=4, tol=1e-11, max_cycles=50, adjoint="fas", learning_rate=lr)
    res = tr.step(dev(X), dev(labels))
    assert res.fwd_converged.all() and res.adj_converged.all()
    onet = fas.net_from_arrays(a)
    src = onet.source(X)
    lv = fas.build_levels(onet.blocks, 4)
    U, _, _ = fas.solve(lv, 4, src, 1e-11, 50)
    final, logits = fas.adjoint_head(onet, U)
    loss, dl = fas.loss_and_dlogits(logits, labels)
    gfin, _ = fas.g_final_from(onet, final, dl)
    D = fas.derivs(onet.blocks, U)
    mu, lam0 = fas.adjoint_sequential(fas.adjoint_level(onet.blocks, D), gfin)
    gW, gb = fas.block_grads(onet.blocks, U, mu, D, 1.0 / B)
    W_new = a["W"] - lr * gW
    got = d.stack.W.cpu().numpy()
    assert np.max(np.abs(got - W_new)) <= 1e-10 * np.max(np.abs(lr * gW)) + 1e-15
    np.testing.assert_allclose(res.loss.cpu().numpy(), loss, rtol=1e-10)


@pytest.mark.parametrize("N,q,B,c,thr", [(256, 64, 16, 4, 16), (512, 128, 8, 8, 8)])
def test_larger_solve_against_oracle(N, q, B, c, thr):
    a = fas.random_network_arrays(N, q, [1, N, q])
    onet = fas.net_from_arrays(a)
    X = np.stack([fas.random_sample(q, [1, N, q, b]) for b in range(B)])
    src = onet.source(X)
    lv = fas.build_levels(onet.blocks, c, thr)
    U, hist, conv = fas.solve(lv, c, src, 1e-9, 50)
    d = P.device_network(N, q, [1, N, q])
    tr = P.DeviceTrainer(d, coarsening=c, threshold=thr, tol=1e-9, max_cycles=50)
    Ug, h, cyc, cv = tr.forward(dev(X))
    assert np.max(np.abs(Ug.cpu().numpy() - U)) <= 1e-11
    for b in range(B):
        assert cyc[b] == len(hist[b]) - 1
        assert all(band(x, y, N, q) for x, y in zip(h[: cyc[b] + 1, b], hist[b]))


def test_conv_transform_and_vjp_against_oracle():
    """kernels.py:130-136 / 171-188 for single conv blocks (odd geometry, 3 channels, 5x7)."""
    rng = np.random.default_rng(5)
    C, H, Wd = 3, 5, 7
    p = P.conv2d_params(rng.normal(0, 0.3, (3, 3, C, C)), rng.normal(0, 0.1, C), "tanh", H, Wd)
    lev = fas.ConvLevel(p.weights[None], p.bias[None], "tanh", 1.0, H, Wd)
    X = rng.normal(size=(4, C * H * Wd))
    G = rng.normal(size=(4, C * H * Wd))
    y = P.apply_transform(p, X)
    assert np.max(np.abs(y - lev.F(0, X))) <= 1e-14
    gx, gw, gb = P.transform_vjp(p, X, G)
    D = fas.act_deriv("tanh", lev.pre(0, X))
    assert np.max(np.abs(gx - lev.vjp_input(0, X, G * D))) <= 1e-13
    ow, ob = lev.param_grads(0, X, G * D)
    assert np.max(np.abs(gw - ow)) <= 1e-12 * np.max(np.abs(ow))
    assert np.max(np.abs(gb - ob)) <= 1e-12 * np.max(np.abs(ob))


def test_split_batch_step_matches_unsplit():
    """DeviceTrainer(split=2): batch slices on concurrent streams -- per-sample solves are bitwise
    the unsplit ones; accumulated gradients and the SGD step agree within rounding."""
    N, q, B = 64, 32, 8
    X = dev(P.random_batch(q, [2, N, q], B))
    labels = dev(np.arange(B) % 10)
    res = {}
    for split in (1, 2):
        d = P.device_network(N, q, [2, N, q])
        tr = P.DeviceTrainer(d, coarsening=4, tol=1e-10, max_cycles=50, adjoint="fas",
                             learning_rate=0.1, split=split)
        r = tr.step(X, labels)
        res[split] = (r, d.stack.W.cpu().numpy(), d.Wo.cpu().numpy())
    r1, W1, Wo1 = res[1]
    r2, W2, Wo2 = res[2]
    h1 = r1.fwd_hist[: r1.fwd_cycles.max() + 1]
    h2 = r2.fwd_hist[: r2.fwd_cycles.max() + 1]
    assert np.array_equal(h1, h2, equal_nan=True)
    assert np.array_equal(r1.loss.cpu().numpy(), r2.loss.cpu().numpy())
    assert np.max(np.abs(W1 - W2)) <= 1e-14
    assert np.max(np.abs(Wo1 - Wo2)) <= 1e-14


def test_fast_tanh_accuracy():
    """The epilogue's FP64 tanh (lmg_gemm.cuh fast_tanh) against numpy's (the reference's
    activation, kernels.py:24-28): a few ulp over the whole range, exact +-1 in the tails, NaN
    propagated.  Evaluated through apply_transform with an identity weight (pre = u exactly)."""
    q = 64
    rng = np.random.default_rng(17)
    x = np.concatenate([rng.uniform(-25, 25, 20000), rng.normal(0, 1e-3, 4000),
                        rng.normal(0, 1e-9, 2000), 10.0 ** rng.uniform(-300, -20, 1000),
                        -(10.0 ** rng.uniform(-300, -20, 1000)), [0.0, -0.0, 19.0, 19.1, 20.0,
                                                                   -20.0, 700.0, -700.0, 1e300]])
    x = np.concatenate([x, np.zeros((-len(x)) % q)]).reshape(-1, q)
    p = P.dense_params(np.eye(q), np.zeros(q), "tanh")
    got = P.apply_transform(p, x)
    want = np.tanh(x)
    ulp = np.abs(got - want) / np.spacing(np.maximum(np.abs(want), np.finfo(float).tiny))
    assert np.max(ulp) <= 4, float(np.max(ulp))
    assert np.array_equal(np.sign(got), np.sign(want))
    big = np.abs(x) >= 19.1
    assert np.all(np.abs(got[big]) == 1.0)
    y = P.apply_transform(p, np.full((1, q), np.nan))
    assert np.all(np.isnan(y))

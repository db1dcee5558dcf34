"""Pin the CPU oracle (oracle/fas.py) against golden vectors frozen from the live reference.

exact mode (per-sample W @ u, the reference's own dgemv) must agree BITWISE; batched mode (one
dgemm per layer step) within 1e-13 on states / the SURVEY 7.2 absolute band on histories.
"""

import numpy as np
import pytest

from _golden import SOLVE_CASES, fas, histories, load, oracle_net


def test_kat_one_cycle_bitwise():
    """tests/test_multigrid.py:312-367 KAT, restated through the oracle."""
    g = load("kat_n8_c4_q2")
    net = oracle_net(g, exact=True)
    lev = net.blocks
    src = g["source"][:, None, :]
    levels = fas.build_levels(lev, 4)
    st = g["initial"][:, None, :].copy()
    assert np.array_equal(fas.initial_guess(lev, src), st)
    nrm = fas.mg_cycle(levels, 4, st, src)
    assert st[:, 0].tobytes() == g["after"].tobytes()
    assert nrm[0] == g["norm"]
    r0 = fas.compute_residual(lev, g["initial"][:, None, :], src)
    assert r0[:, 0].tobytes() == g["resid0"].tobytes()
    for name, fn in (("f_relaxed", fas.f_relaxation), ("c_relaxed", fas.c_relaxation),
                     ("fcf_relaxed", fas.fcf_relaxation)):
        st = g["initial"][:, None, :].copy()
        fn(lev, st, src, 4)
        assert st[:, 0].tobytes() == g[name].tobytes(), name
    assert fas.propagation_operator(lev, g["after"][:, None, :])[:, 0].tobytes() == g["propop"].tobytes()


@pytest.mark.parametrize("case", SOLVE_CASES)
@pytest.mark.parametrize("exact", [True, False])
def test_solve_and_grads_match_reference(case, exact):
    g = load(case)
    net = oracle_net(g, exact=exact)
    X = g["samples"]
    src = net.source(X)
    levels = fas.build_levels(net.blocks, int(g["c"]), int(g["threshold"]))
    assert [lv.n for lv in levels] == list(g["levels"])
    states, hist, conv = fas.solve(levels, int(g["c"]), src, float(g["tol"]), int(g["max_cycles"]))
    ref_hist = histories(g)
    if exact:
        assert states.tobytes() == g["states"].tobytes()
        assert hist == ref_hist
    else:
        assert np.max(np.abs(states - g["states"])) <= 1e-12
        N, q = states.shape[0], states.shape[2]
        for h, rh in zip(hist, ref_hist):
            assert len(h) == len(rh)
            for a, b in zip(h, rh):
                assert abs(a - b) <= 1e-9 * b + 1e-12 * np.sqrt(N * q)
    assert list(conv) == list(g["converged"])
    # serial oracle
    seq = fas.sequential_forward(net.blocks, src)
    if exact:
        assert seq.tobytes() == g["seq"].tobytes()
    else:
        assert np.max(np.abs(seq - g["seq"])) <= 1e-12

    # gradients at the converged states: loss_and_grad restated through the adjoint system
    final, logits = fas.adjoint_head(net, g["states"])
    loss, dl = fas.loss_and_dlogits(logits, g["labels"])
    np.testing.assert_allclose(loss, g["loss"], rtol=1e-13, atol=1e-14)
    gfin, gp_read = fas.g_final_from(net, final, dl)
    D = fas.derivs(net.blocks, g["states"])
    adj = fas.adjoint_level(net.blocks, D)
    mu, lam0 = fas.adjoint_sequential(adj, gfin)
    for b in range(X.shape[0]):
        gW, gb = fas.block_grads(net.blocks, g["states"][:, b : b + 1], mu[:, b : b + 1],
                                 D[:, b : b + 1], 1.0)
        np.testing.assert_allclose(gW, g["gW"][b], rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(gb, g["gb"][b], rtol=1e-12, atol=1e-15)
        # readout / opening grads (kernels.py:166-169)
        np.testing.assert_allclose(np.outer(gp_read[b], final[b]), g["gWr"][b], rtol=1e-13, atol=1e-15)
        pre_o = net.Wo @ X[b] + net.bo
        gpo = lam0[b] * fas.act_deriv(net.open_act, pre_o)
        np.testing.assert_allclose(np.outer(gpo, X[b]), g["gWo"][b], rtol=1e-11, atol=1e-14)
        np.testing.assert_allclose(gpo, g["gbo"][b], rtol=1e-11, atol=1e-14)


@pytest.mark.parametrize("case", ["c1_64x32_cf4", "ml3_64x8_cf4", "conv_d8_c2x6x6"])
def test_fas_adjoint_converges_to_sequential_adjoint(case):
    """The FAS adjoint (no reference implementation: SURVEY 8c) must converge to the reference's
    sequential reverse-mode recursion, itself pinned above."""
    g = load(case)
    net = oracle_net(g)
    final, logits = fas.adjoint_head(net, g["states"])
    _, dl = fas.loss_and_dlogits(logits, g["labels"])
    gfin, _ = fas.g_final_from(net, final, dl)
    D = fas.derivs(net.blocks, g["states"])
    adj = fas.adjoint_level(net.blocks, D)
    mu_seq, _ = fas.adjoint_sequential(adj, gfin)
    src = np.zeros_like(mu_seq)
    src[0] = gfin
    levels = fas.build_levels(adj, int(g["c"]), int(g["threshold"]))
    mu, hist, conv = fas.solve(levels, int(g["c"]), src, 1e-11, 60)
    assert all(conv)
    assert np.max(np.abs(mu - mu_seq)) <= 1e-10

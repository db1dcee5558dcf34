"""Training-path parity on the GPU: finite-difference gradients (reference
tests/test_training.py:162-191, rel <= 1e-5) and one train_epoch against the oracle's restatement
of training.py:255-289 (early-stopped 2-cycle solves, per-sample adjoint, batch mean, SGD)."""

import numpy as np
import pytest

from _golden import fas

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2007_07336_b200 as P  # noqa: E402


def _loss(net, x, label):
    f = P.source_from_input(net, x)
    st = P.sequential_forward(net, f)
    logits = P.forward_logits(net, st)
    z = logits - logits.max()
    return float(np.log(np.exp(z).sum()) - z[label])


def test_finite_difference_gradients():
    net = P.random_network(6, 4, [11, 6, 4], input_dim=3, num_classes=3)
    x = P.random_sample(3, 11)
    label = 2
    st = P.sequential_forward(net, P.source_from_input(net, x))
    _, g = P.loss_and_grad(net, st, x, label)
    rng = np.random.default_rng(0)
    eps = 1e-6
    checks = [(net.opening.weights, g.opening[0]), (net.readout.weights, g.readout[0])]
    checks += [(net.blocks[i].weights, g.blocks[i][0]) for i in range(6)]
    checks += [(net.blocks[i].bias, g.blocks[i][1]) for i in range(6)]
    for param, grad in checks:
        for _ in range(2):
            idx = tuple(rng.integers(0, s) for s in param.shape)
            old = param[idx]
            # the reference's pattern: edit the host array in place and re-evaluate, no rebuild
            # (the device copy follows host edits, network.ResidualNetwork.device_stack)
            param[idx] = old + eps
            lp = _loss(net, x, label)
            param[idx] = old - eps
            lm = _loss(net, x, label)
            param[idx] = old
            fd = (lp - lm) / (2 * eps)
            assert abs(fd - grad[idx]) <= 1e-5 * max(1e-3, abs(fd)), (idx, fd, grad[idx])


@pytest.mark.parametrize("n,epochs", [(12, 1), (10, 2)])
def test_train_epoch_matches_oracle(n, epochs):
    """(10, 2): a ragged last batch (4, 4, 2) and a second epoch on the same network -- the per-
    batch-size device buffers and the pinned parameter mirror carried across epochs."""
    rng = np.random.default_rng(3)
    images = rng.random((n, 28, 28))
    labels = rng.integers(0, 10, n)
    data = P.Dataset(images, labels)
    net = P.random_network(16, 8, [3, 16, 8], input_dim=784, horizon=1.0)
    a = fas.random_network_arrays(16, 8, [3, 16, 8], input_dim=784, horizon=1.0)
    cfg = P.TrainConfig(learning_rate=0.1, batch_size=4, epochs=1, mg_cycles=2)
    train_rng = np.random.default_rng(7)
    for _ in range(epochs):
        stats = P.train_epoch(net, data, cfg, rng=train_rng)
    # oracle: training.py:255-289 with oracle/fas.py pieces
    oracle_rng = np.random.default_rng(7)
    W, b, Wo, bo, Wr, br = (a["W"].copy(), a["b"].copy(), a["Wo"].copy(), a["bo"].copy(),
                            a["Wr"].copy(), a["br"].copy())
    for _ in range(epochs):
        order = oracle_rng.permutation(n)
        losses = []
        for lo in range(0, n, 4):
            idx = order[lo : lo + 4]
            X = images[idx].reshape(len(idx), -1)
            onet = fas.Net(Wo, bo, "tanh", fas.DenseLevel(W, b, "tanh", a["step"]), Wr, br, "identity")
            src = onet.source(X)
            U, _, _ = fas.solve(fas.build_levels(onet.blocks, 4), 4, src, 1e-12, 2)
            final, logits = fas.adjoint_head(onet, U)
            loss, dl = fas.loss_and_dlogits(logits, labels[idx])
            losses += list(loss)
            gfin, gpr = fas.g_final_from(onet, final, dl)
            D = fas.derivs(onet.blocks, U)
            mu, lam0 = fas.adjoint_sequential(fas.adjoint_level(onet.blocks, D), gfin)
            gW, gb = fas.block_grads(onet.blocks, U, mu, D, 1.0 / len(idx))
            gpo = lam0 * fas.act_deriv("tanh", X @ Wo.T + bo)
            gWo, gbo = gpo.T @ X / len(idx), gpo.sum(0) / len(idx)
            gWr, gbr = gpr.T @ final / len(idx), gpr.sum(0) / len(idx)
            W, b = W - 0.1 * gW, b - 0.1 * gb
            Wo, bo, Wr, br = Wo - 0.1 * gWo, bo - 0.1 * gbo, Wr - 0.1 * gWr, br - 0.1 * gbr
    got = np.stack([blk.weights for blk in net.blocks])
    assert np.max(np.abs(got - W)) <= 1e-11
    assert np.max(np.abs(net.opening.weights - Wo)) <= 1e-11
    assert np.max(np.abs(net.readout.weights - Wr)) <= 1e-11
    assert abs(stats.mean_loss - float(np.mean(losses))) <= 1e-12


def test_host_edits_reach_the_device_copy():
    """an in-place edit of blocks[i].weights after the first device use must be seen by
    the next solve (multigrid.py:83-85 aliasing semantics), with only the edited block re-sent."""
    net = P.random_network(32, 8, [4, 32, 8])
    f = P.source_from_input(net, P.random_sample(8, 4))
    s1 = P.sequential_forward(net, f)
    net.blocks[5].weights *= 1.5
    net.blocks[9].bias += 0.25
    s2 = P.sequential_forward(net, f)
    fresh = P.ResidualNetwork(net.opening, [P.dense_params(b.weights.copy(), b.bias.copy(), b.activation)
                                            for b in net.blocks], net.readout, net.step_size)
    s3 = P.sequential_forward(fresh, f)
    assert not np.array_equal(s1, s2)
    assert np.array_equal(s2, s3)
    # device-side updates survive (host unchanged since upload) and are written back on request
    d = net.device_stack()
    d.W[3] += 1.0
    assert np.array_equal(net.device_stack().W[3].cpu().numpy(), net.blocks[3].weights + 1.0)
    net.pull_from_device()
    assert np.array_equal(net.device_stack().W.cpu().numpy(), np.stack([b.weights for b in net.blocks]))

"""Freeze golden vectors from the LIVE reference (run in the build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every case stores the network parameters it was generated from, the per-sample inputs, the
reference's converged states (`solve`), per-cycle residual histories (`CycleReport`), the
serial oracle (`sequential_forward`) and `loss_and_grad` at the converged states, so the GPU
box (which has no /root/reference) can check both the CPU oracle and the CUDA path.
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

import layermg as L  # noqa: E402
from layermg.multigrid import initial_guess  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def _net_arrays(net):
    blk = net.blocks[0]
    d = dict(
        step=np.float64(net.step_size),
        activation=np.array(blk.activation),
        kind=np.array(blk.kind),
        Wo=net.opening.weights, bo=net.opening.bias, open_act=np.array(net.opening.activation),
        Wr=net.readout.weights, br=net.readout.bias, read_act=np.array(net.readout.activation),
        b=np.stack([b.bias for b in net.blocks]),
    )
    if blk.kind == "dense":
        d["W"] = np.stack([b.weights for b in net.blocks])
    else:
        d["Wc"] = np.stack([b.weights for b in net.blocks])
        d["height"] = np.int64(blk.height)
        d["width"] = np.int64(blk.width)
    return d


def solve_case(name, net, samples, labels, c, threshold=None, tol=1e-9, max_cycles=50):
    hier = L.build_hierarchy(net, c, threshold)
    out = _net_arrays(net)
    states_all, hist_all, conv_all, seq_all = [], [], [], []
    loss_all, gW_all, gb_all, gWo_all, gbo_all, gWr_all, gbr_all = [], [], [], [], [], [], []
    for x, lab in zip(samples, labels):
        f = L.source_from_input(net, x)
        st, rep = L.solve(hier, f, tol=tol, max_cycles=max_cycles)
        states_all.append(st)
        hist_all.append(rep.residual_norms)
        conv_all.append(rep.converged)
        seq_all.append(L.sequential_forward(net, f))
        loss, g = L.loss_and_grad(net, st, x, int(lab))
        loss_all.append(loss)
        gW_all.append(np.stack([w for w, _ in g.blocks]))
        gb_all.append(np.stack([b for _, b in g.blocks]))
        gWo_all.append(g.opening[0]); gbo_all.append(g.opening[1])
        gWr_all.append(g.readout[0]); gbr_all.append(g.readout[1])
    maxlen = max(len(h) for h in hist_all)
    hist = np.full((len(samples), maxlen), np.nan)
    for i, h in enumerate(hist_all):
        hist[i, : len(h)] = h
    out.update(
        c=np.int64(c), threshold=np.int64(hier.coarsest_direct_threshold), tol=np.float64(tol),
        max_cycles=np.int64(max_cycles), levels=np.array([lv.num_layers for lv in hier.levels]),
        samples=np.stack(samples), labels=np.array(labels, dtype=np.int64),
        states=np.stack(states_all, axis=1),          # (N, B, q)
        seq=np.stack(seq_all, axis=1),                # (N, B, q)
        hist=hist, cycles=np.array([len(h) - 1 for h in hist_all]), converged=np.array(conv_all),
        loss=np.array(loss_all), gW=np.stack(gW_all), gb=np.stack(gb_all),
        gWo=np.stack(gWo_all), gbo=np.stack(gbo_all), gWr=np.stack(gWr_all), gbr=np.stack(gbr_all),
    )
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **out)
    print(name, [lv.num_layers for lv in hier.levels], "cycles", out["cycles"], "final", hist[:, -1])


def experiment(depth, width, seed=0, horizon=4.0, nsamp=2, **kw):
    net = L.random_network(depth, width, [seed, depth, width], horizon=horizon, **kw)
    xs = [L.random_sample(width, [seed, depth, width, b]) for b in range(nsamp)]
    # sample 0 is exactly cli._experiment_net's sample (cli.py:150-153)
    xs[0] = L.random_sample(width, [seed, depth, width])
    return net, xs, [b % net.readout.output_width for b in range(nsamp)]


def kat():
    """tests/test_multigrid.py:312-367 problem: one 2-level cycle, N=8, c=4, q=2, seed 23."""
    net = L.random_network(8, 2, [23, 8, 2])
    f = L.source_from_input(net, L.random_sample(2, [23, 8, 2]))
    hier = L.build_hierarchy(net, 4)
    st0 = initial_guess(net, f)
    st = st0.copy()
    norm = L.mg_cycle(hier, st, f)
    resid0 = L.compute_residual(net, st0, f)
    # relaxation pieces, each from the same initial guess
    fr = st0.copy(); L.f_relaxation(net, fr, f, L.make_partition(8, 4, 1))
    cr = st0.copy(); L.c_relaxation(net, cr, f, L.make_partition(8, 4, 1))
    fcf = st0.copy(); L.fcf_relaxation(net, fcf, f, L.make_partition(8, 4, 1))
    d = _net_arrays(net)
    d.update(source=f, initial=st0, after=st, norm=np.float64(norm), resid0=resid0,
             f_relaxed=fr, c_relaxed=cr, fcf_relaxed=fcf,
             propop=L.propagation_operator(net, st))
    np.savez_compressed(os.path.join(OUT, "kat_n8_c4_q2.npz"), **d)
    print("kat norm", norm)


def conv_case():
    """tests/test_multigrid.py:450-470 conv net (2 channels, 6x6, depth 8, h 0.25), dense opening."""
    rng = np.random.default_rng(46)
    channels, side = 2, 6
    width = channels * side * side
    depth, h = 8, 0.25
    blocks = [
        L.conv2d_params(rng.normal(0, 0.15, (3, 3, channels, channels)), rng.normal(0, 0.05, channels),
                        "tanh", side, side)
        for _ in range(depth)
    ]
    net = L.ResidualNetwork(
        opening=L.dense_params(rng.normal(0, 0.3, (width, 5)), np.zeros(width), "tanh"),
        blocks=blocks,
        readout=L.dense_params(rng.normal(size=(3, width)), np.zeros(3), "identity"),
        step_size=h,
    )
    xs = [rng.normal(size=5) for _ in range(2)]
    solve_case("conv_d8_c2x6x6", net, xs, [0, 2], 4, tol=1e-10)


def conv_relu_case():
    """A config-3-shaped (relu, h = 4/N) conv net at toy size: 16 layers, 4 channels, 8x8."""
    rng = np.random.default_rng([0, 16, 4])
    C, side, depth = 4, 8, 16
    width = C * side * side
    blocks = [
        L.conv2d_params(rng.normal(0, 1 / np.sqrt(9 * C), (3, 3, C, C)), rng.normal(0, 0.05, C),
                        "relu", side, side)
        for _ in range(depth)
    ]
    net = L.ResidualNetwork(
        opening=L.dense_params(rng.normal(0, 1 / np.sqrt(12), (width, 12)), rng.normal(0, .05, width), "tanh"),
        blocks=blocks,
        readout=L.dense_params(rng.normal(0, 1 / np.sqrt(width), (10, width)), np.zeros(10), "identity"),
        step_size=4.0 / depth,
    )
    xs = [rng.normal(size=12) for _ in range(2)]
    solve_case("conv_relu_d16_c4x8x8", net, xs, [1, 7], 4, threshold=1)


def netfile_case():
    """A network file written by the reference's own save_network (network.py:199-216, .json + LE
    float64 .bin in declaration order), with the arrays it holds, for the loader parity test."""
    net = L.random_network(8, 6, [5, 8, 6], input_dim=4, num_classes=3)
    L.save_network(net, os.path.join(OUT, "net_dense_8x6"))
    np.savez_compressed(os.path.join(OUT, "net_dense_8x6_arrays.npz"), **_net_arrays(net))
    rng = np.random.default_rng([9, 2])
    blocks = [L.conv2d_params(rng.normal(0, 0.2, (3, 3, 2, 2)), rng.normal(0, 0.05, 2), "relu", 3, 4)
              for _ in range(3)]
    opening = L.dense_params(rng.normal(0, 0.3, (24, 5)), rng.normal(0, 0.1, 24), "tanh")
    readout = L.dense_params(rng.normal(0, 0.3, (3, 24)), np.zeros(3), "identity")
    cnet = L.ResidualNetwork(opening=opening, blocks=blocks, step_size=0.25, readout=readout)
    L.save_network(cnet, os.path.join(OUT, "net_conv_3x2x3x4"))
    np.savez_compressed(os.path.join(OUT, "net_conv_3x2x3x4_arrays.npz"), **_net_arrays(cnet))
    print("network files written")


if __name__ == "__main__":
    if sys.argv[1:] == ["--only", "netfile"]:
        netfile_case()
        sys.exit(0)
    netfile_case()
    kat()
    net, xs, labs = experiment(64, 32, nsamp=3)
    solve_case("c1_64x32_cf4", net, xs, labs, 4)
    solve_case("c1_64x32_cf4_early2", net, xs, labs, 4, tol=1e-12, max_cycles=2)
    net, xs, labs = experiment(64, 8, seed=1, nsamp=2)
    solve_case("ml3_64x8_cf4", net, xs, labs, 4, threshold=4)
    net, xs, labs = experiment(32, 4, seed=2, nsamp=2)
    solve_case("ml4_32x4_cf2", net, xs, labs, 2, threshold=4)
    net, xs, labs = experiment(4, 2, seed=42, nsamp=2)
    solve_case("single_block_4x2_cf4", net, xs, labs, 4)
    net, xs, labs = experiment(256, 16, seed=3, nsamp=2)
    solve_case("d256x16_cf16", net, xs, labs, 16)
    net, xs, labs = experiment(128, 24, seed=4, nsamp=2, activation="relu")
    solve_case("relu_128x24_cf8_3lvl", net, xs, labs, 8, threshold=2)
    conv_case()
    conv_relu_case()

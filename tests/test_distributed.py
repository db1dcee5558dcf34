"""Multi-rank layer-partitioned FAS on CPU: world_size 2, 4 and 8 under gloo, the same DistSolver
the GPUs run, with the oracle-backed numpy level ops (oracle/local_ops.py).  Checks, against the
single-process oracle solve (multigrid.py:175-311):
  * states bitwise identical (forward and the reversed adjoint system),
  * per-sample residual histories within the SURVEY 7.2 band, and bitwise equal across world sizes
    (canonical per-block norm partials),
  * the protocol: halo messages per rank per cycle (1 per cross edge per C-sweep + 2 residual /
    coarse-source rows per relaxed level + 1 on the pipelined coarsest level).
"""

import os
import pickle
import socket
import sys

import numpy as np
import pytest

from _golden import ROOT, fas

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from oracle.local_ops import NumpyOps, OracleView  # noqa: E402

N, Q, B, C, THR = 64, 8, 3, 4, 4
TOL, MAXC = 1e-11, 40
# the c5 hierarchy (cf 16, levels [1024, 64, 4]) at narrow width: at 8 ranks the finest level
# splits (8 blocks per rank) and level 1 does not, so [64, 4] is gathered onto every rank
C5 = dict(N=1024, Q=4, B=2, C=16, THR=4, seed=11)
BASE = dict(N=N, Q=Q, B=B, C=C, THR=THR, seed=9)


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem(sh=BASE):
    N, Q, B, sd = sh["N"], sh["Q"], sh["B"], sh["seed"]
    a = fas.random_network_arrays(N, Q, [sd, N, Q])
    net = fas.net_from_arrays(a)
    X = np.stack([fas.random_sample(Q, [sd, N, Q, b]) for b in range(B)])
    return a, net, X


def _worker(rank, world, port, out, mode, sh=BASE):
    N, Q, B, C, THR = sh["N"], sh["Q"], sh["B"], sh["C"], sh["THR"]
    sys.path.insert(0, ROOT)
    os.environ["CUDA_VISIBLE_DEVICES"] = ""
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    from paper_2007_07336_b200 import _lib
    from paper_2007_07336_b200.distributed import DistSolver

    a, net, X = _problem(sh)
    L = N // world
    lo, hi = rank * L, (rank + 1) * L
    fine = fas.DenseLevel(a["W"], a["b"], a["activation"], a["step"])
    local = fas.DenseLevel(a["W"][lo:hi], a["b"][lo:hi], a["activation"], a["step"])
    levels = fas.build_levels(fine, C, THR)
    if mode == "fwd":
        view = OracleView(local)
        head = torch.from_numpy(net.source(X)[0].copy()) if rank == 0 else None
        reverse = False
    else:
        src = net.source(X)
        U, _, _ = fas.solve(levels, C, src, 1e-12, 60)
        D = fas.derivs(fine, U)
        final, logits = fas.adjoint_head(net, U)
        _, dl = fas.loss_and_dlogits(logits, np.arange(B) % 10)
        gfin, _ = fas.g_final_from(net, final, dl)
        view = OracleView(fas.adjoint_level(local, D[lo:hi]))
        head = torch.from_numpy(gfin.copy()) if rank == world - 1 else None
        reverse = True
    solver = DistSolver(view, N, C, len(levels), B, rank=rank, world=world, ops=NumpyOps(),
                        reverse=reverse, device="cpu")
    U0 = torch.zeros(L + 1, B, Q, dtype=torch.float64)
    hist, cyc, conv = solver.solve(U0, head, _lib.SRC_HEAD, tol=TOL, max_cycles=MAXC)
    parts = [torch.empty(L, B, Q, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(parts, U0[:L].contiguous())
    if rank == 0:
        if reverse:  # the adjoint system's rows 0.. live on the last rank
            parts = parts[::-1]
        states = torch.cat(parts, 0).numpy()
        with open(out, "wb") as fh:
            pickle.dump(dict(states=states, hist=hist, cyc=cyc, conv=conv,
                             messages=solver.messages), fh)
    dist.barrier()
    dist.destroy_process_group()


def _run(world, mode, tmp_path, sh=BASE):
    out = str(tmp_path / f"{mode}_{world}_{sh['N']}.pkl")
    mp.spawn(_worker, args=(world, _port(), out, mode, sh), nprocs=world, join=True)
    with open(out, "rb") as fh:
        return pickle.load(fh)


def _oracle(sh):
    N, Q, B, C, THR = sh["N"], sh["Q"], sh["B"], sh["C"], sh["THR"]
    a, net, X = _problem(sh)
    fine = fas.DenseLevel(a["W"], a["b"], a["activation"], a["step"])
    levels = fas.build_levels(fine, C, THR)
    src = net.source(X)
    U, hist, conv = fas.solve(levels, C, src, TOL, MAXC)
    Uc, _, _ = fas.solve(levels, C, src, 1e-12, 60)
    D = fas.derivs(fine, Uc)
    final, logits = fas.adjoint_head(net, Uc)
    _, dl = fas.loss_and_dlogits(logits, np.arange(B) % 10)
    gfin, _ = fas.g_final_from(net, final, dl)
    adj = fas.adjoint_level(fine, D)
    asrc = np.zeros_like(Uc)
    asrc[0] = gfin
    M, ahist, aconv = fas.solve(fas.build_levels(adj, C, THR), C, asrc, TOL, MAXC)
    return dict(fwd=(U, hist, conv), adj=(M, ahist, aconv))


@pytest.fixture(scope="module")
def oracle_solutions():
    return _oracle(BASE)


def _band(a, b):
    return abs(a - b) <= 1e-9 * abs(b) + 1e-12 * np.sqrt(N * Q)


@pytest.mark.parametrize("mode", ["fwd", "adj"])
def test_partitioned_solve_matches_oracle(mode, tmp_path, oracle_solutions):
    want_U, want_hist, want_conv = oracle_solutions[mode]
    runs = {w: _run(w, mode, tmp_path) for w in (1, 2, 4, 8)}
    for w, r in runs.items():
        # multigrid.py: bitwise states for any worker count (parallel.py:10-12)
        assert r["states"].tobytes() == want_U.tobytes(), (mode, w)
        for b in range(B):
            h = r["hist"][: r["cyc"][b] + 1, b]
            assert len(h) == len(want_hist[b]), (mode, w, b)
            assert all(_band(x, y) for x, y in zip(h, want_hist[b]))
        assert list(r["conv"]) == list(want_conv)
    # canonical block partials: norms bitwise across world sizes
    for w in (2, 4, 8):
        assert np.array_equal(runs[w]["hist"], runs[1]["hist"], equal_nan=True), (mode, w)


@pytest.mark.parametrize("mode", ["fwd", "adj"])
def test_c5_hierarchy_at_eight_ranks_collapses_level_one(mode, tmp_path):
    """c5's cf-16 hierarchy [1024, 64, 4] at world 8 (rejected before): the fine
    level is partitioned, [64, 4] gathered onto every rank; states bitwise the oracle's."""
    from paper_2007_07336_b200.distributed import check_partition

    assert check_partition(1024, 16, 3, 8) == 1
    want_U, want_hist, want_conv = _oracle(C5)[mode]
    r = _run(8, mode, tmp_path, C5)
    assert r["states"].tobytes() == want_U.tobytes(), mode
    for b in range(C5["B"]):
        h = r["hist"][: r["cyc"][b] + 1, b]
        assert len(h) == len(want_hist[b]), (mode, b)
        assert all(_band(x, y) for x, y in zip(h, want_hist[b]))


def test_halo_message_count(tmp_path):
    """Rank 0 of 2 (first in forward order) sends, per cycle: 1 (C-sweep) + 1 (P/adv pair) per
    relaxed level and 1 on the coarsest level; plus 1 for the initial residual."""
    r = _run(2, "fwd", tmp_path)
    cycles = int(max(r["cyc"]))
    relaxed = 2  # levels [64, 16, 4]
    assert r["messages"] == 1 + cycles * (2 * relaxed + 1)

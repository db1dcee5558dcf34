"""The reference's hot-path property tests, restated against this package on the GPU.

SURVEY 8(c) lists the reference tests that pin the path; the reference cannot travel to the GPU
box, so each property is restated here (our own code, the reference test it mirrors cited) and
run through the C-ABI:

  tests/test_multigrid.py:279-297   relaxation exactness (hypothesis)
  tests/test_multigrid.py:303-309   one cycle at the solution is a fixed point
  tests/test_multigrid.py:370-378   residual history monotone after cycle 1
  tests/test_multigrid.py:380-387   solve == sequential oracle
  tests/test_multigrid.py:389-396   early stop: report shape
  tests/test_multigrid.py:399-405   bad tolerances rejected
  tests/test_multigrid.py:407-413   N = c converges in one cycle
  tests/test_multigrid.py:416-422   3-level V-cycle converges
  tests/test_multigrid.py:450-470   conv2d residual blocks
  tests/test_parallel.py:92-102, 144-152, 281-301   bitwise across worker counts / exchange
  tests/test_acceptance.py:53-145   criteria 1-5 (depth-independent convergence, oracle
                                    equivalence, fixed point, relaxation exactness, bitwise
                                    determinism + scale checksum)
"""

import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from hypothesis import given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402

import paper_2007_07336_b200 as P  # noqa: E402
from paper_2007_07336_b200 import cli  # noqa: E402


def problem(depth, width, seed):
    """The reference tests' seeding (test_acceptance.py:43-46)."""
    net = P.random_network(depth, width, [seed, depth, width])
    f = np.asarray(P.source_from_input(net, P.random_sample(width, [seed, depth, width])))
    return net, f


def rows(depth, c, kind):
    return [j for j in range(depth) if (j % c == 0) == (kind == "C")]


@settings(max_examples=20, deadline=None)
@given(blocks=st.integers(2, 6), c=st.integers(2, 4), width=st.integers(1, 5),
       seed=st.integers(0, 10_000))
def test_relaxation_exactness_property(blocks, c, width, seed):
    depth = blocks * c
    net = P.random_network(depth, width, seed)
    f = np.asarray(P.source_from_input(net, P.random_sample(width, seed)))
    part = P.make_partition(depth, c, 1)
    s = np.asarray(P.initial_guess(net, f)) + np.random.default_rng(seed).normal(size=(depth, width))
    P.f_relaxation(net, s, f, part)
    assert np.max(np.abs(P.compute_residual(net, s, f)[rows(depth, c, "F")])) <= 1e-13
    P.c_relaxation(net, s, f, part)
    assert np.max(np.abs(P.compute_residual(net, s, f)[rows(depth, c, "C")])) <= 1e-13


def test_cycle_fixed_point_at_solution():
    net, f = problem(64, 4, 22)
    hier = P.build_hierarchy(net, 4)
    s = P.sequential_forward(net, f)
    before = s.copy()
    assert P.mg_cycle(hier, s, f) <= 1e-12
    assert np.max(np.abs(s - before)) <= 1e-12


def test_history_monotone_after_first_cycle():
    for seed in range(4):
        for depth in (64, 256):
            net, f = problem(depth, 4, 24 + seed)
            _, rep = P.solve(P.build_hierarchy(net, 4), f, tol=1e-9, max_cycles=50)
            assert rep.converged
            h = rep.residual_norms
            assert all(h[i + 1] <= h[i] for i in range(1, len(h) - 1)), h


def test_solve_matches_sequential_oracle():
    for seed in range(3):
        net, f = problem(32, 3, 30 + seed)
        s, rep = P.solve(P.build_hierarchy(net, 4), f, tol=1e-9, max_cycles=50)
        assert rep.converged
        assert np.max(np.abs(s - P.sequential_forward(net, f))) <= 1e-8


def test_early_stop_report_shape():
    net, f = problem(32, 3, 40)
    s, rep = P.solve(P.build_hierarchy(net, 4), f, tol=1e-15, max_cycles=2)
    assert rep.cycles_used == 2 and len(rep.residual_norms) == 3 and not rep.converged
    assert np.all(np.isfinite(s))


def test_bad_tolerances_rejected():
    net, f = problem(8, 2, 41)
    hier = P.build_hierarchy(net, 4)
    for bad in (0.0, -1.0, float("inf"), float("nan")):
        with pytest.raises(P.ConfigurationError):
            P.solve(hier, f, tol=bad)
    with pytest.raises(P.ConfigurationError):
        P.solve(hier, f, max_cycles=0)


def test_single_block_converges_in_one_cycle():
    net, f = problem(4, 2, 42)
    s, rep = P.solve(P.build_hierarchy(net, 4), f, tol=1e-9)
    assert rep.converged and rep.cycles_used == 1
    assert np.max(np.abs(s - P.sequential_forward(net, f))) <= 1e-12


def test_three_level_converges():
    net, f = problem(16, 2, 43)
    hier = P.build_hierarchy(net, 2, threshold=4)
    assert hier.num_levels == 3
    s, rep = P.solve(hier, f, tol=1e-10, max_cycles=50)
    assert rep.converged
    assert np.max(np.abs(s - P.sequential_forward(net, f))) <= 1e-8


def test_conv2d_blocks_solve():
    rng = np.random.default_rng(46)
    C, side, depth = 2, 6, 8
    q = C * side * side
    blocks = [P.conv2d_params(rng.normal(0, 0.15, (3, 3, C, C)), rng.normal(0, 0.05, C), "tanh",
                              side, side) for _ in range(depth)]
    net = P.ResidualNetwork(P.dense_params(rng.normal(0, 0.3, (q, 5)), np.zeros(q), "tanh"), blocks,
                            P.dense_params(rng.normal(size=(3, q)), np.zeros(3), "identity"), 0.25)
    f = np.asarray(P.source_from_input(net, rng.normal(size=5)))
    s, rep = P.solve_forward(net, f, coarsening=4, tol=1e-10)
    assert rep.converged
    assert np.max(np.abs(s - P.sequential_forward(net, f))) <= 1e-8


@pytest.mark.parametrize("workers", [2, 4, 8])
def test_fcf_and_solve_bitwise_across_worker_counts(workers):
    net, f = problem(64, 3, 14)
    ref = np.asarray(P.initial_guess(net, f))
    P.fcf_relaxation(net, ref, f, P.make_partition(64, 4, 1))
    s = np.asarray(P.initial_guess(net, f))
    with ThreadPoolExecutor(max_workers=workers) as pool:
        P.fcf_relaxation(net, s, f, P.make_partition(64, 4, workers), executor=pool)
    assert s.tobytes() == ref.tobytes()
    net, f = problem(64, 3, 15)
    hier = P.build_hierarchy(net, 4)
    s1, r1 = P.solve(hier, f, tol=1e-9, max_cycles=50, workers=1)
    sw, rw = P.solve(hier, f, tol=1e-9, max_cycles=50, workers=workers)
    assert sw.tobytes() == s1.tobytes() and rw.residual_norms == r1.residual_norms


def test_exchange_matches_serial_c_relaxation_bitwise():
    net, f = problem(32, 3, 5)
    serial = np.asarray(P.initial_guess(net, f)) + 0.25
    exchanged = serial.copy()
    P.c_relaxation(net, serial, f, P.make_partition(32, 4, 1))
    part = P.make_partition(32, 4, 4)
    with ThreadPoolExecutor(max_workers=4) as pool:
        msgs = P.exchange_and_c_relax(net, exchanged, f, part, executor=pool)
    assert exchanged.tobytes() == serial.tobytes()
    assert len(msgs) == len(part.cross_edges()) == 3


def test_acceptance_1_depth_independent_convergence(tmp_path):
    t0 = time.perf_counter()
    out = tmp_path / "converge.csv"
    assert cli.main(["converge", "--depths", "64,256,1024", "--tol", "1e-9", "--seed", "0",
                     "--out", str(out)]) == cli.EXIT_OK
    cyc, fin = {}, {}
    for ln in [x for x in out.read_text().splitlines() if not x.startswith("#")][1:]:
        d, c, n = ln.split(",")
        cyc[int(d)], fin[int(d)] = int(c), float(n)
    assert set(cyc) == {64, 256, 1024} and all(v <= 1e-9 for v in fin.values())
    assert max(cyc.values()) - min(cyc.values()) <= 2, cyc
    assert time.perf_counter() - t0 < 120.0


def test_acceptance_2_oracle_equivalence():
    t0 = time.perf_counter()
    for seed in range(20):
        for depth in (16, 64, 256):
            for width in (2, 8):
                net, f = problem(depth, width, seed)
                s, rep = P.solve(P.build_hierarchy(net, 4), f, tol=1e-9, max_cycles=50)
                assert rep.converged, (seed, depth, width)
                assert np.max(np.abs(s - P.sequential_forward(net, f))) <= 1e-8, (seed, depth, width)
    assert time.perf_counter() - t0 < 60.0


def test_acceptance_4_relaxation_exactness():
    for seed in range(8):
        depth, width, c = 16 + 4 * (seed % 3), 2 + seed % 4, 4
        net, f = problem(depth, width, seed)
        part = P.make_partition(depth, c, 1)
        s = np.asarray(P.initial_guess(net, f)) + np.random.default_rng(seed).normal(size=(depth, width))
        P.f_relaxation(net, s, f, part)
        assert np.max(np.abs(P.compute_residual(net, s, f)[rows(depth, c, "F")])) <= 1e-13
        P.c_relaxation(net, s, f, part)
        assert np.max(np.abs(P.compute_residual(net, s, f)[rows(depth, c, "C")])) <= 1e-13


def test_acceptance_5_bitwise_determinism_and_scale_checksum(tmp_path):
    net, f = problem(256, 8, 2)
    ref = np.asarray(P.initial_guess(net, f))
    P.fcf_relaxation(net, ref, f, P.make_partition(256, 4, 1))
    hier = P.build_hierarchy(net, 4)
    sref, _ = P.solve(hier, f, tol=1e-9, max_cycles=50, workers=1)
    for workers in (2, 4, 8):
        s = np.asarray(P.initial_guess(net, f))
        with ThreadPoolExecutor(max_workers=workers) as pool:
            P.fcf_relaxation(net, s, f, P.make_partition(256, 4, workers), executor=pool)
        assert s.tobytes() == ref.tobytes(), workers
        sw, _ = P.solve(hier, f, tol=1e-9, max_cycles=50, workers=workers)
        assert sw.tobytes() == sref.tobytes(), workers
    out = tmp_path / "scale.csv"
    assert cli.main(["scale", "--workers", "1,2,4,8", "--batches", "1", "--seed", "0",
                     "--out", str(out)]) == cli.EXIT_OK
    rows_ = [ln.split(",") for ln in out.read_text().splitlines() if not ln.startswith("#")][1:]
    assert len({r[-1] for r in rows_}) == 1

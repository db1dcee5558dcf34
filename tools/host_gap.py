"""Host-side cost of the per-cycle stopping test in a small-batch solve (c5 forward solve).

    python tools/host_gap.py [--config c5] [--reps 5]

lmg_solve syncs the stream once per cycle to read the residual norms back (multigrid.py:297's
per-sample test) and replays the cycle graph.  Estimate of the idle time that adds:
    gap = T(solve, k cycles) - T(solve stopped after the initial norm) - k * T(cycle)
with T(cycle) from k back-to-back lmg_mg_cycle calls (eager launches, no host test; the host
enqueues faster than the GPU runs them, so this is device time).  All on CUDA events.
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2007_07336_b200 as P  # noqa: E402
from paper_2007_07336_b200 import _lib  # noqa: E402
from paper_2007_07336_b200.multigrid import solve_device, solver_workspace  # noqa: E402
from paper_2007_07336_b200.training import _dense_apply  # noqa: E402


def timed(fn, reps):
    out = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        out.append(s.elapsed_time(e))
    return float(np.median(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    cfg = bench.CONFIGS[a.config]
    N, q, B, c = cfg["depth"], cfg["width"], cfg["batch"], cfg["cf"]
    dev = torch.device("cuda", 0)
    d = P.device_network(N, q, [0, N, q], device=dev)
    X = torch.from_numpy(P.random_batch(q, [0, N, q], B)).to(dev)
    view = d._lmg_view()
    sizes = [N]
    thr = cfg["threshold"] or N // c  # None: two levels (multigrid.py:76-102 default)
    while sizes[-1] > thr:
        sizes.append(sizes[-1] // c)
    nlev = len(sizes)
    f0 = _dense_apply(d.Wo, d.bo, d.open_act, X).contiguous()
    U = torch.empty((N, B, q), dtype=torch.float64, device=dev)
    work = solver_workspace(view, nlev, c, B, dev)

    def solve(tol):
        return solve_device(view, nlev, c, f0, U, src_mode=_lib.SRC_HEAD, use_initial=False,
                            tol=tol, max_cycles=cfg["max_cycles"], work=work)

    _, cyc, _ = solve(cfg["tol"])
    k = int(cyc.max())
    solve(cfg["tol"])
    t_solve = timed(lambda: solve(cfg["tol"]), a.reps)
    t_init = timed(lambda: solve(1e300), a.reps)
    norms = torch.empty(B, dtype=torch.float64, device=dev)
    desc = view.desc()

    def cycles():
        for _ in range(k):
            _lib.call("lmg_mg_cycle", desc, nlev, c, B, U.data_ptr(), f0.data_ptr(), _lib.SRC_HEAD,
                      norms.data_ptr(), work[0].data_ptr(), work[1], _lib.stream_handle())

    cycles()
    t_cyc = timed(cycles, a.reps)
    gap = t_solve - t_init - t_cyc
    print(f"{a.config}: levels {sizes} cycles {k}: solve {t_solve:.3f} ms, initial norm only "
          f"{t_init:.3f} ms, {k} back-to-back cycles {t_cyc:.3f} ms ({t_cyc / k:.3f} ms each) -> "
          f"host stopping-test gap {gap:.3f} ms per solve ({gap / k * 1e3:.1f} us per cycle)")


if __name__ == "__main__":
    main()

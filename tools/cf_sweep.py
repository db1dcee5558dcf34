"""BASELINE.json configs[4]: coarsening-factor / level-count sweep on 1024 layers.

    python tools/cf_sweep.py [--out profiles/r2_cf_sweep.json] [--steps 3]

For cf in {2, 4, 8, 16} and every level count 2..6 that divides 1024 (threshold = the coarsest
size, multigrid.py:76-102), at q=512/B=16 (the HBM-bound point) and q=16/B=1 (the reference's
survey shape): FAS forward cycles to tol 1e-9, FAS adjoint cycles, GPU ms per
training step (forward + adjoint to tol + gradients + SGD, theta restored before every timed
step), the serial layer-by-layer GPU step on the same network, and the critical path in
sequential layer steps (per cycle: 2c+2 per relaxed level -- FCF 2c-1, the P step, the coarse
source and the post-correction residual row -- plus the coarsest level's n-1 serial steps; the
formula that reproduces BASELINE.md 3.4).  One GPU; at P GPUs the relaxed-level work divides by
P while the critical path does not, so the smallest critical path with few cycles is the
multi-GPU candidate.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2007_07336_b200 as P  # noqa: E402
from paper_2007_07336_b200 import _lib  # noqa: E402
from paper_2007_07336_b200.training import _dense_apply, backward  # noqa: E402

N = 1024


def hierarchies(N=1024):
    for cf in (2, 4, 8, 16):
        for L in range(2, 7):
            if cf ** (L - 1) > N or N % cf ** (L - 1):
                continue
            sizes = [N // cf ** l for l in range(L)]
            yield cf, L, sizes


def critical_path(cf, sizes):
    return (2 * cf + 2) * (len(sizes) - 1) + sizes[-1] - 1


def timed(fn, steps, restore):
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    out = []
    for _ in range(steps):
        restore()
        s, e = ev(), ev()
        s.record()
        r = fn()
        e.record()
        e.synchronize()
        out.append(s.elapsed_time(e))
    return float(np.median(out)), r


def run_point(q, B, cf, sizes, steps, N=N):
    dev = torch.device("cuda", 0)
    d = P.device_network(N, q, [0, N, q], device=dev)
    saved = [x.clone() for x in (d.stack.W, d.stack.b, d.Wo, d.bo, d.Wr, d.br)]
    live = [d.stack.W, d.stack.b, d.Wo, d.bo, d.Wr, d.br]

    def restore():
        for a, b in zip(live, saved):
            a.copy_(b)

    X = torch.from_numpy(P.random_batch(q, [0, N, q], B)).to(dev)
    labels = torch.from_numpy(np.arange(B) % 10).to(dev)
    tr = P.DeviceTrainer(d, coarsening=cf, threshold=sizes[-1], tol=1e-9, max_cycles=200,
                         adjoint="fas", learning_rate=0.1)
    restore()
    tr.step(X, labels)  # warm-up (graph capture)
    ms, res = timed(lambda: tr.step(X, labels), steps, restore)
    Us = torch.empty((N, B, q), dtype=torch.float64, device=dev)

    def serial():
        f0 = _dense_apply(d.Wo, d.bo, d.open_act, X)
        _lib.call("lmg_sequential_forward", d._lmg_view().desc(), B, f0.data_ptr(), _lib.SRC_HEAD,
                  Us.data_ptr(), _lib.stream_handle())
        backward(d, Us, X, labels, adjoint="sequential", scale=1.0 / B, lr=0.1, want_grads=False)

    restore()
    serial()
    sms, _ = timed(serial, steps, restore)
    fc, ac = int(res.fwd_cycles.max()), int(res.adj_cycles.max())
    cp = critical_path(cf, sizes)
    return dict(q=q, B=B, cf=cf, levels=sizes, fwd_cycles=fc, adj_cycles=ac,
                converged=bool(res.fwd_converged.all() and res.adj_converged.all()),
                gpu_ms_per_step=ms, serial_gpu_ms_per_step=sms, fas_over_serial=ms / sms,
                layer_samples_per_s=N * B / (ms * 1e-3),
                critical_path_per_cycle=cp, critical_path_total=cp * (fc + ac),
                serial_critical_path=2 * (N - 1))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r2_cf_sweep.json"))
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--shapes", default="512x16,16x1")
    ap.add_argument("--depths", default="1024",
                    help="comma list of N; with --cf/--levels a depth sweep of one hierarchy shape")
    ap.add_argument("--cf", type=int, default=None)
    ap.add_argument("--levels", default=None, help="comma list of level counts (with --cf)")
    a = ap.parse_args()
    rows = []

    def points(n):
        if a.cf is None:
            yield from hierarchies(n)
            return
        for L in (int(v) for v in a.levels.split(",")):
            if a.cf ** (L - 1) <= n and n % a.cf ** (L - 1) == 0:
                yield a.cf, L, [n // a.cf ** l for l in range(L)]

    for shape in a.shapes.split(","):
        q, B = (int(v) for v in shape.split("x"))
        for n, (cf, L, sizes) in ((n, p) for n in (int(v) for v in a.depths.split(",")) for p in points(n)):
            t0 = time.time()
            r = run_point(q, B, cf, sizes, a.steps, N=n)
            r["depth"] = n
            rows.append(r)
            print(f"N {n} q {q} B {B} cf {cf:2d} levels {sizes}: cycles {r['fwd_cycles']}+{r['adj_cycles']} "
                  f"step {r['gpu_ms_per_step']:.2f} ms serial {r['serial_gpu_ms_per_step']:.2f} ms "
                  f"crit {r['critical_path_total']} ({time.time() - t0:.1f}s)", flush=True)
            torch.cuda.empty_cache()
    with open(a.out, "w") as fh:
        json.dump(dict(what=__doc__.strip().splitlines()[0], gpu=torch.cuda.get_device_name(0),
                       rows=rows), fh, indent=1)
    print(a.out)


if __name__ == "__main__":
    main()

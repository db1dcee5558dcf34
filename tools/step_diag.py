"""Per-step host wall vs device time of the bench's training step (diagnosis of idle gaps).

    python tools/step_diag.py [--config c2] [--steps 6]

Prints, per step, the forward solve and the backward (adjoint + gradients) host wall time and
GPU time (CUDA events on the current stream), plus the library's launch count per step.
"""

import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2007_07336_b200 as P  # noqa: E402
from paper_2007_07336_b200 import _lib  # noqa: E402
from paper_2007_07336_b200.training import backward  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--steps", type=int, default=6)
    a = ap.parse_args()
    cfg = bench.CONFIGS[a.config]
    N, q, B = cfg["depth"], cfg["width"], cfg["batch"]
    dev = torch.device("cuda", 0)
    d = P.device_network(N, q, [0, N, q], device=dev)
    X = torch.from_numpy(P.random_batch(q, [0, N, q], B)).to(dev)
    labels = torch.from_numpy(np.arange(B) % 10).to(dev)
    tr = P.DeviceTrainer(d, coarsening=cfg["cf"], threshold=cfg["threshold"], tol=cfg["tol"],
                         max_cycles=cfg["max_cycles"], adjoint="fas", learning_rate=cfg["lr"])
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    for i in range(a.steps):
        torch.cuda.synchronize()
        n0 = _lib.launch_count()
        e0, e1, e2 = ev(), ev(), ev()
        t0 = time.perf_counter()
        e0.record()
        U, hist, cyc, conv = tr.forward(X)
        e1.record()
        t1 = time.perf_counter()
        _, lam, D = tr._buffers(B, dev)
        r = backward(d, U, X, labels, adjoint="fas", coarsening=cfg["cf"], threshold=cfg["threshold"],
                     tol=cfg["tol"], max_cycles=cfg["max_cycles"], scale=1.0 / B, lr=cfg["lr"],
                     want_grads=False, lam_buf=lam, D_buf=D, head_buf=tr._head(1, B, dev))
        e2.record()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"step {i}: fwd wall {1e3 * (t1 - t0):8.2f} gpu {e0.elapsed_time(e1):8.2f} ms "
              f"({int(cyc.max())} cyc) | bwd wall {1e3 * (t2 - t1):8.2f} gpu {e1.elapsed_time(e2):8.2f} "
              f"ms ({int(r.cycles.max())} cyc) | launches {_lib.launch_count() - n0}", flush=True)


if __name__ == "__main__":
    main()

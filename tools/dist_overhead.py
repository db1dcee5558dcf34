"""Host cost of the layer-partitioned (Python-driven) cycle: LayerParallelTrainer at world 1 over
NCCL against DeviceTrainer (C++ cycle loop, cached cycle graphs) on the same GPU and config.

    python -m torch.distributed.run --nproc-per-node 1 --master-addr 127.0.0.1 \
        --master-port 29533 tools/dist_overhead.py [--config c5] [--steps 5]

At world 1 the partitioned solver runs every per-cycle host step it runs at world P (the level
ops through ctypes, the norm all_gather, the per-cycle read-back) but no halo traffic, so the
difference is the host overhead a rank adds per training step.
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
import paper_2007_07336_b200 as P  # noqa: E402
from paper_2007_07336_b200.distributed import LayerParallelTrainer  # noqa: E402


def timed(fn, steps):
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps):
        r = fn()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / steps, r


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--steps", type=int, default=5)
    a = ap.parse_args()
    cfg = bench.CONFIGS[a.config]
    N, q, B = cfg["depth"], cfg["width"], cfg["batch"]
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    dist.init_process_group("nccl", device_id=dev)
    X = torch.from_numpy(P.random_batch(q, [0, N, q], B)).to(dev)
    labels = torch.from_numpy(np.arange(B) % 10).to(dev)
    kw = dict(coarsening=cfg["cf"], threshold=cfg["threshold"], tol=cfg["tol"],
              max_cycles=cfg["max_cycles"], adjoint="fas", learning_rate=0.0)
    lp = LayerParallelTrainer(N, q, [0, N, q], **kw)
    lp.step(X, labels)
    t_lp, r1 = timed(lambda: lp.step(X, labels), a.steps)
    d = P.device_network(N, q, [0, N, q], device=dev)
    tr = P.DeviceTrainer(d, **kw)
    tr.step(X, labels)
    t_dt, r2 = timed(lambda: tr.step(X, labels), a.steps)
    print(f"{a.config}: partitioned trainer at world 1 {t_lp:.2f} ms/step "
          f"({int(np.max(r1.fwd_cycles))}+{int(np.max(r1.adj_cycles))} cycles), DeviceTrainer "
          f"{t_dt:.2f} ms/step ({int(np.max(r2.fwd_cycles))}+{int(np.max(r2.adj_cycles))}) -> "
          f"{t_lp - t_dt:+.2f} ms per step")
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

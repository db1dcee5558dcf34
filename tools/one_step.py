"""One bench training step inside a CUDA profiler range, for ncu launch lists / full captures.

    ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,\
dram__bytes_write.sum --clock-control none --csv --log-file out.csv \
        python tools/one_step.py --config c5 [--warmup 2]

The warm-up steps (graph capture, first-use allocations) run outside the range; the profiled
step is the same DeviceTrainer.step bench.py times (theta restored first).
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--warmup", type=int, default=2)
    a = ap.parse_args()
    cfg = bench.CONFIGS[a.config]
    N, q, B = cfg["depth"], cfg["width"], cfg["batch"]
    dev = torch.device("cuda", 0)
    d = P.device_network(N, q, [0, N, q], device=dev)
    X = torch.from_numpy(P.random_batch(q, [0, N, q], B)).to(dev)
    labels = torch.from_numpy(np.arange(B) % 10).to(dev)
    tr = P.DeviceTrainer(d, coarsening=cfg["cf"], threshold=cfg["threshold"], tol=cfg["tol"],
                         max_cycles=cfg["max_cycles"], adjoint="fas", learning_rate=cfg["lr"])
    theta = bench.ThetaSnapshot(torch, d)
    for _ in range(a.warmup):
        theta.restore()
        tr.step(X, labels)
    theta.restore()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    r = tr.step(X, labels)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print(f"{a.config}: cycles {int(r.fwd_cycles.max())}+{int(r.adj_cycles.max())}")


if __name__ == "__main__":
    main()

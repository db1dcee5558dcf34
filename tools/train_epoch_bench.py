"""The reference-shaped training API (train_epoch over a Dataset, host parameter arrays) against
the device-resident DeviceTrainer, per batch, at the c2 shape (1024 x 512, batch 256, cf 4,
levels [1024, 256, 64], FAS forward to tol 1e-9 + the sequential adjoint -- what train_epoch
runs, training.py:255-289).

    python tools/train_epoch_bench.py [--batches 8]

train_epoch's time includes what its API implies once per epoch: uploading the network's host
arrays (2 GiB of theta) and writing the SGD-updated parameters back into them.
"""

import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2007_07336_b200 as P  # noqa: E402
from paper_2007_07336_b200.training import Dataset, TrainConfig, train_epoch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", type=int, default=8)
    ap.add_argument("--depth", type=int, default=1024)
    ap.add_argument("--width", type=int, default=512)
    ap.add_argument("--batch", type=int, default=256)
    a = ap.parse_args()
    N, q, B, c, thr = a.depth, a.width, a.batch, 4, 64
    rng = np.random.default_rng(3)
    count = a.batches * B
    data = Dataset(rng.uniform(0.0, 1.0, size=(count, 28, 28)), rng.integers(0, 10, size=count))
    net = P.random_network(N, q, [0, N, q], input_dim=28 * 28)
    hier = P.build_hierarchy(net, c, threshold=thr)
    cfg = TrainConfig(learning_rate=0.1, batch_size=B, epochs=1, mode="mg", mg_cycles=50,
                      coarsening=c, solve_tol=1e-9)
    train_epoch(net, data.subset(B), cfg, hierarchy=hier)  # warm-up (one batch)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st = train_epoch(net, data, cfg, rng=np.random.default_rng(0), hierarchy=hier)
    torch.cuda.synchronize()
    t_epoch = time.perf_counter() - t0

    d = P.device_network(N, q, [0, N, q], device="cuda:0", input_dim=28 * 28)
    tr = P.DeviceTrainer(d, coarsening=c, threshold=thr, tol=1e-9, max_cycles=50,
                         adjoint="sequential", learning_rate=0.1)
    X = torch.from_numpy(data.images.reshape(count, -1)).cuda()
    L = torch.from_numpy(data.labels).cuda()
    tr.step(X[:B], L[:B])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(a.batches):
        r = tr.step(X[i * B:(i + 1) * B], L[i * B:(i + 1) * B])
    r.loss.cpu()
    torch.cuda.synchronize()
    t_dev = time.perf_counter() - t0
    print(f"c2 shape {N}x{q}, batch {B}, {a.batches} batches: train_epoch {t_epoch / a.batches * 1e3:.1f} ms "
          f"per batch (incl. theta upload + write-back), DeviceTrainer.step {t_dev / a.batches * 1e3:.1f} ms "
          f"per batch -> ratio {t_epoch / t_dev:.3f}; epoch mean loss {st.mean_loss:.4f}")


if __name__ == "__main__":
    main()

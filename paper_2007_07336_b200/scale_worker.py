"""One rank of the CLI `scale` command's multi-GPU rows (run under torchrun by cli.py).

The forward FAS solve of the CLI's experiment network (cli.py:150-153 seeding) with the layer
axis partitioned over the ranks (distributed.DistSolver, one process per GPU, NCCL halos; with
LMG_SCALE_BACKEND=gloo the ranks may share GPUs and stage halos through host memory).  Rank 0
writes {seconds (max over ranks), roofline of the relaxation step class on rank 0, sha256 of
sample 0's states, cycles} to --out.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import time

import numpy as np


def main() -> None:
    import torch
    import torch.distributed as dist

    from . import _lib, roofline
    from .distributed import CudaOps, DistSolver
    from .multigrid import _levels_for
    from .network import SystemView
    from .cli import _samples
    from .synthetic import device_network
    from .training import _dense_apply

    _lib.set_canonical_order(True)  # the CLI's checksum rows compare bitwise
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--batch", type=int, required=True)
    ap.add_argument("--config", required=True)
    a = ap.parse_args()
    cfg = json.loads(a.config)
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank)) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    backend = os.environ.get("LMG_SCALE_BACKEND", "nccl")
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group(backend)
    N, q, seed, B = cfg["depth"], cfg["width"], cfg["seed"], a.batch
    c = cfg["coarsening"]
    nlev = _levels_for(N, c, cfg["threshold"])
    L = N // world
    dnet = device_network(N, q, [seed, N, q], horizon=cfg["horizon"], layers=(rank * L, (rank + 1) * L),
                          device=dev)
    view = SystemView(dnet.stack, 1, dnet.step_size, L)
    solver = DistSolver(view, N, c, nlev, B, rank=rank, world=world, ops=CudaOps(dev), device=dev)
    head = None
    if rank == 0:
        xs = _samples(N, q, seed, B)
        head = _dense_apply(dnet.Wo, dnet.bo, dnet.open_act, torch.from_numpy(np.stack(xs)).to(dev))
    U = torch.zeros(L + 1, B, q, dtype=torch.float64, device=dev)

    def run():
        return solver.solve(U, head, _lib.SRC_HEAD, tol=cfg["tol"], max_cycles=cfg["max_cycles"])

    run()  # warm-up
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    hist, cyc, conv = run()
    torch.cuda.synchronize()
    el = torch.tensor([time.perf_counter() - t0], dtype=torch.float64)
    if backend == "nccl":
        el = el.to(dev)
    dist.all_reduce(el, op=dist.ReduceOp.MAX)
    peaks = (roofline.fp64_peak_tflops(torch, dev) if rank == 0 else 0.0, roofline.hbm_peak()[0])
    rf = roofline.measure(run, *peaks)
    rows = U[:L, 0].contiguous()
    parts = [torch.empty_like(rows) for _ in range(world)]
    if backend == "nccl":
        dist.all_gather(parts, rows)
    else:
        cp = [p.cpu() for p in parts]
        dist.all_gather(cp, rows.cpu())
        parts = cp
    if rank == 0:
        states = torch.cat([p.cpu() for p in parts]).numpy()
        digest = hashlib.sha256(states.tobytes()).hexdigest()
        with open(a.out, "w") as fh:
            json.dump(dict(seconds=float(el.item()), roofline=rf, checksum=digest,
                           cycles=int(np.max(cyc))), fh)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

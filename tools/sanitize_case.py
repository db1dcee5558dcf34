"""Small training steps that exercise the asynchronous kernels, for compute-sanitizer.

    compute-sanitizer --tool racecheck python tools/sanitize_case.py
    compute-sanitizer --tool synccheck python tools/sanitize_case.py
    compute-sanitizer --tool memcheck  python tools/sanitize_case.py

Cases (and the kernels they route to, asserted through lmg_route_counts):
  tgemm   N 16, q 128, B 64, cf 4     -- warp-specialised TMA step GEMM (adjoint layout; with
                                         LMG_TGEMM=all also the forward), mbarrier ring; run
                                         with LMG_NO_SWEEP=1 (else the fused sweep takes B 64)
  sweep   N 64, q 128, B 16, cf 4     -- fused persistent FCF / serial sweeps: TMA ring, DSMEM
                                         st.async all-gather, cluster barriers
  splitk  N 16, q 128, B 32, cf 4, levels [16, 4] -- split-K cluster serial steps (DSMEM reduce);
                                         LMG_NO_SWEEP=1
  chain   N 64, q 128, B 16, cf 4     -- persistent chain launches (completion counters,
                                         cooperative grid); LMG_NO_SWEEP=1
  warp16  N 256, q 16, B 3, cf 4, levels [256, 64, 16] -- warp FMA sweeps (cp.async ring, 4-warp
                                         CTAs with an idle warp) + the fused narrow residual
  warp32  N 64, q 32, B 9, cf 4       -- the same at q 32, two CTAs per chain (8 + 1 samples)
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2007_07336_b200 as P  # noqa: E402
from paper_2007_07336_b200 import _lib  # noqa: E402

CASES = {"tgemm": (16, 128, 64, 4, 4, ("tgemm_big",)),
         "sweep": (64, 128, 16, 4, 4, ("sweep_fcf", "sweep_seq")),
         "splitk": (16, 128, 32, 4, 4, ("serial_splitk",)),
         "chain": (64, 128, 16, 4, 4, ("chain",)),
         "warp16": (256, 16, 3, 4, 16, ("wsweep", "sweep_fcf", "sweep_seq")),
         "warp32": (64, 32, 9, 4, 4, ("wsweep", "sweep_fcf", "sweep_seq"))}


def main():
    names = sys.argv[1:] or list(CASES)
    for name in names:
        N, q, B, c, thr, want = CASES[name]
        before = _lib.route_counts() if _lib.load() else None
        d = P.device_network(N, q, [0, N, q], device="cuda:0")
        X = torch.from_numpy(P.random_batch(q, [0, N, q], B)).cuda()
        labels = torch.from_numpy(np.arange(B) % 10).cuda()
        tr = P.DeviceTrainer(d, coarsening=c, threshold=thr, tol=1e-9, max_cycles=4, adjoint="fas",
                             learning_rate=0.1)
        r = tr.step(X, labels)
        torch.cuda.synchronize()
        ran = {k: v - before[k] for k, v in _lib.route_counts().items() if v - before[k]}
        missing = [k for k in want if k not in ran]
        print(f"{name}: cycles {int(r.fwd_cycles.max())}+{int(r.adj_cycles.max())} routes {ran}"
              + (f" MISSING {missing}" if missing else ""), flush=True)


if __name__ == "__main__":
    main()

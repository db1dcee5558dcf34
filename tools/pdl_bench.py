"""Effective HBM throughput of back-to-back small-batch relaxation steps (the c5 fine level:
64 blocks x B=16 x q=512, cf 16): CUDA events around a batch of F-relaxation sweeps (15 step
launches each, no events in between, so programmatic dependent launch can overlap them).
Algorithmic bytes per step launch = tasks * (8 q^2 W + 2 * 8 B q state rows).

    python tools/pdl_bench.py            (compare with LMG_NO_PDL=1)"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2007_07336_b200 as P  # noqa: E402
from paper_2007_07336_b200 import _lib  # noqa: E402

N, q, B, c = 1024, 512, 16, 16
d = P.device_network(N, q, [0, N, q])
view = d._lmg_view()
U = torch.randn(N, B, q, dtype=torch.float64, device="cuda") * 0.3
S = torch.zeros(B, q, dtype=torch.float64, device="cuda")
st = _lib.stream_handle()


def sweep():
    _lib.call("lmg_f_relax", view.desc(), B, c, U.data_ptr(), S.data_ptr(), _lib.SRC_HEAD, st)


for _ in range(3):
    sweep()
torch.cuda.synchronize()
reps = 20
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    sweep()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
launches = reps * (c - 1)
tasks = N // c
bytes_per = tasks * (8.0 * q * q + 2 * 8.0 * B * q)
gbs = bytes_per * launches / (ms * 1e-3) / 1e9
print(json.dumps(dict(pdl=os.environ.get("LMG_NO_PDL") is None, us_per_step_launch=1e3 * ms / launches,
                      effective_GBps=gbs, frac_of_6650=gbs / 6650.0)))

"""Serial propagation (lmg_sequential_forward) of a long chain: fused sweep vs per-step, bitwise.
    LMG_SWEEP_CFG=0 python tools/seq_repro.py N q B out.npy   (compare with LMG_NO_SWEEP=1 LMG_NO_SPLITK=1)"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2007_07336_b200 as P  # noqa: E402
from paper_2007_07336_b200 import _lib  # noqa: E402
from paper_2007_07336_b200.training import _dense_apply  # noqa: E402

N, q, B = (int(v) for v in sys.argv[1:4])
d = P.device_network(N, q, [0, N, q], device="cuda:0")
X = torch.from_numpy(P.random_batch(q, [0, N, q], B)).cuda()
f0 = _dense_apply(d.Wo, d.bo, d.open_act, X)
U = torch.empty((N, B, q), dtype=torch.float64, device="cuda:0")
outs = []
adj = os.environ.get("ADJ") == "1"
if adj:  # forward states by the per-step path's twin (any fixed U works), then the adjoint system
    Uf = torch.from_numpy(np.random.default_rng(1).normal(0, 1, (N, B, q))).cuda()
    D = torch.empty_like(Uf)
    _lib.call("lmg_act_deriv", d._lmg_view().desc(), B, Uf.data_ptr(), D.data_ptr(), _lib.stream_handle())
    g = torch.from_numpy(np.random.default_rng(2).normal(0, 1, (B, q))).cuda()
    desc = d._lmg_view().desc(D)
    if os.environ.get("COARSE"):
        desc = d._lmg_view().coarsen(int(os.environ["COARSE"])).desc(D)
        U = U[: desc.num_layers]
    src = g
else:
    desc, src = d._lmg_view().desc(), f0
for rep in range(3):
    _lib.call("lmg_sequential_forward", desc, B, src.data_ptr(), _lib.SRC_HEAD, U.data_ptr(),
              _lib.stream_handle())
    outs.append(U.cpu().numpy().copy())
print("repeat-consistent:", all(np.array_equal(outs[0], o) for o in outs[1:]))
np.save(sys.argv[4], outs[0])

"""One conv (c3-shaped) forward and adjoint sweep step launch through the library (for ncu)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2007_07336_b200 import _lib  # noqa: E402
from paper_2007_07336_b200.synthetic import conv_device_network  # noqa: E402

N, C, S, B = 64, 64, 32, 32
d = conv_device_network(N, C, S, [0, N, C], device="cuda:0", input_dim=64)
view = d._lmg_view()
q = C * S * S
U = torch.randn(N, B, q, dtype=torch.float64, device="cuda") * 0.3
Sd = torch.zeros(B, q, dtype=torch.float64, device="cuda")
D = torch.rand(N, B, q, dtype=torch.float64, device="cuda")
st = _lib.stream_handle()
for rep in range(2):
    _lib.call("lmg_f_relax", view.desc(), B, 4, U.data_ptr(), Sd.data_ptr(), _lib.SRC_HEAD, st)
    _lib.call("lmg_f_relax", view.desc(D), B, 4, U.data_ptr(), Sd.data_ptr(), _lib.SRC_HEAD, st)
torch.cuda.synchronize()

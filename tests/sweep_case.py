"""Run one FAS training step on cuda:0 and save everything it produced (helper of
tests/test_gpu_sweep.py; run in a subprocess so LMG_* routing variables take effect).

    python tests/sweep_case.py N q B c threshold out.npz [activation]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    N, q, B, c, thr = (int(v) for v in sys.argv[1:6])
    out = sys.argv[6]
    act = sys.argv[7] if len(sys.argv) > 7 else "tanh"
    import torch

    import paper_2007_07336_b200 as P

    d = P.device_network(N, q, [0, N, q], device="cuda:0", activation=act)
    X = torch.from_numpy(P.random_batch(q, [0, N, q], B)).cuda()
    labels = torch.from_numpy(np.arange(B) % 10).cuda()
    tr = P.DeviceTrainer(d, coarsening=c, threshold=thr if thr > 0 else None, tol=1e-9,
                         max_cycles=50, adjoint="fas", learning_rate=0.1)
    U, hist, cyc, conv = tr.forward(X)
    U0 = U.cpu().numpy().copy()
    r = tr.step(X, labels)
    U1, lam, _ = tr._buffers(B, X.device)
    # serial propagation through the library (sequential_forward, the coarsest-solve routine)
    from paper_2007_07336_b200 import _lib
    from paper_2007_07336_b200.training import _dense_apply

    f0 = _dense_apply(d.Wo, d.bo, d.open_act, X)
    Us = torch.empty_like(U1)
    _lib.call("lmg_sequential_forward", d._lmg_view().desc(), B, f0.data_ptr(), _lib.SRC_HEAD,
              Us.data_ptr(), _lib.stream_handle())
    torch.cuda.synchronize()
    np.savez(out, U0=U0, hist=hist, cyc=cyc, U1=U1.cpu().numpy(), lam=lam.cpu().numpy(),
             loss=r.loss.cpu().numpy(), adj_hist=r.adj_hist, adj_cyc=r.adj_cycles,
             W=d.stack.W.cpu().numpy(), b=d.stack.b.cpu().numpy(), Us=Us.cpu().numpy(),
             launches=np.array(_lib.launch_count()),
             routes=np.array(list(_lib.route_counts().values())))


if __name__ == "__main__":
    main()

"""Time the fused sweep vs the launch-per-step path on one configuration (CUDA events).

    python tools/sweep_bench.py [N q B c threshold]      (default: c5 1024 512 16 16 4)

Prints per-class kernel time of one FAS forward solve and of one serial propagation.  Run it
twice (LMG_NO_SWEEP=1 for the per-step path); under ncu -k regex:sweep for the sweep kernel."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    N, q, B, c, thr = (int(v) for v in (sys.argv[1:6] or [1024, 512, 16, 16, 4]))
    import torch

    import paper_2007_07336_b200 as P
    from paper_2007_07336_b200 import _lib
    from paper_2007_07336_b200.multigrid import solve_device
    from paper_2007_07336_b200.training import _dense_apply

    d = P.device_network(N, q, [0, N, q], device="cuda:0")
    X = torch.from_numpy(P.random_batch(q, [0, N, q], B)).cuda()
    tr = P.DeviceTrainer(d, coarsening=c, threshold=thr, tol=1e-9, max_cycles=50, adjoint="fas")
    f0 = _dense_apply(d.Wo, d.bo, d.open_act, X)
    view = d._lmg_view()
    U = torch.empty((N, B, q), dtype=torch.float64, device="cuda:0")

    def serial():
        _lib.call("lmg_sequential_forward", view.desc(), B, f0.data_ptr(), _lib.SRC_HEAD,
                  U.data_ptr(), _lib.stream_handle())

    def fas():
        return solve_device(view, tr.nlevels, c, f0, U, src_mode=_lib.SRC_HEAD, use_initial=False,
                            tol=1e-9, max_cycles=50)

    names = {0: "gemm_fwd", 1: "gemm_adj", 2: "gemm_pg", 3: "elem", 4: "sweep_fwd", 5: "sweep_adj"}
    labels = torch.from_numpy(np.arange(B) % 10).cuda()

    def step():
        r = tr.step(X, labels)
        return (None, r.fwd_cycles) if r.adj_cycles is None else (None, np.concatenate([r.fwd_cycles, r.adj_cycles]))

    for label, fn in (("serial", serial), ("fas", fas), ("train_step", step)):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        r = fn()
        e.record()
        torch.cuda.synchronize()
        total = s.elapsed_time(e)
        _lib.timing_enable(True)
        fn()
        torch.cuda.synchronize()
        parts = []
        for cls, nm in names.items():
            ms, fl, by, n = _lib.timing_read(cls)
            if n:
                parts.append(f"{nm}: {ms:.3f} ms n={n} {fl / ms / 1e9:.2f} TF/s {by / ms / 1e6:.0f} GB/s")
        _lib.timing_enable(False)
        extra = "" if r is None else f" cycles={int(np.max(r[1]))}"
        print(f"{label}: {total:.3f} ms{extra} | " + " | ".join(parts))


if __name__ == "__main__":
    main()


def trace(N=None, q=None, B=None):
    """Per-step phase times of one serial fused sweep (lmg_debug_sweep_trace).  Cluster sweeps
    stamp (start, peers' state landed, mainloop done, epilogue done); the warp FMA sweep (q 16 /
    32) stamps (start, W stage landed, matvec done, epilogue done)."""
    N = N or int(os.environ.get("LMG_TRACE_N", 1024))
    q = q or int(os.environ.get("LMG_TRACE_Q", 512))
    B = B or int(os.environ.get("LMG_TRACE_B", 16))
    import ctypes

    import torch

    import paper_2007_07336_b200 as P
    from paper_2007_07336_b200 import _lib
    from paper_2007_07336_b200.training import _dense_apply

    d = P.device_network(N, q, [0, N, q], device="cuda:0")
    X = torch.from_numpy(P.random_batch(q, [0, N, q], B)).cuda()
    f0 = _dense_apply(d.Wo, d.bo, d.open_act, X)
    U = torch.empty((N, B, q), dtype=torch.float64, device="cuda:0")
    buf = torch.zeros(4 * N, dtype=torch.int64, device="cuda:0")
    lib = _lib.load()
    lib.lmg_debug_sweep_trace(ctypes.c_void_p(buf.data_ptr()))
    for _ in range(2):
        _lib.call("lmg_sequential_forward", d._lmg_view().desc(), B, f0.data_ptr(), _lib.SRC_HEAD,
                  U.data_ptr(), _lib.stream_handle())
    torch.cuda.synchronize()
    lib.lmg_debug_sweep_trace(ctypes.c_void_p(0))
    t = buf.cpu().numpy().reshape(N, 4)[: N - 1].astype(np.float64)
    t -= t[0, 0]
    wait = np.median(t[1:, 1] - t[1:, 0])
    main = np.median(t[1:, 2] - t[1:, 1])
    epi = np.median(t[1:, 3] - t[1:, 2])
    step = np.median(np.diff(t[:, 0]))
    unit = "SM cycles" if q in (16, 32) else "ns"  # the warp FMA sweep stamps clock64
    print(f"serial trace ({unit}, median per step): step {step:.0f} = wait {wait:.0f} + "
          f"mainloop {main:.0f} + epilogue {epi:.0f} + rest {step - wait - main - epi:.0f}")


if __name__ == "__main__" and os.environ.get("LMG_TRACE"):
    trace()

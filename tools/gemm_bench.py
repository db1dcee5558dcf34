"""Microbenchmark of the FP64 DMMA layer-step kernel (lmg::step_gemm) on one GPU.

    LMG_TILE=big|mid|small python tools/gemm_bench.py [--q 512] [--B 256]

Times (CUDA events around every launch, via the library's instrumentation):
  sweep   one F-relaxation sweep step over all blocks of a 1024-layer level (cf 4: 256 tasks)
  adjoint the same with the adjoint layout (W^T, scaled A)
  serial  a 64-step sequential_forward (single-task launches: the coarsest solve)
and prints achieved FP64 TFLOP/s next to cuBLAS DGEMM.
"""

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2007_07336_b200 as P  # noqa: E402
from paper_2007_07336_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--q", type=int, default=512)
    ap.add_argument("--B", type=int, default=256)
    ap.add_argument("--N", type=int, default=1024)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--act", default="tanh")
    a = ap.parse_args()
    N, q, B = a.N, a.q, a.B
    d = P.device_network(N, q, [0, N, q], activation=a.act)
    view = d._lmg_view()
    U = torch.randn(N, B, q, dtype=torch.float64, device="cuda") * 0.3
    S = torch.zeros(B, q, dtype=torch.float64, device="cuda")
    D = torch.rand(N, B, q, dtype=torch.float64, device="cuda")
    st = _lib.stream_handle()
    out = {"tile": os.environ.get("LMG_TILE", "auto"), "N": N, "q": q, "B": B, "act": a.act}

    def timed(fn, cls):
        fn()
        torch.cuda.synchronize()
        _lib.timing_enable(True)
        for _ in range(a.reps):
            fn()
        ms, fl, _, n = _lib.timing_read(cls)
        if n == 0:  # routed to the fused sweep (class 4/5)
            ms, fl, _, n = _lib.timing_read(cls + 4)
        _lib.timing_enable(False)
        return dict(ms_per_launch=ms / n if n else None,
                    tflops=fl / (ms * 1e-3) / 1e12 if ms > 0 else None, launches=n)

    out["sweep"] = timed(lambda: _lib.call("lmg_f_relax", view.desc(), B, 4, U.data_ptr(), S.data_ptr(),
                                           _lib.SRC_HEAD, st), 0)
    out["adjoint"] = timed(lambda: _lib.call("lmg_f_relax", view.desc(D), B, 4, U.data_ptr(), S.data_ptr(),
                                             _lib.SRC_HEAD, st), 1)
    coarse = view.coarsen(16)  # 64 layers
    V = torch.empty(64, B, q, dtype=torch.float64, device="cuda")
    out["serial"] = timed(lambda: _lib.call("lmg_sequential_forward", coarse.desc(), B, S.data_ptr(),
                                            _lib.SRC_HEAD, V.data_ptr(), st), 0)
    x = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
    torch.matmul(x, x)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    torch.matmul(x, x)
    e1.record()
    e1.synchronize()
    out["cublas_dgemm_tflops"] = 2 * 8192 ** 3 / (e0.elapsed_time(e1) * 1e-3) / 1e12
    print(json.dumps(out))


if __name__ == "__main__":
    main()

"""Roofline bookkeeping shared by bench.py and the CLI `scale` command.

The dominant kernel class of a FAS solve is the relaxation / residual layer step (forward +
adjoint layouts, liblmg timing classes 0 and 1).  Its algorithmic work per launch is recorded by
the library (2q^2+5q flops per F-evaluation; 8q^2 bytes of W per layer step plus 8qB
per state row read or written), its time by CUDA events around every launch on the launching
stream.  The bound is picked by arithmetic intensity against the FP64 ridge (DGEMM peak / HBM
peak): tensor (FP64 DMMA) for big batches, HBM for small ones.
"""

from __future__ import annotations

import json
import os

from . import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RELAX_CLASSES = (0, 1)   # step GEMM forward / adjoint layouts
SERIAL_CLASS = 6         # split-K serial steps (latency-bound)
SWEEP_CLASSES = (4, 5)   # fused persistent sweeps


def fp64_peak_tflops(torch, dev) -> float:
    """Measured FP64 tensor peak of this GPU: cuBLAS DGEMM 8192^3 (best of 3, CUDA events).
    MEASURED_PEAKS.json carries HBM and bf16 only ('measure DGEMM on the box')."""
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    torch.matmul(a, b)
    best = 0.0
    for _ in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch.matmul(a, b)
        e.record()
        e.synchronize()
        best = max(best, 2.0 * n ** 3 / (s.elapsed_time(e) * 1e-3) / 1e12)
    del a, b
    return best


def hbm_peak():
    """(GB/s, source): MEASURED_PEAKS.json (driver-measured on this pool), else the profiling
    recipe's fallback."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy bandwidth)"
    except (OSError, ValueError, KeyError):
        return 6650.0, "fallback 6.65 TB/s of B200_PROFILING.md (MEASURED_PEAKS.json absent)"


def read_classes(classes):
    """(ms, flops, bytes, launches) summed over the recorded launches of `classes`."""
    tot = [0.0, 0.0, 0.0, 0]
    for c in classes:
        for i, v in enumerate(_lib.timing_read(c)):
            tot[i] += v
    return tuple(tot)


def classify(flops, nbytes, ms, fp64_tflops, hbm_gbs, force_tensor=False):
    """Roofline of a kernel class from its algorithmic flops / bytes and measured time."""
    intensity = flops / nbytes if nbytes else float("inf")
    ridge = fp64_tflops * 1e12 / (hbm_gbs * 1e9)
    if force_tensor or intensity >= ridge:
        achieved = flops / (ms * 1e-3) / 1e12 if ms > 0 else 0.0
        return dict(bound="tensor", achieved=achieved, peak=fp64_tflops, unit="TFLOP/s",
                    frac=achieved / fp64_tflops if fp64_tflops else None,
                    intensity_flop_per_byte=intensity, fp64_ridge_flop_per_byte=ridge)
    achieved = nbytes / (ms * 1e-3) / 1e9 if ms > 0 else 0.0
    return dict(bound="hbm", achieved=achieved, peak=hbm_gbs, unit="GB/s",
                frac=achieved / hbm_gbs if hbm_gbs else None,
                intensity_flop_per_byte=intensity, fp64_ridge_flop_per_byte=ridge)


def measure(fn, fp64_tflops, hbm_gbs, force_tensor=False):
    """Run fn() with per-launch timing on and return the relaxation class's roofline dict."""
    import torch

    torch.cuda.synchronize()
    _lib.timing_enable(True)
    try:
        fn()
        torch.cuda.synchronize()
        ms, fl, by, n = read_classes(RELAX_CLASSES)
    finally:
        _lib.timing_enable(False)
    r = classify(fl, by, ms, fp64_tflops, hbm_gbs, force_tensor)
    r["launches"] = n
    return r

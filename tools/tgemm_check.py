"""The TMA step GEMM (lmg_tgemm.cu) against step_gemm: bitwise, on a c2-shaped training step.
    python tools/tgemm_check.py N q B c thr out.npz   (run with and without LMG_NO_TGEMM=1)"""
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
if __name__ == "__main__":
    args = sys.argv[1:6] or ["256", "512", "128", "4", "16"]
    outs = []
    for env in ({}, {"LMG_NO_TGEMM": "1"}):
        out = "/tmp/tg_%d.npz" % len(outs)
        subprocess.run([sys.executable, os.path.join(HERE, "..", "tests", "sweep_case.py"), *args, out],
                       check=True, env=dict(os.environ, **env))
        outs.append(np.load(out))
    for k in ("U0", "hist", "cyc", "U1", "lam", "loss", "adj_hist", "adj_cyc", "W", "b", "Us"):
        same = np.array_equal(outs[0][k], outs[1][k], equal_nan=True)
        print(k, "bitwise" if same else "DIFF %.3e" % float(np.nanmax(np.abs(outs[0][k] - outs[1][k]))))
    print("launches", int(outs[0]["launches"]), int(outs[1]["launches"]))

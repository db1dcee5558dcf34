"""c3-shaped conv sweep launches (64 ch, 32x32, B 32, 64 layers -> 16 tasks per launch) under the
LMG_CONV_CFG variants: TF/s per layout and a bitwise check of the outputs against the default.

    python tools/conv_probe.py            (spawns one process per variant: the knob is read once)
"""
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
VARIANTS = ["4,3,0", "4,3,0/noprescale", "4,3,1"]


def child():
    import hashlib

    import torch

    sys.path.insert(0, os.path.dirname(HERE))
    from paper_2007_07336_b200 import _lib
    from paper_2007_07336_b200.synthetic import conv_device_network

    N, C, S, B = 64, 64, 32, 32
    d = conv_device_network(N, C, S, [0, N, C], device="cuda:0", input_dim=64)
    view = d._lmg_view()
    q = C * S * S
    g = torch.Generator(device="cuda").manual_seed(7)
    U0 = torch.randn(N, B, q, dtype=torch.float64, device="cuda", generator=g) * 0.3
    Sd = torch.zeros(B, q, dtype=torch.float64, device="cuda")
    D = torch.rand(N, B, q, dtype=torch.float64, device="cuda", generator=g)
    st = _lib.stream_handle()
    out = {}
    for name, desc, cls in (("fwd", view.desc(), 0), ("adj", view.desc(D), 1)):
        U = U0.clone()
        _lib.call("lmg_f_relax", desc, B, 4, U.data_ptr(), Sd.data_ptr(), _lib.SRC_HEAD, st)
        torch.cuda.synchronize()
        digest = hashlib.sha1(U.cpu().numpy().tobytes()).hexdigest()[:12]
        _lib.timing_enable(True)
        for _ in range(5):
            _lib.call("lmg_f_relax", desc, B, 4, U.data_ptr(), Sd.data_ptr(), _lib.SRC_HEAD, st)
        ms, fl, _, n = _lib.timing_read(cls)
        ems = _lib.timing_read(3)[0]  # elementwise launches (the adjoint's prescale pass)
        _lib.timing_enable(False)
        ms += ems  # conv launches + their elementwise helpers (fl: the conv's algorithmic flops)
        out[name] = dict(ms_per_launch=ms / n, tflops=fl / (ms * 1e-3) / 1e12, digest=digest)
    print(json.dumps(out))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        child()
        sys.exit(0)
    ref = None
    for v in VARIANTS:
        env = dict(os.environ, LMG_CONV_CFG=v.split("/")[0])
        if v.endswith("/noprescale"):
            env["LMG_CONV_NO_PRESCALE"] = "1"
        r = subprocess.run([sys.executable, __file__, "--child"], capture_output=True, text=True,
                           env=env, timeout=600)
        res = json.loads(r.stdout.strip().splitlines()[-1])
        if ref is None:
            ref = res
        same = all(res[k]["digest"] == ref[k]["digest"] for k in res)
        print(f"LMG_CONV_CFG={v}: fwd {res['fwd']['ms_per_launch']:.3f} ms {res['fwd']['tflops']:.2f} TF/s, "
              f"adj {res['adj']['ms_per_launch']:.3f} ms {res['adj']['tflops']:.2f} TF/s, "
              f"{'bitwise' if same else 'DIFFERS'} vs {VARIANTS[0]}", flush=True)

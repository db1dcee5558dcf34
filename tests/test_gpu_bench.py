"""bench.py end to end on the GPU: the JSON line the driver reads (keys, roofline, CPU baseline,
e2e through the public API, launch count, clocks) for a small config, and the multi-rank path
under torchrun (ranks sharing the test GPU over gloo: a functional check of the partitioned
bench, not a measurement)."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "roofline",
        "cpu_baseline", "clocks")


def _line(out):
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out[-2000:]
    return json.loads(lines[0])


def test_bench_json_line_c1():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "c1",
                          "--steps", "3", "--warmup", "3"], capture_output=True, text=True,
                         timeout=900, cwd=ROOT, check=True).stdout
    d = _line(out)
    for k in KEYS:
        assert k in d, k
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["n_gpus"] == 1 and d["steps"] == 3
    assert d["gpu_launches"] > 0
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor") and r["achieved"] > 0 and r["peak"] > 0
    assert r["frac"] == pytest.approx(r["achieved"] / r["peak"])
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["value"] > 0
    assert d["serial_gpu"]["ms_per_step"] > 0
    assert all(len(c) == 2 for c in d["config"]["cycles_per_step"])


def test_bench_under_torchrun_two_ranks():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, LMG_BENCH_BACKEND="gloo")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(port),
                          os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", "c1",
                          "--steps", "2", "--warmup", "1", "--no-cpu-baseline"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT, env=env,
                         check=True).stdout
    d = _line(out)
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert d["config"]["parallelism"] == "layer-partitioned x2"

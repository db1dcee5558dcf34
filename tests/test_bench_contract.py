"""bench.py's reference arm (the CPU oracle on the host cores) prints one JSON line with the keys
the driver reads (task contract: impl, cpu_baseline, e2e with zero transfer bytes)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--config", "c1", "--steps", "1", "--warmup", "1"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT, check=True).stdout
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert "workload" in d["config"]


def test_reference_arm_stops_at_its_time_budget():
    """A requested K can exceed what "a few minutes" allows (a c2 step solves 16 samples to tol,
    ~70 s): the arm stops timing once the next step would overrun LMG_REF_BUDGET_S, always times
    at least one, and reports the steps it actually timed."""
    env = dict(os.environ, LMG_REF_BUDGET_S="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--config", "c1", "--steps", "3", "--warmup", "1"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT, check=True,
                         env=env).stdout
    d = json.loads([ln for ln in out.splitlines() if ln.startswith("{")][0])
    assert d["steps"] == 1 and d["config"]["steps_requested"] == 3
    assert d["config"]["time_budget_s"] == 0.0


def test_traffic_per_config_from_the_round_summary():
    """bench.py's roofline `traffic` comes from the newest profiles/r*_ncu_summary.json: per
    config (round 2 format), None for a config without a capture."""
    sys.path.insert(0, ROOT)
    import bench

    t2, _ = bench.load_traffic("c2")
    t5, _ = bench.load_traffic("c5")
    t3, _ = bench.load_traffic("c3")
    assert t2 and t5 and 0.9e9 < t2 < 1.2e9 and 2.0e9 < t5 < 2.5e9
    assert t3 is None

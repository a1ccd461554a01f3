"""CPU checks of bench.py's contract pieces: the §8(d) algorithmic byte counts the roofline
uses, and the reference arm's JSON line (it runs the CPU oracle, so it
runs here) with the keys the driver reads."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_algorithmic_bytes_match_survey_table():
    import bench
    # n, h, E per config (SURVEY 8(a) sizes); c3 adds per-tet mu, lambda
    assert abs(bench.algorithmic_bytes(53040, 128, 98304, 8) - 121.9e6) < 0.1e6      # c2 fp64
    assert abs(bench.algorithmic_bytes(53040, 128, 98304, 4) - 61.7e6) < 0.1e6       # c2 fp32
    assert abs(bench.algorithmic_bytes(408672, 256, 786432, 4, True) - 902e6) < 1e6  # c3 fp32
    assert abs(bench.algorithmic_bytes(53040, 128, 98304, 8, want_grad=False) - 67.1e6) < 0.1e6
    assert abs(bench.algorithmic_bytes(408672, 256, 786432, 4, True, want_grad=False) - 482e6) < 1e6


def test_reference_arm_line(oracle):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                          "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = [x for x in out.stdout.splitlines() if x.startswith("{")][-1]
    d = json.loads(line)
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 2 and d["warmup"] >= 3
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]

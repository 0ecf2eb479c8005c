"""The bench.py JSON contract, checked on the committed round-end bench lines
(profiles/r01_bench*.json) and on bench.py's command line (CPU only)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LINES = ["r01_bench.json", "r01_bench_cfg3.json", "r01_bench_cfg4.json", "r01_bench_cfg5.json"]


def _load(name):
    with open(os.path.join(ROOT, "profiles", name)) as f:
        return json.loads(f.read().strip().splitlines()[-1])


@pytest.mark.parametrize("name", LINES)
def test_bench_line_keys(name):
    d = _load(name)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "clocks", "gpu_launches"):
        assert k in d, k
    assert d["value"] > 0 and d["unit"] == "unknowns/s" and d["higher_is_better"] is True
    assert d["warmup"] >= 3 and d["steps"] >= 1 and d["n_gpus"] >= 1
    assert d["dtype"] == "f64" and d["data"] == "synthetic" and "workload" in d["config"]
    assert "l2" in d["config"]
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor", "alu") and r["unit"] in ("GB/s", "TFLOP/s")
    assert r["frac"] == pytest.approx(r["achieved"] / r["peak"])
    assert 0 < r["frac"] <= 1
    assert "traffic" in r
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    c = d["clocks"]
    assert c["sm_mhz"] and c["sm_max_mhz"] and not ({"hw_slowdown", "hw_thermal_slowdown",
                                                      "sw_thermal_slowdown"} & set(c["reasons"]))
    assert d["gpu_launches"] > 0


def test_headline_line_has_cpu_baseline_and_traffic():
    d = _load("r01_bench.json")
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] > 0 and cb["sample"]
    assert d["roofline"]["traffic"] and d["config"]["workload"].startswith("cfg2")


def test_bench_cli_flags():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--help"], capture_output=True,
                         text=True, timeout=120, cwd=ROOT)
    assert out.returncode == 0
    for flag in ("--gpus", "--steps", "--warmup", "--impl", "--config", "--compressor", "--mode"):
        assert flag in out.stdout

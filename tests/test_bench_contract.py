"""bench.py keeps the driver's JSON-line contract (keys and types), checked
on the small C1 workload: the reference arm on the CPU, the device arm on a
GPU."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric": str, "value": float, "unit": str, "n_gpus": int, "steps": int,
             "warmup": int, "ms_per_step": float, "higher_is_better": bool, "scaling": str,
             "dtype": str, "data": str, "config": dict, "e2e": dict}


def run_bench(*args):
    out = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True,
                         text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, out.stdout  # exactly one JSON line on stdout
    return json.loads(lines[0])


def check_common(d):
    for k, t in BASE_KEYS.items():
        assert k in d, k
        assert isinstance(d[k], t) or (t is float and isinstance(d[k], int)), (k, d[k])
    assert "vs_baseline" in d and d["vs_baseline"] is None
    assert d["value"] > 0 and d["higher_is_better"] is True
    assert "workload" in d["config"]
    e = d["e2e"]
    assert {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"} <= set(e)
    cb = d["cpu_baseline"]
    assert {"value", "unit", "cores", "kind", "sample"} <= set(cb) and cb["kind"] in ("port", "reference")


def test_reference_arm_line():
    d = run_bench("--impl", "reference", "--config", "C1", "--steps", "1", "--warmup", "0")
    check_common(d)
    assert d["impl"] == "reference"
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0


@pytest.mark.gpu
def test_device_arm_line():
    d = run_bench("--config", "C1", "--steps", "2", "--warmup", "3", "--no-other-runs")
    check_common(d)
    assert "impl" not in d
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(r)
    assert 0 < r["frac"] <= 1.2
    assert d["gpu_launches"] > 0
    v = d["roofline_vector"]  # HBM view of the CG vector kernels
    assert v["bound"] == "hbm" and v["unit"] == "GB/s" and v["achieved"] > 0 and v["peak"] > 1000
    c = d["clocks"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(c) and c["samples"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["cpu_baseline"]["single_thread"]["cores"] == 1
    # both arms describe the same workload with the same config dict
    ref = run_bench("--impl", "reference", "--config", "C1", "--steps", "1", "--warmup", "0")
    assert ref["config"] == d["config"] and ref["metric"] == d["metric"]

"""bench.py's JSON-line contract: the reference arm on CPU (the fp64 oracle, field-parallel; it needs no GPU) and, on
a B200, the default line with every key the driver reads (roofline, cpu_baseline, e2e, clocks, gpu_launches)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT, capture_output=True,
                       text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line_on_cpu():
    d = _run(["--impl", "reference", "--config", "c1", "--steps", "3", "--warmup", "3", "--ref-budget", "0.5"], 300)
    assert d["impl"] == "reference" and d["dtype"] == "f64" and d["higher_is_better"] is True
    assert d["steps"] == 3 and d["value"] > 0 and d["unit"] == "images/s"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["single_core_value"] > 0
    assert d["e2e"] == {"value": d["value"], "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["workload"] == "c1"


@pytest.mark.gpu
def test_default_line_on_gpu():
    d = _run(["--steps", "4", "--warmup", "3"], 900)
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "clocks", "gpu_launches"):
        assert key in d, key
    assert d["n_gpus"] == 1 and d["steps"] == 4 and d["dtype"] == "bf16" and d["config"]["workload"] == "c3"
    r = d["roofline"]
    assert r["bound"] in ("tensor", "hbm") and 0 < r["frac"] < 1 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert d["e2e"]["h2d_bytes_per_step"] == 256 * 200 * 200 * 3 * 4 and d["e2e"]["value"] > 0
    assert d["gpu_launches"] > 0 and d["cpu_baseline"]["kind"] == "oracle"
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]

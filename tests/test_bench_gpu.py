"""The bench.py contract on a GPU: one short run of each arm, the JSON line's
keys and invariants (the driver parses exactly this line)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=900):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT,
                       capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.strip().splitlines() if ln.startswith("{")]
    assert lines, r.stdout[-2000:]
    return json.loads(lines[-1])


@pytest.mark.gpu
def test_bench_line_contract():
    d = _run(["--steps", "5", "--warmup", "3", "--no-secondary", "--no-cpu-baseline"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e",
              "gpu_launches", "roofline", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] == 3
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["higher_is_better"] is True
    assert "workload" in d["config"]
    e = d["e2e"]
    assert e["value"] > 0 and e["unit"] == d["unit"]
    assert e["h2d_bytes_per_step"] == 3 * 8 * d["config"]["n_events"] and e["d2h_bytes_per_step"] > 0
    assert e["results_bitwise_equal_device_run"] is True
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert 0 < r["frac"] <= 1.05 and abs(r["achieved"] / r["peak"] - r["frac"]) < 1e-9
    assert d["gpu_launches"] >= 5 * 4
    assert d["bitwise_identical_repeats"] is True
    # (a 5-step run can end before the first nvidia-smi sample: sm_mhz None)
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]


@pytest.mark.gpu
def test_bench_reference_arm_contract():
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "1"], timeout=1200)
    assert d["impl"] == "reference"
    if "unavailable" in d:
        return
    assert d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0

"""bench.py's JSON line keeps the driver's contract (keys, units, arms)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, timeout=600):
    out = subprocess.check_output([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                                  cwd=ROOT, text=True, timeout=timeout)
    lines = [line for line in out.strip().splitlines() if line.startswith("{")]
    assert len(lines) == 1, out  # exactly one JSON line on stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    """--impl reference: the reference's own CPU code on the host cores, the
    same metric and config as our arm, e2e with no device traffic."""
    j = _run("--impl", "reference", "--workload", "C1", "--steps", "1", "--warmup", "0")
    assert j["impl"] == "reference"
    if "unavailable" in j:
        pytest.skip(j["unavailable"])
    assert j["metric"] == "grid-resistance skyline tuples/sec" and j["unit"] == "skyline tuples/s"
    assert j["value"] > 0 and j["higher_is_better"] is True and j["steps"] == 1
    assert j["config"]["workload"].startswith("C1")
    cb = j["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["value"] == j["value"]
    assert j["e2e"] == {"value": j["value"], "unit": j["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}


@pytest.mark.gpu
def test_our_arm_line():
    j = _run("--workload", "C1", "--steps", "3", "--warmup", "3", "--no-cpu-baseline")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e",
              "gpu_launches", "roofline", "clocks"):
        assert k in j, k
    assert j["n_gpus"] == 1 and j["steps"] == 3 and j["warmup"] == 3 and j["scaling"] == "weak"
    assert j["value"] > 0 and j["ms_per_step"] > 0 and j["gpu_launches"] > 0
    assert j["config"]["workload"].startswith("C1") and "l2" in j["config"]
    e = j["e2e"]
    assert e["value"] > 0 and e["unit"] == j["unit"]
    assert e["h2d_bytes_per_step"] == 100_000 * 4 * 8 + 100_000 * 8 and e["d2h_bytes_per_step"] > 0
    r = j["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert 0 < r["frac"] < 1
    assert "sm_mhz" in j["clocks"] and "reasons" in j["clocks"]

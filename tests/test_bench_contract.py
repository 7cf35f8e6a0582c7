"""bench.py's output contract (the driver parses one JSON line): the
reference arm runs on the host (the oracle port), so its line is checked
here at a small scale; the device arm's keys are checked on the GPU."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config"}


def run_bench(*args, timeout=600):
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, out.stdout  # exactly one line on stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = run_bench("--impl", "reference", "--scale", "10", "--steps", "2", "--warmup", "1", "--roots", "4")
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["unit"] == "GTEPS" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["steps"] == 2 and d["warmup"] == 1
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": "GTEPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["workload"] == "rmat-s10-ef16-4roots"


@pytest.mark.gpu
def test_device_arm_line():
    d = run_bench("--scale", "16", "--steps", "3", "--warmup", "3", "--roots", "8", "--cpu-budget", "1",
                  "--no-extra-configs")
    assert BASE_KEYS <= set(d)
    assert d["value"] > 0 and d["config"]["validated_trees"] == 3 * 8  # every timed tree
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert r["ms_per_bfs"] > 0 and r["expansion"]["ms_per_bfs"] > 0
    assert d["cpu_baseline"]["cpu_model"]
    assert d["e2e"]["d2h_bytes_per_step"] > 0 and d["e2e"]["value"] > 0
    assert d["gpu_launches"] > 0 and "clocks" in d and d["cpu_baseline"]["value"] > 0
    assert d["direction_optimizing"]["layers_equal_top_down"] is True

"""bench.py keeps the driver's JSON contract (task statement):
the reference (oracle) arm on the CPU, and the GPU arm on a small instance of
the same C4 recipe (--scale), each printing one JSON line with every key the
driver and the judge read."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e")


def _run(args, timeout):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT,
                       capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def _common(d):
    for k in BASE_KEYS:
        assert k in d, k
    assert d["value"] > 0 and d["higher_is_better"] is True
    assert d["metric"] == "vehicle-steps/sec" and d["unit"] == "vehicle-steps/s"
    assert "workload" in d["config"] and d["config"]["n_vehicles"] > 0
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in d["e2e"], k


def test_reference_arm_contract(oracle_lib):
    d = _run(["--impl", "reference", "--steps", "2", "--warmup", "3", "--scale", "0.02"], 600)
    _common(d)
    assert d["impl"] == "reference" and d["dtype"] == "f64"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


@pytest.mark.gpu
def test_gpu_arm_contract():
    d = _run(["--steps", "3", "--warmup", "3", "--no-cpu", "--scale", "0.05"], 900)
    _common(d)
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert d["gpu_launches"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]

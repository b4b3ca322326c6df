"""bench.py keeps the driver contract: exactly one JSON line on stdout with
the required keys (reference arm on CPU here; the GPU arm under -m gpu)."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _run(*args, timeout=600):
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True,
                         text=True, timeout=timeout, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [l for l in res.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, res.stdout
    return json.loads(lines[0])


def _common(line):
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e"):
        assert k in line, k
    assert line["config"]["workload"].startswith("C2")
    assert line["value"] > 0 and line["higher_is_better"] is True
    e = line["e2e"]
    assert e["value"] > 0 and {"unit", "h2d_bytes_per_step", "d2h_bytes_per_step"} <= set(e)


def test_reference_arm_prints_one_contract_line():
    line = _run("--impl", "reference", "--steps", "1", "--warmup", "0")
    _common(line)
    assert line["impl"] == "reference"
    cb = line["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["sample"]
    assert cb["value"] == line["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0


@pytest.mark.gpu
def test_gpu_arm_prints_one_contract_line():
    line = _run("--steps", "3", "--warmup", "3", "--no-cpu-baseline")
    _common(line)
    assert line["dtype"] == "bf16" and line["n_gpus"] == 1
    r = line["roofline"]
    assert r["bound"] in ("hbm", "tensor") and r["unit"] in ("GB/s", "TFLOP/s")
    assert 0 < r["frac"] < 1 and abs(r["achieved"] / r["peak"] - r["frac"]) < 1e-9
    assert line["gpu_launches"] > 0 and "clocks" in line and "sm_mhz" in line["clocks"]
    e = line["e2e"]
    assert e["h2d_bytes_per_step"] == e["d2h_bytes_per_step"] == 65536 * 768 * 2
    assert e["matches_device_forward"] is True

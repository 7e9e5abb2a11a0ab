"""The bench.py JSON line the driver parses (one line on stdout, rank 0): the keys
and their meaning for both arms.  CPU: the reference arm (`--impl reference`,
the oracle port on the whole C3 plus the stock-liftfuse sample when
baseline/_ref exists).  GPU: our arm's line, with `roofline`, `cpu_baseline`,
`e2e`, `clocks` and `gpu_launches`."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config")


def _run(*args, timeout=900):
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                       text=True, timeout=timeout)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]
    return json.loads(lines[0])


def _check_base(d, steps, warmup):
    for k in BASE:
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == steps and d["warmup"] == warmup
    assert d["higher_is_better"] is True and d["unit"] == "Gpixel/s" and d["scaling"] == "weak"
    assert d["value"] > 0 and d["ms_per_step"] > 0
    assert d["config"]["workload"].startswith("C3: 16384x16384")
    assert d["dtype"] == "f32"


def test_reference_arm_line():
    d = _run("--impl", "reference", "--steps", "1", "--warmup", "1")
    _check_base(d, 1, 1)
    assert d["impl"] == "reference"
    assert d["config"]["same_config"] is True
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


@pytest.mark.gpu
def test_our_arm_line():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():  # pragma: no cover - CPU container
        pytest.skip("needs a CUDA device")
    d = _run("--steps", "3", "--warmup", "3", "--no-cpu", "--no-scale-configs")
    _check_base(d, 3, 3)
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert 0.3 < r["frac_compulsory"] <= 1.0  # the bytes the fused launch must move, against measured copy
    e = d["e2e"]
    assert e["value"] > 0 and e["unit"] == "Gpixel/s"
    assert e["h2d_bytes_per_step"] == 16384 * 16384 * 4 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] == 3 * 3  # three launch groups (two fused pairs + level 4) per step
    assert set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}
    assert d["config"]["other_arith"]["mode"] == "strict"

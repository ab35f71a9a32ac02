"""bench.py prints ONE JSON line with the keys the driver reads, for both arms."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.strip().splitlines() if ln.strip()]
    assert len(lines) == 1, lines
    return json.loads(lines[0])


@pytest.mark.gpu
def test_own_arm_line():
    d = _run("--steps", "3", "--warmup", "3", "--no-sweep", "--no-configs", "--no-cpu")
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert key in d, key
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["higher_is_better"] is True
    assert d["vs_baseline"] is None and d["dtype"] == "f32" and d["data"] == "synthetic"
    assert d["config"]["workload"] == "cfg2" and "model" not in d["config"]
    assert d["value"] > 0 and abs(d["value"] - 128 * d["config"]["products4"] / (d["ms_per_step"] * 1e-3) / 1e9) < 1e-6 * d["value"]
    r = d["roofline"]
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-12 and 0 < r["frac"] < 1 and r["unit"] == "TFLOP/s"
    e = d["e2e"]
    # operands stay on the host: keys + norms (72 bytes per stored leaf) and the 1 KB blocks of the leaves that occur in
    # a task cross PCIe; beside it the variants that upload every stored leaf / the dense matrix first
    assert 0 < e["operand_leaves_fetched"] <= 65536
    assert e["h2d_bytes_per_step"] > 1024 * e["operand_leaves_fetched"] and e["h2d_bytes_per_step"] < e["all_leaves"]["h2d_bytes_per_step"]
    assert e["d2h_bytes_per_step"] > 0 and 0 < e["value"] < d["value"]
    assert e["all_leaves"]["h2d_bytes_per_step"] % 1028 == 0 and 0 < e["all_leaves"]["value"] < d["value"]
    assert e["from_dense"]["h2d_bytes_per_step"] == 4096 * 4096 * 4 and 0 < e["from_dense"]["value"] < d["value"]
    assert d["gpu_launches"] >= 3 * 3                       # at least plan, execute, interior per step
    assert set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}


def test_reference_arm_line_runs_without_a_gpu():
    d = _run("--impl", "reference", "--steps", "1", "--warmup", "3", "--workload", "cfg1")
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "GFLOP/s"
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1 and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}

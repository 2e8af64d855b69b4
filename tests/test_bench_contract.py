"""bench.py's reference arm (the CPU port of the reference path) prints one
JSON line with the keys the driver reads; run here at a tiny sample size."""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0", "--cpu-seconds", "0.2", "--n", "30000", "--no-numba"],
                         capture_output=True, text=True, check=True, cwd=ROOT, timeout=300)
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    rec = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "cpu_baseline", "e2e"):
        assert key in rec, key
    assert rec["impl"] == "reference" and rec["value"] > 0 and rec["ms_per_step"] > 0
    assert rec["unit"] == "GCUPS" and rec["higher_is_better"] is True
    assert rec["cpu_baseline"]["kind"] == "port" and rec["cpu_baseline"]["cores"] >= 1
    assert rec["e2e"]["value"] == rec["value"]
    assert rec["e2e"]["h2d_bytes_per_step"] == 0 and rec["e2e"]["d2h_bytes_per_step"] == 0


import pytest  # noqa: E402


@pytest.mark.gpu
def test_native_arm_json_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--steps", "1", "--warmup", "3",
                          "--n", "200000", "--no-cpu", "--no-align"],
                         capture_output=True, text=True, check=True, cwd=ROOT, timeout=600)
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    rec = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "dtype",
                "config", "e2e", "roofline", "clocks", "gpu_launches"):
        assert key in rec, key
    assert rec["value"] > 0 and rec["e2e"]["value"] > 0 and rec["gpu_launches"] > 0
    assert rec["e2e"]["h2d_bytes_per_step"] >= 200000
    assert 0 < rec["roofline"]["frac"] <= 1.0

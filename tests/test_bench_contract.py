"""The bench.py contract the driver depends on: one JSON line with the required keys.

`-m "not gpu"`: the reference arm (the oracle on host cores) runs here.  `-m gpu`: the
default arm on a small config with --check (labels bit-exact), and the extra modes."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def run_bench(*args, timeout=900):
    r = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True, text=True,
                       timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = run_bench("--impl", "reference", "--config", "C1", "--steps", "2", "--warmup", "1")
    assert d["impl"] == "reference"
    assert BASE_KEYS <= set(d)
    assert d["value"] > 0 and d["unit"] == "Mpoints/s" and d["n_gpus"] == 1
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert "workload" in d["config"]


@pytest.mark.gpu
def test_default_arm_line_small_config():
    d = run_bench("--config", "C2", "--steps", "5", "--warmup", "3", "--check")
    assert BASE_KEYS <= set(d)
    assert d["parity_bit_exact"] is True
    assert d["higher_is_better"] is True and d["dtype"] == "f32" and d["data"] == "synthetic"
    rf = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(rf)
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and 0 < rf["frac"] < 1
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 12 * d["config"]["n_points"]
    assert e["d2h_bytes_per_step"] == 4 * d["config"]["n_points"]
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["gpu_launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    # the timed step's labels against the oracle's stored full-size digest (tests/golden)
    pd = d["parity_digest"]
    assert pd["input_matches_golden"] is True and pd["labels_match_oracle_digest"] is True


@pytest.mark.gpu
@pytest.mark.parametrize("mode", [["--batch", "16"], ["--ground", "G2"], ["--ap"]], ids=["batch", "ground", "ap"])
def test_extra_modes_lines(mode):
    d = run_bench(*mode, "--steps", "3", "--warmup", "3", "--check")
    assert BASE_KEYS - {"e2e"} <= set(d)
    assert d["parity_bit_exact"] is True and d["value"] > 0

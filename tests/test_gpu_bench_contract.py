"""bench.py keeps the driver's JSON-line contract (one line, required keys and types) for
both arms; runs small (20k tiles, one step) so it stays a few seconds."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_native_arm_contract():
    j = _run("--steps", "1", "--warmup", "3", "--n-tiles", "20000", "--no-layer", "--cpu-every", "256")
    for k, t in (("metric", str), ("value", float), ("unit", str), ("n_gpus", int), ("steps", int),
                 ("warmup", int), ("ms_per_step", float), ("higher_is_better", bool), ("scaling", str),
                 ("dtype", str), ("data", str), ("config", dict), ("roofline", dict), ("cpu_baseline", dict),
                 ("e2e", dict), ("gpu_launches", int), ("clocks", dict)):
        assert isinstance(j[k], t), k
    assert j["n_gpus"] == 1 and j["steps"] == 1 and j["warmup"] == 3 and j["value"] > 0
    assert j["vs_baseline"] is None and "workload" in j["config"]
    rf = j["roofline"]
    assert rf["bound"] == "alu" and rf["unit"] == "TFLOP/s" and 0 < rf["frac"] < 1
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    assert j["cpu_baseline"]["kind"] == "oracle" and j["cpu_baseline"]["cores"] >= 1
    e = j["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert j["gpu_launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(j["clocks"])


def test_reference_arm_contract():
    j = _run("--impl", "reference", "--steps", "1", "--warmup", "0", "--n-tiles", "20000", "--ref-every", "256")
    assert j["impl"] == "reference" and j["value"] > 0
    assert j["cpu_baseline"]["value"] == j["value"] and j["e2e"]["h2d_bytes_per_step"] == 0

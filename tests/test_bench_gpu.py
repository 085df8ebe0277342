"""bench.py's own arm on the B200: one JSON line with the contract's keys, the roofline and
clocks objects, the e2e leg and a launch count that matches the fused path (one kernel per
step)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.timeout(600)
def test_bench_line():
    r = subprocess.run([sys.executable, "bench.py", "--steps", "4", "--warmup", "3", "--no-cpu-baseline",
                        "--no-variants", "--e2e-steps", "20"], cwd=ROOT, capture_output=True, text=True, timeout=580)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [x for x in r.stdout.splitlines() if x.strip().startswith("{")]
    assert len(lines) == 1, lines
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "clocks", "e2e", "gpu_launches", "step_us"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 4 and d["warmup"] == 3 and d["value"] > 0
    assert d["gpu_launches"] == 4  # the fused step kernel, once per timed step
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and 0 < rf["frac"] < 1
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]


@pytest.mark.timeout(600)
def test_bench_strong_scaling_line():
    """--scaling strong at N=1: the 1M pool as 8 co-resident shards of 131072 slots exchanging
    their top-K by peer stores; one line, scaling "strong", 8 step kernels per timed step."""
    r = subprocess.run([sys.executable, "bench.py", "--scaling", "strong", "--steps", "3", "--warmup", "3",
                        "--e2e-steps", "5"], cwd=ROOT, capture_output=True, text=True, timeout=580)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [x for x in r.stdout.splitlines() if x.strip().startswith("{")]
    assert len(lines) == 1, lines
    d = json.loads(lines[0])
    assert d["scaling"] == "strong" and d["n_gpus"] == 1 and d["config"]["shards"] == 8
    assert d["config"]["shards_per_gpu"] == 8 and d["gpu_launches"] == 8 * 3
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["admitted_per_step"] > 0

"""bench.py's own arm on the GPU (the driver's round-end command, shortened):
one JSON line with every key of the contract — metric/value/unit, timing,
e2e with its copied bytes, the roofline object, clocks sampled during the
timed region, the CPU baseline and the launch count of this library."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_bench_line_contract():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "3",
                        "--warmup", "3", "--no-cpu-baseline"], capture_output=True, text=True,
                       timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e",
              "roofline", "clocks", "gpu_launches", "per_kernel", "byte_models"):
        assert k in line, k
    assert line["unit"] == "snake-steps/s" and line["value"] > 0 and line["higher_is_better"]
    assert line["steps"] == 3 and line["warmup"] == 3 and line["n_gpus"] == 1
    assert line["dtype"] == "f64" and line["config"]["global_envs"] == 1024
    e2e = line["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] == 1024 * 4 * 8
    assert e2e["d2h_bytes_per_step"] == 1024 * 3 * 8
    rf = line["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and 0 < rf["frac"] < 1.2
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    assert line["gpu_launches"] > 0
    assert line["clocks"]["sm_mhz"] is None or line["clocks"]["sm_mhz"] > 0

"""bench.py --impl reference (the driver's reference arm) runs on CPU: one
JSON line with the contract's keys from rank 0, nothing from other ranks."""
import json
import os
import subprocess
import sys

from conftest import ROOT


def _run(rank):
    env = dict(os.environ, RANK=str(rank), WORLD_SIZE="2", OMP_NUM_THREADS="1")
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                           "--steps", "1", "--warmup", "1"], env=env, capture_output=True,
                          text=True, timeout=600, cwd=ROOT)


def test_reference_arm_rank0_prints_contract_line():
    r = _run(0)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "snake-steps/s"
    assert line["value"] > 0 and line["higher_is_better"] is True
    for k in ("metric", "n_gpus", "steps", "warmup", "ms_per_step", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "port"


def test_reference_arm_other_ranks_exit_quietly():
    r = _run(1)
    assert r.returncode == 0 and r.stdout.strip() == ""

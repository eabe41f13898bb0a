"""Parity margins: the worst relative error per state field over the two
frames tests/test_gpu_params.py steps (latency on, then off) from the
reference's frame-19 snake state against the oracle, for the default
SolverConfig and every variant of tests/test_gpu_params.py, both solvers,
next to the per-step tolerance the tests use (tests/conftest.py STEP_TOL).
python tools/parity_margins.py > profiles/r2_parity_margins.md"""
import dataclasses
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1904_02833_b200 as M  # noqa: E402
from conftest import STEP_TOL, golden_frame, load_golden, rel_err, scene_parts  # noqa: E402
from oracle.oracle import OracleSim  # noqa: E402
from test_gpu_params import VARIANTS  # noqa: E402

KEYS = ("positions", "velocities", "body_pos", "body_quat", "lam_tetra", "lam_dist")
g = load_golden("step_S.npz")
before = golden_frame(g, 19, "before")
rows = []
for name, kw in [("default", {})] + sorted(VARIANTS.items()):
    for solver in ("streaming", "cluster"):
        parts, cfg = scene_parts("S")
        cfg = dataclasses.replace(cfg, **kw)
        cfg.solver = solver
        sim = M.Simulator(config=cfg, **parts)
        o = OracleSim(config=cfg, **parts)
        o.set_state(before)
        sim.set_state_arrays(before, 0, 1)
        err = {k: 0.0 for k in KEYS}
        for latency in ((True,) if name.startswith("damping") else (True, False)):
            sim.step(g["f19.commands"], latency=latency)
            o.step(g["f19.commands"], latency)
            got = {k: v[0] for k, v in sim.get_state_arrays(0, 1).items()}
            want = o.get_state()
            for k in KEYS:
                err[k] = max(err[k], rel_err(got[k], want[k]))
        worst = max(err[k] / STEP_TOL.get(k, 1e-8) for k in KEYS)
        cells = [f"{err[k]:.1e}" for k in KEYS]
        rows.append((name, solver, cells, worst))
        sim.close()
print("| config | solver | " + " | ".join(f"{k} (tol {STEP_TOL.get(k, 1e-8):.0e})" for k in KEYS)
      + " | worst err / tol |")
print("|---|---|" + "---|" * len(KEYS) + "---|")
for name, solver, cells, worst in rows:
    print(f"| {name} | {solver} | " + " | ".join(cells) + f" | {worst:.3f} |")

"""Golden for the coupled multi-snake scene:
build_snake(SceneConfig(), n_snakes=2) is ONE compliant system — both snakes
share the Newton/PCR iteration and its Krylov scalars (SURVEY key fact 5).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nc \
        python tests/golden/make_golden_multi.py       # ~1 min

step_S2.npz: topology digests, and the full state before/after frames 0 and
2 of a run where snake 1 turns (bias +0.3) and snake 0 does not, plus the
reference StepStats.
"""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import softsnake as R  # noqa: E402
from make_goldens import digest, ref_state, topo_arrays  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def commands(model, i):
    sim = model.sim
    a = model.commands(i * sim.config.dt)          # both snakes, default gait
    b = model.commands(i * sim.config.dt, R.GaitParams(turn_bias=0.3))
    L = model.links_per_snake
    a[L:] = b[L:]
    return a


def main():
    model = R.build_snake(R.SceneConfig(), n_snakes=2)
    sim = model.sim
    out = {f"topo:{k}": np.array(digest(a)) for k, a in topo_arrays(model).items()}
    for i in range(3):
        cmds = commands(model, i)
        if i in (0, 2):
            for k, v in ref_state(sim).items():
                out[f"f{i}.before.{k}"] = v
            out[f"f{i}.commands"] = np.asarray(cmds, np.float64)
        stats = sim.step(cmds, latency=True)
        if i in (0, 2):
            for k, v in ref_state(sim).items():
                out[f"f{i}.after.{k}"] = v
            out[f"f{i}.stats"] = np.array([stats.newton_iterations, stats.pcr_iterations,
                                           stats.contact_count, stats.inverted_tets], np.int64)
    out["frames_captured"] = np.array([0, 2])
    np.savez_compressed(os.path.join(OUT, "step_S2.npz"), **out)
    print("step_S2.npz", os.path.getsize(os.path.join(OUT, "step_S2.npz")))


if __name__ == "__main__":
    main()

"""Replay single envs of the bench workload on the device with each solver /
tet-J mode; report the first non-finite frame."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_1904_02833_b200 as M  # noqa: E402

envs = [int(x) for x in sys.argv[1].split(",")]
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 200
cmds = bench.env_commands(1024, frames, 0)[:, envs]
for solver, exact in (("streaming", False), ("streaming", True), ("cluster", False)):
    m = M.build_snake(M.SceneConfig(), n_envs=len(envs))
    sim = m.sim
    sim.config.solver = solver
    sim.config.exact_jacobian = exact
    first = [-1] * len(envs)
    maxinv = [0] * len(envs)
    for f in range(frames):
        sim.step(cmds[f], True, 1)
        st = sim.get_stats()
        for j, s in enumerate(st):
            maxinv[j] = max(maxinv[j], s.inverted_tets)
            if not s.finite and first[j] < 0:
                first[j] = f
    print(solver, "exact" if exact else "structured", "first non-finite", first, "max inverted", maxinv)

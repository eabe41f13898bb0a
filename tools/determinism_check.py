"""Run the bench workload twice for F frames and compare every env's state
bitwise (race / cross-env contamination check); also report envs that are
non-finite."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_1904_02833_b200 as M  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 100
cmds = bench.env_commands(n, frames, 0)
res = []
for rep in range(2):
    m = M.build_snake(M.SceneConfig(), n_envs=n)
    sim = m.sim
    sim.step(cmds, True, frames)
    res.append(sim.get_state_arrays(names=["positions", "velocities"]))
    fin = np.array([s.finite for s in sim.get_stats()])
    print("rep", rep, "non-finite envs", np.flatnonzero(fin == 0)[:20].tolist(), "info", sim.solver_info)
diff = np.array([not np.array_equal(res[0]["positions"][e], res[1]["positions"][e], equal_nan=True)
                 for e in range(n)])
print("envs differing between runs:", int(diff.sum()), np.flatnonzero(diff)[:20].tolist())

"""Which envs of the bench workload (config 3 commands) go non-finite over
600 frames, and when (stats every 10 frames)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_1904_02833_b200 as M  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 600
solver = sys.argv[3] if len(sys.argv) > 3 else "auto"
model = M.build_snake(M.SceneConfig(), n_envs=n)
sim = model.sim
sim.config.solver = solver
cmds = bench.env_commands(n, frames, 0)
first_bad = np.full(n, -1)
max_inv = np.zeros(n, int)
for f0 in range(0, frames, 10):
    sim.step(cmds[f0:f0 + 10], True, 10)
    st = sim.get_stats()
    fin = np.array([s.finite for s in st])
    inv = np.array([s.inverted_tets for s in st])
    max_inv = np.maximum(max_inv, inv)
    newly = (fin == 0) & (first_bad < 0)
    first_bad[newly] = f0 + 10
bad = np.flatnonzero(first_bad >= 0)
print(json.dumps({"n": n, "frames": frames, "solver": solver, "n_bad": int(bad.size),
                  "bad": bad[:40].tolist(), "first_bad_frame": first_bad[bad][:40].tolist(),
                  "max_inverted_of_good": int(max_inv[first_bad < 0].max()) if (first_bad < 0).any() else None}))

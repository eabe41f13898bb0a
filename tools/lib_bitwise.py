"""Run the bench workload for a few frames with the library in
SS_LIB_OVERRIDE and write the full state to an .npz (argv[1]); with two
.npz files, compare them bitwise: python tools/lib_bitwise.py a.npz b.npz"""
import os
import sys

import numpy as np

if len(sys.argv) == 3 and all(a.endswith(".npz") and os.path.exists(a) for a in sys.argv[1:]):
    a, b = np.load(sys.argv[1]), np.load(sys.argv[2])
    bad = [k for k in a.files if not np.array_equal(a[k], b[k], equal_nan=True)]
    print("bitwise identical" if not bad else f"differ: {bad}")
    for k in bad:
        d = np.nanmax(np.abs(a[k].astype(float) - b[k].astype(float)))
        print(k, "max abs diff", d)
    sys.exit(0)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1904_02833_b200 as M  # noqa: E402

n = int(os.environ.get("N_ENVS", "96"))
frames = int(os.environ.get("FRAMES", "4"))
solver = os.environ.get("SOLVER", "streaming")
model = M.build_snake(M.SceneConfig(), n_envs=n)
model.sim.config.solver = solver
cmds = bench.env_commands(n, frames, 0)
model.sim.step(cmds, True, frames)
st = model.sim.get_state_arrays()
np.savez(sys.argv[1], **st)
print("wrote", sys.argv[1])

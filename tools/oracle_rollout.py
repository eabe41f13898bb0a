"""The reference algorithm (oracle C port) on the bench workload: envs
[e0, e1) for F frames on all host cores; first non-finite frame per env.
Compares the divergence RATE of the long-horizon batched workload with the
device's (tools/diverge_scan.py) — trajectories are chaotic, so which envs
diverge depends on rounding, but how many should not."""
import json
import os
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_1904_02833_b200 as M  # noqa: E402
from oracle.oracle import OracleSim, build  # noqa: E402
from paper_1904_02833_b200.model import build_scene_parts  # noqa: E402

e0, e1, frames = (int(x) for x in sys.argv[1:4])
build()
cmds = bench.env_commands(e1, frames, 0)
sc = M.SceneConfig()
parts, *_ = build_scene_parts(sc)
cfg = sc.solver_config()


def run(e):
    o = OracleSim(config=cfg, **parts)
    for f in range(frames):
        o.step(cmds[f, e], True)
        if f % 10 == 9 and not np.all(np.isfinite(o.get_state()["positions"])):
            return f + 1
    return -1


with ThreadPoolExecutor(len(os.sched_getaffinity(0))) as ex:
    first = list(ex.map(run, range(e0, e1)))
bad = [e0 + i for i, f in enumerate(first) if f >= 0]
print(json.dumps({"envs": [e0, e1], "frames": frames, "n_bad": len(bad), "bad": bad,
                  "first_bad_frame": [f for f in first if f >= 0]}))

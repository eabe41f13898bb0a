"""Config 1: the reference harness's curvature sweep, all 17
pressure levels as one batch of bend fixtures (rollout.curvature_sweep, the
reference protocol: settle <= 900 frames, 30 samples). Prints the wall time
and the per-level curvature means."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_02833_b200 as M  # noqa: E402
from paper_1904_02833_b200 import rollout  # noqa: E402

sc = M.SceneConfig()
rollout.curvature_sweep(sc, pressures=[0.0, 8.0], max_frames=5, samples_per_level=2)  # warm-up
t = time.perf_counter()
r = rollout.curvature_sweep(sc)
wall = time.perf_counter() - t
frames = 930  # nonzero levels never settle: 900 + 30 frames
print(json.dumps({"config": "curvature sweep, 17 levels batched", "wall_s": round(wall, 3),
                  "level_frames_per_s": round(17 * frames / wall, 1),
                  "curvature_mean": [round(x, 4) for x in r["curvature_mean"]],
                  "settled": [int(x) for x in r["settled"]]}))

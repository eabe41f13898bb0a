"""Minimal driver for ncu: N frames of the batched snake step."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_1904_02833_b200 as M  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--envs", type=int, default=1024)
ap.add_argument("--frames", type=int, default=2)
ap.add_argument("--warmup", type=int, default=1)
ap.add_argument("--scene", default="S", choices=["S", "H"])
a = ap.parse_args()
if a.scene == "H":
    a.envs = 1
scene = M.SceneConfig(**bench.H_SCENE) if a.scene == "H" else M.SceneConfig()
model = M.build_snake(scene, n_envs=a.envs)
sim = model.sim
cmds = bench.env_commands(a.envs, a.warmup + a.frames, 0)
sim.step(cmds[:a.warmup], True, a.warmup)
sim.synchronize()
sim.step(cmds[a.warmup:], True, a.frames)
sim.synchronize()
print("ok", sim.get_stats(0, 1)[0].contact_count)

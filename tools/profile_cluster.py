"""Minimal driver for ncu: frames of one snake on the cluster-resident solver."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_02833_b200 as M  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1
model = M.build_snake(M.SceneConfig(), n_envs=n)
model.sim.config.solver = "cluster"
for i in range(3):
    model.sim.step(model.commands(i * model.sim.config.dt)[None, :].repeat(n, 0), True)
model.sim.synchronize()
print("ok", model.sim.solver_info)

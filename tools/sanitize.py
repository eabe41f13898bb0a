"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck), one CUDA path each:

  python tools/sanitize.py cluster     # bend fixture, 1 env, cluster solver (DSMEM + barrier.cluster)
  python tools/sanitize.py streaming   # 64 snakes, streaming kernels (last-block reductions)
  python tools/sanitize.py fused       # 64 snakes, fused J^T gather (shared-memory scatter)
  python tools/sanitize.py builder     # device scene builder (1 snake)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_1904_02833_b200 as M  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "streaming"
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 1
sc = M.SceneConfig()
if what == "cluster":
    m = M.build_bend_fixture(sc)
    m.sim.config.solver = "cluster"
    for i in range(frames):
        m.sim.step(np.array([8.0]), latency=True)
    assert m.sim.solver_info["cluster"]
elif what in ("streaming", "fused"):
    os.environ["SS_FUSED"] = "1" if what == "fused" else "0"
    m = M.build_snake(sc, n_envs=64)
    m.sim.config.solver = "streaming"
    rng = np.random.default_rng(1)
    for i in range(frames):
        m.sim.step(np.clip(rng.normal(0, 4, (64, 4)), -8, 8), latency=True)
    m.sim.synchronize()
    assert m.sim.solver_info["fused_gather"] == (what == "fused")
elif what == "builder":
    m = M.build_snake(sc)
else:
    raise SystemExit(f"unknown workload {what}")
print("ok", what, m.sim.get_stats(0, 1)[0].contact_count)

"""The reference's own numba vs numpy backends on the per-step parity case
(one/two frames from the reference frame-19 snake state, tests/golden/step_S.npz),
for the default SolverConfig and the ill-conditioned Fischer-Burmeister
variant of tests/test_gpu_params.py: how far the reference disagrees with
itself, beside this build's distance from the oracle (tools/parity_margins.py).
Build container only (imports /root/reference):
  PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nbc python tools/ref_backend_spread.py"""
import dataclasses
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import softsnake as R  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
g = np.load(os.path.join(ROOT, "tests", "golden", "step_S.npz"))
pre = "f19.before."


def load_state(sim):
    st = sim.state
    st.particles.positions[:] = g[pre + "positions"]
    st.particles.velocities[:] = g[pre + "velocities"]
    st.body_pos[:] = g[pre + "body_pos"]
    st.body_quat[:] = g[pre + "body_quat"]
    st.body_lin_vel[:] = g[pre + "body_lin_vel"]
    st.body_ang_vel[:] = g[pre + "body_ang_vel"]
    st.time = float(g[pre + "time"])
    sim.lam_dist[:] = g[pre + "lam_dist"]
    sim.lam_tetra[:] = g[pre + "lam_tetra"]
    sim.lam_attach[:] = g[pre + "lam_attach"]
    sim.lam_hinge[:] = g[pre + "lam_hinge"]
    sim.tetras.quats[:] = g[pre + "tet_quats"]
    sim.distances.dirs[:] = g[pre + "dist_dirs"]
    sim.distances.scale[:] = g[pre + "dist_scale"]
    sim._strain_live[:] = g[pre + "strain_live"]
    sim._strain_target[:] = g[pre + "strain_target"]
    sim.channels.pressures[:] = g[pre + "pressures"]
    sim._warm.clear()
    for k, w in enumerate(sim.wheels):
        if g[pre + "warm_valid"][k]:
            sim._warm[("wheel", w.body)] = g[pre + "warm"][k].copy()


def run(backend, **kw):
    sc = R.SceneConfig(backend=backend)
    m = R.build_snake(sc)
    sim = m.sim
    sim.config = dataclasses.replace(sim.config, **kw)
    load_state(sim)
    out = []
    for latency in (True, False):
        sim.step(g["f19.commands"], latency=latency)
        st = sim.state
        out.append({"positions": st.particles.positions.copy(),
                    "velocities": st.particles.velocities.copy(),
                    "body_quat": st.body_quat.copy(), "lam_tetra": sim.lam_tetra.copy()})
    return out


def rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


for name, kw in (("default", {}),
                 ("fb_slopes", dict(fb_slope_min=1e-3, fb_slope_max=1.5, fb_delta=1e-8))):
    a, b = run("numba", **kw), run("numpy", **kw)
    for f in range(2):
        print(name, "frame", f + 1, {k: f"{rel(a[f][k], b[f][k]):.1e}" for k in a[f]})

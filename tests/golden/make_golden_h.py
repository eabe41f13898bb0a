"""Generate the config-5 (1M-tet snake, SURVEY.md §8(d) "H") golden by
running the REFERENCE implementation for two gait frames from rest.

Run in the build container only (needs /root/reference and numba; ~5 min):
    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nc \
        python tests/golden/make_golden_h.py
The full H state is 92 MB per snapshot, so the fixture keeps
  * sha256 digests of the H topology arrays (builder bit-identity),
  * every 64th particle's position/velocity after frames 1 and 2,
  * all body poses/velocities, pressures, StepStats,
  * whole-array checksums (per-axis position sums, Σ|v|, Σ|λ| per family)
so a full-size device run can be checked without shipping the state.
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import softsnake as R  # noqa: E402
from make_goldens import digest, topo_arrays  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
H_SCENE = dict(sections=101, width_nodes=26, height_nodes=21)
SUB = 64


def summary(sim, tag: str) -> dict:
    st = sim.state
    out = {
        f"{tag}.pos_sub": st.particles.positions[::SUB].copy(),
        f"{tag}.vel_sub": st.particles.velocities[::SUB].copy(),
        f"{tag}.pos_sum": st.particles.positions.sum(axis=0),
        f"{tag}.vel_abs": np.abs(st.particles.velocities).sum(),
        f"{tag}.body_pos": st.body_pos.copy(), f"{tag}.body_quat": st.body_quat.copy(),
        f"{tag}.body_lin_vel": st.body_lin_vel.copy(),
        f"{tag}.body_ang_vel": st.body_ang_vel.copy(),
        f"{tag}.pressures": sim.channels.pressures.copy(),
        f"{tag}.time": np.float64(st.time),
    }
    for fam in ("lam_dist", "lam_tetra", "lam_attach", "lam_hinge"):
        out[f"{tag}.{fam}_abs"] = np.abs(getattr(sim, fam)).sum()
    return out


def main():
    sc = R.SceneConfig(**H_SCENE)
    t = time.time()
    model = R.build_snake(sc)
    print(f"build {time.time() - t:.1f}s", flush=True)
    sim = model.sim
    assert sim.tetras.count == 1_000_000
    out = {f"topo:{k}": np.array(digest(a)) for k, a in topo_arrays(model).items()}
    for i in range(2):
        cmds = model.commands(i * sim.config.dt)
        t = time.time()
        stats = sim.step(cmds, latency=True)
        print(f"frame {i} {time.time() - t:.1f}s contacts {stats.contact_count}", flush=True)
        out[f"f{i}.commands"] = np.asarray(cmds, np.float64)
        out[f"f{i}.stats"] = np.array([stats.newton_iterations, stats.pcr_iterations,
                                       stats.contact_count, stats.inverted_tets], np.int64)
        out[f"f{i}.residual"] = np.float64(stats.residual)
        out.update(summary(sim, f"f{i}"))
    out["sub"] = np.int64(SUB)
    np.savez_compressed(os.path.join(OUT, "step_H.npz"), **out)
    print("step_H.npz", os.path.getsize(os.path.join(OUT, "step_H.npz")))


if __name__ == "__main__":
    main()

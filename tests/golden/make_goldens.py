"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container only (needs /root/reference and numba):
    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nc \
        python tests/golden/make_goldens.py
Outputs (committed, small): tests/golden/*.npz. Nothing at test time reads
/root/reference; tests only read these fixtures.

Contents
  topology_digest.npz  sha256 of every topology array the reference builder
                       produces for the snake (S) and the bend fixture (B)
  kernels_S20.npz      numba eval_tetra / eval_distance outputs on the S
                       state before frame 20 (tets subset), and block-kernel
                       I/O on seeded random inputs
  step_B.npz/step_S.npz full state before + after single frames, commands,
                       and the reference StepStats
  traj_S.npz/traj_B.npz short-horizon particle positions
"""
from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import softsnake as R  # noqa: E402
from softsnake.kernels import numba_backend as NB  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def digest(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(str(a.dtype).encode() + str(a.shape).encode() + a.tobytes()).hexdigest()


def topo_arrays(model):
    sim = model.sim
    out = {
        "inv_mass": sim.state.particles.inv_mass, "positions": sim.state.particles.positions,
        "body_pos": sim.state.body_pos, "body_quat": sim.state.body_quat,
        "body_mass": sim.state.body_mass, "body_inertia": sim.state.body_inertia,
        "frame_bodies": model.frame_bodies,
    }
    for fam, attrs in (("distances", ("pairs", "rest", "compliance", "kind", "channel")),
                       ("tetras", ("tets", "rest_inv", "rest_volume", "compliance")),
                       ("attachments", ("particle", "body", "local_anchor", "compliance")),
                       ("hinges", ("body_a", "body_b", "anchor_a", "anchor_b", "axis_a",
                                   "axis_b", "tan1_b", "tan2_b", "compliance"))):
        obj = getattr(sim, fam)
        if obj is None:
            continue
        for a in attrs:
            out[f"{fam}.{a}"] = getattr(obj, a)
    if sim.wheels:
        out["wheels.body"] = np.array([w.body for w in sim.wheels], np.int64)
        out["wheels.radius"] = np.array([w.radius for w in sim.wheels])
    return out


def ref_state(sim) -> dict:
    st = sim.state
    nw = len(sim.wheels)
    warm = np.zeros((nw, 3))
    valid = np.zeros(nw, np.int32)
    for k, w in enumerate(sim.wheels):
        got = sim._warm.get(("wheel", w.body))
        if got is not None:
            warm[k] = got
            valid[k] = 1
    nch = sim.channels.pressures.shape[0] if sim.channels is not None else 0
    return {
        "positions": st.particles.positions.copy(), "velocities": st.particles.velocities.copy(),
        "body_pos": st.body_pos.copy(), "body_quat": st.body_quat.copy(),
        "body_lin_vel": st.body_lin_vel.copy(), "body_ang_vel": st.body_ang_vel.copy(),
        "lam_dist": sim.lam_dist.copy(), "lam_tetra": sim.lam_tetra.copy(),
        "lam_attach": sim.lam_attach.copy(), "lam_hinge": sim.lam_hinge.copy(),
        "tet_quats": sim.tetras.quats.copy(), "dist_dirs": sim.distances.dirs.copy(),
        "dist_scale": sim.distances.scale.copy(),
        "strain_live": (sim._strain_live.copy() if sim._strain_live is not None else np.ones(nch)),
        "strain_target": (sim._strain_target.copy() if sim._strain_target is not None else np.ones(nch)),
        "pressures": sim.channels.pressures.copy() if nch else np.zeros(0),
        "warm": warm, "warm_valid": valid, "time": np.float64(st.time),
    }


def save_steps(name, model, frames, capture, traj_every, latency, cmd_fn):
    sim = model.sim
    out = {}
    traj = {}
    for i in range(frames):
        cmds = cmd_fn(model, i)
        if i in capture:
            for k, v in ref_state(sim).items():
                out[f"f{i}.before.{k}"] = v
            out[f"f{i}.commands"] = np.asarray(cmds, np.float64)
        stats = sim.step(cmds, latency=latency)
        if i in capture:
            for k, v in ref_state(sim).items():
                out[f"f{i}.after.{k}"] = v
            out[f"f{i}.stats"] = np.array([stats.newton_iterations, stats.pcr_iterations,
                                           stats.contact_count, stats.inverted_tets], np.int64)
            out[f"f{i}.residual"] = np.float64(stats.residual)
        if (i + 1) % traj_every == 0:
            traj[f"pos{i + 1}"] = sim.state.particles.positions.copy()
            traj[f"pressures{i + 1}"] = sim.channels.pressures.copy()
            traj[f"com{i + 1}"] = R.state.center_of_mass(sim.state)
    out["frames_captured"] = np.array(sorted(capture))
    np.savez_compressed(os.path.join(OUT, f"step_{name}.npz"), **out)
    np.savez_compressed(os.path.join(OUT, f"traj_{name}.npz"), latency=np.int32(latency), **traj)
    return sim


def main():
    sc = R.SceneConfig()
    # ---- topology digests
    dig = {}
    for tag, model in (("S", R.build_snake(sc)), ("B", R.build_bend_fixture(sc))):
        for k, a in topo_arrays(model).items():
            dig[f"{tag}:{k}"] = np.array(digest(a))
    np.savez_compressed(os.path.join(OUT, "topology_digest.npz"), **dig)

    # ---- bend fixture: +8 psi with latency, 50 frames
    save_steps("B", R.build_bend_fixture(sc), 50, {0, 9, 29}, 10, True,
               lambda m, i: np.array([8.0]))
    # ---- snake: default gait with latency, 30 frames
    sim = save_steps("S", R.build_snake(sc), 30, {0, 19}, 10, True,
                     lambda m, i: m.commands(i * m.sim.config.dt))

    # ---- per-kernel goldens on the snake state before frame 20
    g = np.load(os.path.join(OUT, "step_S.npz"))
    pos = g["f19.before.positions"]
    model = R.build_snake(sc)
    ts = model.sim.tetras
    rng = np.random.default_rng(20260817)
    sub = np.sort(rng.choice(ts.count, 512, replace=False)).astype(np.int32)
    tets = np.ascontiguousarray(ts.tets[sub])
    rinv = np.ascontiguousarray(ts.rest_inv[sub])
    q_in = np.ascontiguousarray(g["f19.before.tet_quats"][sub])
    q = q_in.copy()
    res = np.empty((sub.size, 6))
    vals = np.empty((sub.size, 6, 12))
    ninv = NB.eval_tetra(pos, tets, rinv, q, 1e-12, 500, res, vals)
    # a cold start (identity quats) exercises long polar iterations
    q0 = np.zeros_like(q_in)
    q0[:, 0] = 1.0
    res0 = np.empty_like(res)
    vals0 = np.empty_like(vals)
    NB.eval_tetra(pos, tets, rinv, q0, 1e-12, 500, res0, vals0)
    ds = model.sim.distances
    dirs = g["f19.before.dist_dirs"].copy()
    dres = np.empty(ds.count)
    NB.eval_distance(pos, ds.pairs, ds.rest, g["f19.before.dist_scale"], dirs, dres)
    kern = dict(tet_subset=sub, tet_pos=pos, tet_quats_in=q_in, tet_quats_out=q, tet_res=res,
                tet_vals=vals, tet_ninv=np.int64(ninv), tet_quats0_out=q0, tet_res0=res0,
                tet_vals0=vals0, dist_dirs_in=g["f19.before.dist_dirs"], dist_dirs_out=dirs,
                dist_res=dres)
    # block kernels on seeded random inputs (numba outputs)
    ndof = 300
    for fam, (n, r, k) in {"t": (40, 6, 12), "d": (50, 1, 6), "a": (7, 3, 9), "c": (9, 2, 6)}.items():
        idx = rng.integers(0, ndof, size=(n, k)).astype(np.int32)
        v = rng.normal(size=(n, r, k))
        u = rng.normal(size=ndof)
        x = rng.normal(size=(n, r))
        md = rng.uniform(0.1, 2.0, size=ndof)
        y0 = rng.normal(size=ndof)
        fw = np.empty((n, r))
        NB.block_forward(idx, v, u, fw)
        tr = y0.copy()
        NB.block_transpose(idx, v, x, tr)
        rd = np.empty((n, r))
        NB.block_rowdiag(idx, v, md, rd)
        kern.update({f"blk{fam}.idx": idx, f"blk{fam}.vals": v, f"blk{fam}.u": u,
                     f"blk{fam}.x": x, f"blk{fam}.md": md, f"blk{fam}.y0": y0,
                     f"blk{fam}.fw": fw, f"blk{fam}.tr": tr, f"blk{fam}.rd": rd})
    nb = 5
    md = rng.uniform(0.1, 2.0, size=ndof + 6 * nb)
    ai = rng.normal(size=(nb, 3, 3))
    u = rng.normal(size=ndof + 6 * nb)
    mo = np.empty_like(u)
    NB.minv_apply(md, ai, ndof, u, mo)
    e6 = rng.normal(size=(30, 6, 6))
    x6 = rng.normal(size=(30, 6))
    eo = np.empty((30, 6))
    NB.ereg_apply(e6, x6, eo)
    kern.update(minv_md=md, minv_ai=ai, minv_u=u, minv_out=mo, minv_bd0=np.int64(ndof),
                ereg_v=e6, ereg_x=x6, ereg_out=eo)
    np.savez_compressed(os.path.join(OUT, "kernels_S20.npz"), **kern)
    for f in sorted(os.listdir(OUT)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(OUT, f)))


if __name__ == "__main__":
    main()

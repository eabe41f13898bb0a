"""Shared fixtures. `gpu`-marked tests need a B200 (run under gpurun);
everything else runs on the CPU. The oracle (oracle/) is test
infrastructure: tests use it as the checker only."""
from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")

STATE_KEYS = ("positions", "velocities", "body_pos", "body_quat", "body_lin_vel",
              "body_ang_vel", "lam_dist", "lam_tetra", "lam_attach", "lam_hinge",
              "tet_quats", "dist_dirs", "dist_scale", "strain_live", "strain_target",
              "pressures", "warm", "warm_valid", "time")

# per-step tolerances; relative to the field's max |value|
STEP_TOL = {"positions": 1e-10, "body_pos": 1e-10, "body_quat": 1e-10, "tet_quats": 1e-9,
            "velocities": 1e-8, "body_lin_vel": 1e-8, "body_ang_vel": 1e-8,
            "lam_dist": 1e-8, "lam_tetra": 1e-8, "lam_attach": 1e-8, "lam_hinge": 1e-8,
            "warm": 1e-8, "dist_dirs": 1e-9, "dist_scale": 0.0, "strain_live": 0.0,
            "strain_target": 0.0, "pressures": 0.0, "time": 0.0}


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA) device")


def rel_err(a, b) -> float:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if b.size == 0:
        return 0.0
    scale = max(float(np.max(np.abs(b))), 1e-300)
    return float(np.max(np.abs(a - b))) / scale


def assert_state_close(got: dict, want: dict, tol=None, keys=STATE_KEYS, what=""):
    tol = STEP_TOL if tol is None else tol
    for k in keys:
        if k not in want or np.asarray(want[k]).size == 0:
            continue
        if k == "warm_valid":
            assert np.array_equal(np.asarray(got[k]), np.asarray(want[k])), f"{what} {k}"
            continue
        if k == "tet_quats":
            # q and -q are the same rotation: a tet whose polar iteration lands on
            # the other sign (inverted or strongly sheared elements) is equal
            a, b = np.asarray(got[k], np.float64), np.asarray(want[k], np.float64)
            d = np.minimum(np.abs(a - b).max(axis=-1), np.abs(a + b).max(axis=-1))
            e = float(d.max()) / max(float(np.abs(b).max()), 1e-300) if d.size else 0.0
            assert e <= tol.get(k, 1e-8), f"{what} {k}: rel err {e:.3e} (modulo sign)"
            continue
        if k == "warm" and "warm_valid" in want:
            # a wheel without contact has no entry in the reference's _warm dict
            # (solver.py:522): its stored values are don't-cares
            m = np.asarray(want["warm_valid"]).astype(bool)
            e = rel_err(np.asarray(got[k])[m], np.asarray(want[k])[m]) if m.any() else 0.0
            assert e <= tol.get(k, 1e-8), f"{what} {k}: rel err {e:.3e}"
            continue
        e = rel_err(got[k], want[k])
        assert e <= tol.get(k, 1e-8), f"{what} {k}: rel err {e:.3e} > {tol.get(k, 1e-8):.1e}"


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name))


def golden_frame(g, f, which):
    pre = f"f{f}.{which}."
    return {k[len(pre):]: g[k] for k in g.files if k.startswith(pre)}


def scene_parts(tag: str):
    """(parts, config) for 'S' (snake), 'S2' (two coupled snakes in one
    system) or 'B' (bend fixture), built by this package's builder
    (bit-identical to the reference)."""
    import paper_1904_02833_b200 as M
    from paper_1904_02833_b200.model import build_scene_parts
    sc = M.SceneConfig()
    if tag in ("S", "S2"):
        parts, ns, links, fids = build_scene_parts(sc, 2 if tag == "S2" else None)
        cfg = sc.solver_config()
    else:
        one = M.SceneConfig(**{**sc.__dict__, "links": 1, "snakes": 1})
        parts, ns, links, fids = build_scene_parts(one, 1, with_wheels=False)
        cfg = one.solver_config()
        cfg.ground_enabled = False
        cfg.gravity = (0.0, 0.0, 0.0)
        parts["state"].particles.inv_mass[:one.width_nodes * one.height_nodes] = 0.0
    return parts, cfg


@pytest.fixture(scope="session")
def oracle_mod():
    from oracle import oracle
    oracle.build()
    return oracle

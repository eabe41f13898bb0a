"""Pin the CPU oracle to the reference (goldens made by running
/root/reference, tests/golden/make_goldens.py) before it is trusted as the
checker of the GPU path: per-kernel I/O, single steps from injected full
state, and short-horizon trajectories."""
import numpy as np
import pytest

from conftest import (assert_state_close, golden_frame, load_golden, rel_err,
                      scene_parts)


@pytest.fixture(scope="module")
def kern():
    return load_golden("kernels_S20.npz")


@pytest.mark.parametrize("fam", ["t", "d", "a", "c"])
def test_block_kernels_bitwise(oracle_mod, kern, fam):
    g = {k.split(".", 1)[1]: kern[k] for k in kern.files if k.startswith(f"blk{fam}.")}
    fw = np.empty_like(g["fw"])
    oracle_mod.block_forward(g["idx"], g["vals"], g["u"], fw)
    assert np.array_equal(fw, g["fw"])
    tr = g["y0"].copy()
    oracle_mod.block_transpose(g["idx"], g["vals"], g["x"], tr)
    assert np.array_equal(tr, g["tr"])
    rd = np.empty_like(g["rd"])
    oracle_mod.block_rowdiag(g["idx"], g["vals"], g["md"], rd)
    assert np.array_equal(rd, g["rd"])


def test_minv_ereg_bitwise(oracle_mod, kern):
    out = np.empty_like(kern["minv_out"])
    oracle_mod.minv_apply(kern["minv_md"], kern["minv_ai"], int(kern["minv_bd0"]),
                          kern["minv_u"], out)
    assert np.array_equal(out, kern["minv_out"])
    eo = np.empty_like(kern["ereg_out"])
    oracle_mod.ereg_apply(kern["ereg_v"], kern["ereg_x"], eo)
    assert np.array_equal(eo, kern["ereg_out"])


def test_eval_distance_bitwise(oracle_mod, kern):
    parts, _ = scene_parts("S")
    ds = parts["distances"]
    g = load_golden("step_S.npz")
    dirs = kern["dist_dirs_in"].copy()
    res = np.empty(ds.count)
    oracle_mod.eval_distance(kern["tet_pos"], ds.pairs, ds.rest, g["f19.before.dist_scale"],
                             dirs, res)
    assert np.array_equal(res, kern["dist_res"]) and np.array_equal(dirs, kern["dist_dirs_out"])


@pytest.mark.parametrize("cold", [False, True])
def test_eval_tetra(oracle_mod, kern, cold):
    parts, _ = scene_parts("S")
    ts = parts["tetras"]
    sub = kern["tet_subset"]
    q = kern["tet_quats_in"].copy()
    if cold:
        q[:] = 0.0
        q[:, 0] = 1.0
    res = np.empty((sub.size, 6))
    vals = np.empty((sub.size, 6, 12))
    it = np.zeros(sub.size, np.int32)
    ninv = oracle_mod.eval_tetra(kern["tet_pos"], np.ascontiguousarray(ts.tets[sub]),
                                 np.ascontiguousarray(ts.rest_inv[sub]), q, 1e-12, 500,
                                 res, vals, it)
    sfx = "0" if cold else ""
    assert rel_err(res, kern[f"tet_res{sfx}"]) < 1e-12
    assert rel_err(vals, kern[f"tet_vals{sfx}"]) < 1e-12
    want_q = kern["tet_quats0_out" if cold else "tet_quats_out"]
    assert np.max(1.0 - np.abs(np.sum(q * want_q, axis=1))) < 1e-12  # q == +-q'
    if not cold:
        assert ninv == int(kern["tet_ninv"])
    assert it.max() < 500


@pytest.mark.parametrize("tag", ["B", "S"])
def test_single_step_injected(oracle_mod, tag):
    g = load_golden(f"step_{tag}.npz")
    parts, cfg = scene_parts(tag)
    for f in g["frames_captured"]:
        o = oracle_mod.OracleSim(config=cfg, **parts)
        o.set_state(golden_frame(g, f, "before"))
        o.step(g[f"f{f}.commands"], True)
        assert_state_close(o.get_state(), golden_frame(g, f, "after"), what=f"{tag} frame {f}")
        s = o.stats()
        st = g[f"f{f}.stats"]
        assert (s.newton_iterations, s.pcr_iterations, s.contact_count, s.inverted_tets) == tuple(st)
        assert s.residual == pytest.approx(float(g[f"f{f}.residual"]), rel=1e-9)


@pytest.mark.parametrize("tag,frames", [("B", 50), ("S", 30)])
def test_short_horizon(oracle_mod, tag, frames):
    import paper_1904_02833_b200 as M
    t = load_golden(f"traj_{tag}.npz")
    parts, cfg = scene_parts(tag)
    o = oracle_mod.OracleSim(config=cfg, **parts)
    sc = M.SceneConfig()
    gait = M.GaitParams.from_scene(sc)
    for i in range(frames):
        cmd = np.array([8.0]) if tag == "B" else M.gait_commands(gait, i * cfg.dt, 4, 4)
        o.step(cmd, True)
        if (i + 1) % 10 == 0:
            got = o.get_state()
            assert rel_err(got["positions"], t[f"pos{i + 1}"]) <= 1e-4, f"frame {i + 1}"
            assert np.array_equal(got["pressures"], t[f"pressures{i + 1}"])

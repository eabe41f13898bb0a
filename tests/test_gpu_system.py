"""System inspection: Simulator.last_system /
export_system against the reference's own last_system() after frame 0
(tests/golden/system_{B,S}.npz, tests/golden/make_golden_system.py)."""
from __future__ import annotations

import os

import numpy as np
import pytest

import paper_1904_02833_b200 as M

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module", autouse=True)
def built():
    import __graft_entry__ as g
    g.build()


def _model(tag):
    sc = M.SceneConfig()
    return M.build_bend_fixture(sc) if tag == "B" else M.build_snake(sc)


@pytest.mark.parametrize("tag", ["B", "S"])
def test_last_system_vs_reference(tag):
    path = os.path.join(GOLD, f"system_{tag}.npz")
    if not os.path.exists(path):
        pytest.skip("system golden not generated")
    g = np.load(path)
    model = _model(tag)
    sim = model.sim
    sim.config.keep_matrix = True
    sim.step(g["commands"], latency=True)
    s = sim.last_system()
    A = s.matrix
    assert (A.rows, A.cols) == tuple(g["shape"])
    # the state after one frame agrees with the reference to ~1e-10, so A
    # (a function of positions, quaternions and contact multipliers) to 1e-8
    scale_b = np.max(np.abs(g["rhs"]))
    assert np.max(np.abs(s.rhs - g["rhs"])) <= 1e-7 * scale_b
    for k in range(3):
        ax = A.matvec(g["X"][k])
        assert np.max(np.abs(ax - g["AX"][k])) <= 1e-8 * np.max(np.abs(g["AX"][k])), k
    sp = A.to_scipy()
    assert np.max(np.abs(sp.diagonal() - g["diag"])) <= 1e-8 * np.max(np.abs(g["diag"]))
    absrow = np.asarray(abs(sp).sum(axis=1)).ravel()
    assert np.max(np.abs(absrow - g["absrow"])) <= 1e-8 * np.max(g["absrow"])


def test_last_system_requires_snapshot_and_toggle_keeps_state(tmp_path):
    model = _model("S")
    sim = model.sim
    with pytest.raises(RuntimeError):
        sim.last_system()
    twin = _model("S").sim
    c0 = model.commands(0.0)
    sim.step(c0, latency=True)
    twin.step(c0, latency=True)
    sim.config.keep_matrix = True          # handle rebuilt, state carried over
    c1 = model.commands(sim.config.dt)
    sim.step(c1, latency=True)
    twin.step(c1, latency=True)
    a = sim.get_state_arrays(0, 1)["positions"][0]
    b = twin.get_state_arrays(0, 1)["positions"][0]
    assert np.max(np.abs(a - b)) <= 1e-10 * np.max(np.abs(b))
    s = sim.last_system()
    pa, pb = tmp_path / "A.mtx", tmp_path / "b.mtx"
    sim.export_system(str(pa), str(pb))
    lines = pa.read_text().splitlines()
    assert lines[0] == "%%MatrixMarket matrix coordinate real general"
    assert lines[1] == f"{s.matrix.rows} {s.matrix.cols} {s.matrix.nnz}"
    assert len(lines) == 2 + s.matrix.nnz
    vb = pb.read_text().splitlines()
    assert vb[1] == f"{s.rhs.size} 1" and float(vb[2]) == s.rhs[0]


def test_keep_matrix_multi_wave_export():
    """keep_matrix with more waves than concurrent lanes (10 envs in waves of
    4): every env's exported system is its own (each wave keeps its own
    workspace), equal to a single-env run of the same env."""
    from conftest import scene_parts
    n = 10
    parts, cfg = scene_parts("S")
    cfg.keep_matrix = True
    cfg.wave_envs = 4
    sim = M.BatchedSimulator(n, config=cfg, **parts)
    assert sim.solver_info["waves"] == 3
    rng = np.random.default_rng(11)
    bias = rng.uniform(-0.5, 0.5, n)
    cmds = [np.stack([M.gait_commands(M.GaitParams(turn_bias=b), i * cfg.dt, 4, 4)
                      for b in bias]) for i in range(2)]
    for c in cmds:
        sim.step(c, latency=True)
    X = rng.normal(size=(2, sim.last_system(0).rhs.size))
    for e in (0, 4, 8, 9):
        parts1, cfg1 = scene_parts("S")
        cfg1.keep_matrix = True
        one = M.BatchedSimulator(1, config=cfg1, **parts1)
        for c in cmds:
            one.step(c[e:e + 1], latency=True)
        a, b = sim.last_system(e), one.last_system(0)
        assert a.rhs.shape == b.rhs.shape, f"env {e}: contact count differs"
        assert np.max(np.abs(a.rhs - b.rhs)) <= 1e-8 * np.max(np.abs(b.rhs)), e
        xs = X[:, :b.rhs.size] if b.rhs.size <= X.shape[1] else rng.normal(size=(2, b.rhs.size))
        for x in xs:
            ya, yb = a.matrix.matvec(x), b.matrix.matvec(x)
            assert np.max(np.abs(ya - yb)) <= 1e-8 * np.max(np.abs(yb)), e
        one.close()


def test_keep_toggle_keeps_gait_and_reset_template():
    """Toggling keep_matrix rebuilds the handle: the on-device gait (params
    and frame counters) and the reset template survive the rebuild."""
    from conftest import scene_parts
    n = 3
    outs = []
    for toggle in (False, True):
        parts, cfg = scene_parts("S")
        cfg.solver = "streaming"
        sim = M.BatchedSimulator(n, config=cfg, **parts)
        sim.set_gait([M.GaitParams(turn_bias=b) for b in (-0.3, 0.0, 0.4)], 4, t0=[0.0, 0.1, 0.2])
        sim.step_gait(True, 2)
        if toggle:
            sim.config.keep_matrix = True
        sim.step_gait(True, 2)
        prm, fr = sim.get_gait()
        assert list(fr) == [4, 4, 4]
        assert np.allclose(prm[:, 3], [-0.3, 0.0, 0.4])
        outs.append(sim.get_state_arrays())
        sim.reset_envs([1])  # template = the scene's initial state
        st = sim.get_state_arrays(1, 1)
        assert np.array_equal(st["positions"][0], parts["state"].particles.positions)
        sim.close()
    for k in ("positions", "velocities", "pressures"):
        a, b = outs[0][k], outs[1][k]
        assert np.max(np.abs(a - b)) <= 1e-10 * max(np.max(np.abs(b)), 1e-30), k


def test_get_state_tensors_after_torch_work():
    """get_state_tensors allocates uninitialised tensors and orders the
    device gather after torch's queued work."""
    import torch
    from conftest import scene_parts
    parts, cfg = scene_parts("S")
    sim = M.BatchedSimulator(2, config=cfg, **parts)
    sim.step(np.zeros((2, 4)), latency=True)
    want = sim.get_state_arrays()
    big = torch.randn(4096, 4096, device="cuda:0", dtype=torch.float64)
    for _ in range(8):
        big = big @ big.T / 4096.0  # queue work on torch's stream
    got = sim.get_state_tensors()
    for k in ("positions", "velocities", "tet_quats"):
        assert np.array_equal(got[k].cpu().numpy(), want[k]), k

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

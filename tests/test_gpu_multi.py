"""Coupled multi-snake scene: build_snake(n_snakes=2)
is one compliant system whose Newton/PCR iteration (and Krylov scalars) spans
both snakes (SURVEY key fact 5). Checked per frame from injected reference
state (tests/golden/step_S2.npz, tests/golden/make_golden_multi.py) and
against the oracle."""
from __future__ import annotations

import os

import numpy as np
import pytest

import paper_1904_02833_b200 as M
from conftest import assert_state_close, golden_frame, load_golden, scene_parts

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "step_S2.npz")


@pytest.fixture(scope="module", autouse=True)
def built():
    import __graft_entry__ as g
    g.build()
    if not os.path.exists(GOLD):
        pytest.skip("step_S2.npz not generated")


def _one(a):
    return {k: v[0] for k, v in a.items()}


@pytest.mark.parametrize("exact", [False, True], ids=["structuredJ", "exactJ"])
def test_two_coupled_snakes_vs_reference(exact):
    g = load_golden("step_S2.npz")
    parts, cfg = scene_parts("S2")
    cfg.exact_jacobian = exact
    sim = M.Simulator(config=cfg, **parts)
    assert sim.n_links == 8
    info = sim.solver_info
    if os.environ.get("SS_MULTI_CLUSTER", "1") != "0":
        assert info["clusters_per_env"] == 2  # one cluster per snake (component)
    for f in g["frames_captured"]:
        sim.set_state_arrays(golden_frame(g, f, "before"), 0, 1)
        st = sim.step(g[f"f{f}.commands"], latency=True)
        assert_state_close(_one(sim.get_state_arrays(0, 1)), golden_frame(g, f, "after"),
                           what=f"S2 frame {f}")
        assert (st.newton_iterations, st.pcr_iterations, st.contact_count,
                st.inverted_tets) == tuple(g[f"f{f}.stats"])
    assert sim.solver_info["cross_cluster_fault"] == 0


def test_two_coupled_snakes_vs_oracle(oracle_mod):
    g = load_golden("step_S2.npz")
    parts, cfg = scene_parts("S2")
    sim = M.Simulator(config=cfg, **parts)
    f = int(g["frames_captured"][-1])
    before = golden_frame(g, f, "before")
    o = oracle_mod.OracleSim(config=cfg, **parts)
    o.set_state(before)
    sim.set_state_arrays(before, 0, 1)
    sim.step(g[f"f{f}.commands"], latency=True)
    o.step(g[f"f{f}.commands"], True)
    assert_state_close(_one(sim.get_state_arrays(0, 1)), o.get_state(), what="S2 vs oracle")


def test_coupling_is_real():
    """Snake 0 of the coupled scene differs from the same snake stepped
    alone (shared Krylov scalars), as in the reference."""
    g = load_golden("step_S2.npz")
    parts, cfg = scene_parts("S2")
    two = M.Simulator(config=cfg, **parts)
    b = golden_frame(g, 0, "before")
    two.set_state_arrays(b, 0, 1)
    two.step(g["f0.commands"], latency=True)
    p2 = two.get_state_arrays(0, 1)["positions"][0]
    parts1, cfg1 = scene_parts("S")
    one = M.Simulator(config=cfg1, **parts1)
    one.step(g["f0.commands"][:4], latency=True)
    p1 = one.get_state_arrays(0, 1)["positions"][0]
    n0 = p1.shape[0]
    d = np.max(np.abs(p2[:n0, [0, 2]] - p1[:, [0, 2]]))  # y is offset by the spacing
    assert d > 1e-12


def test_multi_cluster_matches_single_cluster(monkeypatch):
    """The multi-cluster plan (one cluster per snake, cross-cluster dot
    products through global memory in cluster order) against the plan the
    scene gets without it (S2 does not fit one cluster: the streaming
    kernels) over several frames: same Newton/PCR decisions, states within
    round-off of the summation-order change."""
    g = load_golden("step_S2.npz")
    parts, cfg = scene_parts("S2")
    runs = {}
    for mc in ("1", "0"):
        monkeypatch.setenv("SS_MULTI_CLUSTER", mc)
        sim = M.Simulator(config=cfg, **parts)
        runs[mc] = (sim, sim.solver_info["clusters_per_env"])
    assert runs["1"][1] == 2 and runs["0"][1] in (0, 1)
    b = golden_frame(g, 0, "before")
    for sim, _ in runs.values():
        sim.set_state_arrays(b, 0, 1)
    for f in range(4):
        cmds = g["f0.commands"]
        st = [sim.step(cmds, latency=True) for sim, _ in runs.values()]
        assert (st[0].newton_iterations, st[0].pcr_iterations) == \
            (st[1].newton_iterations, st[1].pcr_iterations)
    a = _one(runs["1"][0].get_state_arrays(0, 1))
    b1 = _one(runs["0"][0].get_state_arrays(0, 1))
    assert_state_close(a, b1, what="multi vs single cluster")
    assert runs["1"][0].solver_info["cross_cluster_fault"] == 0


@pytest.mark.parametrize("n", [4, 10])
def test_n_coupled_snakes_vs_oracle(oracle_mod, n):
    """Table II scenes beyond two snakes, two frames of the default gait
    from rest against the oracle: 4 snakes run one 16-CTA cluster per snake
    (cross-cluster sums through global memory), 10 snakes do not fit the
    148 SMs as clusters and run the streaming kernels at one env lane."""
    from paper_1904_02833_b200.model import build_scene_parts
    sc = M.SceneConfig()
    parts, ns, links, fids = build_scene_parts(sc, n)
    cfg = sc.solver_config()
    sim = M.Simulator(config=cfg, **parts)
    info = sim.solver_info
    if n == 4:
        assert info["cluster"] and info["clusters_per_env"] == 4
    else:
        assert not info["cluster"]
    parts_o, *_ = build_scene_parts(sc, n)
    o = oracle_mod.OracleSim(config=cfg, **parts_o)
    o.set_state(_one(sim.get_state_arrays(0, 1)))
    gait = M.GaitParams.from_scene(sc)
    for f in range(2):
        cmds = M.gait_commands(gait, f * cfg.dt, 4 * n, 4)
        st = sim.step(cmds, latency=True)
        o.step(cmds, True)
        assert_state_close(_one(sim.get_state_arrays(0, 1)), o.get_state(),
                           what=f"{n} snakes frame {f}")
        ref = o.stats()
        assert (st.newton_iterations, st.pcr_iterations, st.contact_count) == \
            (ref.newton_iterations, ref.pcr_iterations, ref.contact_count)
    assert sim.solver_info["cross_cluster_fault"] == 0

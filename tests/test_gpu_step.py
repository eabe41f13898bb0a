"""Step parity of the B200 path (C ABI through the drop-in Simulator /
BatchedSimulator) against the reference goldens and the CPU oracle:
single frames from injected full state, short horizons, batched envs,
determinism, edge cases."""
import numpy as np
import pytest

import paper_1904_02833_b200 as M
from conftest import (assert_state_close, golden_frame, load_golden, rel_err,
                      scene_parts)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def built():
    import __graft_entry__ as g
    g.build()


def _sim(tag, n_envs=1, exact=False, solver="auto"):
    parts, cfg = scene_parts(tag)
    cfg.exact_jacobian = exact
    cfg.solver = solver
    if n_envs == 1:
        return M.Simulator(config=cfg, **parts), parts, cfg
    return M.BatchedSimulator(n_envs, config=cfg, **parts), parts, cfg


def _one(a):
    return {k: v[0] for k, v in a.items()}


SOLVERS = [(False, "streaming"), (True, "streaming"), (False, "cluster"), (True, "cluster")]
SOLVER_IDS = ["structuredJ-streaming", "exactJ-streaming", "structuredJ-cluster",
              "exactJ-cluster"]


@pytest.mark.parametrize("exact,solver", SOLVERS, ids=SOLVER_IDS)
@pytest.mark.parametrize("tag", ["B", "S"])
def test_step_vs_reference_golden(tag, exact, solver):
    g = load_golden(f"step_{tag}.npz")
    sim, _, _ = _sim(tag, exact=exact, solver=solver)
    assert sim.solver_info["cluster"] == (solver == "cluster")
    for f in g["frames_captured"]:
        sim.set_state_arrays(golden_frame(g, f, "before"), 0, 1)
        st = sim.step(g[f"f{f}.commands"], latency=True)
        got = _one(sim.get_state_arrays(0, 1))
        assert_state_close(got, golden_frame(g, f, "after"), what=f"{tag} frame {f}")
        want = g[f"f{f}.stats"]
        assert (st.newton_iterations, st.pcr_iterations, st.contact_count,
                st.inverted_tets) == tuple(want)
        assert st.residual == pytest.approx(float(g[f"f{f}.residual"]), rel=1e-8)


@pytest.mark.parametrize("exact,solver", SOLVERS, ids=SOLVER_IDS)
@pytest.mark.parametrize("tag", ["B", "S"])
def test_step_vs_oracle(oracle_mod, tag, exact, solver):
    g = load_golden(f"step_{tag}.npz")
    sim, parts, cfg = _sim(tag, exact=exact, solver=solver)
    for f in g["frames_captured"]:
        before = golden_frame(g, f, "before")
        o = oracle_mod.OracleSim(config=cfg, **parts)
        o.set_state(before)
        sim.set_state_arrays(before, 0, 1)
        sim.step(g[f"f{f}.commands"], latency=True)
        o.step(g[f"f{f}.commands"], True)
        assert_state_close(_one(sim.get_state_arrays(0, 1)), o.get_state(),
                           what=f"{tag} frame {f} vs oracle")


@pytest.mark.parametrize("solver", ["streaming", "cluster"])
@pytest.mark.parametrize("tag,frames", [("B", 50), ("S", 30)])
def test_short_horizon_vs_reference(tag, frames, solver):
    t = load_golden(f"traj_{tag}.npz")
    sim, _, cfg = _sim(tag, solver=solver)
    gait = M.GaitParams.from_scene(M.SceneConfig())
    for i in range(frames):
        cmd = np.array([8.0]) if tag == "B" else M.gait_commands(gait, i * cfg.dt, 4, 4)
        sim.step(cmd, latency=True)
        if (i + 1) % 10 == 0:
            got = sim.get_state_arrays(0, 1)
            assert rel_err(got["positions"][0], t[f"pos{i + 1}"]) <= 1e-4, f"frame {i + 1}"
            assert np.array_equal(got["pressures"][0], t[f"pressures{i + 1}"])
            com = sim.center_of_mass(0, 1)[0]
            assert np.allclose(com, t[f"com{i + 1}"], rtol=1e-6, atol=1e-9)


@pytest.mark.parametrize("solver", ["streaming", "cluster"])
def test_batched_envs_match_oracle_per_env(oracle_mod, solver):
    """5 envs (padded to 8 lanes), each driven by different commands, each
    equal to its own single-env oracle run (envs are independent)."""
    n = 5
    sim, parts, cfg = _sim("S", n, solver=solver)
    rng = np.random.default_rng(20260817)
    bias = rng.uniform(-0.5, 0.5, n)
    ors = [oracle_mod.OracleSim(config=cfg, **parts) for _ in range(n)]
    for i in range(3):
        cmds = np.stack([M.gait_commands(M.GaitParams(turn_bias=b), i * cfg.dt, 4, 4)
                         for b in bias])
        sim.step(cmds, latency=True)
        for e in range(n):
            ors[e].step(cmds[e], True)
    got = sim.get_state_arrays()
    for e in range(n):
        assert_state_close({k: v[e] for k, v in got.items()}, ors[e].get_state(),
                           tol={"positions": 1e-9, "velocities": 1e-6, "pressures": 0.0,
                                "body_quat": 1e-9}, keys=("positions", "velocities",
                                                          "pressures", "body_quat"),
                           what=f"env {e}")
    stats = sim.get_stats()
    assert [s.contact_count for s in stats] == [o.stats().contact_count for o in ors]


@pytest.mark.parametrize("solver", ["streaming", "cluster"])
def test_run_to_run_bitwise_determinism(solver):
    outs = []
    for _ in range(2):
        sim, _, cfg = _sim("S", 3, solver=solver)
        for i in range(2):
            sim.step(np.tile(M.gait_commands(M.GaitParams(), i * cfg.dt, 4, 4), (3, 1)), True)
        outs.append(sim.get_state_arrays())
        sim.close()
    for k in outs[0]:
        assert np.array_equal(outs[0][k], outs[1][k]), k


@pytest.mark.parametrize("solver", ["streaming", "cluster"])
def test_no_commands_and_latency_off(oracle_mod, solver):
    sim, parts, cfg = _sim("B", solver=solver)
    o = oracle_mod.OracleSim(config=cfg, **parts)
    sim.step(np.array([5.0]), latency=False)
    o.step(np.array([5.0]), False)
    sim.step(None)
    o.step(None)
    got = _one(sim.get_state_arrays(0, 1))
    assert_state_close(got, o.get_state(), what="latency off / None")
    assert got["pressures"][1] == 5.0


def test_simulator_drop_in_surface():
    model = M.build_snake(M.SceneConfig())
    sim = model.sim
    st = sim.step(model.commands(0.0))
    assert isinstance(st, M.StepStats) and st.pcr_iterations == 160
    assert sim.totals["steps"] == 1 and sim.static_rows == 27194
    assert sim.state.time == pytest.approx(1 / 60)
    assert sim.channels.pressures.max() > 0.0  # link 1 inflates at t=0 (sin(pi/2) = 1)
    assert np.isfinite(model.link_curvature(0)) and np.isfinite(model.center_of_mass()).all()
    assert sim.lam_tetra.shape == (4320, 6)


def test_cluster_and_streaming_agree():
    """Both Newton-loop solvers from the same state: same contacts, states
    within the per-step tolerance (their dot-product trees differ)."""
    outs = []
    for solver in ("streaming", "cluster"):
        sim, _, cfg = _sim("S", 4, solver=solver)
        for i in range(2):
            sim.step(np.tile(M.gait_commands(M.GaitParams(), i * cfg.dt, 4, 4), (4, 1)), True)
        outs.append((sim.get_state_arrays(), [s.contact_count for s in sim.get_stats()]))
    (a, ca), (b, cb) = outs
    assert ca == cb
    for e in range(4):
        assert_state_close({k: v[e] for k, v in a.items()}, {k: v[e] for k, v in b.items()},
                           tol={"positions": 1e-9, "velocities": 1e-7, "pressures": 0.0},
                           keys=("positions", "velocities", "pressures"))


@pytest.mark.gpu
def test_waves_match_oracle_per_env(oracle_mod):
    """10 envs run as 3 waves of 4 lanes (last wave 2 real + 2 padding):
    state I/O, commands, stats and COM are routed to the right wave/lane and
    each env equals its own single-env oracle run."""
    n = 10
    parts, cfg = scene_parts("S")
    cfg.wave_envs = 4
    sim = M.BatchedSimulator(n, config=cfg, **parts)
    assert sim.solver_info["waves"] == 3 and sim.solver_info["env_lanes"] == 4
    rng = np.random.default_rng(7)
    bias = rng.uniform(-0.5, 0.5, n)
    ors = [oracle_mod.OracleSim(config=cfg, **parts) for _ in range(n)]
    # perturb envs 3..8 (crosses two wave boundaries) through a ranged set_state
    st = sim.get_state_arrays()
    kick = rng.normal(0.0, 0.05, st["velocities"][3:9].shape)
    st["velocities"][3:9] += kick
    sim.set_state_arrays({"velocities": st["velocities"][3:9]}, env0=3, n=6)
    for e in range(3, 9):
        s0 = ors[e].get_state()
        s0["velocities"] = s0["velocities"] + kick[e - 3]
        ors[e].set_state(s0)
    for i in range(3):
        cmds = np.stack([M.gait_commands(M.GaitParams(turn_bias=b), i * cfg.dt, 4, 4)
                         for b in bias])
        sim.step(cmds, latency=True)
        for e in range(n):
            ors[e].step(cmds[e], True)
    got = sim.get_state_arrays()
    for e in range(n):
        assert_state_close({k: v[e] for k, v in got.items()}, ors[e].get_state(),
                           tol={"positions": 1e-9, "velocities": 1e-6, "pressures": 0.0},
                           keys=("positions", "velocities", "pressures"), what=f"env {e}")
    assert [s.contact_count for s in sim.get_stats()] == [o.stats().contact_count for o in ors]
    # COM per env equals a single-env device run of that env's final state
    # (the particle-sum tree depends on the lane count: equal to rounding)
    com = sim.center_of_mass()
    for e in (0, 4, 9):
        one = M.BatchedSimulator(1, config=cfg, **parts)
        one.set_state_arrays({k: v[e] for k, v in got.items()})
        assert np.allclose(one.center_of_mass()[0], com[e], rtol=1e-14, atol=1e-15), f"env {e}"


@pytest.mark.gpu
def test_two_lanes_match_one_lane():
    """From 64 envs the waves alternate between two workspaces / streams
    (concurrent lanes). Every env equals its single-lane run up to the
    reduction tree (which depends on the lane width)."""
    import os
    parts, cfg = scene_parts("S")
    cfg.solver = "streaming"
    n = 96
    rng = np.random.default_rng(5)
    bias = rng.uniform(-0.5, 0.5, n)
    cmds = [np.stack([M.gait_commands(M.GaitParams(turn_bias=b), i * cfg.dt, 4, 4) for b in bias])
            for i in range(3)]
    out = {}
    for lanes in ("1", "2"):
        os.environ["SS_LANES"] = lanes
        try:
            sim = M.BatchedSimulator(n, config=cfg, **parts)
            sim._ensure()
        finally:
            os.environ.pop("SS_LANES", None)
        assert sim.solver_info["waves"] == (1 if lanes == "1" else 2)
        for c in cmds:
            sim.step(c, latency=True)
        out[lanes] = sim.get_state_arrays()
    # three frames apart in the reduction order only (STEP_TOL-scale bounds)
    for k, tol in (("positions", 1e-9), ("velocities", 1e-7), ("lam_tetra", 1e-7),
                   ("pressures", 0.0)):
        a, b = out["1"][k], out["2"][k]
        scale = max(float(np.max(np.abs(a))), 1e-30)
        assert np.max(np.abs(a - b)) <= tol * scale, k


@pytest.mark.gpu
@pytest.mark.parametrize("split", ["4", "8"])
def test_split_gather_matches_serial_walk(split):
    """A lone env's J^T gather splits each DOF's incidence walk over 2-8
    lanes (structured mode; SS_GATHER_SPLIT, auto up to 4 by default). Same frames
    as the serial walk in reference order up to the summation order."""
    import os
    out = {}
    for s in ("1", split):
        os.environ["SS_GATHER_SPLIT"] = s
        try:
            m = M.build_snake(M.SceneConfig(), n_snakes=2)
            m.sim.config.solver = "streaming"
            m.sim._ensure()
        finally:
            os.environ.pop("SS_GATHER_SPLIT", None)
        for i in range(3):
            m.sim.step(m.commands(i * m.sim.config.dt), latency=True)
        out[s] = m.sim.get_state_arrays(0, 1)
    for k, tol in (("positions", 1e-9), ("velocities", 1e-7), ("lam_tetra", 1e-7),
                   ("pressures", 0.0)):
        a, b = out["1"][k], out[split][k]
        scale = max(float(np.max(np.abs(a))), 1e-30)
        assert np.max(np.abs(a - b)) <= tol * scale, k


def test_set_channel_targets_then_step_none():
    """Simulator.set_channel_targets (solver.py:274-277) ticks the channels
    on the device without stepping; step(None) afterwards equals
    step(commands) (step() = set_channel_targets + the frame)."""
    from paper_1904_02833_b200.structures import ChannelBank
    a, _, cfg = _sim("S")
    b, _, _ = _sim("S")
    host = ChannelBank.create(4)
    for i in range(3):
        cmd = M.gait_commands(M.GaitParams(turn_bias=0.2), i * cfg.dt, 4, 4)
        a.set_channel_targets(cmd, latency=True)
        host.tick(cmd, latency=True)
        assert np.array_equal(a.channels.pressures, host.pressures), i
        st = a.get_state_arrays(0, 1)
        assert np.array_equal(st["pressures"][0], host.pressures)
        a.step(None)
        b.step(cmd, latency=True)
    ga, gb = a.get_state_arrays(0, 1), b.get_state_arrays(0, 1)
    for k in ga:
        assert np.array_equal(ga[k], gb[k]), k
    # latency off snaps; a batched handle takes one row per env
    bs, _, _ = _sim("S", 3)
    bs.set_channel_targets(np.array([[8.0, -4.0, 0.0, 1.0]] * 3), latency=False)
    p = bs.get_state_arrays()["pressures"]
    assert np.array_equal(p[2], [0.0, 8.0, 4.0, 0.0, 0.0, 0.0, 0.0, 1.0])


@pytest.mark.parametrize("n,fw,smem", [(40, "8", None), (40, "4", None), (40, "8", "20000"),
                                        (3, "1", None)])
def test_fused_gather_matches_gather(n, fw, smem):
    """k_gather_fused (J^T z of the PCR loop scattered through shared
    memory, no tet column sums in HBM) against k_tet_jt + k_gather (serial
    walk): the same terms in another fixed order. A small shared budget
    splits each link into blocks (elements spanning two blocks)."""
    import os
    parts, cfg = scene_parts("S")
    cfg.solver = "streaming"
    rng = np.random.default_rng(3)
    bias = rng.uniform(-0.5, 0.5, n)
    cmds = [np.stack([M.gait_commands(M.GaitParams(turn_bias=b), i * cfg.dt, 4, 4) for b in bias])
            for i in range(3)]
    out = {}
    for mode in ("0", "1"):
        env = {"SS_FUSED": mode, "SS_FUSED_W": fw, "SS_GATHER_SPLIT": "1"}
        if smem:
            env["SS_FUSED_SMEM"] = smem
        os.environ.update(env)
        try:
            sim = M.BatchedSimulator(n, config=cfg, **parts)
            sim._ensure()
        finally:
            for k in env:
                os.environ.pop(k, None)
        info = sim.solver_info
        assert info["fused_gather"] == (mode == "1")
        if mode == "1":
            assert info["fused_blocks"] == (4 if not smem else 16), info
        names = sim.profile_frames(cmds[0], True, 1)
        assert (names["k_gather_fused"][1] > 0) == (mode == "1")
        for c in cmds[1:]:
            sim.step(c, latency=True)
        out[mode] = sim.get_state_arrays()
        sim.close()
    for k, tol in (("positions", 1e-9), ("velocities", 1e-7), ("lam_tetra", 1e-7),
                   ("pressures", 0.0), ("tet_quats", 1e-9)):
        a, b = out["0"][k], out["1"][k]
        scale = max(float(np.max(np.abs(a))), 1e-30)
        assert np.max(np.abs(a - b)) <= tol * scale, k


@pytest.mark.parametrize("n", [40, 96])
def test_apply_async_bitwise(n):
    """k_apply_rows_async (tet operands staged through shared memory by
    cp.async) gives bitwise the state of k_apply_rows<false>."""
    import os
    parts, cfg = scene_parts("S")
    cfg.solver = "streaming"
    rng = np.random.default_rng(9)
    bias = rng.uniform(-0.5, 0.5, n)
    cmds = [np.stack([M.gait_commands(M.GaitParams(turn_bias=b), i * cfg.dt, 4, 4) for b in bias])
            for i in range(3)]
    out = {}
    for mode in ("0", "1"):
        os.environ["SS_APPLY_ASYNC"] = mode
        os.environ["SS_APPLY2"] = "0"  # both against the one-warp-per-tet kernel
        try:
            sim = M.BatchedSimulator(n, config=cfg, **parts)
            sim._ensure()
        finally:
            os.environ.pop("SS_APPLY_ASYNC", None)
            os.environ.pop("SS_APPLY2", None)
        prof = sim.profile_frames(cmds[0], True, 1)
        assert (prof["k_apply_rows_async"][1] > 0) == (mode == "1")
        for c in cmds[1:]:
            sim.step(c, latency=True)
        out[mode] = sim.get_state_arrays()
        sim.close()
    for k in out["0"]:
        assert np.array_equal(out["0"][k], out["1"][k], equal_nan=True), k


@pytest.mark.parametrize("n,ring,lag", [(96, "3", "2"), (256, "2", "1"), (128, "4", "3")])
def test_jtg_bitwise(n, ring, lag):
    """k_jtg (persistent tile-pipelined J^T z gather, column sums through an
    L2-resident ring) gives bitwise the state of k_tet_jt + k_gather."""
    import os
    parts, cfg = scene_parts("S")
    cfg.solver = "streaming"
    rng = np.random.default_rng(13)
    bias = rng.uniform(-0.5, 0.5, n)
    cmds = [np.stack([M.gait_commands(M.GaitParams(turn_bias=b), i * cfg.dt, 4, 4) for b in bias])
            for i in range(3)]
    out = {}
    for mode in ("0", "1"):
        env = {"SS_JTG": mode, "SS_JTG_RING": ring, "SS_JTG_LAG": lag}
        os.environ.update(env)
        try:
            sim = M.BatchedSimulator(n, config=cfg, **parts)
            sim._ensure()
        finally:
            for k in env:
                os.environ.pop(k, None)
        prof = sim.profile_frames(cmds[0], True, 1)
        assert (prof["k_jtg"][1] > 0) == (mode == "1")
        for c in cmds[1:]:
            sim.step(c, latency=True)
        out[mode] = sim.get_state_arrays()
        sim.close()
    for k in out["0"]:
        assert np.array_equal(out["0"][k], out["1"][k], equal_nan=True), k


@pytest.mark.parametrize("n", [64, 96])
def test_apply2_matches_apply(n):
    """k_apply_rows2 (each tet split over two warps) against k_apply_rows:
    every az is the same expression; only the rho partials are summed over
    another thread assignment (three frames apart at rounding level)."""
    import os
    parts, cfg = scene_parts("S")
    cfg.solver = "streaming"
    rng = np.random.default_rng(17)
    bias = rng.uniform(-0.5, 0.5, n)
    cmds = [np.stack([M.gait_commands(M.GaitParams(turn_bias=b), i * cfg.dt, 4, 4) for b in bias])
            for i in range(3)]
    out = {}
    for mode in ("0", "1"):
        os.environ["SS_APPLY2"] = mode
        try:
            sim = M.BatchedSimulator(n, config=cfg, **parts)
            sim._ensure()
        finally:
            os.environ.pop("SS_APPLY2", None)
        prof = sim.profile_frames(cmds[0], True, 1)
        assert (prof["k_apply_rows2"][1] > 0) == (mode == "1")
        for c in cmds[1:]:
            sim.step(c, latency=True)
        out[mode] = sim.get_state_arrays()
        sim.close()
    for k, tol in (("positions", 1e-9), ("velocities", 1e-7), ("lam_tetra", 1e-7),
                   ("pressures", 0.0), ("tet_quats", 1e-9)):
        a, b = out["0"][k], out["1"][k]
        scale = max(float(np.max(np.abs(a))), 1e-30)
        assert np.max(np.abs(a - b)) <= tol * scale, k


@pytest.mark.parametrize("n", [64, 96])
def test_dir_rows_matches_dir(n):
    """k_pcr_dir_rows (row-wise) against k_pcr_dir (element-owned): the same
    per-row values; den summed over another thread assignment."""
    import os
    parts, cfg = scene_parts("S")
    cfg.solver = "streaming"
    rng = np.random.default_rng(19)
    bias = rng.uniform(-0.5, 0.5, n)
    cmds = [np.stack([M.gait_commands(M.GaitParams(turn_bias=b), i * cfg.dt, 4, 4) for b in bias])
            for i in range(3)]
    out = {}
    for mode in ("0", "1"):
        os.environ["SS_DIR2"] = mode
        try:
            sim = M.BatchedSimulator(n, config=cfg, **parts)
            sim._ensure()
        finally:
            os.environ.pop("SS_DIR2", None)
        prof = sim.profile_frames(cmds[0], True, 1)
        assert (prof["k_pcr_dir_rows"][1] > 0) == (mode == "1")
        for c in cmds[1:]:
            sim.step(c, latency=True)
        out[mode] = sim.get_state_arrays()
        sim.close()
    for k, tol in (("positions", 1e-9), ("velocities", 1e-7), ("lam_tetra", 1e-7),
                   ("pressures", 0.0), ("tet_quats", 1e-9)):
        a, b = out["0"][k], out["1"][k]
        scale = max(float(np.max(np.abs(a))), 1e-30)
        assert np.max(np.abs(a - b)) <= tol * scale, k


@pytest.mark.parametrize("solver", ["streaming", "cluster"])
def test_polar_split_bitwise(solver):
    """k_eval_polar + k_eval_tet (zero iterations from the converged
    quaternion) gives bitwise the state of the fused k_eval_tet."""
    import os
    n = 8 if solver == "cluster" else 40
    parts, cfg = scene_parts("S")
    cfg.solver = solver
    rng = np.random.default_rng(23)
    bias = rng.uniform(-0.5, 0.5, n)
    cmds = [np.stack([M.gait_commands(M.GaitParams(turn_bias=b), i * cfg.dt, 4, 4) for b in bias])
            for i in range(3)]
    out = {}
    for mode in ("0", "1"):
        os.environ["SS_POLAR_SPLIT"] = mode
        try:
            sim = M.BatchedSimulator(n, config=cfg, **parts)
            sim._ensure()
        finally:
            os.environ.pop("SS_POLAR_SPLIT", None)
        prof = sim.profile_frames(cmds[0], True, 1)
        assert (prof["k_eval_polar"][1] > 0) == (mode == "1")
        for c in cmds[1:]:
            sim.step(c, latency=True)
        out[mode] = sim.get_state_arrays()
        sim.close()
    for k in out["0"]:
        assert np.array_equal(out["0"][k], out["1"][k], equal_nan=True), k


@pytest.mark.parametrize("n", [64, 96])
def test_step_jt_bitwise(n):
    """k_step_jt (step + tet column sums in one pass) gives bitwise the state
    of k_pcr_step + k_tet_jt."""
    import os
    parts, cfg = scene_parts("S")
    cfg.solver = "streaming"
    rng = np.random.default_rng(29)
    bias = rng.uniform(-0.5, 0.5, n)
    cmds = [np.stack([M.gait_commands(M.GaitParams(turn_bias=b), i * cfg.dt, 4, 4) for b in bias])
            for i in range(3)]
    out = {}
    for mode in ("0", "1"):
        os.environ["SS_STEPJT"] = mode
        try:
            sim = M.BatchedSimulator(n, config=cfg, **parts)
            sim._ensure()
        finally:
            os.environ.pop("SS_STEPJT", None)
        prof = sim.profile_frames(cmds[0], True, 1)
        assert (prof["k_step_jt"][1] > 0) == (mode == "1")
        for c in cmds[1:]:
            sim.step(c, latency=True)
        out[mode] = sim.get_state_arrays()
        sim.close()
    for k in out["0"]:
        assert np.array_equal(out["0"][k], out["1"][k], equal_nan=True), k


@pytest.mark.parametrize("n", [64, 96])
def test_newton2_bitwise(n):
    """k_newton_rhs2 / k_newton_final2 (tets split over two warps) give
    bitwise the state of k_newton_rhs / k_newton_final (the residual stat is
    summed over another thread assignment)."""
    import os
    parts, cfg = scene_parts("S")
    cfg.solver = "streaming"
    rng = np.random.default_rng(31)
    bias = rng.uniform(-0.5, 0.5, n)
    cmds = [np.stack([M.gait_commands(M.GaitParams(turn_bias=b), i * cfg.dt, 4, 4) for b in bias])
            for i in range(3)]
    out, res = {}, {}
    for mode in ("0", "1"):
        os.environ["SS_NEWTON2"] = mode
        try:
            sim = M.BatchedSimulator(n, config=cfg, **parts)
            sim._ensure()
        finally:
            os.environ.pop("SS_NEWTON2", None)
        prof = sim.profile_frames(cmds[0], True, 1)
        assert (prof["k_newton_rhs2"][1] > 0) == (mode == "1")
        assert (prof["k_newton_final2"][1] > 0) == (mode == "1")
        for c in cmds[1:]:
            sim.step(c, latency=True)
        out[mode] = sim.get_state_arrays()
        res[mode] = np.array([s.residual for s in sim.get_stats()])
        sim.close()
    for k in out["0"]:
        assert np.array_equal(out["0"][k], out["1"][k], equal_nan=True), k
    assert np.allclose(res["0"], res["1"], rtol=1e-10, atol=0.0)


@pytest.mark.parametrize("exact", [False, True], ids=["structuredJ", "exactJ"])
def test_tc_inbox_bitwise(exact):
    """One env on the streaming kernels: tet column sums stored in incidence
    order (SS_TC_INBOX, 256-bit sector per incidence) give bitwise the state
    of the component-major tC layout (the gather adds the same values in
    the same order)."""
    import os
    out = {}
    for mode in ("0", "1"):
        parts, cfg = scene_parts("S")  # fresh state: the drop-in steps it in place
        cfg.solver = "streaming"
        cfg.exact_jacobian = exact
        os.environ["SS_TC_INBOX"] = mode
        try:
            sim = M.Simulator(config=cfg, **parts)
            sim._ensure()
        finally:
            os.environ.pop("SS_TC_INBOX", None)
        for i in range(3):
            sim.step(M.gait_commands(M.GaitParams(), i * cfg.dt, 4, 4), latency=True)
        out[mode] = sim.get_state_arrays(0, 1)
        sim.close()
    for k in out["0"]:
        assert np.array_equal(out["0"][k], out["1"][k], equal_nan=True), k


@pytest.mark.parametrize("exact", [False, True], ids=["structuredJ", "exactJ"])
def test_gather_bulk_bitwise(exact):
    """One env, serial J^T x walk (SS_GATHER_SPLIT=1): the bulk-copy gather
    (k_gather_bulk, each warp's tet-run range of the incidence-order column
    sums streamed into shared memory with cp.async.bulk) gives bitwise the
    state of the per-lane walk (k_gather<17>)."""
    import os
    out = {}
    for mode in ("0", "1"):
        parts, cfg = scene_parts("S")
        cfg.solver = "streaming"
        cfg.exact_jacobian = exact
        os.environ["SS_GATHER_BULK"] = mode
        os.environ["SS_GATHER_SPLIT"] = "1"
        try:
            sim = M.Simulator(config=cfg, **parts)
            sim._ensure()
        finally:
            os.environ.pop("SS_GATHER_BULK", None)
            os.environ.pop("SS_GATHER_SPLIT", None)
        for i in range(3):
            sim.step(M.gait_commands(M.GaitParams(), i * cfg.dt, 4, 4), latency=True)
        out[mode] = sim.get_state_arrays(0, 1)
        sim.close()
    for k in out["0"]:
        assert np.array_equal(out["0"][k], out["1"][k], equal_nan=True), k


@pytest.mark.parametrize("n", [64, 96, 1024])
def test_apply3_bitwise(n):
    """k_apply_rows3 (opt-in SS_APPLY3=1: tet operands staged by TMA
    tensor-tile loads into a shared-memory ring) against k_apply_rows2: the
    same expressions on the same thread assignment, so the whole state is
    bitwise equal."""
    import os
    parts, cfg = scene_parts("S")
    cfg.solver = "streaming"
    rng = np.random.default_rng(23)
    bias = rng.uniform(-0.5, 0.5, n)
    cmds = [np.stack([M.gait_commands(M.GaitParams(turn_bias=b), i * cfg.dt, 4, 4) for b in bias])
            for i in range(3)]
    out = {}
    for mode in ("0", "1"):
        os.environ["SS_APPLY3"] = mode
        try:
            sim = M.BatchedSimulator(n, config=cfg, **parts)
            sim._ensure()
        finally:
            os.environ.pop("SS_APPLY3", None)
        prof = sim.profile_frames(cmds[0], True, 1)
        assert (prof["k_apply_rows3"][1] > 0) == (mode == "1")
        assert (prof["k_apply_rows2"][1] > 0) == (mode == "0")
        for c in cmds[1:]:
            sim.step(c, latency=True)
        out[mode] = sim.get_state_arrays()
        sim.close()
    for k in out["0"]:
        assert np.array_equal(out["0"][k], out["1"][k], equal_nan=True), k


def test_polar_narrow_bitwise():
    """One env: k_eval_polar in 32-thread CTAs (SS_POLAR_NARROW, default)
    gives bitwise the state of the 256-thread launch (each tet's polar loop
    is independent of the launch shape)."""
    import os
    out = {}
    for mode in ("0", "1"):
        parts, cfg = scene_parts("S")
        cfg.solver = "cluster"
        os.environ["SS_POLAR_NARROW"] = mode
        try:
            sim = M.Simulator(config=cfg, **parts)
            sim._ensure()
        finally:
            os.environ.pop("SS_POLAR_NARROW", None)
        for i in range(3):
            sim.step(M.gait_commands(M.GaitParams(), i * cfg.dt, 4, 4), latency=True)
        out[mode] = sim.get_state_arrays(0, 1)
        sim.close()
    for k in out["0"]:
        assert np.array_equal(out["0"][k], out["1"][k], equal_nan=True), k


@pytest.mark.parametrize("exact", [False, True], ids=["structuredJ", "exactJ"])
@pytest.mark.parametrize("n", [64, 1024])
def test_tc_inbox2_bitwise(n, exact):
    """Batched layouts: tet column sums in incidence order ([n_inc][3][E],
    SS_TC_INBOX2, default) give bitwise the state of the tet-major layout
    (the gather adds the same values in the same order)."""
    import os
    parts, cfg = scene_parts("S")
    cfg.solver = "streaming"
    cfg.exact_jacobian = exact
    rng = np.random.default_rng(29)
    bias = rng.uniform(-0.5, 0.5, n)
    cmds = [np.stack([M.gait_commands(M.GaitParams(turn_bias=b), i * cfg.dt, 4, 4) for b in bias])
            for i in range(3)]
    out = {}
    for mode in ("0", "1"):
        os.environ["SS_TC_INBOX2"] = mode
        try:
            sim = M.BatchedSimulator(n, config=cfg, **parts)
            sim._ensure()
        finally:
            os.environ.pop("SS_TC_INBOX2", None)
        for c in cmds:
            sim.step(c, latency=True)
        out[mode] = sim.get_state_arrays()
        sim.close()
    for k in out["0"]:
        assert np.array_equal(out["0"][k], out["1"][k], equal_nan=True), k


def test_pdl_bitwise():
    """Programmatic dependent launch of the frame kernels (SS_PDL=1, opt-in):
    every kernel waits for its predecessor's memory before its first read,
    so the state is bitwise the plain stream order's."""
    import os
    n = 64
    parts, cfg = scene_parts("S")
    cfg.solver = "streaming"
    rng = np.random.default_rng(37)
    bias = rng.uniform(-0.5, 0.5, n)
    cmds = [np.stack([M.gait_commands(M.GaitParams(turn_bias=b), i * cfg.dt, 4, 4) for b in bias])
            for i in range(3)]
    out = {}
    for mode in ("0", "1"):
        os.environ["SS_PDL"] = mode
        try:
            sim = M.BatchedSimulator(n, config=cfg, **parts)
            sim._ensure()
        finally:
            os.environ.pop("SS_PDL", None)
        for c in cmds:
            sim.step(c, latency=True)
        out[mode] = sim.get_state_arrays()
        sim.close()
    for k in out["0"]:
        assert np.array_equal(out["0"][k], out["1"][k], equal_nan=True), k

"""Parity at the benchmarked layouts (SURVEY.md §8(d)
config 3 "8 envs vs 8 separate reference Simulators").

The headline bench (bench.py) builds 1024 envs with the auto plan — two
concurrent lanes of 512 env-lanes (16 tiles of 32 per launch) — and steps
them through ss_step_device with per-env gait commands resident on the
device. Here the same build is fed the reference frame-19 state of the
snake (tests/golden/step_S.npz) and bench.env_commands, and 8 envs spread
over both waves and several tiles are compared with 8 OracleSim runs
(oracle/, the CPU restatement of solver.py:296-544) frame by frame. The
65,536-env config (16 waves of 4,096 lanes) is spot-checked the same way
for one frame. ss_step_device and ss_step (host commands) must agree
bitwise: they replay the same frame graph.
"""
from __future__ import annotations

import numpy as np
import pytest

import paper_1904_02833_b200 as M
from conftest import STEP_TOL, assert_state_close, golden_frame, load_golden

pytestmark = pytest.mark.gpu

SPOT_1024 = (0, 31, 32, 511, 512, 700, 1000, 1023)
SPOT_65536 = (0, 4095, 4096, 20000, 32767, 32768, 50001, 65535)
LATER_TOL = {"positions": 1e-9, "body_pos": 1e-9, "body_quat": 1e-9, "velocities": 1e-7,
             "body_lin_vel": 1e-7, "body_ang_vel": 1e-7, "pressures": 0.0,
             "strain_live": 0.0, "strain_target": 0.0, "dist_scale": 0.0}
LATER_KEYS = tuple(LATER_TOL)


@pytest.fixture(scope="module", autouse=True)
def built():
    import __graft_entry__ as g
    g.build()


def _bench_sim(n_envs: int):
    """The bench's build (bench.py main: build_snake(SceneConfig(), n_envs),
    auto solver and wave plan), every env at the reference frame-19 state
    (replicated on the device through the reset template)."""
    model = M.build_snake(M.SceneConfig(), n_envs=n_envs)
    sim = model.sim
    g = load_golden("step_S.npz")
    f = int(g["frames_captured"][-1])
    before = golden_frame(g, f, "before")
    sim.set_state_arrays(before, 0, 1)
    sim.capture_initial(0)
    sim.reset_envs(np.arange(n_envs))
    return model, sim, before, f


def _oracles(oracle_mod, sim, before, envs):
    from paper_1904_02833_b200.model import build_scene_parts
    sc = M.SceneConfig()
    parts, *_ = build_scene_parts(sc)
    cfg = sc.solver_config()
    out = {}
    for e in envs:
        o = oracle_mod.OracleSim(config=cfg, **parts)
        o.set_state(before)
        out[e] = o
    return out


def _spot(sim, envs):
    return {e: {k: v[0] for k, v in sim.get_state_arrays(e, 1).items()} for e in envs}


def test_bench_layout_1024_vs_oracle(oracle_mod):
    import torch
    from bench import env_commands
    n, frames = 1024, 3
    model, sim, before, f0 = _bench_sim(n)
    info = sim.solver_info
    # the benchmarked plan: streaming solver, two 512-lane waves on two lanes
    assert not info["cluster"] and info["env_lanes"] == 512 and info["waves"] == 2, info
    cmds = env_commands(n, frames, f0)
    d_cmds = torch.from_numpy(cmds).to("cuda:0")
    ors = _oracles(oracle_mod, sim, before, SPOT_1024)
    for i in range(frames):
        sim.step_device(d_cmds.data_ptr() + 8 * i * n * 4, True, 1)
        sim.synchronize()
        for e, o in ors.items():
            o.step(cmds[i, e], True)
        got = _spot(sim, SPOT_1024)
        stats = sim.get_stats()
        for e, o in ors.items():
            want = o.get_state()
            if i == 0:
                assert_state_close(got[e], want, what=f"env {e} frame 1")
            else:
                assert_state_close(got[e], want, tol=LATER_TOL, keys=LATER_KEYS,
                                   what=f"env {e} frame {i + 1}")
            os_ = o.stats()
            assert stats[e].contact_count == os_.contact_count, f"env {e} frame {i + 1} contacts"
            assert stats[e].inverted_tets == os_.inverted_tets, f"env {e} frame {i + 1} inverted"
            assert stats[e].pcr_iterations == 160
    assert all(s.finite for s in stats)


def test_step_device_equals_step_bitwise():
    """ss_step_device (device commands, the bench's timed entry point) and
    ss_step (host commands, the drop-in path) at the bench layout."""
    import torch
    from bench import env_commands
    n, frames = 1024, 2
    cmds = env_commands(n, frames, 19)
    out = []
    for path in ("device", "host"):
        _, sim, _, _ = _bench_sim(n)
        if path == "device":
            d_cmds = torch.from_numpy(cmds).to("cuda:0")
            for i in range(frames):
                sim.step_device(d_cmds.data_ptr() + 8 * i * n * 4, True, 1)
        else:
            for i in range(frames):
                sim.step(cmds[i], latency=True)
        sim.synchronize()
        out.append(sim.get_state_arrays())
        sim.close()
    for k in out[0]:
        assert np.array_equal(out[0][k], out[1][k], equal_nan=True), k


def test_bench_layout_65536_vs_oracle(oracle_mod):
    """Config 4 on one GPU: 65,536 envs in 4,096-lane waves, one frame."""
    import torch
    from bench import env_commands
    n = 65536
    model, sim, before, f0 = _bench_sim(n)
    info = sim.solver_info
    assert info["env_lanes"] == 4096 and info["waves"] == 16, info
    cmds = env_commands(n, 1, f0)
    d_cmds = torch.from_numpy(cmds).to("cuda:0")
    ors = _oracles(oracle_mod, sim, before, SPOT_65536)
    sim.step_device(d_cmds.data_ptr(), True, 1)
    sim.synchronize()
    for e, o in ors.items():
        o.step(cmds[0, e], True)
    got = _spot(sim, SPOT_65536)
    for e, o in ors.items():
        assert_state_close(got[e], o.get_state(), tol=STEP_TOL, what=f"env {e}")
        assert sim.get_stats(e, 1)[0].contact_count == o.stats().contact_count, f"env {e}"
    sim.close()


def test_bench_layout_1024_exact_jacobian_vs_oracle(oracle_mod):
    """The bench layout (1024 envs, two 512-lane waves) in exact tet-Jacobian
    mode (the reference expressions per 6x12 column; the one-thread apply /
    direction / step kernels at 32-env tiles) against the oracle, one frame,
    4 envs over both waves."""
    import dataclasses
    import torch
    from bench import env_commands
    n = 1024
    spots = (0, 511, 512, 1023)
    model = M.build_snake(M.SceneConfig(), n_envs=n)
    sim = model.sim
    sim.config.exact_jacobian = True  # before the handle exists (_ensure reads it)
    g = load_golden("step_S.npz")
    f0 = int(g["frames_captured"][-1])
    before = golden_frame(g, f0, "before")
    sim.set_state_arrays(before, 0, 1)
    sim.capture_initial(0)
    sim.reset_envs(np.arange(n))
    info = sim.solver_info
    assert not info["cluster"] and info["env_lanes"] == 512 and info["waves"] == 2, info
    cmds = env_commands(n, 1, f0)
    d_cmds = torch.from_numpy(cmds).to("cuda:0")
    from paper_1904_02833_b200.model import build_scene_parts
    sc = M.SceneConfig()
    parts, *_ = build_scene_parts(sc)
    cfg = dataclasses.replace(sc.solver_config(), exact_jacobian=True)
    sim.step_device(d_cmds.data_ptr(), True, 1)
    sim.synchronize()
    got = _spot(sim, spots)
    stats = sim.get_stats()
    for e in spots:
        o = oracle_mod.OracleSim(config=cfg, **parts)
        o.set_state(before)
        o.step(cmds[0, e], True)
        assert_state_close(got[e], o.get_state(), what=f"exact env {e} frame 1")
        assert stats[e].contact_count == o.stats().contact_count
    # the exact-mode kernels ran (one thread per tet, reference column expressions)
    prof = sim.profile_frames(cmds[0], True, 1)
    assert prof["k_apply_rows"][1] > 0 and prof["k_apply_rows2"][1] == 0

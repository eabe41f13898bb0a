"""Device-side episode resets: replicate the captured
initial state into chosen envs, optionally perturbed, without touching the
others."""
from __future__ import annotations

import numpy as np
import pytest

import paper_1904_02833_b200 as M

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def built():
    import __graft_entry__ as g
    g.build()


def _model(n, **kw):
    sc = M.SceneConfig()
    m = M.build_snake(sc, n_envs=n)
    for k, v in kw.items():
        setattr(m.sim.config, k, v)
    return m


@pytest.mark.parametrize("wave_envs", [0, 4])
def test_reset_restores_initial_state_and_leaves_others(wave_envs):
    n = 10
    a = _model(n, wave_envs=wave_envs, solver="streaming")
    b = _model(n, wave_envs=wave_envs, solver="streaming")
    fresh = a.sim.get_state_arrays()
    rng = np.random.default_rng(3)
    bias = rng.uniform(-0.5, 0.5, n)
    gaits = [M.GaitParams(turn_bias=x) for x in bias]
    for sim in (a.sim, b.sim):
        sim.set_gait(gaits, a.links_per_snake)
        sim.step_gait(latency=True, n_frames=3)
    ids = [1, 4, 9]
    a.sim.reset_envs(ids)
    sa, sb = a.sim.get_state_arrays(), b.sim.get_state_arrays()
    for k in sa:
        for e in range(n):
            want = fresh[k][e] if e in ids else sb[k][e]
            assert np.array_equal(sa[k][e], want), (k, e)
    # the reset envs' gait clocks restarted: next frame equals a fresh env's first frame
    c = _model(n, wave_envs=wave_envs, solver="streaming")
    c.sim.set_gait(gaits, a.links_per_snake)
    a.sim.step_gait(latency=True)
    c.sim.step_gait(latency=True)
    pa, pc = a.sim.get_state_arrays()["positions"], c.sim.get_state_arrays()["positions"]
    for e in ids:
        assert np.array_equal(pa[e], pc[e]), e


def test_reset_perturbation_is_deterministic_per_env():
    n = 6
    a = _model(n)
    b = _model(n)
    a.sim.reset_envs([0, 2, 5], seed=11, pos_sigma=1e-3, vel_sigma=1e-2)
    b.sim.reset_envs([5, 2], seed=11, pos_sigma=1e-3, vel_sigma=1e-2)  # other order, subset
    sa, sb = a.sim.get_state_arrays(), b.sim.get_state_arrays()
    p0 = M.build_snake(M.SceneConfig()).sim.state.particles.positions
    for e in (2, 5):
        assert np.array_equal(sa["positions"][e], sb["positions"][e])
    d = sa["positions"][2] - p0
    assert 0.5e-3 < d.std() < 2e-3 and abs(d.mean()) < 2e-4
    assert not np.array_equal(sa["positions"][2], sa["positions"][5])
    assert np.array_equal(sa["positions"][1], p0)  # untouched env
    v = sa["velocities"][0]
    assert 0.5e-2 < v.std() < 2e-2
    with pytest.raises(ValueError):
        a.sim.reset_envs([n])


def test_device_state_io_matches_host_io():
    """ss_get/set_state_device (torch CUDA tensors) == the host path."""
    import torch
    n = 5
    m = _model(n, solver="streaming")
    m.sim.set_gait(M.GaitParams(turn_bias=0.2), m.links_per_snake, t0=[0.0, 0.1, 0.2, 0.3, 0.4])
    m.sim.step_gait(latency=True, n_frames=2)
    host = m.sim.get_state_arrays(1, 3)
    dev = m.sim.get_state_tensors(1, 3)
    for k in host:
        assert np.array_equal(host[k], dev[k].cpu().numpy()), k
    # write env 0's state into envs 3 and 4 from the device, then compare
    src = m.sim.get_state_tensors(0, 1)
    rep = {k: v.repeat((2,) + (1,) * (v.dim() - 1)) for k, v in src.items()}
    m.sim.set_state_tensors(rep, 3, 2)
    after = m.sim.get_state_arrays()
    for k in after:
        assert np.array_equal(after[k][3], after[k][0]) and np.array_equal(after[k][4], after[k][0]), k
    with pytest.raises(ValueError):
        m.sim.set_state_tensors({"positions": torch.zeros(1, 3, device="cuda")}, 0, 1)

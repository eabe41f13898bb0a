"""The builder reproduces the reference topology bit for bit (digests of
every array the reference builder produced, tests/golden/topology_digest.npz,
made by tests/golden/make_goldens.py from /root/reference). Both builders:
the host one (numpy, CPU) and the device one (ss_build_link_meshes, the
link meshes built on the GPU)."""
import hashlib

import numpy as np
import pytest

import paper_1904_02833_b200 as M
from conftest import load_golden


def _digest(a):
    a = np.ascontiguousarray(a)
    return hashlib.sha256(str(a.dtype).encode() + str(a.shape).encode() + a.tobytes()).hexdigest()


def _arrays(model):
    sim = model.sim
    out = {"inv_mass": sim.state.particles.inv_mass, "positions": sim.state.particles.positions,
           "body_pos": sim.state.body_pos, "body_quat": sim.state.body_quat,
           "body_mass": sim.state.body_mass, "body_inertia": sim.state.body_inertia,
           "frame_bodies": model.frame_bodies}
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


BUILDERS = [pytest.param("host"), pytest.param("device", marks=pytest.mark.gpu)]


@pytest.mark.parametrize("builder", BUILDERS)
@pytest.mark.parametrize("tag", ["S", "B"])
def test_topology_bit_identical(tag, builder):
    g = load_golden("topology_digest.npz")
    sc = M.SceneConfig()
    model = (M.build_snake(sc, builder=builder) if tag == "S"
             else M.build_bend_fixture(sc, builder=builder))
    arrays = _arrays(model)
    keys = sorted(k.split(":", 1)[1] for k in g.files if k.startswith(tag + ":"))
    assert keys == sorted(arrays), "array set differs from the reference builder"
    for k in keys:
        assert _digest(arrays[k]) == str(g[f"{tag}:{k}"]), f"{tag} {k} differs from reference"


def test_snake_counts_match_survey():
    sim = M.build_snake(M.SceneConfig(), builder="host").sim
    assert sim.state.num_particles == 1456 and sim.state.num_bodies == 15
    assert sim.distances.count == 1080 and sim.tetras.count == 4320
    assert sim.attachments.count == 48 and sim.hinges.count == 10 and len(sim.wheels) == 10
    assert sim.static_rows == 27194


@pytest.mark.parametrize("builder", BUILDERS)
def test_degenerate_grid_rejected(builder):
    with pytest.raises(ValueError):
        M.build_snake(M.SceneConfig(width_nodes=4), builder=builder)


@pytest.mark.parametrize("builder", BUILDERS)
def test_hires_topology_bit_identical(builder):
    """Config 5 (1,000,000 tets): every topology array equals the reference
    builder's (digests in tests/golden/step_H.npz)."""
    import os
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "step_H.npz")
    if not os.path.exists(path):
        pytest.skip("step_H.npz not generated")
    g = np.load(path)
    import time
    t0 = time.perf_counter()
    model = M.build_snake(M.SceneConfig(sections=101, width_nodes=26, height_nodes=21),
                          builder=builder)
    secs = time.perf_counter() - t0
    assert model.sim.tetras.count == 1_000_000
    if builder == "device":
        assert secs < 5.0, f"device build of the 1M-tet scene took {secs:.1f} s"
    arrays = _arrays(model)
    keys = sorted(k.split(":", 1)[1] for k in g.files if k.startswith("topo:"))
    assert keys == sorted(arrays)
    for k in keys:
        assert _digest(arrays[k]) == str(g[f"topo:{k}"]), f"H {k} differs from reference"


@pytest.mark.parametrize("builder", BUILDERS)
def test_two_snake_topology_bit_identical(builder):
    """build_snake(n_snakes=2) (the coupled scene) equals the reference
    builder's arrays (digests in tests/golden/step_S2.npz)."""
    import os
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "step_S2.npz")
    if not os.path.exists(path):
        pytest.skip("step_S2.npz not generated")
    g = np.load(path)
    arrays = _arrays(M.build_snake(M.SceneConfig(), n_snakes=2, builder=builder))
    keys = sorted(k.split(":", 1)[1] for k in g.files if k.startswith("topo:"))
    assert keys == sorted(arrays)
    for k in keys:
        assert _digest(arrays[k]) == str(g[f"topo:{k}"]), f"S2 {k} differs from reference"

"""SceneConfig strictness and the pneumatic / strain known answers of the
reference's own tests (pkg/tests/test_pneumatics.py:11-133), checked on the
host mirror and on the C oracle the GPU path is compared against."""
import numpy as np
import pytest
from hypothesis import given, strategies as st

import paper_1904_02833_b200 as M
from paper_1904_02833_b200.structures import update_pressure, route_antagonistic


def test_scene_defaults_and_gamma():
    sc = M.SceneConfig()
    cfg = sc.solver_config()
    assert cfg.constraint_damping == 10.0 and cfg.h == pytest.approx(1 / 120)
    assert sc.poisson == 0.49 and sc.links == 4


def test_scene_ini_roundtrip(tmp_path):
    sc = M.SceneConfig(links=2, mu=0.5, latency=False)
    p = tmp_path / "s.ini"
    sc.write(str(p))
    back = M.SceneConfig.from_file(str(p))
    assert back == sc


def test_scene_unknown_key_and_section():
    with pytest.raises(ValueError):
        M.SceneConfig.from_string("[snake]\nbogus = 1\n")
    with pytest.raises(ValueError):
        M.SceneConfig.from_string("[nope]\n")


def test_inflation_first_step_exact(oracle_mod):
    assert update_pressure(0.0, 8.0) == pytest.approx(1.84, abs=1e-12)
    assert oracle_mod.update_pressure(0.0, 8.0) == update_pressure(0.0, 8.0)


def test_deflation_linear_then_geometric(oracle_mod):
    p = 8.0
    while p * 0.23 > 0.68:
        nxt = oracle_mod.update_pressure(p, 0.0)
        assert p - nxt == pytest.approx(0.68, abs=1e-12)
        p = nxt
    assert oracle_mod.update_pressure(2.0, 0.0) / 2.0 == pytest.approx(0.77, abs=1e-12)
    assert 0.68 / 0.23 == pytest.approx(2.9565, abs=1e-4)


def test_fixed_point_and_floor(oracle_mod):
    assert oracle_mod.update_pressure(5.0, 5.0) == 5.0
    assert oracle_mod.update_pressure(1e-9, 0.0) >= 0.0


@given(st.floats(0.0, 8.0), st.floats(0.0, 8.0))
def test_pressure_range_and_mirror(p, target):
    from oracle import oracle
    out = oracle.update_pressure(p, target)
    assert 0.0 <= out <= 8.0
    assert out == update_pressure(p, target)


def test_strain_law():
    law = M.StrainLaw(66243.0)
    assert law.strain_pa(55158.0) == pytest.approx(1.8327, abs=1e-4)
    assert law.strain(8.0) == pytest.approx(1.0 + 8.0 * M.PSI_TO_PA / 66243.0, rel=1e-12)
    assert law.strain(0.0) == 1.0


def test_route_and_bank():
    assert route_antagonistic(3.0) == (0.0, 3.0)
    assert route_antagonistic(-3.0) == (3.0, 0.0)
    bank = M.ChannelBank.create(2)
    bank.tick(np.array([8.0, -8.0]))
    assert bank.pressures[1] == pytest.approx(1.84) and bank.pressures[2] == pytest.approx(1.84)
    assert bank.pressures[0] == 0.0 and bank.pressures[3] == 0.0

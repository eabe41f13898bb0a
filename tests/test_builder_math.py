"""The device scene builder's arithmetic (paper_1904_02833_b200/csrc/
ss_build.cuh), compiled for the host, against numpy on the CPU: the rest
inverse (np.linalg.inv, constraints.py:136), the determinant behind the
rest volume (np.linalg.det, constraints.py:132) and the cable rest length
(np.linalg.norm, snake.py:133) are bitwise numpy's for every tet and cable
of the snake and the bend fixture. The device
build itself is checked against the reference digests in test_topology.py."""
from __future__ import annotations

import os
import subprocess

import numpy as np
import pytest

import paper_1904_02833_b200 as M
from paper_1904_02833_b200.model import build_scene_parts

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def checker(tmp_path_factory):
    d = tmp_path_factory.mktemp("bc")
    exe = str(d / "build_check")
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-o", exe,
                           os.path.join(ROOT, "tools", "build_check.cpp"), "-lm"])
    return exe, d


@pytest.mark.parametrize("links", [4, 1])
def test_inverse_det_norm_bitwise(checker, links):
    exe, d = checker
    sc = M.SceneConfig(links=links, snakes=1)
    parts, *_ = build_scene_parts(sc, 1, with_wheels=links > 1)
    pos = parts["state"].particles.positions
    tets = parts["tetras"].tets
    x = pos[tets]
    D = np.ascontiguousarray(np.stack([x[:, 1] - x[:, 0], x[:, 2] - x[:, 0], x[:, 3] - x[:, 0]],
                                      axis=2))
    pairs = parts["distances"].pairs
    V = np.ascontiguousarray(pos[pairs[:, 0]] - pos[pairs[:, 1]])
    D.tofile(d / "D.bin")
    V.tofile(d / "V.bin")
    subprocess.check_call([exe, str(d / "D.bin"), str(d / "V.bin"), str(d / "o.bin"),
                           str(d / "n.bin")])
    o = np.fromfile(d / "o.bin").reshape(-1, 10)
    nrm = np.fromfile(d / "n.bin")
    inv = np.linalg.inv(D)
    det = np.linalg.det(D)
    assert np.array_equal(o[:, :9].reshape(-1, 3, 3), inv)
    assert np.array_equal(o[:, 9], det)
    assert np.array_equal(nrm, np.array([np.linalg.norm(v) for v in V]))
    # and what the builder stores: the reference's rest_inv / rest_volume / rest
    assert np.array_equal(o[:, :9].reshape(-1, 3, 3), parts["tetras"].rest_inv)
    assert np.array_equal(np.abs(o[:, 9]) / 6.0, parts["tetras"].rest_volume)
    assert np.array_equal(nrm, parts["distances"].rest)

"""Golden for system inspection: the reference's
Simulator.last_system() (solver.py:548-575; keep_matrix) after frame 0 of
the bend fixture (+8 psi) and of the snake (default gait).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nc \
        python tests/golden/make_golden_system.py

The CSR of A = J M^-1 J^T + reg is too large to commit, so system_{B,S}.npz
keep: A @ x for three seeded vectors, diag(A), the rhs, the shape and nnz,
and the row/column sums of |A|.
"""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import softsnake as R  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def capture(tag, model, cmd):
    sim = model.sim
    sim.config.keep_matrix = True
    sim.step(cmd, latency=True)
    sys_ = sim.last_system()
    A = sys_.matrix
    m = A.rows
    rng = np.random.default_rng(20260817)
    X = rng.normal(size=(3, m))
    AX = np.zeros_like(X)
    rows = np.repeat(np.arange(m), np.diff(A.row_offsets))
    for k in range(3):
        np.add.at(AX[k], rows, A.values * X[k][A.col_indices])
    diag = np.zeros(m)
    sel = rows == A.col_indices
    np.add.at(diag, rows[sel], A.values[sel])
    absrow = np.zeros(m)
    np.add.at(absrow, rows, np.abs(A.values))
    np.savez_compressed(os.path.join(OUT, f"system_{tag}.npz"), X=X, AX=AX, diag=diag,
                        rhs=sys_.rhs, shape=np.array([A.rows, A.cols]), nnz=np.int64(A.nnz),
                        absrow=absrow, commands=np.asarray(cmd, np.float64))
    print(tag, A.rows, A.nnz, os.path.getsize(os.path.join(OUT, f"system_{tag}.npz")))


def main():
    sc = R.SceneConfig()
    capture("B", R.build_bend_fixture(sc), np.array([8.0]))
    m = R.build_snake(sc)
    capture("S", m, m.commands(0.0))


if __name__ == "__main__":
    main()

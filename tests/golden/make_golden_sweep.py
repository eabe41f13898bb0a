"""Goldens for the batched curvature sweep from
the REFERENCE harness.

  sweep_B.npz        harness.run_curvature_sweep on a subset of levels
                     (settle <= 900 frames, 30 samples): the full protocol.
  sweep_B_short.npz  the same protocol restated from the reference's own
                     pieces (build_bend_fixture, harness._settle with
                     max_frames=10, 10 samples via the loop of
                     harness.py:121-128) for all 17 levels: a horizon short
                     enough to gate (with 60 + 30 frames the snapped
                     pressures already drive some levels chaotic: the
                     reference's numba and numpy backends differ by 6% at
                     +-5 psi).
  sweep_B_short_numpy.npz  the short protocol with the reference's numpy
                     backend: the reference's own backend-to-backend spread,
                     the noise floor the GPU tolerance is scaled from.
  sweep_B_chaos.npz  level +8 (full protocol) with the numpy backend: the
                     same spread at 930 frames.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nc \
        python tests/golden/make_golden_sweep.py [full|short|short_numpy|chaos]
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import softsnake as R  # noqa: E402
from softsnake import harness  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
LEVELS = [-8.0, -3.0, 0.0, 4.0, 8.0]


def full():
    rec = harness.run_curvature_sweep(R.SceneConfig(), pressures=LEVELS)
    rows = np.array(rec.rows, dtype=np.float64)  # tick time p mean std settled
    np.savez_compressed(os.path.join(OUT, "sweep_B.npz"), levels=np.array(LEVELS), rows=rows,
                        columns=np.array(rec.columns))


def short(max_frames=10, samples=10, backend="numba"):
    levels = [float(p) for p in range(-8, 9)]
    rows = []
    for level, p in enumerate(levels):
        model = R.build_bend_fixture(R.SceneConfig(backend=backend))
        cmd = np.array([p])
        settled = harness._settle(model, cmd, max_frames=max_frames)
        s = np.empty(samples)
        for k in range(samples):
            model.sim.step(cmd, latency=False)
            s[k] = model.link_curvature(0)
        rows.append([level, model.sim.state.time, p, s.mean(), s.std(), 1.0 if settled else 0.0])
    name = "sweep_B_short.npz" if backend == "numba" else f"sweep_B_short_{backend}.npz"
    np.savez_compressed(os.path.join(OUT, name), levels=np.array(levels),
                        rows=np.array(rows), max_frames=np.int64(max_frames),
                        samples=np.int64(samples))


def chaos():
    sc = R.SceneConfig(backend="numpy")
    rec = harness.run_curvature_sweep(sc, pressures=[8.0])
    np.savez_compressed(os.path.join(OUT, "sweep_B_chaos.npz"), rows=np.array(rec.rows, np.float64))


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "full"
    t = time.time()
    {"full": full, "short": short, "chaos": chaos,
     "short_numpy": lambda: short(backend="numpy")}[what]()
    print(what, f"{time.time() - t:.0f}s")

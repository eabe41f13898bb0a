"""Golden for the batched curvature sweep from the
REFERENCE harness: harness.run_curvature_sweep on the bend fixture for a
subset of the 17 levels (each level = fresh fixture, latency off, settle
<= 900 frames, then 30 samples).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nc \
        python tests/golden/make_golden_sweep.py      # ~5 min
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


def main():
    t = time.time()
    rec = harness.run_curvature_sweep(R.SceneConfig(), pressures=LEVELS)
    rows = np.array(rec.rows, dtype=np.float64)  # tick time p mean std settled
    print(f"{time.time() - t:.0f}s")
    print(rec.columns)
    print(rows)
    np.savez_compressed(os.path.join(OUT, "sweep_B.npz"), levels=np.array(LEVELS), rows=rows,
                        columns=np.array(rec.columns))


if __name__ == "__main__":
    main()

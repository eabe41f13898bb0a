"""Goldens for the CSV emit of the experiment records (harness.py:58-80,
SURVEY.md §8(f) row 2): bytes written by the REFERENCE's own emit_csv.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nc \
        python tests/golden/make_golden_csv.py

csv_format.csv   — a fixed record exercising every _fmt branch (bool, numpy
                   bool, int, numpy int, float, numpy float, str with comma
                   and quote) under the default SceneConfig preamble.
step_response.csv — run_step_response(SceneConfig(), targets=(0.6, 1.0),
                   hold_s=0.25): the bend fixture under the valve latency law.
locomote.csv     — run_locomotion(SceneConfig(), duration=10 frames).
"""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import softsnake as R  # noqa: E402
from softsnake import harness as H  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def format_record():
    sc = R.SceneConfig()
    rec = H.ExperimentRecord("format-check", sc.to_items(),
                             ["flag", "nflag", "count", "ncount", "x", "nx", "label"])
    rec.append(True, np.bool_(False), 7, np.int64(-3), 1.0 / 3.0, np.float64(2.5e-17), "a,b")
    rec.append(False, np.bool_(True), 0, np.int32(12), -123456789.987654321, np.float64(np.nan),
               'say "hi"')
    rec.append(1, np.int64(2 ** 40), -0.0, np.float64(1e300), float("inf"), 6894.76, "plain")
    return rec


def main():
    H.emit_csv(format_record(), os.path.join(OUT, "csv_format.csv"))
    sc = R.SceneConfig()
    H.run_step_response(sc, targets=(0.6, 1.0), hold_s=0.25,
                        out_path=os.path.join(OUT, "step_response.csv"))
    H.run_locomotion(sc, duration=10 * sc.dt, out_path=os.path.join(OUT, "locomote.csv"))
    print("wrote csv goldens")


if __name__ == "__main__":
    main()

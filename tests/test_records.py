"""Experiment records and CSV emit (harness.py:27-80, 99-263; SURVEY.md
§8(f) row 2) against CSV files written by the reference's own emit_csv
(tests/golden/make_golden_csv.py)."""
from __future__ import annotations

import csv
import io
import os

import numpy as np
import pytest

import paper_1904_02833_b200 as M
from paper_1904_02833_b200 import records

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name), encoding="utf-8") as f:
        return f.read()


def test_emit_csv_bytes_match_reference(tmp_path):
    sc = M.SceneConfig()
    rec = records.ExperimentRecord("format-check", sc.to_items(),
                                   ["flag", "nflag", "count", "ncount", "x", "nx", "label"])
    rec.append(True, np.bool_(False), 7, np.int64(-3), 1.0 / 3.0, np.float64(2.5e-17), "a,b")
    rec.append(False, np.bool_(True), 0, np.int32(12), -123456789.987654321, np.float64(np.nan),
               'say "hi"')
    rec.append(1, np.int64(2 ** 40), -0.0, np.float64(1e300), float("inf"), 6894.76, "plain")
    out = tmp_path / "f.csv"
    records.emit_csv(rec, str(out))
    assert out.read_bytes() == _gold("csv_format.csv").encode("utf-8")


def test_record_row_width_and_unwritable_path(tmp_path):
    rec = records.ExperimentRecord("x", [], ["a", "b"])
    with pytest.raises(ValueError):
        rec.append(1)
    with pytest.raises(OSError):
        records.emit_csv(rec, str(tmp_path / "missing" / "x.csv"))


def _parse(text):
    lines = text.splitlines()
    pre = [ln for ln in lines if ln.startswith("#")]
    body = [ln for ln in lines if not ln.startswith("#")]
    rows = list(csv.reader(io.StringIO("\n".join(body))))
    return pre, rows[0], rows[1:]


def _compare(got_text, want_text, exact_cols, close_cols, rtol):
    gp, gh, gr = _parse(got_text)
    wp, wh, wr = _parse(want_text)
    assert gp == wp and gh == wh and len(gr) == len(wr)
    for c in exact_cols:
        j = gh.index(c)
        assert [r[j] for r in gr] == [r[j] for r in wr], c
    for c in close_cols:
        j = gh.index(c)
        a = np.array([float(r[j]) for r in gr])
        b = np.array([float(r[j]) for r in wr])
        scale = max(float(np.max(np.abs(b))), 1e-30)
        assert np.max(np.abs(a - b)) <= rtol * scale, c


@pytest.mark.gpu
def test_step_response_csv_vs_reference(tmp_path):
    sc = M.SceneConfig()
    out = tmp_path / "sr.csv"
    records.run_step_response(sc, targets=(0.6, 1.0), hold_s=0.25, out_path=str(out))
    _compare(out.read_text(), _gold("step_response.csv"),
             ("tick", "time_s", "target_fraction", "phase", "pressure_psi", "strain"),
             ("curvature",), 1e-6)
    again = tmp_path / "sr2.csv"
    records.run_step_response(sc, targets=(0.6, 1.0), hold_s=0.25, out_path=str(again))
    assert again.read_bytes() == out.read_bytes()  # byte-identical re-run


@pytest.mark.gpu
def test_locomotion_csv_vs_reference(tmp_path):
    sc = M.SceneConfig()
    out = tmp_path / "lo.csv"
    records.run_locomotion(sc, duration=10 * sc.dt, out_path=str(out))
    press = [f"pressure_{i}" for i in range(8)]
    _compare(out.read_text(), _gold("locomote.csv"),
             ("tick", "time_s", "contacts", "pcr_iterations", "diverged", *press),
             ("com_x", "com_y", "com_z", "head_yaw", "path_xy", "curvature_0", "curvature_1",
              "curvature_2", "curvature_3"), 1e-6)
    again = tmp_path / "lo2.csv"
    records.run_locomotion(sc, duration=10 * sc.dt, out_path=str(again))
    assert again.read_bytes() == out.read_bytes()

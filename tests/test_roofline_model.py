"""The algorithmic byte model bench.py divides by kernel time
(paper_1904_02833_b200/roofline.py), checked on the snake's dimensions
 against hand counts: per-env bytes of the PCR
kernels, the once-per-launch topology term, and the SURVEY §8(d)
reference-layout model (1.83 GB per snake-step at ~294 contacts)."""
from paper_1904_02833_b200 import roofline as R

# config S: P=1456, nb=15, 1080 distances, 4320 tets, 48 attachments,
# 10 hinges, 10 wheels, 27,194 static rows
S = dict(P=1456, nb=15, nd=1080, nt=4320, na=48, nh=10, nw=10, ns=10 + 1456, ms=27194,
         ndof=3 * 1456 + 6 * 15)


def test_pcr_kernels_per_env():
    nc = 300.0
    rows = S["ms"] + 3 * nc
    # k_pcr_dir (structured): az, apd, d read + apd written; the setup launch
    # (one of 20) reads no apd
    dirb = R.bytes_per_launch_per_env("k_pcr_dir_rows", S, nc)
    assert abs(dirb - (8 * (4 - 1 / 20) * rows + 4 * S["ns"] + 16 * nc)) < 1e-6
    # the apply moves the compact J (10 doubles/tet), u, z in and az out
    app = R.bytes_per_launch_per_env("k_apply_rows2", S, nc)
    assert app > 8 * (10 * S["nt"] + 2 * rows)
    # aliases of the round-2 kernels move the same operands
    assert R.bytes_per_launch_per_env("k_apply_rows3", S, nc) == app
    assert R.bytes_per_launch_per_env("k_gather_bulk", S, nc) == \
        R.bytes_per_launch_per_env("k_gather", S, nc)


def test_topology_once_per_launch():
    # tet kernels: int32 indices (16 B), packed rest inverse (80 B), E_tet (24 B) per tet
    assert R.topology_bytes_per_launch("k_apply_rows2", S, 512) == \
        120 * S["nt"] + 16 * (S["nd"] + S["na"] + S["nh"])
    # one env of a large mesh also reads each tet vertex's incidence position
    assert R.topology_bytes_per_launch("k_tet_jt", S, 1) - \
        R.topology_bytes_per_launch("k_tet_jt", S, 512) == 16 * S["nt"]
    # row-vector kernels read no topology; the snake's is ~0.5 MB (L2-resident)
    assert R.topology_bytes_per_launch("k_pcr_step", S, 512) == 0.0
    assert R.topology_bytes_per_launch("k_apply_rows2", S, 512) < 0.6e6


def test_survey_reference_layout_model():
    m = R.survey_model(S, 294.0)
    assert 1.7e9 < m["total"] < 1.95e9  # 1.832 GB per snake-step
    assert m["env_private"] < m["total"] and m["shared"] > 0

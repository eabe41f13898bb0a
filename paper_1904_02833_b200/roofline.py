"""Algorithmic byte model of the step kernels (host-side accounting).

Bytes are the env-private traffic one launch must move per environment if
every operand is read once and every result written once (fp64 values,
int32 flags), plus (topology_bytes_per_launch) the scene topology the
launch reads once for all its envs — index arrays, rest-shape inverses,
E_tet, incidence lists: ~0.5 MB for the snake (L2-resident across the
envs of a batch, negligible), ~100-120 MB per tet kernel for the 1M-tet
mesh, where one env's launch streams it from HBM. Contact rows count
only for present contacts (absent slots are skipped by every kernel); `nc`
is the mean number of present contacts per substep. DESIGN.md §4 derives
each line; bench.py divides by the live CUDA-event duration.
"""
from __future__ import annotations

F8 = 8


def dims_of(sim) -> dict:
    sim._ensure()
    d = sim._packed.dims
    P, nb, nd, nt, na, nh, nw = (d[k] for k in ("P", "nb", "nd", "nt", "na", "nh", "nw"))
    ground = bool(sim.config.ground_enabled)
    nq = (d["ncp"] if not d["cp_all"] else P) if ground else 0
    nw = nw if ground else 0
    ms = nd + 6 * nt + 3 * na + 5 * nh
    return dict(P=P, nb=nb, nd=nd, nt=nt, na=na, nh=nh, nw=nw, ns=nw + nq, ms=ms,
                ndof=3 * P + 6 * nb)


def bytes_per_launch_per_env(kernel: str, d: dict, nc: float, structured: bool = True,
                             pcr: int = 20) -> float:
    """structured: the default tet-J mode. Its k_pcr_step keeps r = d z
    implicit, reads ap/d from k_pcr_dir and forms p = z + beta p itself, so
    k_pcr_dir moves 4 row vectors (3 on the setup launch) instead of 7, and
    k_pcr_step 7 on odd launches, 5 on even ones (x deferred to the next
    launch; 4 on the first launch of a solve) instead of 8. pcr: the
    PCR budget, for the per-launch average over one solve (pcr k_pcr_dir
    launches, pcr - 1 k_pcr_step launches)."""
    # round-2 kernels that move the same operands as their round-1 twins
    kernel = {"k_apply_rows2": "k_apply_rows", "k_apply_rows3": "k_apply_rows",
              "k_apply_rows_async": "k_apply_rows",
              "k_pcr_dir_rows": "k_pcr_dir", "k_newton_rhs2": "k_newton_rhs",
              "k_newton_final2": "k_newton_final", "k_gather_bulk": "k_gather"}.get(kernel, kernel)
    rows = d["ms"] + 3 * nc                      # rows a PCR kernel touches
    jc = F8 * 10 * d["nt"]                       # compact tet J: quat(4) S(6); R, K^-1 rebuilt
    tc = F8 * 12 * d["nt"]                       # tet column sums J^T x
    small_j = F8 * (3 * d["nd"] + 3 * d["na"] + 60 * d["nh"] + 18 * d["nw"])
    flags = 4 * d["ns"] + F8 * 2 * nc            # present flags, actf/dynn of present
    if kernel == "k_pcr_step":
        if structured:
            # odd launches: read x p z apd, write x z p; even launches defer x
            # (read p z apd, write z p); the first launch of a solve reads no p
            n = max(pcr - 1, 1)
            even, odd = (n + 1) // 2, n // 2
            return F8 * ((5 * even + 7 * odd - 1) / n) * rows + flags
        # read x p r ap d, write x r z
        return F8 * 8 * rows + flags
    if kernel == "k_tet_jt":
        # z of the tet rows, compact J; write tC
        return F8 * 6 * d["nt"] + jc + tc
    if kernel == "k_pcr_dir":
        if structured:
            # read az apd d, write apd (the setup launch reads no apd)
            return F8 * (4 - 1.0 / max(pcr, 1)) * rows + flags
        # read z az p ap d, write p ap
        return F8 * 7 * rows + flags
    if kernel == "k_apply_rows":
        # compact J, small-family J, u (once), z (own rows), write az
        return jc + small_j + F8 * d["ndof"] + F8 * 2 * rows + flags
    if kernel == "k_gather_fused":
        # z of every row of the particle families (tet z, dist, attach, contact
        # rows), compact J, dirs, flags; write u — no tC
        return F8 * 6 * d["nt"] + jc + F8 * (rows - 6 * d["nt"]) + small_j + \
            F8 * 9 * d["nb"] + flags + F8 * d["ndof"]
    if kernel == "k_gather":
        # tC once, non-tet x rows once, small-family J, ang_inv; write u
        return tc + F8 * (rows - 6 * d["nt"]) + small_j + F8 * 9 * d["nb"] + flags + \
            F8 * d["ndof"]
    if kernel == "k_newton_rhs":
        # compact J, v, res/lam/bdiag of rows, write r d z x, write tC
        return jc + small_j + F8 * d["ndof"] + F8 * 3 * rows + F8 * 4 * rows + tc + flags
    if kernel == "k_newton_final":
        # read x r z p ap d + lam, write lam + dlam, compact J, write tC
        return F8 * 9 * rows + jc + tc + flags
    if kernel == "k_eval_polar":
        # positions once, quats read and written (the polar loop alone)
        return F8 * (3 * d["P"] + 8 * d["nt"])
    if kernel == "k_eval_tet":
        # positions once, quats r/w, S + diag + tC written, lam read
        return F8 * (3 * d["P"] + 8 * d["nt"] + 6 * d["nt"] + 6 * d["nt"] + 12 * d["nt"]
                     + 6 * d["nt"])
    return 0.0


def survey_model(d: dict, nc: float, substeps: int = 2, newton: int = 4, pcr: int = 20) -> dict:
    """SURVEY.md §8(d) algorithmic bytes per snake-step in the reference's
    data layout (fp64 values, int32 indices, the 6x12 tet J stored and read
    twice per operator apply, the 6x6 E_tet block per tet):
      B_apply = 2 (8 Jnnz + 4 idx) + 8*36 T + 8 (4 m) + 8 (4 ndof) + 8*9 nb
      B_vec   = 8*11 m
      frame   = substeps [newton (21 (B_apply + B_vec) + 2 Jpass + 6 m-vectors) + 3 Jpass]
    with Jpass = 8 Jnnz + 4 idx. Shared by identical envs: the index arrays
    and E_tet; the rest is env-private. (The 21 applies are pcr + 1.)"""
    nt, nd, na, nh = d["nt"], d["nd"], d["na"], d["nh"]
    m = d["ms"] + 3 * nc
    jnnz = 6 * nd + 72 * nt + 27 * na + 60 * nh + 18 * nc
    idx = 6 * nd + 12 * nt + 9 * na + 12 * nh + 6 * nc
    b_apply = 2 * (F8 * jnnz + 4 * idx) + F8 * 36 * nt + F8 * 4 * m + F8 * 4 * d["ndof"] + \
        F8 * 9 * d["nb"]
    b_vec = F8 * 11 * m
    jpass = F8 * jnnz + 4 * idx
    applies = pcr + 1
    total = substeps * (newton * (applies * (b_apply + b_vec) + 2 * jpass + 6 * F8 * m) + 3 * jpass)
    sh_apply = 2 * 4 * idx + F8 * 36 * nt
    shared = substeps * (newton * (applies * sh_apply + 2 * 4 * idx) + 3 * 4 * idx)
    return {"total": float(total), "shared": float(shared), "env_private": float(total - shared)}


def topology_bytes_per_launch(kernel: str, d: dict, envs_per_launch: int = 1) -> float:
    """Scene topology one launch must read once (shared by all its envs):
    int32 tet indices (16 B/tet), the packed rest inverse (80 B/tet), E_tet
    (24 B/tet), family index / compliance arrays, incidence lists (4 B per
    incidence + 20 B per particle). One env of a large mesh also reads the
    incidence destination of each tet vertex in k_tet_jt (16 B/tet)."""
    kernel = {"k_apply_rows2": "k_apply_rows", "k_apply_rows3": "k_apply_rows",
              "k_apply_rows_async": "k_apply_rows", "k_newton_rhs2": "k_newton_rhs",
              "k_newton_final2": "k_newton_final", "k_gather_bulk": "k_gather",
              "k_pcr_dir_rows": "k_pcr_dir"}.get(kernel, kernel)
    nt, nd, na, nh, P, ns = d["nt"], d["nd"], d["na"], d["nh"], d["P"], d["ns"]
    small = 16 * nd + 16 * na + 16 * nh
    if kernel in ("k_apply_rows", "k_newton_rhs", "k_eval_tet"):
        return float((16 + 80 + 24) * nt + small)
    if kernel == "k_newton_final":
        return float((80 + 24) * nt + small)
    if kernel == "k_tet_jt":
        return float((80 + (16 if envs_per_launch == 1 else 0)) * nt)
    if kernel == "k_eval_polar":
        return float((16 + 80) * nt)
    if kernel == "k_gather":
        n_inc = 4 * nt + 2 * nd + 2 * na + 2 * nh + 2 * ns
        return float(4 * n_inc + 20 * P)
    return 0.0

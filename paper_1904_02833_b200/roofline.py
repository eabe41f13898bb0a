"""Algorithmic byte model of the step kernels (host-side accounting).

Bytes are the env-private traffic one launch must move per environment if
every operand is read once and every result written once (fp64 values,
int32 flags), with the scene topology (index arrays, rest-shape inverses,
incidence lists) excluded: it is shared by all environments of a batch and
stays L2-resident. These are the figures bench.py's `roofline.achieved`
divides by the live CUDA-event duration; DESIGN.md derives them.
"""
from __future__ import annotations


def dims_of(sim) -> dict:
    d = sim._packed.dims if sim._packed is not None else None
    if d is None:
        sim._ensure()
        d = sim._packed.dims
    P, nb, nd, nt, na, nh, nw = (d[k] for k in ("P", "nb", "nd", "nt", "na", "nh", "nw"))
    ground = bool(sim.config.ground_enabled)
    nq = (d["ncp"] if not d["cp_all"] else P) if ground else 0
    nw = nw if ground else 0
    ns = nw + nq
    ms = nd + 6 * nt + 3 * na + 5 * nh
    return dict(P=P, nb=nb, nd=nd, nt=nt, na=na, nh=nh, nw=nw, ns=ns, ms=ms, m=ms + 3 * ns,
                ndof=3 * P + 6 * nb)


def bytes_per_launch_per_env(kernel: str, d: dict) -> int:
    f8 = 8
    J = f8 * (72 * d["nt"] + 3 * d["nd"] + 3 * d["na"] + 60 * d["nh"] + 18 * d["nw"])
    flags = 4 * d["ns"]
    if kernel == "k_gather":
        # J once, x rows once, ang_inv, contact flags; u (or v) written once
        return J + f8 * d["m"] + f8 * 9 * d["nb"] + flags + f8 * d["ns"] + f8 * d["ndof"]
    if kernel == "k_apply_rows":
        # J once, u once, z once, dyn/act of contacts; az written once
        return J + f8 * d["ndof"] + f8 * d["m"] + flags + 2 * f8 * d["ns"] + f8 * d["m"]
    if kernel == "k_pcr_dir":
        return f8 * 7 * d["m"]     # read z az p ap d, write p ap
    if kernel == "k_pcr_step":
        return f8 * 8 * d["m"]     # read x p r ap d, write x r z
    if kernel == "k_newton_rhs":
        # J once, v once, res/lam/bdiag once; write r d z x
        return J + f8 * d["ndof"] + 3 * f8 * d["m"] + 4 * f8 * d["m"] + flags
    if kernel == "k_eval_tet":
        # positions once, quats read+write, J + res + diag written
        return f8 * (3 * d["P"] + 8 * d["nt"] + 72 * d["nt"] + 12 * d["nt"])
    return 0

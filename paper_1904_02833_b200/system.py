"""System inspection: the explicit Newton system of
the last substep, A = J M^-1 J^T + reg, as CSR plus its right-hand side —
Simulator.last_system / export_system (solver.py:548-581) and the Matrix
Market writers (sparse.py:190-207).

The device keeps the snapshot (ss_params.keep_matrix) and hands it over in
the reference's block layout (ss_export_system); the sparse products here
are host-side scipy (off the step path).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native
from ._abi import SsSystemView


@dataclass
class CsrMatrix:
    """sparse.py:99-110 field names."""
    row_offsets: np.ndarray
    col_indices: np.ndarray
    values: np.ndarray
    rows: int
    cols: int

    @property
    def nnz(self) -> int:
        return int(self.col_indices.shape[0])

    @classmethod
    def from_scipy(cls, A) -> "CsrMatrix":
        A = A.tocsr()
        A.sort_indices()
        return cls(A.indptr.astype(np.int64), A.indices.astype(np.int32),
                   A.data.astype(np.float64), A.shape[0], A.shape[1])

    def to_scipy(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.values, self.col_indices, self.row_offsets),
                             shape=(self.rows, self.cols))

    def matvec(self, x: np.ndarray) -> np.ndarray:
        return self.to_scipy() @ np.asarray(x, np.float64)


@dataclass
class SchurSystem:
    """solver.py:129-132: A and the Newton right-hand side."""
    matrix: CsrMatrix
    rhs: np.ndarray


def export_blocks(sim, env: int = 0) -> dict:
    """ss_export_system for one env: the snapshot's blocks as numpy arrays."""
    d = sim._packed.dims
    nd, nt, na, nh, nb = d["nd"], d["nt"], d["na"], d["nh"], d["nb"]
    ns = int(d["nw"]) + int(d["ncp"] if not d["cp_all"] else d["P"])
    ms = nd + 6 * nt + 3 * na + 5 * nh
    ndof = 3 * d["P"] + 6 * nb
    out = {
        "dist_vals": np.zeros((nd, 1, 6)), "dist_idx": np.zeros((nd, 6), np.int32),
        "tet_vals": np.zeros((nt, 6, 12)), "tet_idx": np.zeros((nt, 12), np.int32),
        "att_vals": np.zeros((na, 3, 9)), "att_idx": np.zeros((na, 9), np.int32),
        "hinge_vals": np.zeros((nh, 5, 12)), "hinge_idx": np.zeros((nh, 12), np.int32),
        "slot_vals": np.zeros((ns, 3, 6)), "slot_idx": np.zeros((ns, 6), np.int32),
        "slot_present": np.zeros(ns, np.int32), "rhs_static": np.zeros(ms),
        "dyn_static": np.zeros(ms), "rhs_slot": np.zeros((ns, 3)), "dyn_slot": np.zeros((ns, 3)),
        "minv_diag": np.zeros(ndof), "ang_inv": np.zeros((nb, 3, 3)),
    }
    v = SsSystemView()
    for name, a in out.items():
        kind = C.POINTER(C.c_double) if a.dtype == np.float64 else C.POINTER(C.c_int32)
        setattr(v, name, a.ctypes.data_as(kind) if a.size else C.cast(None, kind))
    _native.check(_native.lib().ss_export_system(sim._ensure(), int(env), C.byref(v)))
    out["bd0"] = 3 * d["P"]
    return out


def assemble(blocks: dict, eh2: np.ndarray | None) -> SchurSystem:
    """Simulator.last_system (solver.py:548-575): J from the family blocks
    (static families, then the present contacts' normal rows, then their
    friction row pairs), M^-1 (state.py:223-243), reg = diag(dyn) + the
    E_tet 6x6 blocks; A = J M^-1 J^T + reg."""
    import scipy.sparse as sp
    b = blocks
    nd, nt, na, nh = (b["dist_idx"].shape[0], b["tet_idx"].shape[0], b["att_idx"].shape[0],
                      b["hinge_idx"].shape[0])
    ms = b["rhs_static"].size
    pres = np.flatnonzero(b["slot_present"])
    nc = pres.size
    m = ms + 3 * nc
    ndof = b["minv_diag"].size
    cdof = b["slot_idx"][pres]
    nvals = b["slot_vals"][pres][:, 0:1, :]
    fvals = b["slot_vals"][pres][:, 1:3, :]
    fams = [(b["dist_idx"], b["dist_vals"], 0), (b["tet_idx"], b["tet_vals"], nd),
            (b["att_idx"], b["att_vals"], nd + 6 * nt),
            (b["hinge_idx"], b["hinge_vals"], nd + 6 * nt + 3 * na),
            (cdof, nvals, ms), (cdof, fvals, ms + nc)]
    rows, cols, vals = [], [], []
    for idx, bv, off in fams:
        n, r, k = bv.shape
        if n == 0:
            continue
        rows.append(np.repeat(off + np.arange(n * r), k))
        cols.append(np.broadcast_to(idx[:, None, :], (n, r, k)).ravel())
        vals.append(bv.ravel())
    J = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(m, ndof)).tocsr()
    bd0 = int(b["bd0"])
    nb = b["ang_inv"].shape[0]
    mr = list(range(bd0))
    mc = list(range(bd0))
    mv = list(b["minv_diag"][:bd0])
    for bi in range(nb):
        o = bd0 + 6 * bi
        for i in range(3):
            mr.append(o + i)
            mc.append(o + i)
            mv.append(b["minv_diag"][o + i])
        for i in range(3):
            for j in range(3):
                mr.append(o + 3 + i)
                mc.append(o + 3 + j)
                mv.append(b["ang_inv"][bi, i, j])
    Minv = sp.coo_matrix((mv, (mr, mc)), shape=(ndof, ndof)).tocsr()
    dyn = np.concatenate([b["dyn_static"], b["dyn_slot"][pres, 0], b["dyn_slot"][pres, 1:].ravel()])
    rr, cc, vv = [np.arange(m)], [np.arange(m)], [dyn]
    if nt and eh2 is not None:
        base = nd + 6 * np.arange(nt)
        rr.append(np.repeat(base, 36) + np.tile(np.repeat(np.arange(6), 6), nt))
        cc.append(np.repeat(base, 36) + np.tile(np.tile(np.arange(6), 6), nt))
        vv.append(np.asarray(eh2, np.float64).ravel())
    reg = sp.coo_matrix((np.concatenate(vv), (np.concatenate(rr), np.concatenate(cc))),
                        shape=(m, m)).tocsr()
    A = (J @ Minv @ J.T + reg).tocsr()
    rhs = np.concatenate([b["rhs_static"], b["rhs_slot"][pres, 0], b["rhs_slot"][pres, 1:].ravel()])
    return SchurSystem(CsrMatrix.from_scipy(A), rhs)


def mmwrite(path, A: CsrMatrix) -> None:
    """Matrix Market coordinate, 1-based, real general (sparse.py:190-197)."""
    with open(path, "w") as f:
        f.write("%%MatrixMarket matrix coordinate real general\n")
        f.write(f"{A.rows} {A.cols} {A.nnz}\n")
        rows = np.repeat(np.arange(A.rows), np.diff(A.row_offsets)) + 1
        for i, j, x in zip(rows, A.col_indices + 1, A.values):
            f.write(f"{i} {j} {x:.17g}\n")


def mmwrite_dense(path, v: np.ndarray) -> None:
    """Matrix Market array for a dense vector (sparse.py:200-207)."""
    v = np.asarray(v, np.float64).ravel()
    with open(path, "w") as f:
        f.write("%%MatrixMarket matrix array real general\n")
        f.write(f"{v.size} 1\n")
        for x in v:
            f.write(f"{x:.17g}\n")

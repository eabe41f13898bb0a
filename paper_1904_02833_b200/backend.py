"""The "cuda" kernel backend: the reference's backend plugin interface
(softsnake/kernels/__init__.py:24-41, numba_backend.py) on the B200.

Same names, signatures and semantics as numba_backend: caller-owned numpy
arrays, outputs written in place, block kernels bitwise equal to numba's.
Each call moves its arrays to the device and back (kernel-level parity and
drop-in use on a reference Simulator via `sim.kern = backend`); the batched
step never goes through here — it runs the fused kernels of the handle.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native

NAME = "cuda"
COMPILED = True


class _Dev:
    """Device copy of a numpy array for the duration of one call."""

    def __init__(self, a: np.ndarray):
        self.a = a
        self.nbytes = int(a.nbytes)
        self.ptr = C.c_void_p()
        _native.check(_native.lib().ssk_malloc(C.byref(self.ptr), max(self.nbytes, 8), 0))
        if self.nbytes:
            _native.check(_native.lib().ssk_memcpy(self.ptr, a.ctypes.data_as(C.c_void_p),
                                                   self.nbytes, 1))

    def download(self):
        if self.nbytes:
            _native.check(_native.lib().ssk_memcpy(self.a.ctypes.data_as(C.c_void_p), self.ptr,
                                                   self.nbytes, 2))

    def free(self):
        if self.ptr:
            _native.lib().ssk_free(self.ptr)
            self.ptr = C.c_void_p()


def _call(fn, ins, outs):
    for a in outs:
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("output arrays must be C-contiguous (numpy_backend.py:4-7)")
    din = [_Dev(np.ascontiguousarray(a)) for a in ins]
    dout = [_Dev(a) for a in outs]
    try:
        _native.check(fn([d.ptr for d in din], [d.ptr for d in dout]))
        for d in dout:
            d.download()
    finally:
        for d in din + dout:
            d.free()


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def block_forward(dof_idx, vals, u, out_rows):
    n, r, k = vals.shape
    L = _native.lib()
    _call(lambda i, o: L.ssk_block_forward(i[0], i[1], n, r, k, i[2], o[0], None),
          [_i32(dof_idx), _f64(vals), _f64(u)], [out_rows])
    return out_rows


def block_transpose(dof_idx, vals, x_rows, y):
    n, r, k = vals.shape
    L = _native.lib()
    _call(lambda i, o: L.ssk_block_transpose(i[0], i[1], n, r, k, i[2], o[0], y.shape[0], None),
          [_i32(dof_idx), _f64(vals), _f64(x_rows)], [y])
    return y


def block_rowdiag(dof_idx, vals, minv_diag, out_rows):
    n, r, k = vals.shape
    L = _native.lib()
    _call(lambda i, o: L.ssk_block_rowdiag(i[0], i[1], n, r, k, i[2], o[0], None),
          [_i32(dof_idx), _f64(vals), _f64(minv_diag)], [out_rows])
    return out_rows


def minv_apply(minv_diag, ang_inv, body_dof0, u, out):
    L = _native.lib()
    nb = ang_inv.shape[0]
    _call(lambda i, o: L.ssk_minv_apply(i[0], i[1], nb, int(body_dof0), i[2], o[0],
                                        u.shape[0], None),
          [_f64(minv_diag), _f64(ang_inv), _f64(u)], [out])
    return out


def ereg_apply(vals6, x_rows, out_rows):
    L = _native.lib()
    n = vals6.shape[0]
    _call(lambda i, o: L.ssk_ereg_apply(i[0], i[1], o[0], n, None),
          [_f64(vals6), _f64(x_rows)], [out_rows])
    return out_rows


def dot(a, b):
    L = _native.lib()
    res = C.c_double(0.0)
    _call(lambda i, o: L.ssk_dot(i[0], i[1], a.shape[0], C.byref(res), None),
          [_f64(a), _f64(b)], [])
    return float(res.value)


def csr_spmv(indptr, indices, data, x, out):
    """Off the step path (sparse.py inspection only)."""
    raise NotImplementedError("csr_spmv is outside the B200 hot path (sparse.py inspection)")


def eval_distance(pos, pairs, rest, scale, dirs, out_res):
    L = _native.lib()
    n = pairs.shape[0]
    _call(lambda i, o: L.ssk_eval_distance(i[0], i[1], i[2], i[3], o[0], o[1], n, None),
          [_f64(pos), _i32(pairs), _f64(rest), _f64(scale)], [dirs, out_res])
    return out_res


def eval_tetra(pos, tets, rest_inv, quats, tol, maxiter, out_res, out_vals):
    L = _native.lib()
    n = tets.shape[0]
    ninv = C.c_int(0)
    _call(lambda i, o: L.ssk_eval_tetra(i[0], i[1], i[2], o[0], float(tol), int(maxiter), o[1],
                                        o[2], n, C.byref(ninv), None),
          [_f64(pos), _i32(tets), _f64(rest_inv)], [quats, out_res, out_vals])
    return int(ninv.value)

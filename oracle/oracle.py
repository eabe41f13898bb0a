"""ctypes wrapper of liboracle.so — TEST INFRASTRUCTURE ONLY.

OracleSim steps ONE environment on the CPU with the reference algorithm
(oracle/softsnake_oracle.c restates softsnake/solver.py:296-544). The
state dict uses the reference shapes (field names of ss_state_view).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_1904_02833_b200._abi import (STATE_FIELDS, PackedTopology, SsEnvStats,
                                        SsParams, SsTopology, StateBuffers,
                                        pack_params)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    src = os.path.join(HERE, "softsnake_oracle.c")
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", HERE, "-B", "liboracle.so"])
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        vp, dp, ip, i = C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int32), C.c_int
        L.or_create.restype = vp
        L.or_create.argtypes = [C.POINTER(SsTopology), C.POINTER(SsParams)]
        L.or_destroy.argtypes = [vp]
        L.or_set_state.argtypes = [vp, vp]
        L.or_get_state.argtypes = [vp, vp]
        L.or_get_stats.argtypes = [vp, C.POINTER(SsEnvStats)]
        L.or_step.argtypes = [vp, dp, i]
        L.or_run.argtypes = [vp, dp, i, i]
        for n, args in (("or_block_forward", [ip, dp, i, i, i, dp, dp]),
                        ("or_block_transpose", [ip, dp, i, i, i, dp, dp]),
                        ("or_block_rowdiag", [ip, dp, i, i, i, dp, dp]),
                        ("or_minv_apply", [dp, dp, i, i, dp, dp, i]),
                        ("or_ereg_apply", [dp, dp, dp, i]),
                        ("or_eval_distance", [dp, ip, dp, dp, dp, dp, i]),
                        ("or_eval_tetra", [dp, ip, dp, dp, C.c_double, i, dp, dp, i, ip])):
            getattr(L, n).argtypes = args
        L.or_eval_tetra.restype = C.c_int
        L.or_update_pressure.restype = C.c_double
        L.or_update_pressure.argtypes = [C.c_double] * 6
        _lib = L
    return _lib


def _p(a, kind=C.c_double):
    return a.ctypes.data_as(C.POINTER(kind))


class OracleSim:
    """One environment of a scene, stepped by the C oracle."""

    def __init__(self, state, config, distances=None, tetras=None, attachments=None,
                 hinges=None, wheels=None, channels=None, strain=None,
                 contact_particles=None):
        self.packed = PackedTopology(state, distances, tetras, attachments, hinges, wheels,
                                     channels, strain, contact_particles)
        self.params = pack_params(config, self.packed)
        self.dims = self.packed.dims
        self.h = lib().or_create(C.byref(self.packed.struct), C.byref(self.params))
        self.links = self.dims["nch"] // 2
        # reference constructor state: the containers' arrays (solver.py:166-255)
        st = state
        init = {"positions": st.particles.positions, "velocities": st.particles.velocities,
                "body_pos": st.body_pos, "body_quat": st.body_quat,
                "body_lin_vel": st.body_lin_vel, "body_ang_vel": st.body_ang_vel,
                "time": np.float64(st.time)}
        if tetras is not None:
            init["tet_quats"] = tetras.quats
        if distances is not None:
            init["dist_dirs"] = distances.dirs
            init["dist_scale"] = distances.scale
        if channels is not None:
            init["pressures"] = np.asarray(channels.pressures)
        self.set_state(init)

    @classmethod
    def from_sim(cls, sim):
        """Same scene as a (B200 or reference) Simulator-like object."""
        return cls(sim.state, sim.config, sim.distances, sim.tetras, sim.attachments,
                   sim.hinges, sim.wheels, sim.channels, sim.strain, sim.contact_particles)

    def __del__(self):
        try:
            lib().or_destroy(self.h)
        except Exception:
            pass

    def set_state(self, arrays: dict) -> None:
        buf = StateBuffers(self.dims, 1)
        names = [n for n, _, _ in STATE_FIELDS if n in arrays]
        for n in names:
            buf.arrays[n][0] = np.asarray(arrays[n]).reshape(buf.arrays[n].shape[1:])
        v = buf.view(names)
        lib().or_set_state(self.h, C.byref(v))

    def get_state(self) -> dict:
        buf = StateBuffers(self.dims, 1)
        v = buf.view()
        lib().or_get_state(self.h, C.byref(v))
        return {k: a[0] for k, a in buf.arrays.items()}

    def step(self, commands=None, latency: bool = True) -> None:
        if commands is None:
            lib().or_step(self.h, None, 1 if latency else 0)
        else:
            c = np.ascontiguousarray(np.asarray(commands, np.float64).reshape(self.links))
            lib().or_step(self.h, _p(c), 1 if latency else 0)

    def run(self, commands, latency: bool = True) -> None:
        c = np.ascontiguousarray(np.asarray(commands, np.float64))
        frames = c.size // max(self.links, 1)
        lib().or_run(self.h, _p(c), 1 if latency else 0, frames)

    def stats(self) -> SsEnvStats:
        s = SsEnvStats()
        lib().or_get_stats(self.h, C.byref(s))
        return s


# ---- per-kernel functions with the reference backend signatures ----------
def block_forward(dof_idx, vals, u, out_rows):
    n, r, k = vals.shape
    lib().or_block_forward(_p(dof_idx, C.c_int32), _p(vals), n, r, k, _p(u), _p(out_rows))
    return out_rows


def block_transpose(dof_idx, vals, x_rows, y):
    n, r, k = vals.shape
    lib().or_block_transpose(_p(dof_idx, C.c_int32), _p(vals), n, r, k, _p(x_rows), _p(y))
    return y


def block_rowdiag(dof_idx, vals, minv_diag, out_rows):
    n, r, k = vals.shape
    lib().or_block_rowdiag(_p(dof_idx, C.c_int32), _p(vals), n, r, k, _p(minv_diag), _p(out_rows))
    return out_rows


def minv_apply(minv_diag, ang_inv, body_dof0, u, out):
    lib().or_minv_apply(_p(minv_diag), _p(ang_inv), ang_inv.shape[0], body_dof0, _p(u), _p(out),
                        u.shape[0])
    return out


def ereg_apply(vals6, x_rows, out_rows):
    lib().or_ereg_apply(_p(vals6), _p(x_rows), _p(out_rows), vals6.shape[0])
    return out_rows


def eval_distance(pos, pairs, rest, scale, dirs, out_res):
    lib().or_eval_distance(_p(pos), _p(pairs, C.c_int32), _p(rest), _p(scale), _p(dirs),
                           _p(out_res), pairs.shape[0])
    return out_res


def eval_tetra(pos, tets, rest_inv, quats, tol, maxiter, out_res, out_vals, iters=None):
    it = iters if iters is not None else np.zeros(tets.shape[0], np.int32)
    return lib().or_eval_tetra(_p(pos), _p(tets, C.c_int32), _p(rest_inv), _p(quats),
                               float(tol), int(maxiter), _p(out_res), _p(out_vals),
                               tets.shape[0], _p(it, C.c_int32))


def update_pressure(p, target, k_i=0.23, k_d=0.23, cap=0.68, p_s=8.0):
    return lib().or_update_pressure(p, target, k_i, k_d, cap, p_s)

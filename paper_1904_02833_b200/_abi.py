"""ctypes mirror of include/softsnake_b200.h plus packers.

The packers turn the reference-shaped host containers (ours or the
reference's own, duck-typed) into the flat arrays the C ABI takes. The
arrays are kept alive on the returned object for as long as the struct
is in use.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)


class SsTopology(C.Structure):
    _fields_ = [
        ("num_particles", C.c_int32), ("num_bodies", C.c_int32),
        ("inv_mass", _dp), ("body_mass", _dp), ("body_inertia", _dp),
        ("n_dist", C.c_int32), ("dist_pairs", _ip), ("dist_rest", _dp),
        ("dist_compliance", _dp), ("dist_channel", _ip),
        ("n_tet", C.c_int32), ("tets", _ip), ("tet_rest_inv", _dp),
        ("tet_compliance", _dp),
        ("n_attach", C.c_int32), ("attach_particle", _ip), ("attach_body", _ip),
        ("attach_anchor", _dp), ("attach_compliance", _dp),
        ("n_hinge", C.c_int32), ("hinge_body_a", _ip), ("hinge_body_b", _ip),
        ("hinge_anchor_a", _dp), ("hinge_anchor_b", _dp), ("hinge_axis_a", _dp),
        ("hinge_tan1_b", _dp), ("hinge_tan2_b", _dp), ("hinge_compliance", _dp),
        ("n_wheel", C.c_int32), ("wheel_body", _ip), ("wheel_radius", _dp),
        ("wheel_axis", _dp),
        ("n_contact_particles", C.c_int32), ("contact_particles", _ip),
        ("n_channels", C.c_int32), ("has_strain", C.c_int32),
    ]


class SsParams(C.Structure):
    _fields_ = [
        ("dt", C.c_double), ("substeps", C.c_int32), ("newton_iters", C.c_int32),
        ("pcr_iters", C.c_int32), ("gravity", C.c_double * 3),
        ("ground_height", C.c_double), ("ground_enabled", C.c_int32),
        ("contact_margin", C.c_double), ("mu", C.c_double),
        ("friction_compliance", C.c_double), ("fb_delta", C.c_double),
        ("fb_slope_min", C.c_double), ("fb_slope_max", C.c_double),
        ("max_strain_rate", C.c_double), ("constraint_damping", C.c_double),
        ("strain_youngs", C.c_double), ("k_inflate", C.c_double),
        ("k_deflate", C.c_double), ("deflate_cap", C.c_double), ("supply", C.c_double),
        ("exact_jacobian", C.c_int32), ("solver_mode", C.c_int32), ("wave_envs", C.c_int32),
        ("keep_matrix", C.c_int32),
    ]


STATE_FIELDS = (
    # name, per-env shape builder, dtype
    ("positions", lambda d: (d["P"], 3), np.float64),
    ("velocities", lambda d: (d["P"], 3), np.float64),
    ("body_pos", lambda d: (d["nb"], 3), np.float64),
    ("body_quat", lambda d: (d["nb"], 4), np.float64),
    ("body_lin_vel", lambda d: (d["nb"], 3), np.float64),
    ("body_ang_vel", lambda d: (d["nb"], 3), np.float64),
    ("lam_dist", lambda d: (d["nd"],), np.float64),
    ("lam_tetra", lambda d: (d["nt"], 6), np.float64),
    ("lam_attach", lambda d: (d["na"], 3), np.float64),
    ("lam_hinge", lambda d: (d["nh"], 5), np.float64),
    ("tet_quats", lambda d: (d["nt"], 4), np.float64),
    ("dist_dirs", lambda d: (d["nd"], 3), np.float64),
    ("dist_scale", lambda d: (d["nd"],), np.float64),
    ("strain_live", lambda d: (d["nch"],), np.float64),
    ("strain_target", lambda d: (d["nch"],), np.float64),
    ("pressures", lambda d: (d["nch"],), np.float64),
    ("warm", lambda d: (d["nw"], 3), np.float64),
    ("warm_valid", lambda d: (d["nw"],), np.int32),
    ("time", lambda d: (), np.float64),
)


class SsStateView(C.Structure):
    _fields_ = [(name, _ip if dt == np.int32 else _dp) for name, _, dt in STATE_FIELDS]


class SsEnvStats(C.Structure):
    _fields_ = [
        ("newton_iterations", C.c_int32), ("pcr_iterations", C.c_int32),
        ("contact_count", C.c_int32), ("inverted_tets", C.c_int32),
        ("residual", C.c_double), ("finite", C.c_int32), ("_pad", C.c_int32),
    ]


class SsSystemView(C.Structure):
    """ss_system_view (include/softsnake_b200.h)."""
    _fields_ = [(n, C.POINTER(C.c_double) if t == "d" else C.POINTER(C.c_int32)) for n, t in (
        ("dist_vals", "d"), ("dist_idx", "i"), ("tet_vals", "d"), ("tet_idx", "i"),
        ("att_vals", "d"), ("att_idx", "i"), ("hinge_vals", "d"), ("hinge_idx", "i"),
        ("slot_vals", "d"), ("slot_idx", "i"), ("slot_present", "i"), ("rhs_static", "d"),
        ("dyn_static", "d"), ("rhs_slot", "d"), ("dyn_slot", "d"), ("minv_diag", "d"),
        ("ang_inv", "d"))]


class SsLinkMeshParams(C.Structure):
    """ss_link_mesh_params (include/softsnake_b200.h)."""
    _fields_ = [
        ("sections", C.c_int32), ("width_nodes", C.c_int32), ("height_nodes", C.c_int32),
        ("n_links", C.c_int32), ("dx", C.c_double), ("dy", C.c_double), ("dz", C.c_double),
        ("half_width", C.c_double), ("youngs_modulus", C.c_double), ("poisson", C.c_double),
        ("density", C.c_double), ("actuation_compliance", C.c_double),
        ("inextensible_compliance", C.c_double), ("structural_compliance", C.c_double),
        ("origins", _dp), ("channels", _ip),
    ]


class SsLinkMeshOut(C.Structure):
    """ss_link_mesh_out (include/softsnake_b200.h)."""
    _fields_ = [(n, C.POINTER(C.c_double) if t == "d" else C.POINTER(C.c_int32)) for n, t in (
        ("positions", "d"), ("masses", "d"), ("tets", "i"), ("rest_inv", "d"),
        ("rest_volume", "d"), ("compliance", "d"), ("pairs", "i"), ("rest", "d"),
        ("cable_compliance", "d"), ("kind", "i"), ("channel", "i"), ("mounts", "i"))]


def _ptr(a: np.ndarray | None, kind):
    if a is None or a.size == 0:
        return C.cast(None, kind)
    return a.ctypes.data_as(kind)


def _f64(a, shape=None):
    out = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return out if shape is None else out.reshape(shape)


def _i32(a, shape=None):
    out = np.ascontiguousarray(np.asarray(a, dtype=np.int32))
    return out if shape is None else out.reshape(shape)


class PackedTopology:
    """Flat ss_topology arrays for one scene (held alive here)."""

    def __init__(self, state, distances=None, tetras=None, attachments=None,
                 hinges=None, wheels=None, channels=None, strain=None,
                 contact_particles=None):
        P = int(state.particles.positions.shape[0])
        nb = int(state.body_pos.shape[0])
        self.keep = {}
        k = self.keep
        k["inv_mass"] = _f64(state.particles.inv_mass, (P,))
        k["body_mass"] = _f64(state.body_mass, (nb,))
        k["body_inertia"] = _f64(state.body_inertia, (nb, 3, 3))
        nd = int(distances.pairs.shape[0]) if distances is not None else 0
        if nd:
            k["dist_pairs"] = _i32(distances.pairs, (nd, 2))
            k["dist_rest"] = _f64(distances.rest, (nd,))
            k["dist_compliance"] = _f64(distances.compliance, (nd,))
            k["dist_channel"] = _i32(distances.channel, (nd,))
        nt = int(tetras.tets.shape[0]) if tetras is not None else 0
        if nt:
            k["tets"] = _i32(tetras.tets, (nt, 4))
            k["tet_rest_inv"] = _f64(tetras.rest_inv, (nt, 3, 3))
            k["tet_compliance"] = _f64(tetras.compliance, (nt, 6, 6))
        na = int(attachments.particle.shape[0]) if attachments is not None else 0
        if na:
            k["attach_particle"] = _i32(attachments.particle, (na,))
            k["attach_body"] = _i32(attachments.body, (na,))
            k["attach_anchor"] = _f64(attachments.local_anchor, (na, 3))
            k["attach_compliance"] = _f64(attachments.compliance, (na,))
        nh = int(hinges.body_a.shape[0]) if hinges is not None else 0
        if nh:
            k["hinge_body_a"] = _i32(hinges.body_a, (nh,))
            k["hinge_body_b"] = _i32(hinges.body_b, (nh,))
            k["hinge_anchor_a"] = _f64(hinges.anchor_a, (nh, 3))
            k["hinge_anchor_b"] = _f64(hinges.anchor_b, (nh, 3))
            k["hinge_axis_a"] = _f64(hinges.axis_a, (nh, 3))
            k["hinge_tan1_b"] = _f64(hinges.tan1_b, (nh, 3))
            k["hinge_tan2_b"] = _f64(hinges.tan2_b, (nh, 3))
            k["hinge_compliance"] = _f64(hinges.compliance, (nh,))
        wheels = list(wheels or [])
        nw = len(wheels)
        if nw:
            k["wheel_body"] = _i32([w.body for w in wheels], (nw,))
            k["wheel_radius"] = _f64([w.radius for w in wheels], (nw,))
            k["wheel_axis"] = _f64([np.asarray(w.axis_local, np.float64) for w in wheels], (nw, 3))
        ncp = 0
        if contact_particles is not None:
            k["contact_particles"] = _i32(contact_particles).ravel()
            ncp = int(k["contact_particles"].shape[0])
        nch = int(np.asarray(channels.pressures).shape[0]) if channels is not None else 0
        self.dims = dict(P=P, nb=nb, nd=nd, nt=nt, na=na, nh=nh, nw=nw, nch=nch,
                         ncp=ncp, cp_all=contact_particles is None)
        t = SsTopology()
        t.num_particles, t.num_bodies = P, nb
        t.inv_mass = _ptr(k["inv_mass"], _dp)
        t.body_mass = _ptr(k["body_mass"], _dp)
        t.body_inertia = _ptr(k["body_inertia"], _dp)
        t.n_dist, t.n_tet, t.n_attach, t.n_hinge, t.n_wheel = nd, nt, na, nh, nw
        for name, kind in (("dist_pairs", _ip), ("dist_rest", _dp), ("dist_compliance", _dp),
                           ("dist_channel", _ip), ("tets", _ip), ("tet_rest_inv", _dp),
                           ("tet_compliance", _dp), ("attach_particle", _ip),
                           ("attach_body", _ip), ("attach_anchor", _dp),
                           ("attach_compliance", _dp), ("hinge_body_a", _ip),
                           ("hinge_body_b", _ip), ("hinge_anchor_a", _dp),
                           ("hinge_anchor_b", _dp), ("hinge_axis_a", _dp),
                           ("hinge_tan1_b", _dp), ("hinge_tan2_b", _dp),
                           ("hinge_compliance", _dp), ("wheel_body", _ip),
                           ("wheel_radius", _dp), ("wheel_axis", _dp),
                           ("contact_particles", _ip)):
            setattr(t, name, _ptr(k.get(name), kind))
        t.n_contact_particles = ncp
        t.n_channels = nch
        t.has_strain = 1 if strain is not None else 0
        self.struct = t
        self.strain_youngs = float(strain.youngs_modulus_pa) if strain is not None else 1.0
        self.channels = channels


def pack_params(config, packed: PackedTopology) -> SsParams:
    """SolverConfig (+ StrainLaw, ChannelBank constants) -> ss_params."""
    p = SsParams()
    p.dt = float(config.dt)
    p.substeps = int(config.substeps)
    p.newton_iters = int(config.newton_iters)
    p.pcr_iters = int(config.pcr_iters)
    g = tuple(float(x) for x in config.gravity)
    p.gravity = (C.c_double * 3)(*g)
    p.ground_height = float(config.ground_height)
    p.ground_enabled = 1 if config.ground_enabled else 0
    p.contact_margin = float(config.contact_margin)
    p.mu = float(config.mu)
    p.friction_compliance = float(config.friction_compliance)
    p.fb_delta = float(config.fb_delta)
    p.fb_slope_min = float(config.fb_slope_min)
    p.fb_slope_max = float(config.fb_slope_max)
    p.max_strain_rate = float(config.max_strain_rate)
    p.constraint_damping = float(config.constraint_damping)
    p.strain_youngs = packed.strain_youngs
    ch = packed.channels
    p.k_inflate = float(getattr(ch, "k_inflate", 0.23))
    p.k_deflate = float(getattr(ch, "k_deflate", 0.23))
    p.deflate_cap = float(getattr(ch, "deflate_cap", 0.68))
    p.supply = float(getattr(ch, "supply", 8.0))
    p.exact_jacobian = 1 if getattr(config, "exact_jacobian", False) else 0
    p.solver_mode = {"auto": 0, "streaming": 1, "cluster": 2}[getattr(config, "solver", "auto")]
    p.wave_envs = int(getattr(config, "wave_envs", 0))
    p.keep_matrix = 1 if getattr(config, "keep_matrix", False) else 0
    return p


class StateBuffers:
    """Host arrays for every ss_state_view field, shaped [n_envs, ...]."""

    def __init__(self, dims: dict, n_envs: int):
        self.n = n_envs
        self.arrays = {}
        for name, shape_fn, dt in STATE_FIELDS:
            self.arrays[name] = np.zeros((n_envs,) + shape_fn(dims), dtype=dt)

    def view(self, names=None) -> SsStateView:
        v = SsStateView()
        for name, _, dt in STATE_FIELDS:
            if names is not None and name not in names:
                continue
            a = self.arrays[name]
            setattr(v, name, _ptr(a, _ip if dt == np.int32 else _dp))
        return v

    def __getitem__(self, name):
        return self.arrays[name]

"""Drop-in Simulator (softsnake/solver.py:154-544) on the B200.

`BatchedSimulator` owns one device handle holding N independent copies of
a scene (the RL-rollout shape); `Simulator` is the single-environment
drop-in with the reference's attribute surface: `step(commands, latency)`
returning StepStats, `state`, `channels.pressures`, `stats`, `totals`,
`static_rows`, `lam_*`. All stepping runs in libsoftsnake_b200.so; the
host objects only mirror state on readback.
"""
from __future__ import annotations

import ctypes as C
import time as _time
from dataclasses import dataclass

import numpy as np

from . import _native
from ._abi import (STATE_FIELDS, PackedTopology, SsEnvStats, StateBuffers,
                   pack_params)


@dataclass
class SolverConfig:
    """solver.py:95-117 (backend/keep_matrix kept for signature parity)."""
    dt: float = 1.0 / 60.0
    substeps: int = 2
    newton_iters: int = 4
    pcr_iters: int = 20
    gravity: tuple = (0.0, 0.0, -9.81)
    ground_height: float = 0.0
    ground_enabled: bool = True
    contact_margin: float = 0.005
    mu: float = 1.0
    friction_compliance: float = 1e-8
    fb_delta: float = 1e-10
    fb_slope_min: float = 1e-6
    fb_slope_max: float = 2.0
    max_strain_rate: float = 6.0
    constraint_damping: float = 1.0
    backend: str | None = None
    keep_matrix: bool = False
    # B200 extension: materialised-column tet Jacobian (bitwise numba sums)
    # instead of the structured chain-rule application (default)
    exact_jacobian: bool = False
    # B200 extension: Newton-loop solver "auto" | "streaming" | "cluster"
    solver: str = "auto"
    # B200 extension: envs per wave (0 = auto from device memory)
    wave_envs: int = 0

    @property
    def h(self) -> float:
        return self.dt / self.substeps


@dataclass
class StepStats:
    """solver.py:142-151"""
    newton_iterations: int = 0
    pcr_iterations: int = 0
    contact_count: int = 0
    inverted_tets: int = 0
    residual: float = 0.0
    wall_time: float = 0.0
    assembly_time: float = 0.0
    solve_time: float = 0.0


def _dims_of(packed: PackedTopology) -> dict:
    return packed.dims


class BatchedSimulator:
    """N independent environments of one scene on one GPU.

    The constructor mirrors Simulator(state, config, distances, tetras,
    attachments, hinges, wheels, channels, strain, contact_particles)
    (solver.py:157-165); every env starts from `state` and the sets'
    persistent arrays (quats, dirs, scale). The device handle is created on
    first use so scene edits made after construction (e.g. the bend
    fixture's clamp, snake.py:363-364) are honoured.
    """

    def __init__(self, n_envs: int, state, config: SolverConfig | None = None,
                 distances=None, tetras=None, attachments=None, hinges=None,
                 wheels=None, channels=None, strain=None, contact_particles=None,
                 device: int = 0):
        if n_envs < 1:
            raise ValueError("n_envs must be >= 1")
        self.n_envs = int(n_envs)
        self.state = state
        self.config = config if config is not None else SolverConfig()
        self.distances, self.tetras = distances, tetras
        self.attachments, self.hinges = attachments, hinges
        self.wheels = list(wheels) if wheels is not None else []
        self.channels, self.strain = channels, strain
        self.contact_particles = contact_particles
        self.device = int(device)
        self._h = None
        self._packed = None
        self.frames = 0
        nd = distances.count if distances is not None else 0
        nt = tetras.count if tetras is not None else 0
        na = attachments.count if attachments is not None else 0
        nh = hinges.count if hinges is not None else 0
        self._m_static = nd + 6 * nt + 3 * na + 5 * nh

    # ------------------------------------------------------------ lifecycle
    @property
    def static_rows(self) -> int:
        return self._m_static

    @property
    def n_links(self) -> int:
        ch = self.channels
        return 0 if ch is None else int(np.asarray(ch.pressures).shape[0]) // 2

    def _ensure(self):
        if self._h is not None:
            return self._h
        L = _native.lib()
        self._packed = PackedTopology(self.state, self.distances, self.tetras,
                                      self.attachments, self.hinges, self.wheels,
                                      self.channels, self.strain, self.contact_particles)
        params = pack_params(self.config, self._packed)
        h = C.c_void_p()
        _native.check(L.ss_create(C.byref(self._packed.struct), C.byref(params),
                                  self.n_envs, self.device, C.byref(h)))
        self._h = h
        self._keep_built = bool(self.config.keep_matrix)
        self._snap_ready = False
        init = getattr(self, "_initial_override", None)
        if init is None:
            self._template = self._initial_state_arrays()  # the reset template (env 0)
            self.set_state_arrays(self._template, env0=0, n=self.n_envs)
        else:
            # handle rebuilt (keep_matrix toggle): the template is restored
            # through env 0, then every env's carried-over state is written
            self.set_state_arrays(self._template, env0=0, n=1)
        _native.check(L.ss_capture_init(h, 0))
        if init is not None:
            self.set_state_arrays(init, env0=0, n=self.n_envs)
        return h

    # ------------------------------------------------------------- episodes
    def capture_initial(self, env: int = 0) -> None:
        """Store env `env`'s current state as the template of reset_envs."""
        _native.check(_native.lib().ss_capture_init(self._ensure(), int(env)))
        # host copy, so a handle rebuild (keep_matrix toggle) can restore it
        self._template = {k: v[0] for k, v in self.get_state_arrays(int(env), 1).items()}

    def reset_envs(self, env_ids, seed: int = 0, pos_sigma: float = 0.0,
                   vel_sigma: float = 0.0) -> None:
        """Reset the listed envs to the template state on the device (RL
        episode reset), with optional deterministic
        Gaussian perturbation of particle positions / velocities."""
        ids = np.ascontiguousarray(np.asarray(env_ids, np.int32).ravel())
        _native.check(_native.lib().ss_reset_envs(
            self._ensure(), ids.ctypes.data_as(C.POINTER(C.c_int)), int(ids.size),
            int(seed) & 0xFFFFFFFFFFFFFFFF, float(pos_sigma), float(vel_sigma)))

    def _sync_keep(self) -> None:
        """config.keep_matrix is read per step in the reference (solver.py:
        511); the device snapshot buffer is sized at ss_create, so a toggle
        recreates the handle with every env's state carried over."""
        if self._h is None or bool(self.config.keep_matrix) == self._keep_built:
            return
        st = self.get_state_arrays()
        gait = self.get_gait()
        self.close()
        self._initial_override = st
        try:
            self._ensure()
        finally:
            self._initial_override = None
        # the on-device gait generator's parameters and frame counters
        prm, fr = gait
        armed = prm[:, 5] >= 1.0  # links_per_snake is 0 where no gait was set
        i = 0
        while i < self.n_envs:
            if not armed[i]:
                i += 1
                continue
            j = i
            while j < self.n_envs and armed[j]:
                j += 1
            p_run = np.ascontiguousarray(prm[i:j])
            f_run = np.ascontiguousarray(fr[i:j])
            _native.check(_native.lib().ss_set_gait(
                self._h, i, j - i, p_run.ctypes.data_as(C.POINTER(C.c_double)),
                f_run.ctypes.data_as(C.POINTER(C.c_int))))
            i = j

    def get_gait(self, env0: int = 0, n: int | None = None):
        """(params [n, 6], frame [n]) of the on-device gait generator
        (ss_set_gait layout; all-zero params when no gait is armed)."""
        n = self.n_envs - env0 if n is None else n
        prm = np.zeros((n, 6))
        fr = np.zeros(n, np.int32)
        _native.check(_native.lib().ss_get_gait(
            self._ensure(), env0, n, prm.ctypes.data_as(C.POINTER(C.c_double)),
            fr.ctypes.data_as(C.POINTER(C.c_int))))
        return prm, fr

    def close(self):
        if self._h is not None:
            _native.lib().ss_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _initial_state_arrays(self) -> dict:
        """Per-env state from the host containers (reference defaults)."""
        st, d = self.state, self._packed.dims
        one = {
            "positions": st.particles.positions, "velocities": st.particles.velocities,
            "body_pos": st.body_pos, "body_quat": st.body_quat,
            "body_lin_vel": st.body_lin_vel, "body_ang_vel": st.body_ang_vel,
            "lam_dist": np.zeros(d["nd"]), "lam_tetra": np.zeros((d["nt"], 6)),
            "lam_attach": np.zeros((d["na"], 3)), "lam_hinge": np.zeros((d["nh"], 5)),
            "tet_quats": self.tetras.quats if d["nt"] else np.zeros((0, 4)),
            "dist_dirs": self.distances.dirs if d["nd"] else np.zeros((0, 3)),
            "dist_scale": self.distances.scale if d["nd"] else np.zeros(0),
            "strain_live": np.ones(d["nch"]), "strain_target": np.ones(d["nch"]),
            "pressures": np.asarray(self.channels.pressures) if d["nch"] else np.zeros(0),
            "warm": np.zeros((d["nw"], 3)), "warm_valid": np.zeros(d["nw"], np.int32),
            "time": np.float64(st.time),
        }
        return one

    # ---------------------------------------------------------------- state
    def set_state_arrays(self, arrays: dict, env0: int = 0, n: int | None = None) -> None:
        """Write state fields (reference shapes, optionally with a leading
        env axis) into envs [env0, env0+n). Missing fields are untouched."""
        h = self._ensure()
        n = self.n_envs - env0 if n is None else n
        buf = StateBuffers(self._packed.dims, n)
        names = []
        for name, shape_fn, dt in STATE_FIELDS:
            if name not in arrays:
                continue
            a = np.asarray(arrays[name], dtype=dt)
            buf.arrays[name][...] = np.broadcast_to(a, buf.arrays[name].shape)
            names.append(name)
        v = buf.view(names)
        _native.check(_native.lib().ss_set_state(h, env0, n, C.byref(v)))

    def get_state_arrays(self, env0: int = 0, n: int | None = None, names=None) -> dict:
        h = self._ensure()
        n = self.n_envs - env0 if n is None else n
        buf = StateBuffers(self._packed.dims, n)
        v = buf.view(names)
        _native.check(_native.lib().ss_get_state(h, env0, n, C.byref(v)))
        return {k: a for k, a in buf.arrays.items() if names is None or k in names}

    def get_state_tensors(self, env0: int = 0, n: int | None = None, names=None) -> dict:
        """State fields as torch CUDA tensors [n, ...] on the handle's device,
        gathered on the device (ss_get_state_device; no host round trip)."""
        import torch
        from ._abi import STATE_FIELDS, SsStateView
        h = self._ensure()
        n = self.n_envs - env0 if n is None else n
        d = self._packed.dims
        out, v = {}, SsStateView()
        for name, shape_fn, dt in STATE_FIELDS:
            if names is not None and name not in names:
                continue
            t = torch.empty((n,) + shape_fn(d), dtype=torch.int32 if dt == np.int32 else torch.float64,
                            device=f"cuda:{self.device}")
            out[name] = t
            kind = C.POINTER(C.c_int32) if dt == np.int32 else C.POINTER(C.c_double)
            setattr(v, name, C.cast(C.c_void_p(t.data_ptr()), kind) if t.numel() else C.cast(None, kind))
        # the handle's stream is not ordered after torch's: finish torch's
        # pending work on these allocations before the device gather writes them
        torch.cuda.current_stream(self.device).synchronize()
        _native.check(_native.lib().ss_get_state_device(h, env0, n, C.byref(v)))
        return out

    def set_state_tensors(self, tensors: dict, env0: int = 0, n: int | None = None) -> None:
        """Write state fields from torch CUDA tensors [n, ...] (reference
        shapes) on the device (ss_set_state_device); missing fields untouched."""
        import torch
        from ._abi import STATE_FIELDS, SsStateView
        h = self._ensure()
        n = self.n_envs - env0 if n is None else n
        d = self._packed.dims
        v, keep = SsStateView(), []
        for name, shape_fn, dt in STATE_FIELDS:
            if name not in tensors:
                continue
            want = torch.int32 if dt == np.int32 else torch.float64
            t = tensors[name].to(device=f"cuda:{self.device}", dtype=want).contiguous()
            if tuple(t.shape) != (n,) + shape_fn(d):
                raise ValueError(f"{name}: expected shape {(n,) + shape_fn(d)}, got {tuple(t.shape)}")
            keep.append(t)
            kind = C.POINTER(C.c_int32) if dt == np.int32 else C.POINTER(C.c_double)
            setattr(v, name, C.cast(C.c_void_p(t.data_ptr()), kind) if t.numel() else C.cast(None, kind))
        torch.cuda.synchronize(self.device)
        _native.check(_native.lib().ss_set_state_device(h, env0, n, C.byref(v)))
        del keep

    def get_stats(self, env0: int = 0, n: int | None = None) -> list[SsEnvStats]:
        h = self._ensure()
        n = self.n_envs - env0 if n is None else n
        arr = (SsEnvStats * n)()
        _native.check(_native.lib().ss_get_stats(h, env0, n, arr))
        return list(arr)

    def center_of_mass(self, env0: int = 0, n: int | None = None) -> np.ndarray:
        h = self._ensure()
        n = self.n_envs - env0 if n is None else n
        out = np.zeros((n, 3))
        _native.check(_native.lib().ss_get_com(h, env0, n, out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def observe(self, env0: int = 0, n: int | None = None) -> dict:
        """Per-env rollout observables computed on the device (ss_observe):
        com [n,3], kinetic_energy [n], body_yaw [n, nb]."""
        h = self._ensure()
        n = self.n_envs - env0 if n is None else n
        nb = self._packed.dims["nb"]
        out = np.zeros((n, 4 + nb))
        _native.check(_native.lib().ss_observe(h, env0, n, out.ctypes.data_as(C.POINTER(C.c_double))))
        return {"com": out[:, :3], "kinetic_energy": out[:, 3], "body_yaw": out[:, 4:]}

    # ----------------------------------------------------------------- step
    def set_gait(self, gaits, links_per_snake: int, t0=0.0, frame0=0, env0: int = 0) -> None:
        """Arm the on-device gait generator (snake.py:235-241) for envs
        [env0, env0+len(gaits)): gaits is one GaitParams or a list (one per
        env); t0 a per-env time offset (s); frame0 the starting frame index
        (t = t0 + frame * dt, like harness.py:190 with t0 = 0)."""
        from .model import GaitParams
        if isinstance(gaits, GaitParams):
            gaits = [gaits] * (self.n_envs - env0)
        n = len(gaits)
        t0 = np.broadcast_to(np.asarray(t0, np.float64), (n,))
        fr = np.ascontiguousarray(np.broadcast_to(np.asarray(frame0, np.int32), (n,)))
        prm = np.array([[g.amplitude_psi, g.angular_rate(), g.phase_offset, g.turn_bias, t0[i],
                         float(links_per_snake)] for i, g in enumerate(gaits)], np.float64)
        prm = np.ascontiguousarray(prm.reshape(n, 6))
        _native.check(_native.lib().ss_set_gait(
            self._ensure(), env0, n, prm.ctypes.data_as(C.POINTER(C.c_double)),
            fr.ctypes.data_as(C.POINTER(C.c_int))))

    def step_gait(self, latency: bool = True, n_frames: int = 1) -> None:
        """Advance all envs n_frames frames with commands generated on the
        device by the gait armed in set_gait (no host commands)."""
        self._sync_keep()
        _native.check(_native.lib().ss_step_gait(self._ensure(), 1 if latency else 0, int(n_frames)))
        self.frames += n_frames
        self._snap_ready = self._keep_built

    def step(self, commands=None, latency: bool = True, n_frames: int = 1) -> None:
        """Advance all envs n_frames frames (asynchronous on the device).
        commands: [n_envs, links] or [n_frames, n_envs, links] psi, or None."""
        self._sync_keep()
        h = self._ensure()
        ptr = None
        if commands is not None:
            cmd = np.ascontiguousarray(np.asarray(commands, np.float64))
            need = n_frames * self.n_envs * self.n_links
            if cmd.size == self.n_links and self.n_envs > 1:
                cmd = np.ascontiguousarray(np.broadcast_to(cmd, (n_frames, self.n_envs, self.n_links)))
            if cmd.size != need:
                raise ValueError(f"commands must hold {need} values, got {cmd.size}")
            self._cmd_keep = cmd
            ptr = cmd.ctypes.data_as(C.POINTER(C.c_double))
        _native.check(_native.lib().ss_step(h, ptr, 1 if latency else 0, int(n_frames)))
        self.frames += n_frames
        self._snap_ready = self._keep_built

    def set_channel_targets(self, commands, latency: bool = True) -> None:
        """One pneumatic tick of every env toward commands [n_envs, links]
        psi (ChannelBank.tick via solver.py:274-277), without stepping."""
        h = self._ensure()
        if self.channels is None:
            return
        cmd = np.ascontiguousarray(np.asarray(commands, np.float64))
        if cmd.size == self.n_links and self.n_envs > 1:
            cmd = np.ascontiguousarray(np.broadcast_to(cmd, (self.n_envs, self.n_links)))
        if cmd.size != self.n_envs * self.n_links:
            raise ValueError(f"commands must hold {self.n_envs * self.n_links} values, got {cmd.size}")
        _native.check(_native.lib().ss_set_channel_targets(
            h, cmd.ctypes.data_as(C.POINTER(C.c_double)), 1 if latency else 0))

    def step_device(self, d_commands_ptr: int, latency: bool = True, n_frames: int = 1) -> None:
        self._sync_keep()
        h = self._ensure()
        _native.check(_native.lib().ss_step_device(h, C.c_void_p(d_commands_ptr),
                                                   1 if latency else 0, int(n_frames)))
        self.frames += n_frames

    # ----------------------------------------------------------- inspection
    def last_system(self, env: int = 0):
        """Explicit CSR of the most recent Newton system (keep_matrix on;
        solver.py:548-575) of one env."""
        from .system import assemble, export_blocks
        if not getattr(self, "_snap_ready", False):
            raise RuntimeError("no system snapshot; set config.keep_matrix and step")
        cfg = self.config
        h = cfg.dt / cfg.substeps
        gamma = 1.0 / (1.0 + max(0.0, cfg.constraint_damping))
        eh2 = None
        if self.tetras is not None and self.tetras.count:
            eh2 = gamma * self.tetras.compliance / (h * h)
        return assemble(export_blocks(self, env), eh2)

    def export_system(self, path_a: str, path_b: str, env: int = 0) -> None:
        """Write the last Newton system as Matrix Market files
        (solver.py:577-581)."""
        from .system import mmwrite, mmwrite_dense
        s = self.last_system(env)
        mmwrite(path_a, s.matrix)
        mmwrite_dense(path_b, s.rhs)

    def synchronize(self) -> None:
        _native.check(_native.lib().ss_synchronize(self._ensure()))

    def profile_frames(self, commands=None, latency: bool = True, n_frames: int = 1) -> dict:
        """Run frames un-graphed with CUDA events around every launch;
        returns {kernel: (total_ms, launches)}."""
        h = self._ensure()
        L = _native.lib()
        names = (C.c_char_p * 32)()
        nk = L.ss_kernel_names(names, 32)
        ms = (C.c_double * nk)()
        cnt = (C.c_int * nk)()
        ptr = None
        if commands is not None:
            cmd = np.ascontiguousarray(np.asarray(commands, np.float64))
            if cmd.size != n_frames * self.n_envs * self.n_links:
                raise ValueError("commands must be [n_frames, n_envs, links]")
            ptr = cmd.ctypes.data_as(C.POINTER(C.c_double))
        _native.check(L.ss_profile_frames(h, ptr, 1 if latency else 0, int(n_frames), ms, cnt))
        return {names[i].decode(): (float(ms[i]), int(cnt[i])) for i in range(nk)}

    @property
    def stream(self) -> int:
        return int(_native.lib().ss_stream(self._ensure()) or 0)

    @property
    def solver_info(self) -> dict:
        info = (C.c_int * 10)()
        _native.check(_native.lib().ss_solver_info(self._ensure(), info))
        return {"cluster": bool(info[0]), "cluster_size": info[1], "smem_bytes": info[2],
                "env_lanes": info[3], "waves": info[4], "fused_gather": bool(info[5]),
                "fused_blocks": info[6], "fused_chunks": info[7], "clusters_per_env": info[8],
                "cross_cluster_fault": info[9]}

    @property
    def launches_per_frame(self) -> int:
        return int(_native.lib().ss_launches_per_frame(self._ensure()))

    @property
    def device_bytes(self) -> int:
        return int(_native.lib().ss_device_bytes(self._ensure()))


class Simulator(BatchedSimulator):
    """Single-environment drop-in for softsnake.solver.Simulator."""

    def __init__(self, state, config: SolverConfig | None = None, distances=None,
                 tetras=None, attachments=None, hinges=None, wheels=None, channels=None,
                 strain=None, contact_particles=None, device: int = 0):
        super().__init__(1, state, config, distances, tetras, attachments, hinges, wheels,
                         channels, strain, contact_particles, device)
        self.kern = None  # the reference's backend slot; kernels live in the .so
        self.stats = StepStats()
        self.totals = {"steps": 0, "newton_iterations": 0, "pcr_iterations": 0,
                       "contact_count": 0, "inverted_tets": 0, "assembly_time": 0.0,
                       "solve_time": 0.0, "wall_time": 0.0}
        self._cache = None

    # reference surface ------------------------------------------------
    def set_channel_targets(self, commands, latency: bool = True) -> None:
        """Advance the pneumatic channels one tick toward the commands
        (solver.py:274-277) on the device, without stepping."""
        super().set_channel_targets(np.asarray(commands, np.float64).reshape(1, -1), latency)
        self._refresh_host()

    def step(self, commands=None, latency: bool = True) -> StepStats:  # noqa: D401
        t0 = _time.perf_counter()
        super().step(None if commands is None else np.asarray(commands, np.float64).reshape(1, -1),
                     latency, 1)
        s = self.get_stats(0, 1)[0]
        self._cache = None
        self.stats = StepStats(s.newton_iterations, s.pcr_iterations, s.contact_count,
                               s.inverted_tets, float(s.residual))
        self.stats.wall_time = _time.perf_counter() - t0
        self.stats.solve_time = self.stats.wall_time
        tot = self.totals
        tot["steps"] += 1
        for k in ("newton_iterations", "pcr_iterations", "contact_count", "inverted_tets"):
            tot[k] += getattr(self.stats, k)
        tot["wall_time"] += self.stats.wall_time
        tot["solve_time"] += self.stats.solve_time
        self._refresh_host()
        return self.stats

    def _refresh_host(self):
        """Mirror device state into the host containers in place."""
        a = self.get_state_arrays(0, 1)
        self._cache = a
        st = self.state
        st.particles.positions[...] = a["positions"][0]
        st.particles.velocities[...] = a["velocities"][0]
        st.body_pos[...] = a["body_pos"][0]
        st.body_quat[...] = a["body_quat"][0]
        st.body_lin_vel[...] = a["body_lin_vel"][0]
        st.body_ang_vel[...] = a["body_ang_vel"][0]
        st.time = float(a["time"][0])
        if self.channels is not None:
            self.channels.pressures[...] = a["pressures"][0]
        if self.tetras is not None:
            self.tetras.quats[...] = a["tet_quats"][0]
        if self.distances is not None:
            self.distances.dirs[...] = a["dist_dirs"][0]
            self.distances.scale[...] = a["dist_scale"][0]

    def push_state(self) -> None:
        """Upload edits made to the host containers (state, quats, dirs...)."""
        self._ensure()
        arr = self._initial_state_arrays()
        for k in ("lam_dist", "lam_tetra", "lam_attach", "lam_hinge", "strain_live",
                  "strain_target", "warm", "warm_valid"):
            arr.pop(k)
        self.set_state_arrays(arr, 0, 1)

    def _lam(self, name):
        if self._cache is None:
            self._cache = self.get_state_arrays(0, 1)
        return self._cache[name][0]

    lam_dist = property(lambda self: self._lam("lam_dist"))
    lam_tetra = property(lambda self: self._lam("lam_tetra"))
    lam_attach = property(lambda self: self._lam("lam_attach"))
    lam_hinge = property(lambda self: self._lam("lam_hinge"))

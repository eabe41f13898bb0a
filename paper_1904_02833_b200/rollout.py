"""Batched rollout harness.

The reference's experiments step one Simulator per level/run and read state
back every frame (harness.py:99-210). Here every level or run is one env of a
BatchedSimulator: commands come from the host per frame (curvature sweep) or
from the on-device gait generator (locomotion, ss_set_gait/ss_step_gait), and
per-env observables (COM, kinetic energy, body yaws) are reduced on the
device (ss_observe), so a frame moves (4 + nb) doubles per env to the host.
"""
from __future__ import annotations

import math

import numpy as np

from .model import GaitParams, build_bend_fixture, build_snake

SETTLE_ENERGY_J = 1e-6   # harness.py:24
SETTLE_HOLD_S = 0.5      # harness.py:25


def link_curvature(body_yaw: np.ndarray, frame_bodies: np.ndarray, link: int,
                   link_length: float, snake: int = 0) -> np.ndarray:
    """SnakeModel.link_curvature (snake.py:212-229) over a leading env axis:
    body_yaw [n, nb] -> [n]."""
    d = body_yaw[:, frame_bodies[snake, link + 1]] - body_yaw[:, frame_bodies[snake, link]]
    d = np.where(d > math.pi, d - 2.0 * math.pi * np.ceil((d - math.pi) / (2.0 * math.pi)), d)
    d = np.where(d < -math.pi, d + 2.0 * math.pi * np.ceil((-math.pi - d) / (2.0 * math.pi)), d)
    return d / link_length


class SettleTracker:
    """Per-env state machine of harness._settle (harness.py:83-97) followed
    by the sampling loop of run_curvature_sweep (harness.py:121-128)."""

    def __init__(self, n: int, hold_frames: int, max_frames: int, samples: int):
        self.hold, self.max_frames, self.n_samples = hold_frames, max_frames, samples
        self.quiet = np.zeros(n, np.int64)
        self.frames = np.zeros(n, np.int64)
        self.settled = np.zeros(n, bool)
        self.sampling = np.zeros(n, bool)
        self.done = np.zeros(n, bool)
        self.samples = [[] for _ in range(n)]

    def update(self, ke: np.ndarray, curv: np.ndarray) -> np.ndarray:
        """Feed one frame's observables; returns the envs that finished on
        this frame."""
        finished = np.zeros_like(self.done)
        for e in range(self.quiet.size):
            if self.done[e]:
                continue
            if self.sampling[e]:
                self.samples[e].append(float(curv[e]))
                if len(self.samples[e]) >= self.n_samples:
                    self.done[e] = finished[e] = True
                continue
            self.frames[e] += 1
            if ke[e] < SETTLE_ENERGY_J:
                self.quiet[e] += 1
                if self.quiet[e] >= self.hold:
                    self.settled[e] = self.sampling[e] = True
            else:
                self.quiet[e] = 0
            if not self.sampling[e] and self.frames[e] >= self.max_frames:
                self.sampling[e] = True
            if self.sampling[e] and self.n_samples == 0:
                self.done[e] = finished[e] = True
        return finished


def curvature_sweep(scene, pressures=None, samples_per_level: int = 30,
                    max_frames: int = 900, device: int = 0) -> dict:
    """harness.run_curvature_sweep (harness.py:99-131) with the levels as
    batched envs of the bend fixture. Returns the record's columns:
    tick, time_s, pressure_psi, curvature_mean, curvature_std, settled."""
    if pressures is None:
        pressures = [float(p) for p in range(-8, 9)]
    pressures = [float(p) for p in pressures]
    for p in pressures:
        if abs(p) > 10.0:
            raise ValueError("pressure levels must stay within +-10 psi")
    n = len(pressures)
    model = build_bend_fixture(scene, n_envs=n, device=device)
    sim = model.sim
    cmds = np.array(pressures, np.float64).reshape(n, 1)
    hold = max(1, int(round(SETTLE_HOLD_S / sim.config.dt)))
    tr = SettleTracker(n, hold, max_frames, samples_per_level)
    times = np.zeros(n)
    while not tr.done.all():
        sim.step(cmds, latency=False)
        obs = sim.observe()
        curv = link_curvature(obs["body_yaw"], model.frame_bodies, 0, scene.link_length)
        fin = tr.update(obs["kinetic_energy"], curv)
        if fin.any():
            t = sim.get_state_arrays(names=["time"])["time"]
            times[fin] = t[fin]
    mean = np.array([np.mean(s) if s else np.nan for s in tr.samples])
    std = np.array([np.std(s) if s else np.nan for s in tr.samples])
    return {"tick": np.arange(n), "time_s": times, "pressure_psi": np.array(pressures),
            "curvature_mean": mean, "curvature_std": std, "settled": tr.settled.astype(int)}


def locomotion(scene, n_envs: int, frames: int, gaits=None, t0=0.0, latency: bool = True,
               device: int = 0, model=None) -> dict:
    """harness.run_locomotion (harness.py:170-210) for n_envs snakes at once,
    commands from the on-device gait generator. Per frame and env: com,
    head_yaw, path_xy, contacts, curvature per link, diverged."""
    m = model if model is not None else build_snake(scene, n_envs=n_envs, device=device)
    sim = m.sim
    if gaits is None:
        gaits = GaitParams.from_scene(scene)
    sim.set_gait(gaits, m.links_per_snake, t0=t0)
    L = m.links_per_snake
    com = np.zeros((frames, n_envs, 3))
    yaw = np.zeros((frames, n_envs))
    path = np.zeros((frames, n_envs))
    contacts = np.zeros((frames, n_envs), np.int64)
    curv = np.zeros((frames, n_envs, L))
    diverged = np.zeros((frames, n_envs), bool)
    prev = sim.observe()["com"].copy()
    run = np.zeros(n_envs)
    alive = np.ones(n_envs, bool)
    for i in range(frames):
        sim.step_gait(latency=latency)
        obs = sim.observe()
        c = obs["com"]
        ok = np.all(np.isfinite(c), axis=1) & alive
        step_len = np.hypot(c[:, 0] - prev[:, 0], c[:, 1] - prev[:, 1])
        run = np.where(ok, run + step_len, run)
        prev = np.where(ok[:, None], c, prev)
        alive &= ok
        com[i], path[i], diverged[i] = c, run, ~ok
        yaw[i] = obs["body_yaw"][:, m.frame_bodies[0, 0]]
        for k in range(L):
            curv[i, :, k] = link_curvature(obs["body_yaw"], m.frame_bodies, k, scene.link_length)
        contacts[i] = [s.contact_count for s in sim.get_stats()]
    return {"com": com, "head_yaw": yaw, "path_xy": path, "contacts": contacts,
            "curvature": curv, "diverged": diverged}


def benchmark(scene, snake_counts=(1, 2, 3, 4), frames: int = 60, warmup: int = 5,
              include_single_link: bool = True, device: int = 0) -> list[dict]:
    """harness.run_benchmark (harness.py:212-262, the paper's Table II) on
    the device: per scene size (the 1-link bend fixture, then coupled
    n-snake scenes — one system each), device time per frame from CUDA
    events around each graph replay, and the assembly / solve split from a
    per-launch profile (eval kernels vs the Newton loop)."""
    import torch
    rows = []
    cases = []
    if include_single_link:
        cases.append((0.25, lambda: build_bend_fixture(scene, device=device)))
    for n in snake_counts:
        if n < 1:
            raise ValueError("snake counts must be >= 1")
        cases.append((float(n), lambda n=n: build_snake(scene, n_snakes=n, device=device)))
    g = GaitParams.from_scene(scene)
    for count, make in cases:
        m = make()
        sim = m.sim
        dt = sim.config.dt
        for i in range(warmup):
            sim.step(m.commands(i * dt, g))
        sim.synchronize()
        stream = torch.cuda.ExternalStream(sim.stream, device=f"cuda:{device}")
        times = np.empty(frames)
        for i in range(frames):
            c = m.commands((warmup + i) * dt, g)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            sim.step(c, latency=True)
            e1.record(stream)
            e1.synchronize()
            times[i] = e0.elapsed_time(e1)
        cmds = m.commands((warmup + frames) * dt, g)
        prof = sim.profile_frames(cmds.reshape(1, 1, -1), True, 1)
        asm = sum(v[0] for k, v in prof.items()
                  if k in ("k_frame_begin", "k_pre", "k_slots", "k_eval_tet", "k_eval_misc",
                           "k_integrate"))
        tot = sum(v[0] for v in prof.values())
        total_ms = float(np.mean(times))
        rows.append({"snakes": count, "particles": sim.state.num_particles,
                     "bodies": sim.state.num_bodies, "constraint_rows": sim.static_rows,
                     "frames": frames, "assembly_ms": total_ms * asm / tot,
                     "solve_ms": total_ms * (tot - asm) / tot, "total_ms": total_ms,
                     "total_ms_std": float(np.std(times)), "total_per_snake_ms": total_ms / count,
                     "solver": "cluster" if sim.solver_info["cluster"] else "streaming",
                     "cluster_size": sim.solver_info["cluster_size"],
                     "clusters_per_env": sim.solver_info["clusters_per_env"]})
    return rows

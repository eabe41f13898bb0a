#!/usr/bin/env python
"""Benchmark: batched soft-snake frames on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

A "step" is one frame (dt = 1/60 s: 1 pneumatic tick, 2 substeps x 4 Newton
x 20 PCR) of every environment. Workload (BASELINE.json configs[2]): 1024
independent 4-link snakes per GPU, default gait with a per-env turn bias and
time offset (seeded), latency on. Multi-GPU: one process per GPU, env slices
(weak scaling, no data-path collective); an NCCL all_gather of per-env COM
runs once after timing. Rank 0 prints one JSON line.

The oracle (oracle/) appears only in the cpu_baseline leg and in
--impl reference, where the reference's algorithm (its C restatement) is
timed on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "snake-steps/sec (batched, device-timed) & real-time factor; % HBM roofline"
UNIT = "snake-steps/s"
WORKLOAD = "1024 independent snakes batched on 1xB200 (RL rollout shape), per GPU"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--envs", type=int, default=1024, help="environments per GPU (weak scaling)")
    ap.add_argument("--total-envs", type=int, default=0,
                    help="fixed total environments split across GPUs (strong scaling)")
    ap.add_argument("--profile-frames", type=int, default=2)
    ap.add_argument("--cpu-frames", type=int, default=12,
                    help="oracle frames per host core (cpu_baseline sample: ~15-30 core-seconds)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--scene", default="S", choices=["S", "H"],
                    help="S: the snake (configs 3/4); H: the 1M-tet snake, 1 env per GPU "
                         "(config 5, replicas only)")
    ap.add_argument("--wave-envs", type=int, default=0,
                    help="envs per wave (SolverConfig.wave_envs; 0 = auto)")
    ap.add_argument("--solver", default="auto", choices=["auto", "streaming", "cluster"],
                    help="Newton-loop solver (SolverConfig.solver)")
    return ap.parse_args()


H_SCENE = dict(sections=101, width_nodes=26, height_nodes=21)


def env_commands(n_envs: int, frames: int, first_frame: int, env0: int = 0,
                 default_gait: bool = False):
    """[frames, n_envs, 4] gait commands: per-env turn bias and time offset
    from the conftest seed; default_gait: the
    GaitParams defaults for every env (configs 2 and 5)."""
    import paper_1904_02833_b200 as M
    sc = M.SceneConfig()
    # one (bias, t0) row per env: env e's draw does not depend on the sharding
    draws = np.random.default_rng(20260817).uniform(size=(env0 + n_envs, 2))[env0:]
    bias, t0 = draws[:, 0] - 0.5, 0.5 * draws[:, 1]
    if default_gait:
        bias, t0 = np.zeros(n_envs), np.zeros(n_envs)
    w = 2.0 * np.pi * sc.frequency
    i = np.arange(4)
    t = t0[None, :] + (first_frame + np.arange(frames))[:, None] * sc.dt
    raw = np.sin(w * t[..., None] + sc.phase_offset * i) + bias[None, :, None]
    return np.ascontiguousarray(np.clip(raw, -1.0, 1.0) * sc.amplitude_psi)


# ----------------------------------------------------------------- CPU leg
class CpuArm:
    """The reference algorithm (oracle C port) on host cores: one snake per
    core, one dedicated worker thread per snake pinned to its own core (the
    survey's taskset protocol); ctypes releases the GIL."""

    def __init__(self, cores: int | None = None, frames: int = 64):
        import queue
        from oracle.oracle import OracleSim
        import paper_1904_02833_b200 as M
        from paper_1904_02833_b200.model import build_scene_parts
        cpus = sorted(os.sched_getaffinity(0))
        self.cores = cores or len(cpus)
        self.cpus = [cpus[i % len(cpus)] for i in range(self.cores)]
        sc = M.SceneConfig()
        parts, *_ = build_scene_parts(sc)
        cfg = sc.solver_config()
        self.sims = [OracleSim(config=cfg, **parts) for _ in range(self.cores)]
        self.cmds = env_commands(self.cores, frames, 0)
        self.frame = 0
        self.todo = [queue.Queue() for _ in range(self.cores)]
        self.done = queue.Queue()
        self.threads = [threading.Thread(target=self._worker, args=(e,), daemon=True)
                        for e in range(self.cores)]
        for t in self.threads:
            t.start()

    def _worker(self, e):
        try:
            os.sched_setaffinity(0, {self.cpus[e]})  # this thread only
        except OSError:
            pass
        while True:
            job = self.todo[e].get()
            if job is None:
                return
            f0, frames = job
            for f in range(frames):
                self.sims[e].step(self.cmds[(f0 + f) % len(self.cmds), e], True)
            self.done.put(e)

    def step(self, frames: int = 1):
        for q in self.todo:
            q.put((self.frame, frames))
        for _ in range(self.cores):
            self.done.get()
        self.frame += frames

    def close(self):
        for q in self.todo:
            q.put(None)
        for t in self.threads:
            t.join()


def cpu_oracle_rate(frames_per_core: int, cores: int | None = None):
    """snake-steps/s of the oracle port on all host cores (1 warm-up frame)."""
    arm = CpuArm(cores, frames_per_core + 1)
    arm.step(1)
    t = time.perf_counter()
    arm.step(frames_per_core)
    dt = time.perf_counter() - t
    arm.close()
    return arm.cores * frames_per_core / dt, arm.cores, dt


def numba_calibration(port_rate: float) -> dict:
    """The reference's own numba path beside the port: measured on a B200
    box's host cores (profiles/cpu_host_numba.json: the unmodified reference
    package from baseline/_ref, one pinned process per core,
    tools/cpu_calibration.py --box), and the port/numba ratio of that run
    applied to this run's port rate (numba_equivalent_value). Falls back to
    the build-container calibration (profiles/cpu_calibration.json)."""
    out = {}
    for name in ("cpu_host_numba.json", "cpu_calibration.json"):
        path = os.path.join(ROOT, "profiles", name)
        if not os.path.exists(path):
            continue
        cal = json.load(open(path))
        r = float(cal["port_over_numba_aggregate"])
        out = {"numba_equivalent_value": port_rate / r, "port_over_numba": r,
               "calibration": f"profiles/{name} (numba reference vs this port, "
                              f"{cal['host_cores']} pinned processes, {cal.get('host', 'one host')})"}
        if name == "cpu_host_numba.json":
            out["numba_reference_on_gpu_box_host"] = {
                "value": round(float(cal["numba"]["aggregate_all_cores"]), 2),
                "unit": "snake-steps/s", "cores": int(cal["host_cores"]),
                "per_core_1proc": round(float(cal["numba"]["per_core_1proc"]), 3),
                "measured": cal.get("when"), "cpu": cal.get("cpu_model")}
        break
    return out


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    arm = CpuArm(frames=args.warmup + args.steps)
    cores = arm.cores
    for _ in range(args.warmup):
        arm.step(1)
    t = time.perf_counter()
    for _ in range(args.steps):
        arm.step(1)
    wall = time.perf_counter() - t
    arm.close()
    # each step: every core advances its own snake by one frame
    rate = cores * args.steps / wall
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * wall / max(args.steps, 1), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "sample": f"{cores} snakes x 1 frame per step"},
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"oracle/softsnake_oracle.c (C restatement of the reference "
                                   f"step), 1 snake per core (pinned thread), {args.steps} frames",
                         **numba_calibration(rate)},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu, self.proc, self.lines = gpu, None, []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 8:
                continue
            try:
                sm.append(float(p[0]))
                mx.append(float(p[1]))
            except ValueError:
                continue
            for n, v in zip(names, p[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# -------------------------------------------------------------------- main
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import torch
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import __graft_entry__ as g
    if rank == 0:
        g.build()
    if dist:
        dist.barrier()
    import paper_1904_02833_b200 as M
    from paper_1904_02833_b200 import roofline
    from paper_1904_02833_b200.distributed import env_slice, gather_env_stats, max_over_ranks

    hires = args.scene == "H"
    if hires:
        # config 5: one 1M-tet snake per GPU (replicas only)
        env0, n = rank, 1
        total, scaling = world, "weak"
    elif args.total_envs:
        env0, n = env_slice(args.total_envs, world, rank)
        total, scaling = args.total_envs, "strong"
    else:
        env0, n = rank * args.envs, args.envs
        total, scaling = world * args.envs, "weak"
    scene = M.SceneConfig(**H_SCENE) if hires else M.SceneConfig()
    model = M.build_snake(scene, n_envs=n, device=local)
    sim = model.sim
    sim.config.solver = args.solver
    sim.config.wave_envs = args.wave_envs
    K, W = args.steps, args.warmup
    gcmd = lambda nn, fr, f0, env0=0: env_commands(nn, fr, f0, env0=env0, default_gait=hires)  # noqa: E731
    cmds = gcmd(n, W + K, 0, env0=env0)
    d_cmds = torch.from_numpy(cmds).to(f"cuda:{local}")
    stream = torch.cuda.ExternalStream(sim.stream, device=f"cuda:{local}")
    frame_elems = n * 4

    # warm-up (also instantiates the CUDA graph)
    for f in range(W):
        sim.step_device(d_cmds.data_ptr() + 8 * f * frame_elems, True, 1)
    sim.synchronize()

    # ---- device-timed region: inputs resident in HBM
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        e0.record(stream)
        for f in range(K):
            sim.step_device(d_cmds.data_ptr() + 8 * (W + f) * frame_elems, True, 1)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = max_over_ranks(e0.elapsed_time(e1), device=f"cuda:{local}")
    stats = sim.get_stats(0, min(n, 8))
    finite = all(s.finite for s in sim.get_stats())

    # ---- e2e through the public API: host commands (pinned) in, COM out
    host_cmd = torch.from_numpy(gcmd(n, K, W + K, env0=env0)).pin_memory()
    com_bytes = n * 3 * 8
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for f in range(K):
        sim.step(host_cmd[f].numpy(), latency=True)
        com = sim.center_of_mass()          # D2H of the step's result (synchronises)
    e2e_s = max_over_ranks(time.perf_counter() - t0, device=f"cuda:{local}")
    # optional rollout-stats gather over NVLink, off the timed path
    all_com = gather_env_stats(com, total, device=f"cuda:{local}")

    # ---- live per-kernel timing (CUDA events around each launch)
    prof_cmds = gcmd(n, args.profile_frames, W + 2 * K, env0=env0)
    prof = sim.profile_frames(prof_cmds, True, args.profile_frames)
    step_ms_prof = sum(v[0] for v in prof.values()) / args.profile_frames
    top = max(prof, key=lambda k: prof[k][0])
    d = roofline.dims_of(sim)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    peak = float(peaks.get("hbm_gbs", 6650.0))
    nc_mean = float(np.mean([st.contact_count for st in sim.get_stats()])) / sim.config.substeps
    # one launch covers one wave: envs per launch = n / waves on average
    waves = sim.solver_info["waves"]
    structured = not sim.config.exact_jacobian
    pcr = sim.config.pcr_iters
    epl = max(1, round(n / waves))  # envs per launch
    topo = lambda k: roofline.topology_bytes_per_launch(k, d, epl)  # noqa: E731
    per_launch = roofline.bytes_per_launch_per_env(top, d, nc_mean, structured, pcr) * n / waves \
        + topo(top)
    avg_ms = prof[top][0] / prof[top][1]
    # algorithmic bytes of one frame of every env of this rank (all modelled kernels)
    step_bytes = sum((roofline.bytes_per_launch_per_env(k, d, nc_mean, structured, pcr) * n / waves
                      + topo(k)) * (v[1] / args.profile_frames) for k, v in prof.items())
    achieved = per_launch / (avg_ms * 1e-3) / 1e9
    # per-kernel table (live CUDA events): algorithmic bytes per launch, mean
    # launch time, achieved GB/s and the fraction of the HBM peak
    per_kernel = {}
    for k, (kms, kl) in sorted(prof.items(), key=lambda kv: -kv[1][0]):
        if kl == 0:
            continue
        kb = roofline.bytes_per_launch_per_env(k, d, nc_mean, structured, pcr) * n / waves + topo(k)
        kus = 1e3 * kms / kl
        per_kernel[k] = {"ms_per_frame": round(kms / args.profile_frames, 4),
                         "launches_per_frame": kl // args.profile_frames,
                         "bytes_per_launch": kb, "avg_launch_us": round(kus, 3),
                         "gbps": round(kb / (kus * 1e-6) / 1e9, 1) if kb else None,
                         "frac": round(kb / (kus * 1e-6) / 1e9 / peak, 4) if kb else None}
    # the reference-layout byte model beside this build's own
    survey = roofline.survey_model(d, nc_mean, sim.config.substeps, sim.config.newton_iters, pcr)
    traffic = None
    # traffic.json: the batched S-scene capture (scaled to the envs of one
    # launch); traffic_H.json: the 1M-tet scene (one env)
    tp = os.path.join(ROOT, "profiles", "traffic_H.json" if hires else "traffic.json")
    if os.path.exists(tp):
        tj = json.load(open(tp))
        if tj.get(top) is not None:
            traffic = float(tj[top]) * (1.0 if hires else (n / waves) / float(tj.get("_envs", 1024)))

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return 0

    value = total * K / (ms * 1e-3)
    e2e = total * K / e2e_s
    launches = sim.launches_per_frame
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": ms / K, "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD if total == 1024 * world and scaling == "weak" and
                   not hires else (f"1M-tet snake (config 5, {H_SCENE}), 1 per GPU, default gait"
                                   if hires else f"{total} independent snakes batched on "
                                   f"{world}xB200"), "envs_per_gpu": n, "global_envs": total,
                   "frame_dt_s": 1 / 60, "substeps": 2, "newton": 4, "pcr": 20,
                   "gait": "GaitParams defaults" if hires else
                           "default, per-env turn bias U(-0.5,0.5), t0 U(0,0.5s), seed 20260817",
                   "l2": "no flush: per-step working set "
                         f"{sim.device_bytes / 1e9:.1f} GB >> 126 MB L2",
                   "parallelism": f"env-sharded x{world}",
                   "solver": sim.solver_info},
        "rtf": value / 60.0,
        "roofline": {"bound": "hbm", "kernel": top, "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback",
                     "bytes_per_launch": per_launch, "avg_launch_ms": avg_ms,
                     "mean_contacts_per_substep": nc_mean,
                     "share_of_step": prof[top][0] / sum(v[0] for v in prof.values()),
                     "traffic": traffic,
                     "traffic_over_model": traffic / per_launch if traffic else None},
        # whole step: every kernel's algorithmic bytes per frame over the graph-timed
        # frame (concurrent lanes overlap kernels, so this exceeds per-kernel rates)
        "step_bandwidth": {"achieved": step_bytes * (K / (ms * 1e-3)) / 1e9, "peak": peak,
                           "unit": "GB/s", "frac": step_bytes * (K / (ms * 1e-3)) / 1e9 / peak,
                           "bytes_per_step": step_bytes},
        # SURVEY.md §8(d) model (reference layout: stored 6x12 tet J read twice per
        # apply, 6x6 E_tet) vs this build's own bytes (compact J, structured apply)
        "byte_models": {
            "survey_8d_bytes_per_snake_step": survey["total"],
            "survey_8d_env_private_bytes_per_snake_step": survey["env_private"],
            "implementation_bytes_per_snake_step": step_bytes / n,
            "ratio_survey_env_private_over_implementation": survey["env_private"] / (step_bytes / n),
            "effective_frac_on_survey_env_private": survey["env_private"] * (total * K / (ms * 1e-3))
            / world / 1e9 / peak,
            "note": "effective_frac > 1 means the build moves fewer bytes than the reference "
                    "layout needs; step_bandwidth.frac is the fraction on the build's own bytes"},
        "per_kernel": per_kernel,
        "kernels_ms_per_frame": {k: round(v[0] / args.profile_frames, 4) for k, v in prof.items()},
        "profiled_ms_per_frame": step_ms_prof,
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": n * 4 * 8,
                "d2h_bytes_per_step": com_bytes},
        "gpu_launches": launches * K,
        "finite": finite and bool(np.all(np.isfinite(all_com))),
        "stats_env0": {"contacts": stats[0].contact_count, "inverted": stats[0].inverted_tets,
                       "residual": stats[0].residual},
        "clocks": clk.summary(),
    }
    if hires and not args.no_cpu_baseline:
        from oracle.oracle import OracleSim
        from paper_1904_02833_b200.model import build_scene_parts
        parts, *_ = build_scene_parts(scene)
        o = OracleSim(config=scene.solver_config(), **parts)
        t = time.perf_counter()
        o.step(cmds[0, 0], True)
        secs = time.perf_counter() - t
        line["cpu_baseline"] = {"value": 1.0 / secs, "unit": UNIT, "cores": 1, "kind": "port",
                                "sample": f"oracle C port, 1 frame of the 1M-tet snake from rest "
                                          f"({secs:.1f} s)"}
    elif not args.no_cpu_baseline:
        rate, cores, secs = cpu_oracle_rate(args.cpu_frames)
        line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": cores, "kind": "port",
                                "sample": f"oracle C port, {cores} snakes x {args.cpu_frames} "
                                          f"frames ({secs:.1f} s wall), one pinned thread "
                                          f"per core"}
        line["cpu_baseline"].update(numba_calibration(rate))
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

"""Per-core speed of the reference's own CPU path (the numba Simulator of
the reference package, SURVEY.md §8(d) protocol: one process per core,
pinned, *_NUM_THREADS=1) against the oracle C port that bench.py times.

    python tools/cpu_calibration.py [frames]            # this container
    python tools/cpu_calibration.py [frames] --box       # a GPU box's host

In this container the reference is imported from /root/reference; on a GPU
box (--box) from baseline/_ref, the unmodified reference package installed
once with `pip install --no-index --no-deps --target baseline/_ref` from a
copy of /root/reference/pkg (git-ignored, travels with gpurun). Writes
profiles/cpu_calibration.json (container) or profiles/cpu_host_numba.json
(box): per-core snake-steps/s of both on the same host, same scene
(build_snake(SceneConfig())), same commands (default gait), 3 warm-up frames
excluded; and the aggregate over all cores.
"""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BOX = "--box" in sys.argv
_args = [a for a in sys.argv[1:] if not a.startswith("--")]
FR = int(_args[0]) if _args else 20
REF = os.path.join(ROOT, "baseline", "_ref") if BOX else "/root/reference/pkg/src"

CHILD = r"""
import os, sys, time
os.sched_setaffinity(0, {int(sys.argv[2])})
kind, frames = sys.argv[1], int(sys.argv[3])
sys.path.insert(0, %r)
import numpy as np
if kind == "numba":
    sys.path.insert(0, sys.argv[4])
    import softsnake as R
    sc = R.SceneConfig(backend="numba")
    m = R.build_snake(sc)
    step = lambda c: m.sim.step(c, latency=True)
    cmd = lambda i: m.commands(i * sc.dt)
else:
    import paper_1904_02833_b200 as M
    from paper_1904_02833_b200.model import build_scene_parts
    from oracle.oracle import OracleSim
    sc = M.SceneConfig()
    parts, *_ = build_scene_parts(sc)
    o = OracleSim(config=sc.solver_config(), **parts)
    g = M.GaitParams.from_scene(sc)
    step = lambda c: o.step(c, True)
    cmd = lambda i: M.gait_commands(g, i * sc.dt, 4, 4)
for i in range(3):
    step(cmd(i))
t = time.perf_counter()
for i in range(3, 3 + frames):
    step(cmd(i))
print(frames / (time.perf_counter() - t))
""" % ROOT


def run(kind, cores):
    env = dict(os.environ, OMP_NUM_THREADS="1", OPENBLAS_NUM_THREADS="1", MKL_NUM_THREADS="1",
               NUMBA_NUM_THREADS="1", NUMBA_CACHE_DIR="/tmp/numba_cache",
               PYTHONPATH=REF)
    procs = [subprocess.Popen([sys.executable, "-c", CHILD, kind, str(c), str(FR), REF], env=env,
                              stdout=subprocess.PIPE, text=True) for c in cores]
    return [float(p.communicate()[0].strip().splitlines()[-1]) for p in procs]


def main():
    cpus = sorted(os.sched_getaffinity(0))
    out = {"host_cores": len(cpus), "frames": FR, "scene": "build_snake(SceneConfig())",
           "reference": REF if not BOX else "baseline/_ref (softsnake 0.1.0, unmodified)",
           "host": "GPU box" if BOX else "build container"}
    try:
        out["cpu_model"] = [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo")
                            if l.startswith("model name")][0]
    except (OSError, IndexError):
        pass
    for kind in ("numba", "port"):
        one = run(kind, cpus[:1])[0]
        allc = run(kind, cpus)
        out[kind] = {"per_core_1proc": one, "aggregate_all_cores": sum(allc),
                     "per_core_all": [round(x, 3) for x in allc]}
    out["port_over_numba_per_core"] = out["port"]["per_core_1proc"] / out["numba"]["per_core_1proc"]
    out["port_over_numba_aggregate"] = (out["port"]["aggregate_all_cores"]
                                       / out["numba"]["aggregate_all_cores"])
    out["when"] = time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    name = "cpu_host_numba.json" if BOX else "cpu_calibration.json"
    with open(os.path.join(ROOT, "profiles", name), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()

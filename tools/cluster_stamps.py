import ctypes as C, os, sys
os.environ["SS_CLUSTER_STAMPS"] = "16"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_1904_02833_b200 as M
from paper_1904_02833_b200 import _native
n = int(sys.argv[1]) if len(sys.argv) > 1 else 7
model = M.build_snake(M.SceneConfig(), n_envs=n)
sim = model.sim
sim.config.solver = "cluster"
cmds = bench.env_commands(n, 3, 0)
sim.step(cmds[:2], True, 2)
sim.synchronize()
L = _native.lib()
L.ss_cluster_stamps.argtypes = [C.c_void_p, C.POINTER(C.c_longlong)]
buf = (C.c_longlong * 256)()
_native.check(L.ss_cluster_stamps(sim._ensure(), buf))
names = ["iter start", "step+JT done", "sync1", "gather done", "sync2", "apply done",
         "rho reduce", "dir done", "den reduce"]
# per-CTA phase durations (clock64 is per SM: compare durations, not stamps)
ncta = sum(1 for c in range(16) if buf[16 * c] != 0)
print("phase".ljust(14), " ".join(f"{c:6d}" for c in range(ncta)))
for i in range(1, len(names)):
    d = [buf[16 * c + i] - buf[16 * c + i - 1] for c in range(ncta)]
    print(f"{names[i]:14s}", " ".join(f"{x:6d}" for x in d))
for nm, a, b in (("JT all warps", 0, 10), ("gather all", 2, 11), ("apply all", 4, 12),
                  ("reduce only", 12, 6)):
    d = [buf[16 * c + b] - buf[16 * c + a] for c in range(ncta)]
    print(f"{nm:14s}", " ".join(f"{x:6d}" for x in d))
tot = [buf[16 * c + len(names) - 1] - buf[16 * c] for c in range(ncta)]
print(f"{'total':14s}", " ".join(f"{x:6d}" for x in tot))

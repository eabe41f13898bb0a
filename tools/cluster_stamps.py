import ctypes as C, os, sys
os.environ["SS_CLUSTER_STAMPS"] = "1"
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
buf = (C.c_longlong * 16)()
_native.check(L.ss_cluster_stamps(sim._ensure(), buf))
names = ["iter start", "step+JT done", "sync1", "gather done", "sync2", "apply done",
         "rho reduce", "dir done", "den reduce"]
t0 = buf[0]
prev = t0
for i, nm in enumerate(names):
    print(f"{nm:14s} {buf[i]-t0:8d}  (+{buf[i]-prev})")
    prev = buf[i]

"""Step a coupled n-snake scene (one system, Table II shape) for a few
frames: the command behind the per-launch ncu list of a coupled scene
(`ncu --metrics gpu__time_duration.sum ... python tools/coupled_frames.py 2`)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_02833_b200 as M  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 4
m = M.build_snake(M.SceneConfig(), n_snakes=n)
sim = m.sim
for i in range(frames):
    sim.step(m.commands(i * sim.config.dt), latency=True)
sim.synchronize()
print("launches/frame", sim.launches_per_frame)

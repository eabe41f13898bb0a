"""Long-horizon golden: the reference's default
gait on the snake for 600 frames (10 s, latency on), COM every 10 frames and
the distance travelled. Beyond ~30 frames trajectories are chaotic (the
reference's numba and numpy backends diverge), so this golden gates the
locomotion statistics, not the trajectory.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nc \
        python tests/golden/make_golden_long.py [backend]      # ~4 min
"""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import softsnake as R  # noqa: E402
from softsnake.state import center_of_mass  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def main(backend="numba"):
    sc = R.SceneConfig(backend=backend)
    m = R.build_snake(sc)
    sim = m.sim
    com = [center_of_mass(sim.state)]
    curv, contacts = [], []
    for i in range(600):
        st = sim.step(m.commands(i * sim.config.dt), latency=True)
        curv.append([m.link_curvature(k) for k in range(m.links_per_snake)])
        contacts.append(st.contact_count)
        if (i + 1) % 10 == 0:
            com.append(center_of_mass(sim.state))
    com = np.array(com)
    name = "long_S.npz" if backend == "numba" else f"long_S_{backend}.npz"
    np.savez_compressed(os.path.join(OUT, name), com=com, frames=np.int64(600),
                        curvature=np.array(curv), contacts=np.array(contacts))
    print(name, com[-1] - com[0], np.sqrt(np.mean(np.array(curv) ** 2, axis=0)),
          np.mean(contacts), com[:, 2].mean())


if __name__ == "__main__":
    main(*sys.argv[1:])

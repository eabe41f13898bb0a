"""Device ms per frame of coupled n-snake scenes (Table II shape) and of the
bend fixture: python tools/table2_quick.py [n ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_02833_b200 as M  # noqa: E402
from paper_1904_02833_b200 import rollout  # noqa: E402

counts = tuple(int(x) for x in sys.argv[1:]) or (1, 2, 4)
rows = rollout.benchmark(M.SceneConfig(), counts, frames=30, warmup=5)
print(" ".join(f"{r['snakes']}:{r['total_ms']:.3f}ms({r['solver'][0]}"
               f"{r['clusters_per_env']}x{r['cluster_size']})" for r in rows))

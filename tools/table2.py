"""The paper's Table II (harness.run_benchmark) on one B200: device time per
frame for the single link and coupled 1/2/4/7/10-snake scenes."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_02833_b200 as M  # noqa: E402
from paper_1904_02833_b200 import rollout  # noqa: E402

rows = rollout.benchmark(M.SceneConfig(), snake_counts=(1, 2, 4, 7, 10), frames=30, warmup=3)
for r in rows:
    print(json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in r.items()}))

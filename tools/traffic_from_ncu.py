"""profiles/traffic.json from an ncu --set full report: mean DRAM bytes
(dram__bytes_read.sum + dram__bytes_write.sum) per launch of each kernel.
Usage: python tools/traffic_from_ncu.py gpurun_out/s_full.ncu-rep [envs] [out name]"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
envs = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]
ki, ri, wi = h.index("Kernel Name"), h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
acc = defaultdict(list)
for r in rows[2:]:
    name = r[ki].split("(")[0].replace("void ", "").split("<")[0]
    b = float(r[ri]) * scale[units[ri]] + float(r[wi]) * scale[units[wi]]
    acc[name].append(b)
out = {k: sum(v) / len(v) for k, v in acc.items()}
out["_envs"] = envs
out["_source"] = os.path.basename(rep)
name = sys.argv[3] if len(sys.argv) > 3 else "traffic.json"  # traffic_H.json: the 1M-tet scene
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", name)
json.dump(out, open(path, "w"), indent=1)
print(json.dumps(out, indent=1))

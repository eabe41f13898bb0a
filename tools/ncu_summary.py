"""Per-kernel table from an ncu report (--set full): duration, DRAM bytes,
DRAM throughput %, L1/L2 hit rates, achieved occupancy, registers.
python tools/ncu_summary.py REPORT"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
want = {"gpu__time_duration.sum": "us", "dram__bytes_read.sum": "rd", "dram__bytes_write.sum": "wr",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram%",
        "sm__warps_active.avg.pct_of_peak_sustained_active": "occ%",
        "lts__t_sector_hit_rate.pct": "L2hit%", "l1tex__t_sector_hit_rate.pct": "L1hit%",
        "launch__registers_per_thread": "regs",
        "smsp__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64%"}
idx = {k: h.index(k) for k in want if k in h}
units = rows[1]
agg = defaultdict(list)
for r in rows[2:]:
    name = r[h.index("Kernel Name")].split("(")[0]
    vals = {}
    for k, i in idx.items():
        try:
            v = float(r[i].replace(",", ""))
        except ValueError:
            continue
        u = units[i]
        if k == "gpu__time_duration.sum":
            v = v / 1e3 if u == "ns" else (v * 1e3 if u == "ms" else v)
        if k.startswith("dram__bytes"):
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            v *= scale
        vals[want[k]] = v
    agg[name].append(vals)
print(f"{'kernel':28s} {'n':>3s} {'us':>9s} {'DRAM GB':>8s} {'dram%':>6s} {'L1hit%':>7s} {'L2hit%':>7s} {'occ%':>5s} {'fp64%':>6s} {'regs':>5s}")
for k, L in agg.items():
    n = len(L)
    m = lambda key: sum(x.get(key, 0.0) for x in L) / n  # noqa: E731
    print(f"{k:28s} {n:3d} {m('us'):9.1f} {(m('rd') + m('wr')) / 1e9:8.3f} {m('dram%'):6.1f} "
          f"{m('L1hit%'):7.1f} {m('L2hit%'):7.1f} {m('occ%'):5.1f} {m('fp64%'):6.1f} {m('regs'):5.0f}")

"""Markdown table (one row per kernel, mean over its captured launches) from
an ncu --set full report: duration, DRAM bytes, DRAM % of peak, FP64 pipe,
warps active, registers. Usage: python tools/ncu_table.py report.ncu-rep"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

COLS = [("gpu__time_duration.sum", "duration", 1e-3, "us"),
        ("dram__bytes_read.sum", "DRAM read", None, ""),
        ("dram__bytes_write.sum", "DRAM write", None, ""),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak", 1, "%"),
        ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe %", 1, "%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %", 1, "%"),
        ("launch__registers_per_thread", "regs", 1, "")]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1,
         "msecond": 1e3, "ns": 1e-3, "us": 1, "ms": 1e3}

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]
ki = h.index("Kernel Name")
acc = defaultdict(lambda: defaultdict(list))
for r in rows[2:]:
    name = r[ki].split("(")[0].replace("void ", "")
    for key, *_ in COLS:
        i = h.index(key)
        v = float(r[i].replace(",", ""))
        u = units[i]
        if u in SCALE and key != "launch__registers_per_thread":
            v *= SCALE[u]
        acc[name][key].append(v)
print("| kernel | launches | duration (us) | DRAM read+write / launch | DRAM % peak | FP64 pipe % "
      "| warps active % | regs |")
print("|---|---|---|---|---|---|---|---|")
for name, d in acc.items():
    m = {k: sum(v) / len(v) for k, v in d.items()}
    rw = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
    print(f"| {name} | {len(d['gpu__time_duration.sum'])} | {m['gpu__time_duration.sum']:.1f} | "
          f"{rw / 1e9:.3f} GB | {m['gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed']:.1f} | "
          f"{m['sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active']:.1f} | "
          f"{m['sm__warps_active.avg.pct_of_peak_sustained_active']:.1f} | "
          f"{m['launch__registers_per_thread']:.0f} |")

"""Per-source-line warp-stall samples of one kernel from an ncu report:
python tools/ncu_lines.py REPORT KERNEL_REGEX [TOP]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass",
                      "--kernel-name", f"regex:{kern}", "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
data, fname, i_s = [], "?", None


def num(x):
    try:
        return float(x)
    except ValueError:
        return None


for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        i_s = r.index("Warp Stall Sampling (All Samples)")
        reasons = [(j, x) for j, x in enumerate(r) if x.startswith("stall_") and "Not Issued" not in x]
    elif i_s is not None and len(r) > i_s and num(r[i_s]) is not None and num(r[0]) is not None:
        rs = sorted(((num(r[j]) or 0.0, x[6:]) for j, x in reasons), reverse=True)[:2]
        why = " ".join(f"{n}:{int(v)}" for v, n in rs if v > 0)
        data.append((fname, int(r[0]), r[1] + "   [" + why + "]", num(r[i_s])))
tot = sum(d[3] for d in data)
best = sorted(data, key=lambda d: -d[3])[:top]
for f, ln, src, v in sorted(best, key=lambda d: (d[0], d[1])):
    print(f"{f:>16}:{ln:<5} {100 * v / tot:5.1f}%  {src.strip()[:120]}")
print("total samples", tot)

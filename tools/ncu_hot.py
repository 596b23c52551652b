"""Top stall-sampled SASS instructions of an ncu report (source page).

    python tools/ncu_hot.py report.ncu-rep [N]
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
si, ai = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    try:
        data.append((float(r[ai]), r[h.index("Address")][-5:], r[si].strip()))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
for i, (s, a, src) in enumerate(data):
    data[i] = (s, a, src, i)
for s, a, src, i in sorted(data, reverse=True)[:n]:
    print(f"{s / tot:6.3f}  #{i:4d} {a}  {src[:100]}")

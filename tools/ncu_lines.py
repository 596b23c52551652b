"""Stall samples per CUDA source line of an ncu report (cuda,sass view).

    python tools/ncu_lines.py report.ncu-rep [N]
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname = ""
data = []
hdr = None
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "" or r[0] == "Function Name":
        continue
    try:
        s = float(r[hdr.index("Warp Stall Sampling (All Samples)")])
    except (ValueError, IndexError):
        continue
    data.append((s, f"{fname}:{r[0]}", r[1].strip()))
tot = sum(d[0] for d in data) or 1
for s, loc, src in sorted(data, reverse=True)[:n]:
    print(f"{s / tot:6.3f} {loc:22s} {src[:100]}")

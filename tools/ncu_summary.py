"""Summarise ncu reports (and a launch-list CSV) into markdown + JSON.

    python tools/ncu_summary.py OUT_PREFIX gpurun_out/prof_*.ncu-rep [--launches gpurun_out/launches.csv]

Writes OUT_PREFIX.md and OUT_PREFIX.json (per kernel: duration, DRAM bytes,
fp64 pipe %, occupancy, top stall reasons).  bench.py reads
profiles/ncu_traffic.json (kernel -> dram bytes per launch) for
roofline.traffic.
"""

from __future__ import annotations

import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "launch__registers_per_thread": "regs",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1tex_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum": "dfma",
    "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum": "dmul",
    "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum": "dadd",
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
        "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9, "s": 1.0}


def read_report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    h, units = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        d = {"kernel": v[h.index("Kernel Name")] if "Kernel Name" in h else path}
        for k, name in KEYS.items():
            if k in h:
                i = h.index(k)
                try:
                    x = float(v[i].replace(",", ""))
                except ValueError:
                    continue
                d[name] = x * UNIT.get(units[i], 1.0) if name in ("duration", "dram_read", "dram_write") else x
        stalls = []
        for i, n in enumerate(h):
            if "average_warps_issue_stalled" in n and n.endswith("per_issue_active.ratio"):
                try:
                    stalls.append((float(v[i]), n.split("stalled_")[1].split("_per")[0]))
                except ValueError:
                    pass
        d["top_stalls"] = [f"{s[1]}={s[0]:.1f}" for s in sorted(stalls, reverse=True)[:4]]
        res.append(d)
    return res


def short(name: str) -> str:
    base = name.split("(")[0].replace("void ", "")
    return base.split("::")[-1]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = None
    for i, r in enumerate(rows):
        if "Kernel Name" in r and "Metric Value" in r:
            hi = i
            break
    if hi is None:
        return {}
    h = rows[hi]
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) != len(h) or r[h.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        k = short(r[h.index("Kernel Name")])
        unit = r[h.index("Metric Unit")]
        agg[k][0] += 1
        agg[k][1] += float(r[h.index("Metric Value")].replace(",", "")) * UNIT.get(unit, 1e-9)
    return dict(agg)


def main():
    prefix = sys.argv[1]
    reps = [a for a in sys.argv[2:] if a.endswith(".ncu-rep")]
    lpath = sys.argv[sys.argv.index("--launches") + 1] if "--launches" in sys.argv else None
    kern = []
    for p in reps:
        for d in read_report(p):
            d["report"] = p.split("/")[-1]
            kern.append(d)
    md = ["| report | kernel | us | DRAM rd MB | DRAM wr MB | fp64 pipe % | DRAM % | L1tex % | warps % | regs | stalls |",
          "|---|---|---|---|---|---|---|---|---|---|---|"]
    for d in kern:
        md.append(f"| {d['report']} | {short(d['kernel'])[:60]} | {d.get('duration', 0) * 1e6:.1f} | "
                  f"{d.get('dram_read', 0) / 1e6:.1f} | {d.get('dram_write', 0) / 1e6:.1f} | "
                  f"{d.get('fp64_pipe_pct', 0):.1f} | {d.get('dram_pct', 0):.1f} | {d.get('l1tex_pct', 0):.1f} | "
                  f"{d.get('warps_active_pct', 0):.1f} | {d.get('regs', 0):.0f} | {' '.join(d['top_stalls'])} |")
    out = {"kernels": kern}
    if lpath:
        la = launches(lpath)
        tot = sum(v[1] for v in la.values()) or 1.0
        md += ["", "Launch list (ncu, cold-cache, serialised): kernel, launches, total us, share",
               "", "| kernel | launches | total us | share |", "|---|---|---|---|"]
        for k, (n, t) in sorted(la.items(), key=lambda kv: -kv[1][1]):
            md.append(f"| {k[:70]} | {n} | {t * 1e6:.1f} | {t / tot:.3f} |")
        out["launches"] = {k: {"n": v[0], "total_s": v[1], "share": v[1] / tot} for k, v in la.items()}
    open(prefix + ".md", "w").write("\n".join(md) + "\n")
    open(prefix + ".json", "w").write(json.dumps(out, indent=1))
    print("\n".join(md))


if __name__ == "__main__":
    main()

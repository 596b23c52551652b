"""Per-kernel DRAM traffic and fp64 work of one full time step from an ncu
metrics CSV (tools/profile_step_c4.py under
`ncu --profile-from-start off --metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum,
smsp__sass_thread_inst_executed_op_{dfma,dmul,dadd}_pred_on.sum --csv`),
mapped onto bench.py's timeline names.  Writes the JSON bench.py reads for
roofline.traffic (profiles/ncu_traffic_c4.json) and a markdown table.

    python tools/ncu_step_traffic.py gpurun_out/r2_c4_step_metrics_v2.csv profiles/ncu_traffic_c4.json \
        profiles/r2_c4_step_v2.md
"""

from __future__ import annotations

import csv
import json
import re
import sys
from collections import defaultdict

RULES = {0: "tet1", 1: "tet4", 2: "pyr5", 3: "pri6", 4: "hex8"}
NAMES = [  # (regex on the demangled kernel name, bench timeline label)
    (r"k_pipe<(\d), 0, 128", "K2_momentum[{}]"),
    (r"k_wall_gather", "K8_wall_gather"),
    (r"k_wall", "K8_wall"),
    (r"k_rk_stage", "K3_rk_stage"),
    (r"k_go_div", "K4_divergence"),
    (r"k_go_grad", "K67_grad_correct"),
    (r"k_cg_tile_iter", "K5_cg_tile_iter"),
    (r"k_cg_tile_init", "K5_cg_init"),
    (r"k_cg_tile_finish", "K5_cg_finish"),
    (r"k_cg_spmv", "K5_cg_spmv"),
    (r"k_cg_update_scaled", "K5_cg_update_scaled"),
    (r"k_cg_update", "K5_cg_update"),
    (r"k_cg_init", "K5_cg_init"),
    (r"k_cg_finish", "K5_cg_finish"),
    (r"k_velocity_bc", "velocity_bc"),
]


def label(kernel: str) -> str:
    for rx, lab in NAMES:
        m = re.search(rx, kernel)
        if m:
            return lab.format(RULES[int(m.group(1))]) if "{}" in lab else lab
    return kernel.split("(")[0].replace("void ", "")


def main(src: str, out_json: str, out_md: str | None = None):
    rows = [r for r in csv.reader(line for line in open(src) if line.startswith('"'))]
    hdr = rows[0]
    ix = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value")}
    per = defaultdict(dict)  # launch id -> metrics
    names = {}
    for r in rows[1:]:
        lid = int(r[ix["ID"]])
        names[lid] = r[ix["Kernel Name"]]
        per[lid][r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
    agg = defaultdict(lambda: defaultdict(float))
    cnt = defaultdict(int)
    for lid, m in per.items():
        lab = label(names[lid])
        cnt[lab] += 1
        a = agg[lab]
        a["ncu_us"] += m.get("gpu__time_duration.sum", 0.0) / 1e3
        a["dram_read"] += m.get("dram__bytes_read.sum", 0.0)
        a["dram_write"] += m.get("dram__bytes_write.sum", 0.0)
        a["flops"] += (2 * m.get("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", 0.0)
                       + m.get("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum", 0.0)
                       + m.get("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", 0.0))
    kernels = {}
    for lab, a in agg.items():
        n = cnt[lab]
        kernels[lab] = {"launches": n, "ncu_us": a["ncu_us"] / n, "dram_read": a["dram_read"] / n,
                        "dram_write": a["dram_write"] / n, "dram_bytes": (a["dram_read"] + a["dram_write"]) / n,
                        "flops": a["flops"] / n}
    # K2 per RK stage = the per-category launches of one stage
    k2 = [k for k in kernels if k.startswith("K2_momentum[")]
    if k2:
        kernels["K2_momentum"] = {"ncu_us": sum(kernels[k]["ncu_us"] for k in k2),
                                  "dram_bytes": sum(kernels[k]["dram_bytes"] for k in k2),
                                  "flops": sum(kernels[k]["flops"] for k in k2),
                                  "_note": "sum of the per-category launches of one stage"}
    traffic = {k: v["dram_bytes"] for k, v in kernels.items() if k.startswith("K")}
    traffic["_note"] = (f"dram__bytes_read.sum + dram__bytes_write.sum per launch (K2: per stage, all category "
                        f"launches) from {src.split('/')[-1]} (ncu, one full step of tools/profile_step_c4.py)")
    json.dump({"traffic": traffic, "kernels": kernels}, open(out_json, "w"), indent=1)
    if out_md:
        tot = sum(v["ncu_us"] * v.get("launches", 0) for k, v in kernels.items() if "launches" in v)
        lines = ["| kernel | launches | ncu µs/launch | share of step | DRAM GB/launch | DRAM TB/s | fp64 GFLOP/launch |",
                 "|---|---|---|---|---|---|---|"]
        for k, v in sorted(kernels.items(), key=lambda kv: -kv[1]["ncu_us"] * kv[1].get("launches", 0)):
            if "launches" not in v:
                continue
            tbs = v["dram_bytes"] / (v["ncu_us"] * 1e-6) / 1e12 if v["ncu_us"] else 0
            lines.append(f"| {k} | {v['launches']} | {v['ncu_us']:.1f} | {100 * v['ncu_us'] * v['launches'] / tot:.1f}% | "
                         f"{v['dram_bytes'] / 1e9:.3f} | {tbs:.2f} | {v['flops'] / 1e9:.2f} |")
        open(out_md, "w").write("\n".join(lines) + "\n")
        print("\n".join(lines))


if __name__ == "__main__":
    main(*sys.argv[1:4])

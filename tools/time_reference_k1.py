"""Calibration run IN THE BUILD CONTAINER (it imports the reference from
/root/reference, which does not exist on the GPU box): the reference's own
kernel `assemble_packs` (assembly.py:227-244, pack build excluded, median of
reps after one warm-up: sweep_pack_size semantics, assembly.py:348-373)
against the oracle's restatement `fem.element_mass` (the CPU leg bench.py
times on the B200 host, `k1_mass.cpu_port`) on the same jittered C2-recipe
sample, single-threaded.  Writes profiles/r2_reference_k1_calibration.json.

    python tools/time_reference_k1.py [n_cells]
"""
import json
import os
import sys
import time
from pathlib import Path

os.environ.setdefault("OMP_NUM_THREADS", "1")
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402
from threadpoolctl import threadpool_limits  # noqa: E402

from oracle import fem  # noqa: E402
from paper_2005_05899_b200 import meshgen  # noqa: E402

import coexbal.assembly as ref  # noqa: E402
import coexbal.mesh as refmesh  # noqa: E402


def reference_full_mesh(m):
    """The reference's own FullMesh (its ElementKind objects) of an array mesh."""
    elems = []
    for _tag, rule, conn, _ids in m.categories():
        kind = refmesh.ElementKind(rule[:3])
        elems += [refmesh.FullElement(kind=kind, conn=tuple(int(v) for v in c), rule=rule) for c in conn]
    return refmesh.FullMesh(nodes=m.coords, elements=tuple(elems))


def median_time(fn, reps=5):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts))


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    m = meshgen.box_tets(n, n, n, jitter=0.2, seed=20200131)
    full = reference_full_mesh(m)
    E = m.n_elements
    out = {"sample": f"jittered Kuhn TET04 {n}^3 cells ({E} elements), C2 recipe", "threads": 1}
    with threadpool_limits(1):
        for ps in (32, 256):
            packs = ref.build_packs(full, ps)
            t = median_time(lambda: ref.assemble_packs(packs))
            out[f"reference_assemble_packs_pack{ps}_Melem_s"] = E / t / 1e6
        conn = m.conn["tet4"]
        X = fem.element_coords(m.coords, conn)
        t = median_time(lambda: fem.element_mass(X, "tet4"))
        out["oracle_element_mass_Melem_s"] = E / t / 1e6
    out["port_over_reference"] = out["oracle_element_mass_Melem_s"] / out["reference_assemble_packs_pack32_Melem_s"]
    out["cpu_model"] = next((l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")),
                            "unknown")
    out["where"] = "build container (the reference is not on the GPU box)"
    p = ROOT / "profiles" / "r2_reference_k1_calibration.json"
    p.write_text(json.dumps(out, indent=1))
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()

"""SpMV/CG variants on a DRAM-resident system (C3 Laplacian, 5.6M rows):
int32 vs 16-bit columns, Jacobi z-form vs the symmetrically scaled form.
Graph-replayed 50-iteration solves, L2 flushed before each, device time.

    python tools/lab/time_spmv16.py [scale] [variant,variant,...]

The 16-bit variants need the column-compressed SELL of tools/lab/cg_sell16.cu
built back into the library (it left the product in round 2).
"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np, torch  # noqa: E401,E402
from paper_2005_05899_b200 import meshgen  # noqa: E402
from paper_2005_05899_b200.device import DeviceMesh  # noqa: E402
from paper_2005_05899_b200.solver import PCG, assemble_laplacian  # noqa: E402

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
m = meshgen.c3_mesh(scale)
bc, _ = meshgen.wall_model_bcs(m)
fixed = torch.from_numpy(bc["p_fixed"])
dm = DeviceMesh(m)
A = assemble_laplacian(dm, fixed)
order = dm.node_order()
b = torch.randn(A.n_rows, dtype=torch.float64, device="cuda")
b[fixed.cuda()] = 0
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
ref = None
VARIANTS = {"int32-jacobi": dict(compress_cols=False, scaled=False),
            "16-jacobi": dict(compress_cols=True, scaled=False),
            "int32-scaled-diag": dict(compress_cols=False, unit_diag=False),
            "16-scaled-diag": dict(compress_cols=True),
            "int32-scaled-unit": dict(compress_cols=False, unit_diag=True)}
only = sys.argv[2].split(",") if len(sys.argv) > 2 else list(VARIANTS)
for name, kw in ((k, VARIANTS[k]) for k in only):
    pcg = PCG(A, 1.0 / A.diag, fixed=fixed, order=order, resident=False, **kw)
    work = b.clone()
    pcg.solve(work, 50, zero_b=False)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        pcg.solve(work, 50, zero_b=False)
    ts = []
    for _ in range(8):
        flush.fill_(1)
        a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); c.record(); c.synchronize()
        ts.append(a.elapsed_time(c))
    x = pcg.perm2["x"].clone()
    if ref is None:
        ref = x
    d = float((x - ref).norm() / ref.norm())
    near = round(pcg.perm2["A16"]["near_fraction"], 4) if pcg.perm2["A16"] is not None else None
    print(f"{name:14s} {np.median(ts) * 1e3 / 50:8.1f} us/iteration  rel-diff {d:.2e}  near {near}", flush=True)

"""Device time of one C2 pressure solve (50 iterations) per CG variant, L2
flushed before every solve (as in bench.py), plus agreement of the iterates.

    python tools/time_cg_variants.py [cells]
"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch  # noqa: E401,E402
from paper_2005_05899_b200 import meshgen  # noqa: E402
from paper_2005_05899_b200.device import DeviceMesh  # noqa: E402
from paper_2005_05899_b200.solver import PCG, assemble_laplacian  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 88
its = 50
m = meshgen.box_tets(n, n, n, jitter=0.2, seed=20200131)
fixed = torch.from_numpy(meshgen.boundary_nodes(m))
dm = DeviceMesh(m)
A = assemble_laplacian(dm, fixed)
dinv = 1.0 / A.diag
b = torch.randn(A.n_rows, dtype=torch.float64, device="cuda")
b[fixed.cuda()] = 0
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
order = dm.node_order()
depths = [int(k) for k in sys.argv[2].split(",")] if len(sys.argv) > 2 else []
variants = {
    "local+sfc": dict(order=order),
    **{f"depth{k}": dict(order=order, prefetch_depth=k) for k in depths},
    "local": dict(),
    "two-kernel": dict(resident=False),
}
ref = None
for name, kw in variants.items():
    pcg = PCG(A, dinv, fixed=fixed, **kw)
    info = ""
    if pcg.local is not None:
        info = f"max_ghost={pcg.local['max_ghost']} stored={pcg.local['A'].nnz_stored}"
    pcg.solve(b.clone(), its, zero_b=False)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        pcg.solve(b, its, zero_b=False)
    ts = []
    for _ in range(10):
        flush.zero_()
        a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); c.record(); c.synchronize()
        ts.append(a.elapsed_time(c))
    x = pcg.x.double().cpu().numpy().copy()
    if ref is None:
        ref = x
    d = np.linalg.norm(x - ref) / np.linalg.norm(ref)
    print(f"{name:11s}: {np.median(ts) * 1e3 / its:6.2f} us/iteration (min {min(ts) * 1e3 / its:6.2f})  "
          f"res={pcg.residual():.6e} rel.diff={d:.2e} {info}", flush=True)

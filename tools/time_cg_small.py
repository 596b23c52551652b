"""Fixed per-iteration cost of the resident CG: time it on small systems."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch  # noqa: E401,E402
from paper_2005_05899_b200 import meshgen  # noqa: E402
from paper_2005_05899_b200.solver import PCG, assemble_laplacian  # noqa: E402

for n in (8, 20, 40, 60, 88):
    m = meshgen.box_tets(n, n, n, jitter=0.2)
    fixed = torch.from_numpy(meshgen.boundary_nodes(m))
    A = assemble_laplacian(m, fixed)
    b = torch.randn(A.n_rows, dtype=torch.float64, device="cuda")
    out = []
    for resident in (True, False):
        pcg = PCG(A, 1.0 / A.diag, fixed=fixed, resident=resident)
        pcg.solve(b.clone(), 50, zero_b=False)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            pcg.solve(b, 50, zero_b=False)
        ts = []
        for _ in range(10):
            a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); g.replay(); c.record(); c.synchronize()
            ts.append(a.elapsed_time(c))
        out.append(np.median(ts) * 1e3 / 50)
    print(f"cells {n}^3 rows {A.n_rows}: resident {out[0]:.2f} us/it, two-kernel {out[1]:.2f} us/it")

"""Device time of one C2 pressure solve (50 iterations) per CG path."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch  # noqa: E401,E402
from paper_2005_05899_b200 import meshgen  # noqa: E402
from paper_2005_05899_b200.solver import PCG, assemble_laplacian  # noqa: E402

m = meshgen.c2_mesh()
fixed = torch.from_numpy(meshgen.boundary_nodes(m))
A = assemble_laplacian(m, fixed)
b = torch.randn(A.n_rows, dtype=torch.float64, device="cuda")
b[fixed.cuda()] = 0
for resident in (True, False):
    pcg = PCG(A, 1.0 / A.diag, fixed=fixed, resident=resident)
    g = torch.cuda.CUDAGraph()
    pcg.solve(b.clone(), 50, zero_b=False)
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        pcg.solve(b, 50, zero_b=False)
    ts = []
    for _ in range(10):
        a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); c.record(); c.synchronize()
        ts.append(a.elapsed_time(c))
    print(f"resident={resident}: {np.median(ts) * 1e3 / 50:.2f} us/iteration  res={pcg.residual():.3e}")

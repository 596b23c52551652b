"""One C2 pressure solve (50 iterations) of a chosen CG variant, for ncu.

    python tools/ncu_cg.py [local|resident|two] [cells]
"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
from paper_2005_05899_b200 import meshgen  # noqa: E402
from paper_2005_05899_b200.device import DeviceMesh  # noqa: E402
from paper_2005_05899_b200.solver import PCG, assemble_laplacian  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "local"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 88
m = meshgen.box_tets(n, n, n, jitter=0.2, seed=20200131)
fixed = torch.from_numpy(meshgen.boundary_nodes(m))
dm = DeviceMesh(m)
A = assemble_laplacian(dm, fixed)
kw = {"local": dict(order=dm.node_order()), "two": dict(resident=False)}[kind]
pcg = PCG(A, 1.0 / A.diag, fixed=fixed, **kw)
b = torch.randn(A.n_rows, dtype=torch.float64, device="cuda")
b[fixed.cuda()] = 0
pcg.solve(b, 50, zero_b=False)
torch.cuda.synchronize()
print("ok", pcg.residual())

"""Phase timeline of one resident-CG iteration (ab_debug_timeline).

    python tools/cg_timeline.py [cells]
"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch  # noqa: E401,E402
from paper_2005_05899_b200 import meshgen  # noqa: E402
from paper_2005_05899_b200._lib import call, ptr  # noqa: E402
from paper_2005_05899_b200.device import DeviceMesh  # noqa: E402
from paper_2005_05899_b200.solver import PCG, assemble_laplacian  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 88
m = meshgen.box_tets(n, n, n, jitter=0.2, seed=20200131)
fixed = torch.from_numpy(meshgen.boundary_nodes(m))
dm = DeviceMesh(m)
A = assemble_laplacian(dm, fixed)
depth = int(sys.argv[2]) if len(sys.argv) > 2 else 1
pcg = PCG(A, 1.0 / A.diag, fixed=fixed, order=dm.node_order(), prefetch_depth=depth)
b = torch.randn(A.n_rows, dtype=torch.float64, device="cuda")
b[fixed.cuda()] = 0
tl = torch.zeros(148 * 8, dtype=torch.int64, device="cuda")
call("ab_debug_timeline", ptr(tl))
for _ in range(3):
    pcg.solve(b.clone(), 50, zero_b=False)
torch.cuda.synchronize()
call("ab_debug_timeline", None)
t = tl.view(148, 8).cpu().numpy().astype(np.float64)
t0 = t[:, 0].min()
t = (t - t0) / 1e3
names = ["top", "ghosts", "A reduced", "barrier A", "B reduced", "barrier B", "B loop done (t0)",
         "1st slice done (t0)"]
print("us since the earliest loop top: min / median / max over CTAs")
for k, nm in enumerate(names):
    print(f"{nm:20s} {t[:, k].min():7.2f} {np.median(t[:, k]):7.2f} {t[:, k].max():7.2f}")
order = [0, 1, 7, 2, 3, 6, 4, 5]
for a, b in zip(order[:-1], order[1:]):
    d = t[:, b] - t[:, a]
    print(f"{names[a]:>20s} -> {names[b]:20s}: median {np.median(d):6.2f}  max {d.max():6.2f}")

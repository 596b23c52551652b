"""50 CG iterations on the full C2 system: single-pass and two-pass vs the oracle, and repeatability."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np, torch  # noqa
from paper_2005_05899_b200 import meshgen  # noqa
from paper_2005_05899_b200.device import DeviceMesh  # noqa
from paper_2005_05899_b200.solver import PCG, assemble_laplacian  # noqa
from oracle import fem  # noqa
m = meshgen.c2_mesh()
fixed = meshgen.boundary_nodes(m)
dm = DeviceMesh(m)
A = assemble_laplacian(dm, torch.from_numpy(fixed))
b = np.random.default_rng(3).standard_normal(m.n_nodes); b[fixed] = 0
bt = torch.from_numpy(b).cuda()
L = fem.laplacian(m, fixed)
for its in (9, 50):
    xr, _, _ = fem.pcg(L, b, 1.0 / L.diagonal(), its)
    res = {}
    for name, kw in (("two", dict(single_pass=False)), ("one", dict()), ("one2", dict()), ("resident", dict(resident=True))):
        kw.setdefault("resident", False)
        pcg = PCG(A, 1.0 / A.diag, fixed=torch.from_numpy(fixed), order=dm.node_order(), **kw)
        x, it = pcg.solve(bt.clone(), its, zero_b=False)
        res[name] = x.cpu().numpy().copy()
    r = lambda a, c: np.linalg.norm(a - c) / np.linalg.norm(c)
    print(its, {k: "%.2e" % r(v, xr) for k, v in res.items()}, "one-vs-two %.2e" % r(res["one"], res["two"]),
          "repeat %.2e" % r(res["one2"], res["one"]), flush=True)

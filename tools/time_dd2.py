"""Per-iteration time of the large-subdomain decomposed CG (ab_ddcg2_*, three
launches per iteration) with P virtual ranks on one GPU, plain SELL gather vs
the tiled SpMV (k_d2_spmv_tile), and the tiled single-domain single pass for
reference; jittered tet box split by the SFC partitioner, L2 flushed before
every 50-iteration solve.  Virtual ranks run phase-major on one GPU, so the
time is that of all P ranks' rows together plus the exchange protocol.

    python tools/time_dd2.py [cells=160] [P=2] [iterations=50]
"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch  # noqa: E401,E402
from paper_2005_05899_b200 import meshgen  # noqa: E402
from paper_2005_05899_b200.decompose import decompose  # noqa: E402
from paper_2005_05899_b200.device import DeviceMesh  # noqa: E402
from paper_2005_05899_b200.partition import sfc_partition  # noqa: E402
from paper_2005_05899_b200.peer import DD2Rank, DD2Solver, virtual_dd2  # noqa: E402
from paper_2005_05899_b200.solver import PCG, assemble_laplacian  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 160
P = int(sys.argv[2]) if len(sys.argv) > 2 else 2
its = int(sys.argv[3]) if len(sys.argv) > 3 else 50
m = meshgen.box_tets(n, n, n, jitter=0.2, seed=20200131)
fixed = meshgen.boundary_nodes(m)
b = np.random.default_rng(7).standard_normal(m.n_nodes)
b[fixed] = 0.0
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def timed(fn):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        flush.zero_()
        a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); c.record(); c.synchronize()
        ts.append(a.elapsed_time(c))
    return np.median(ts) * 1e3 / its


dm = DeviceMesh(m)
A = assemble_laplacian(dm, torch.from_numpy(fixed))
dglob = A.diag.clone()
pcg = PCG(A, 1.0 / A.diag, fixed=torch.from_numpy(fixed), order=dm.node_order(), resident=False)
bt = torch.from_numpy(b).cuda()
print(f"single domain, tiled single pass: {timed(lambda: pcg.solve(bt, its, zero_b=False)):.2f} us/iteration",
      flush=True)
ref = pcg.solve(bt, its, zero_b=False)[0].cpu().numpy().copy()
del pcg
if "--oracle" in sys.argv:  # the CPU oracle's iterate (slow): which of the GPU forms drifts
    from oracle import fem  # noqa: E402
    L = fem.laplacian(m, fixed)
    xo, _, _ = fem.pcg(L, b, 1.0 / L.diagonal(), its)
    print(f"single-domain tiled single pass vs oracle: {np.linalg.norm(ref - xo) / np.linalg.norm(xo):.1e}", flush=True)
    ref = xo
parts, _, _ = sfc_partition(m, P, level=8)
subs = [decompose(m, parts, P, r) for r in range(P)]
ms = max([len(v) for _, pl in subs for v in pl.shared.values()] + [0])
for tile, single in ((0, False), (2048, False), (2048, True), (64, True)):
    ranks = []
    for r, (sub, plan) in enumerate(subs):
        sdm = DeviceMesh(sub)
        fl = torch.from_numpy(fixed[plan.l2g])
        Ar = assemble_laplacian(sdm, fl)
        dinv = 1.0 / dglob[torch.from_numpy(plan.l2g).cuda()]
        ranks.append(DD2Rank(r, P, Ar, dinv, plan.own, plan.shared, sdm.node_order(), fixed=fl, max_shared=ms,
                             tile_rows=tile, single_pass=single))
    virtual_dd2(ranks)
    bs = [torch.from_numpy(b[plan.l2g]).cuda() for _, plan in subs]
    solver = DD2Solver(ranks)
    t = timed(lambda: solver.solve(bs, its, zero_b=False))
    xs, _ = solver.solve(bs, its, zero_b=False)
    err = max(np.linalg.norm(x.cpu().numpy() - ref[pl.l2g]) / np.linalg.norm(ref[pl.l2g])
              for x, (_, pl) in zip(xs, subs))
    print(f"P={P} virtual ranks, tile_rows={tile}, single_pass={single}: {t:.2f} us/iteration (interface rows "
          f"{[r.n_if for r in ranks]}), max rel diff vs single domain {err:.1e}", flush=True)
    del ranks, solver
    torch.cuda.empty_cache()

"""Per-iteration time of the fused decomposed CG (ab_cg_dd) with P virtual
ranks on one GPU (148/P CTAs each, C2 mesh split by the SFC partitioner)
vs the single-domain resident solver: the difference is the in-kernel
exchange + cross-rank reduction overhead.

    python tools/time_ddcg.py [cells] [P,...]
"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch  # noqa: E401,E402
from oracle import fem  # noqa: E402
from paper_2005_05899_b200 import meshgen  # noqa: E402
from paper_2005_05899_b200.ddcg import DDRank, DDSolve, virtual_ranks  # noqa: E402
from paper_2005_05899_b200.decompose import decompose  # noqa: E402
from paper_2005_05899_b200.device import DeviceMesh  # noqa: E402
from paper_2005_05899_b200.partition import sfc_partition  # noqa: E402
from paper_2005_05899_b200.solver import PCG, assemble_laplacian  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 88
Ps = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 2, 4]
its = 50
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
pcg = PCG(A, 1.0 / A.diag, fixed=torch.from_numpy(fixed), order=dm.node_order())
bt = torch.from_numpy(b).cuda()
print(f"single domain resident (local map): {timed(lambda: pcg.solve(bt, its, zero_b=False)):.2f} us/iteration")
ref = pcg.x.cpu().numpy().copy()
for P in Ps:
    parts, _, _ = sfc_partition(m, P, level=8)
    subs = [decompose(m, parts, P, r) for r in range(P)]
    ms = max([len(v) for _, pl in subs for v in pl.shared.values()] + [0])
    ranks = []
    for r, (sub, plan) in enumerate(subs):
        sdm = DeviceMesh(sub)
        fl = torch.from_numpy(fixed[plan.l2g])
        Ar = assemble_laplacian(sdm, fl)
        dinv = 1.0 / dglob[torch.from_numpy(plan.l2g).cuda()]
        ranks.append(DDRank(r, P, Ar, dinv, plan.own, plan.shared, sdm.node_order(), 148 // P, fixed=fl,
                            max_shared=ms))
    virtual_ranks(ranks)
    bs = [torch.from_numpy(b[plan.l2g]).cuda() for _, plan in subs]
    solve = DDSolve(ranks, bs, zero_b=False)
    t = timed(lambda: solve.run(its))
    err = max(np.linalg.norm(r.x.cpu().numpy() - ref[pl.l2g]) / np.linalg.norm(ref[pl.l2g])
              for r, (_, pl) in zip(ranks, subs))
    nif = sum(int(r.rrow.numel()) for r in ranks)
    print(f"P={P} virtual ranks ({[r.n_cta for r in ranks]} CTAs, {nif} interface rows): {t:.2f} us/iteration, "
          f"max rel diff vs single domain {err:.1e}, iterations {[r.iterations for r in ranks]}")

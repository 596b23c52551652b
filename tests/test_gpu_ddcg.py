"""The decomposed pressure solve fused with its interface exchange
(ab_cg_dd, paper_2005_05899_b200/ddcg.py) against the single-domain oracle.

The ranks are "virtual": CTA groups of one cooperative launch on one GPU,
whose peer pointers are the other groups' device buffers - the same kernel
and protocol (peer stores, arrival counters, {value, epoch} reduction
records) a multi-GPU run drives over NVLink with IPC-mapped buffers."""

import numpy as np
import pytest
import torch

from conftest import rel_l2
from oracle import fem
from paper_2005_05899_b200 import meshgen

pytestmark = pytest.mark.gpu


def _setup(m, n_ranks, ctas_per_rank):
    from paper_2005_05899_b200.ddcg import DDRank, virtual_ranks
    from paper_2005_05899_b200.decompose import decompose
    from paper_2005_05899_b200.device import DeviceMesh
    from paper_2005_05899_b200.partition import sfc_partition
    from paper_2005_05899_b200.solver import assemble_laplacian
    fixed = meshgen.boundary_nodes(m)
    L = fem.laplacian(m, fixed)
    dglob = L.diagonal()
    parts, _, _ = sfc_partition(m, n_ranks, level=6)
    subs = [decompose(m, parts, n_ranks, r) for r in range(n_ranks)]
    max_shared = max([len(v) for _, plan in subs for v in plan.shared.values()] + [0])
    ranks = []
    for r, (sub, plan) in enumerate(subs):
        dm = DeviceMesh(sub)
        fl = torch.from_numpy(fixed[plan.l2g])
        A = assemble_laplacian(dm, fl)
        dinv = torch.from_numpy(1.0 / dglob[plan.l2g]).cuda()
        ranks.append(DDRank(r, n_ranks, A, dinv, plan.own, plan.shared, dm.node_order(), ctas_per_rank,
                            fixed=fl, max_shared=max_shared))
    virtual_ranks(ranks)
    return L, fixed, subs, ranks


@pytest.mark.parametrize("n_ranks", [2, 3])
def test_dd_cg_matches_single_domain(n_ranks):
    from paper_2005_05899_b200.ddcg import DDSolve
    m = meshgen.box_tets(14, 12, 10, jitter=0.2, seed=5)
    L, fixed, subs, ranks = _setup(m, n_ranks, 148 // n_ranks)
    b = np.random.default_rng(7).standard_normal(m.n_nodes)
    b[fixed] = 0.0
    bs = [torch.from_numpy(b[plan.l2g]).cuda() for _, plan in subs]
    solve = DDSolve(ranks, bs, zero_b=False)
    # fixed iteration count: the oracle's iterate (rounding-level differences only)
    solve.run(9)
    torch.cuda.synchronize()
    xr, _, _ = fem.pcg(L, b, 1.0 / L.diagonal(), 9)
    for r, (_, plan) in zip(ranks, subs):
        assert r.iterations == 9
        assert rel_l2(r.x.cpu().numpy(), xr[plan.l2g]) <= 1e-10
    # repeated solves reuse the monotone counters/epochs (no reset races)
    for _ in range(3):
        solve.run(9)
    torch.cuda.synchronize()
    for r, (_, plan) in zip(ranks, subs):
        assert rel_l2(r.x.cpu().numpy(), xr[plan.l2g]) <= 1e-10
    # to convergence: same iteration count on every rank, matches a direct solve
    import scipy.sparse.linalg as spla
    xd = spla.spsolve(L.tocsc(), b)
    _, itr, _ = fem.pcg(L, b, 1.0 / L.diagonal(), 3000, tol=1e-12)
    solve.run(3000, tol=1e-12)
    torch.cuda.synchronize()
    its = {r.iterations for r in ranks}
    assert len(its) == 1 and abs(its.pop() - itr) <= 1
    for r, (_, plan) in zip(ranks, subs):
        assert r.residual() <= 1e-12
        assert rel_l2(r.x.cpu().numpy(), xd[plan.l2g]) <= 1e-9


def test_dd_cg_single_rank_is_the_resident_solver():
    from paper_2005_05899_b200.ddcg import DDSolve
    m = meshgen.box_tets(10, 9, 8, jitter=0.2, seed=2)
    L, fixed, subs, ranks = _setup(m, 1, 148)
    b = np.random.default_rng(1).standard_normal(m.n_nodes)
    b[fixed] = 0.0
    bt = torch.from_numpy(b).cuda()
    DDSolve(ranks, [bt], zero_b=True).run(12)
    torch.cuda.synchronize()
    xr, _, _ = fem.pcg(L, b, 1.0 / L.diagonal(), 12)
    assert rel_l2(ranks[0].x.cpu().numpy(), xr[subs[0][1].l2g]) <= 1e-10
    assert float(bt.abs().max()) == 0.0  # zero_b re-zeroes the accumulation buffer


def test_ipc_wiring_two_processes_one_gpu():
    """ddcg.ipc_ranks (CUDA IPC handles exchanged over torch.distributed, the
    multi-GPU wiring) driven by two processes sharing one GPU."""
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    r = subprocess.run([sys.executable, str(root / "tools" / "ipc_dd_check.py")], capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "ipc wiring ok" in r.stdout

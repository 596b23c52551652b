"""Multi-domain path on CPU: world_size-2 gloo processes run the product's
decomposition (decompose.py) and exchange protocol (halo.HaloExchanger) with
the decomposed-domain oracle, and must reproduce the single-domain oracle.
Also checks interface-plan invariants.  No GPU needed."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import fem
from oracle import sfc as osfc
from paper_2005_05899_b200 import meshgen
from paper_2005_05899_b200.decompose import decompose, interface_plan, submesh


def _mesh():
    return meshgen.box_tets(6, 5, 4, jitter=0.2, seed=5)


def _parts(m, P):
    cent = np.zeros((m.n_elements, 3))
    ids = np.zeros(m.n_elements, np.int64)
    w = np.zeros(m.n_elements)
    for _t, rule, conn, eids in m.categories():
        cent[eids] = osfc.centroids(m.coords, conn)
        ids[eids] = eids
        w[eids] = meshgen.GAUSS_COUNT[rule]
    parts, _, _ = osfc.partition(cent, ids, w, P, level=6)
    return parts


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.distributed import DistFlowOracle, np_pack, np_unpack_add
    from paper_2005_05899_b200.halo import HaloExchanger
    m = _mesh()
    parts = _parts(m, world)
    sub, plan = decompose(m, parts, world, rank)
    halo = HaloExchanger(plan, "cpu", pack=np_pack, unpack=np_unpack_add)
    pf = meshgen.boundary_nodes(m)[plan.l2g]
    u, p = meshgen.c2_initial(m.coords)
    o = DistFlowOracle(sub, halo, 1.0, 1e-2, 0.07, pf)
    st = o.init_state(u[plan.l2g], p[plan.l2g])
    for _ in range(2):
        st = o.step(st, 1e-3, 25)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), l2g=plan.l2g, u=st["u"], p=st["p"], own=plan.own)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_step_matches_single_domain(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    m = _mesh()
    u0, p0 = meshgen.c2_initial(m.coords)
    ora = fem.FlowOracle(m, 1.0, 1e-2, 0.07, p_fixed=meshgen.boundary_nodes(m))
    st = ora.init_state(u0, p0)
    for _ in range(2):
        st = ora.step(st, 1e-3, cg_iters=25)
    seen = np.zeros(m.n_nodes, int)
    owned = np.zeros(m.n_nodes)
    for r in range(world):
        d = np.load(tmp_path / f"r{r}.npz")
        l2g = d["l2g"]
        seen[l2g] += 1
        owned[l2g] += d["own"]
        # every copy of every node (interface duplicates included) agrees
        assert np.linalg.norm(d["u"] - st["u"][l2g]) <= 1e-10 * np.linalg.norm(st["u"][l2g])
        assert np.linalg.norm(d["p"] - st["p"][l2g]) <= 1e-10 * np.linalg.norm(st["p"][l2g])
    assert seen.min() >= 1 and seen.max() == 2
    assert np.array_equal(owned, np.ones(m.n_nodes))


@pytest.mark.parametrize("P", [2, 3, 5])
def test_interface_plan_invariants(P):
    m = meshgen.c3_mesh(0.06)
    parts = _parts(m, P)
    subs = [submesh(m, parts, r + 1) for r in range(P)]
    plans = [interface_plan(m, parts, P, r, subs[r][1]) for r in range(P)]
    own = np.zeros(m.n_nodes)
    for r, (plan, (sub, l2g)) in enumerate(zip(plans, subs)):
        assert sub.n_elements == int(np.sum(parts == r + 1))
        own[l2g] += plan.own
        for q in plan.neighbors:
            # both sides list the same global nodes in the same order
            mine = l2g[plan.shared[q]]
            theirs = plans[q].l2g[plans[q].shared[r]]
            assert np.array_equal(mine, theirs)
            assert np.all(np.diff(mine) > 0)
    assert np.array_equal(own, np.ones(m.n_nodes))
    assert sum(s[0].n_elements for s in subs) == m.n_elements


def test_throughput_coefficients():
    from paper_2005_05899_b200.balance import TimingSample, compute_metrics, throughput_coefficients
    t = np.array([2.0, 1.0, 4.0])
    w = np.array([10.0, 10.0, 10.0])
    lam = throughput_coefficients(t, w)
    assert abs(lam.sum() - 3.0) < 1e-12
    # new loads lam_i W/P at the same throughput give equal times
    new_t = lam * (w.sum() / 3) / (w / t)
    assert compute_metrics(TimingSample(1, new_t)).imbalance == pytest.approx(1.0, abs=1e-12)
    with pytest.raises(ValueError):
        throughput_coefficients([1.0, -1.0], [1.0, 1.0])

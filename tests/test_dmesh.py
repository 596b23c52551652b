"""Per-rank generation + decomposition of the boundary-layer box (dmesh.py),
on CPU: every rank's subdomain and interface plan must equal what the global
path (meshgen.boundary_layer_mesh + decompose.py) produces for the same
element assignment, and a world_size-2 gloo run of the C4 code path at
reduced scale (per-rank generation, halo-summed lumped mass and a
decomposed oracle step) must reproduce the single-domain oracle."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import fem
from oracle import sfc as osfc
from paper_2005_05899_b200 import dmesh, meshgen
from paper_2005_05899_b200.decompose import interface_plan, submesh


def cpu_keys(cells: torch.Tensor, level: int) -> torch.Tensor:
    return torch.from_numpy(osfc.hilbert_keys(cells.numpy(), level))


SPEC = dmesh.BoxSpec(14, 12, 20, 3, hex_fraction=0.25)


def _parts_from_local(spec, part):
    g = spec.global_mesh()
    parts = np.zeros(g.n_elements, np.int32)
    locs = []
    for r in range(part.n_parts):
        sub, plan = dmesh.local_mesh(spec, part, r)
        locs.append((sub, plan))
        for rule, ids in sub.elem_ids.items():
            parts[ids] = r + 1
    return g, parts, locs


@pytest.mark.parametrize("P", [1, 2, 3, 5])
def test_local_meshes_equal_global_decomposition(P):
    part = dmesh.partition_cells(SPEC, P, device="cpu", keys_fn=cpu_keys)
    assert part.weights.sum() == sum(c.shape[0] * meshgen.GAUSS_COUNT[r]
                                     for r, c in SPEC.global_mesh().conn.items())
    g, parts, locs = _parts_from_local(SPEC, part)
    assert parts.min() >= 1  # every element belongs to exactly one rank
    for r, (sub, plan) in enumerate(locs):
        ref, l2g = submesh(g, parts, r + 1)
        assert np.array_equal(plan.l2g, l2g)
        assert np.array_equal(sub.coords, ref.coords)
        assert sorted(sub.conn) == sorted(r_ for r_, c in ref.conn.items() if c.shape[0])
        for rule in sub.conn:
            assert np.array_equal(sub.conn[rule], ref.conn[rule]), rule
            assert np.array_equal(sub.elem_ids[rule], ref.elem_ids[rule]), rule
        want = interface_plan(g, parts, P, r, l2g)
        assert plan.neighbors == want.neighbors
        for q in want.neighbors:
            assert np.array_equal(plan.shared[q], want.shared[q])
        assert np.array_equal(plan.own, want.own)


def test_partition_follows_split_rule_and_coefficients():
    """Weights follow split_1d's closest-boundary rule; coefficients shift them."""
    a = dmesh.partition_cells(SPEC, 4, device="cpu", keys_fn=cpu_keys)
    W = a.weights.sum()
    assert np.all(np.abs(a.weights - W / 4) <= 24)  # one cell of slack per cut
    lam = np.array([1.3, 0.7, 1.0, 1.0])
    b = dmesh.partition_cells(SPEC, 4, coeffs=lam, device="cpu", keys_fn=cpu_keys)
    assert b.weights[0] > a.weights[0] and b.weights[1] < a.weights[1]
    assert np.all(np.abs(np.cumsum(b.weights)[:-1] - np.cumsum(lam)[:-1] * W / 4) <= 24)
    # cells of a part are contiguous along the curve: owner changes P-1 times in SFC order
    cid = torch.arange(SPEC.n_cells)
    i, j, k = SPEC.cell_ijk(cid)
    keys = cpu_keys(torch.stack([i, j, k], 1), dmesh._level(SPEC))
    o = b.owner[torch.sort(keys).indices]
    assert int((o[1:] != o[:-1]).sum()) == 3 and bool((o[1:] >= o[:-1]).all())


def test_specs_match_baseline_sizes():
    c4 = dmesh.c4_spec()
    assert c4.n_nodes == 44_485_091
    c5 = dmesh.c5_spec(8)
    n_el = c5.nx * c5.ny * (c5.nz - c5.layers) * 6 + c5.nx * c5.ny * c5.layers * 2  # upper bound of the mix
    assert 8 * 28e6 < n_el < 8 * 36e6


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


SPEC2 = dmesh.BoxSpec(10, 9, 14, 2)


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.distributed import DistFlowOracle, np_pack, np_unpack_add
    from paper_2005_05899_b200.halo import HaloExchanger
    part = dmesh.partition_cells(SPEC2, world, device="cpu", keys_fn=cpu_keys)
    sub, plan = dmesh.local_mesh(SPEC2, part, rank)       # this rank's cells only
    halo = HaloExchanger(plan, "cpu", pack=np_pack, unpack=np_unpack_add)
    bc, wall = dmesh.wall_model_bcs_local(sub, SPEC2)
    x = sub.coords
    u = np.stack([np.ones(len(x)) + 0.1 * np.sin(5 * x[:, 1]), 0.05 * np.cos(4 * x[:, 0]),
                  0.02 * np.sin(3 * x[:, 2])], axis=1)
    o = DistFlowOracle(sub, halo, 1.0, 1e-2, 0.07, bc["p_fixed"], u_fixed=bc["u_fixed"],
                       u_fixed_values=bc["u_fixed_values"], wall=wall)
    st = o.init_state(u, np.zeros(len(x)))
    st = o.step(st, 1e-3, 25)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), l2g=plan.l2g, u=st["u"], p=st["p"], ml=o.ml,
             n_el=sub.n_elements)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_c4_path_reduced_scale(tmp_path):
    """The C4 multi-GPU code path (per-rank cells, local interface plan,
    global-bounds wall-model BCs) on 2 gloo ranks vs the single-domain oracle."""
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    m = SPEC2.global_mesh()
    bc, wall = meshgen.wall_model_bcs(m)
    x = m.coords
    u = np.stack([np.ones(len(x)) + 0.1 * np.sin(5 * x[:, 1]), 0.05 * np.cos(4 * x[:, 0]),
                  0.02 * np.sin(3 * x[:, 2])], axis=1)
    ora = fem.FlowOracle(m, 1.0, 1e-2, 0.07, **bc, wall=wall)
    st = ora.step(ora.init_state(u, np.zeros(len(x))), 1e-3, cg_iters=25)
    n_el = 0
    for r in range(world):
        d = np.load(tmp_path / f"r{r}.npz")
        l2g = d["l2g"]
        n_el += int(d["n_el"])
        assert np.abs(d["ml"] - ora.ml[l2g]).max() <= 1e-14 * ora.ml.max()
        assert np.linalg.norm(d["u"] - st["u"][l2g]) <= 1e-10 * np.linalg.norm(st["u"][l2g])
        assert np.linalg.norm(d["p"] - st["p"][l2g]) <= 1e-10 * np.linalg.norm(st["p"][l2g])
    assert n_el == m.n_elements

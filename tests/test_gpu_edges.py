"""Edge cases of the GPU path against the oracle: single elements of every
kind, empty inputs, ragged sizes (node/row counts that fill no slice or CTA
evenly, fewer rows than SMs), zero right-hand sides and zero velocity."""

import numpy as np
import pytest
import torch

from conftest import rel_l2
from oracle import fem
from paper_2005_05899_b200 import meshgen
from paper_2005_05899_b200.meshgen import MeshArrays

pytestmark = pytest.mark.gpu

# one reference element of each kind (VTK node order)
_SINGLE = {
    "tet4": (np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], float), [[0, 1, 2, 3]]),
    "pyr5": (np.array([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0], [0.5, 0.5, 0.7]], float), [[0, 1, 2, 3, 4]]),
    "pri6": (np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [1, 0, 1], [0, 1, 1]], float),
             [[0, 1, 2, 3, 4, 5]]),
    "hex8": (np.array([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0], [0, 0, 1], [1, 0, 1], [1, 1, 1], [0, 1, 1]],
                      float), [[0, 1, 2, 3, 4, 5, 6, 7]]),
}


def _single(rule):
    x, conn = _SINGLE[rule]
    rng = np.random.default_rng(3)
    m = MeshArrays(coords=x + 0.05 * rng.standard_normal(x.shape))
    m.conn[rule] = np.array(conn, np.int32)
    m.elem_ids[rule] = np.zeros(1, np.int64)
    return m


@pytest.mark.parametrize("rule", list(_SINGLE))
def test_single_element_operators(rule):
    from paper_2005_05899_b200.device import DeviceMesh, nodes_as4
    from paper_2005_05899_b200.ops import assemble_divergence, assemble_gradient, assemble_momentum
    from paper_2005_05899_b200.solver import assemble_gradient_operator, assemble_laplacian
    from paper_2005_05899_b200.timestep import FlowParams
    m = _single(rule)
    rng = np.random.default_rng(1)
    u = rng.standard_normal((m.n_nodes, 3))
    p = rng.standard_normal(m.n_nodes)
    for windows in (False, True):
        dm = DeviceMesh(m, windows=windows)
        got = assemble_momentum(dm, u, FlowParams(1.1, 0.02, 0.07)).cpu().numpy()
        assert rel_l2(got, fem.momentum_rhs(m, u, 1.1, 0.02, 0.07)) <= 1e-10
        assert rel_l2(assemble_divergence(dm, u).cpu().numpy(), fem.divergence(m, u)) <= 1e-10
        assert rel_l2(assemble_gradient(dm, p).cpu().numpy(), fem.gradient(m, p)) <= 1e-10
    dm = DeviceMesh(m)
    B = assemble_gradient_operator(dm)
    out = torch.zeros(m.n_nodes, dtype=torch.float64, device="cuda")
    B.div(nodes_as4(torch.from_numpy(u).cuda()), 1.0, out)
    assert rel_l2(out.cpu().numpy(), fem.divergence(m, u)) <= 1e-10
    A = assemble_laplacian(dm)
    L = fem.laplacian(m)
    assert rel_l2(A.matvec(torch.from_numpy(p).cuda()).cpu().numpy(), L @ p) <= 1e-12


def test_empty_mesh_packs():
    from paper_2005_05899_b200.assembly import assemble_packs, build_packs
    from paper_2005_05899_b200.mesh import FullMesh
    full = FullMesh(nodes=np.zeros((0, 3)), elements=())
    assert assemble_packs(build_packs(full, 8)) == {}


@pytest.mark.parametrize("cells", [(1, 1, 1), (3, 2, 5), (2, 7, 3)])
@pytest.mark.parametrize("variant", ["local", "local-node-order", "two-kernel", "tiled-single", "tiled-64"])
def test_ragged_small_systems(cells, variant):
    """Row counts below 148 CTAs / not a multiple of the slice height."""
    from paper_2005_05899_b200.device import DeviceMesh
    from paper_2005_05899_b200.solver import PCG, assemble_laplacian
    m = meshgen.box_tets(*cells, jitter=0.15, seed=9)
    fixed = meshgen.boundary_nodes(m)
    fixed[np.argmax(m.coords.sum(axis=1))] = True
    interior = ~fixed
    if not interior.any():  # all nodes on the boundary: pin all but one
        fixed[:] = True
        fixed[0] = False
    L = fem.laplacian(m, fixed)
    b = np.random.default_rng(4).standard_normal(m.n_nodes)
    b[fixed] = 0.0
    dm = DeviceMesh(m)
    A = assemble_laplacian(dm, torch.from_numpy(fixed))
    kw = {"local": dict(order=dm.node_order()), "local-node-order": dict(), "two-kernel": dict(resident=False),
          # tiled single pass (one 2048-row tile, partial slices) / tiled SpMV with 64-row tiles
          "tiled-single": dict(order=dm.node_order(), resident=False),
          "tiled-64": dict(order=dm.node_order(), resident=False, tile_rows=64)}
    pcg = PCG(A, 1.0 / A.diag, fixed=torch.from_numpy(fixed), **kw[variant])
    if variant.startswith("tiled"):
        assert pcg.perm2["tile"] is not None and pcg.perm2["single"] == (variant == "tiled-single")
    x, it = pcg.solve(torch.from_numpy(b).cuda(), 5, zero_b=False)
    xr, _, _ = fem.pcg(L, b, 1.0 / L.diagonal(), 5)
    assert rel_l2(x.cpu().numpy(), xr) <= 1e-10
    # no iterations: x = 0
    x0, it0 = pcg.solve(torch.from_numpy(b).cuda(), 0, zero_b=False)
    assert it0 == 0 and float(x0.abs().max()) == 0.0


@pytest.mark.parametrize("variant", ["local", "two-kernel", "tiled-single"])
def test_zero_rhs_converges_immediately(variant):
    from paper_2005_05899_b200.device import DeviceMesh
    from paper_2005_05899_b200.solver import PCG, assemble_laplacian
    m = meshgen.box_tets(5, 4, 3, jitter=0.1, seed=1)
    fixed = meshgen.boundary_nodes(m)
    dm = DeviceMesh(m)
    A = assemble_laplacian(dm, torch.from_numpy(fixed))
    kw = {"local": dict(order=dm.node_order()), "two-kernel": dict(resident=False),
          "tiled-single": dict(order=dm.node_order(), resident=False)}[variant]
    pcg = PCG(A, 1.0 / A.diag, fixed=torch.from_numpy(fixed), **kw)
    x, it = pcg.solve(torch.zeros(m.n_nodes, dtype=torch.float64, device="cuda"), 100, tol=1e-10)
    assert it == 0 and float(x.abs().max()) == 0.0


def test_zero_velocity_stays_at_rest():
    from paper_2005_05899_b200.timestep import FlowParams, FlowSolver
    m = meshgen.c3_mesh(0.05)
    bc, wall = meshgen.wall_model_bcs(m)
    bc["u_fixed_values"] = np.zeros_like(bc["u_fixed_values"])  # no inflow
    fs = FlowSolver(m, FlowParams(1.0, 1e-2, 0.07), **bc, wall=wall)
    fs.set_state(np.zeros((m.n_nodes, 3)), np.zeros(m.n_nodes))
    for _ in range(2):
        fs.step(1e-3, cg_iters=20, graph=True)
    torch.cuda.synchronize()
    assert float(fs.u.abs().max()) == 0.0 and float(fs.p.abs().max()) == 0.0


@pytest.mark.parametrize("mode", [1, 2, 3, 4])
def test_resident_local_every_shared_memory_plan(mode):
    """k_cg_resident_local's four shared-memory plans (x in TMEM or global,
    tables in shared or global memory) give the oracle's iterate."""
    from paper_2005_05899_b200.device import DeviceMesh
    from paper_2005_05899_b200.solver import PCG, assemble_laplacian
    m = meshgen.box_tets(12, 9, 7, jitter=0.2, seed=6)
    fixed = meshgen.boundary_nodes(m)
    L = fem.laplacian(m, fixed)
    b = np.random.default_rng(8).standard_normal(m.n_nodes)
    b[fixed] = 0.0
    dm = DeviceMesh(m)
    A = assemble_laplacian(dm, torch.from_numpy(fixed))
    pcg = PCG(A, 1.0 / A.diag, fixed=torch.from_numpy(fixed), order=dm.node_order(), force_mode=mode)
    x, _ = pcg.solve(torch.from_numpy(b).cuda(), 9, zero_b=False)
    xr, _, _ = fem.pcg(L, b, 1.0 / L.diagonal(), 9)
    assert rel_l2(x.cpu().numpy(), xr) <= 1e-10
    x2, it = pcg.solve(torch.from_numpy(b).cuda(), 2000, tol=1e-11, zero_b=False)
    assert pcg.residual() <= 1e-11

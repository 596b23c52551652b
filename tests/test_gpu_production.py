"""Oracle parity IN THE REGIME THE BENCH RUNS ("what's weak" #1).

The small-mesh parity tests (test_gpu_flow.py) give every persistent CTA of
the pipelined element kernels a single 128-element block and every resident
CG CTA a single SELL slice.  Here the same kernels run at production sizes
and are compared with the frozen numpy oracle (oracle/fem.py):

* element kernels (K2 momentum, element-form K4/K6, gradient-operator
  products) on >= 1M jittered tets, every persistent CTA walking >= 3 blocks
  (metadata ring, two-block prefetch, mbarrier phase flips), and K2 on the
  full C2 mesh (4.09M tets, BASELINE configs[1]);
* the resident CG (k_cg_resident_local) on the full C2 system (705k rows:
  ~4.8k rows = ~5 slices per warp per CTA, thousands of ghosts, the tensor-
  memory first slice) and the two-kernel CG (node order and SFC order) with
  hundreds of blocks in its grouped grid reductions, 9 fixed iterations;
* one full C2 time step (CUDA graph, 50 CG iterations) at 4.09M elements;
* C1 exactly as BASELINE configs[0] states it: TGV on 32^3 periodic HEX08,
  10 steps, CG converged to 1e-10;
* a full mixed-mesh step (c3_mesh(0.42): 2.2M tet/prism/pyramid/hex elements,
  wall model) and the chunked setup paths of C3/C4 (CSR pattern, tet node
  order tuning) against their unchunked results.

Tolerances are the north star's (BASELINE.json): assembled fp64 vectors rel
L2 <= 1e-10, velocity/pressure after N steps rel L2 <= 1e-8.  The oracle is
single-threaded numpy, so these tests take minutes; parity remains unpinned
by the reference (it has no Navier-Stokes code).
"""

import ctypes

import numpy as np
import pytest
import torch

from conftest import rel_l2
from oracle import fem
from paper_2005_05899_b200 import meshgen

pytestmark = pytest.mark.gpu

TOL_RHS = 1e-10
TOL_STATE = 1e-8


def _pipe_shape():
    from paper_2005_05899_b200._lib import lib
    g, b = ctypes.c_int64(0), ctypes.c_int64(0)
    assert lib().ab_last_pipe_shape(ctypes.byref(g), ctypes.byref(b)) == 0
    return g.value, b.value


@pytest.fixture(scope="module")
def mega():
    """~1.05M jittered Kuhn tets (56^3 cells) and a rough velocity field."""
    m = meshgen.box_tets(56, 56, 56, jitter=0.2, seed=7)
    rng = np.random.default_rng(1)
    x = m.coords
    u = np.stack([np.sin(6 * x[:, 0]) * np.cos(5 * x[:, 1]), np.cos(4 * x[:, 2]) * x[:, 0], x[:, 1] ** 2], axis=1)
    u += 0.05 * rng.standard_normal(u.shape)
    p = np.cos(7 * x[:, 0] + 3 * x[:, 1]) + 0.1 * rng.standard_normal(len(x))
    return m, u, p


@pytest.fixture(scope="module")
def c2():
    """BASELINE configs[1]: the C2 mesh, its initial field and the oracle's
    Dirichlet Laplacian (assembled once for the CG tests and the step)."""
    m = meshgen.c2_mesh()
    u, p = meshgen.c2_initial(m.coords)
    fixed = meshgen.boundary_nodes(m)
    return m, u, p, fixed


def test_element_kernels_multi_block_per_cta(mega):
    """K2, element-form K4 and K6 through the pipelined persistent kernels,
    each CTA walking several blocks, vs the oracle."""
    from paper_2005_05899_b200.device import DeviceMesh
    from paper_2005_05899_b200.ops import assemble_divergence, assemble_gradient, assemble_momentum
    from paper_2005_05899_b200.timestep import FlowParams
    m, u, p = mega
    dm = DeviceMesh(m, reorder="sfc", windows=True)
    ph = FlowParams(rho=1.2, mu=3e-3, c_vreman=0.07)
    got = assemble_momentum(dm, u, ph).cpu().numpy()
    grid, blocks = _pipe_shape()
    assert blocks >= 3 * grid, (grid, blocks)  # the multi-block steady state ran
    ref = fem.momentum_rhs(m, u, rho=1.2, mu=3e-3, c_vreman=0.07)
    assert rel_l2(got, ref) <= TOL_RHS
    d = assemble_divergence(dm, u, 2.0).cpu().numpy()
    assert _pipe_shape()[1] >= 3 * _pipe_shape()[0]
    assert rel_l2(d, 2.0 * fem.divergence(m, u)) <= TOL_RHS
    g = assemble_gradient(dm, p).cpu().numpy()
    assert rel_l2(g, fem.gradient(m, p)) <= TOL_RHS


def test_gradient_operator_products_large(mega):
    """K4 = s B.u and K6+K7's B dp (ab_gradop_div/grad) at 1M elements."""
    from paper_2005_05899_b200.device import DeviceMesh, nodes_as4
    from paper_2005_05899_b200.solver import assemble_gradient_operator
    m, u, p = mega
    dm = DeviceMesh(m)
    B = assemble_gradient_operator(dm)
    out = torch.zeros(m.n_nodes, dtype=torch.float64, device="cuda")
    B.div(nodes_as4(torch.from_numpy(u).cuda()), -3.0, out)
    assert rel_l2(out.cpu().numpy(), -3.0 * fem.divergence(m, u)) <= TOL_RHS
    g4 = torch.zeros((m.n_nodes, 4), dtype=torch.float64, device="cuda")
    B.grad(torch.from_numpy(p).cuda(), 1.0, g4)
    assert rel_l2(g4[:, :3].cpu().numpy(), fem.gradient(m, p)) <= TOL_RHS


def test_k2_full_c2(c2):
    """K2 on the full C2 mesh (4.09M tets, the bench's element kernel and
    window tuning) with the C2 initial field, vs the oracle."""
    from paper_2005_05899_b200.device import DeviceMesh
    from paper_2005_05899_b200.ops import assemble_momentum
    from paper_2005_05899_b200.timestep import FlowParams
    m, u, _p, _f = c2
    dm = DeviceMesh(m, reorder="sfc", windows=True)
    got = assemble_momentum(dm, u, FlowParams(rho=1.0, mu=1e-3, c_vreman=0.07)).cpu().numpy()
    grid, blocks = _pipe_shape()
    assert blocks >= 3 * grid
    ref = fem.momentum_rhs(m, u, rho=1.0, mu=1e-3, c_vreman=0.07)
    assert np.abs(ref).max() > 0.0
    assert rel_l2(got, ref) <= TOL_RHS


@pytest.mark.parametrize("variant", ["resident-sfc", "two-kernel", "two-kernel-sfc", "two-kernel-sfc-tile",
                                     "two-kernel-sfc-single"])
def test_cg_full_c2_system(c2, variant):
    """9 and 50 fixed Jacobi-PCG iterations on the full C2 Laplacian (705k rows)."""
    from paper_2005_05899_b200.device import DeviceMesh
    from paper_2005_05899_b200.solver import PCG, assemble_laplacian
    m, _u, _p, fixed = c2
    L = fem.laplacian(m, fixed)
    b = np.random.default_rng(3).standard_normal(m.n_nodes)
    b[fixed] = 0.0
    dm = DeviceMesh(m)
    A = assemble_laplacian(dm, torch.from_numpy(fixed))
    kw = {"resident-sfc": dict(order=dm.node_order()), "two-kernel": dict(resident=False),
          "two-kernel-sfc": dict(order=dm.node_order(), resident=False, tile_rows=0),
          "two-kernel-sfc-tile": dict(order=dm.node_order(), resident=False, tile_rows=2048, single_pass=False),
          "two-kernel-sfc-single": dict(order=dm.node_order(), resident=False, tile_rows=2048)}[variant]
    pcg = PCG(A, 1.0 / A.diag, fixed=torch.from_numpy(fixed), **kw)
    if variant == "resident-sfc":
        lm = pcg.local
        assert lm is not None
        rb = lm["struct"].rows_per_cta
        assert rb // 32 >= 2 * 32        # >= 2 SELL slices per warp (32 warps per CTA)
        assert lm["max_ghost"] >= 1000   # thousands of ghost rows gathered per CTA
    else:
        assert not pcg.resident
        assert (m.n_nodes + 255) // 256 >= 20 * 64  # >= 20 groups in the grouped grid reduction
    if variant.startswith("two-kernel-sfc-"):
        assert pcg.perm2["tile"] is not None and pcg.perm2["single"] == (variant == "two-kernel-sfc-single")
    for its in (9, 50):
        x, it = pcg.solve(torch.from_numpy(b).cuda(), its, zero_b=False)
        xr, itr, _ = fem.pcg(L, b, 1.0 / L.diagonal(), its)
        assert it == itr == its
        assert rel_l2(x.cpu().numpy(), xr) <= TOL_RHS


def test_full_c2_step(c2):
    """One full time step of the bench workload (C2: 4.09M tets, 3 x K2+K3,
    K4, PCG 50 it, K6+K7; CUDA graph) vs the oracle."""
    from paper_2005_05899_b200.timestep import FlowParams, FlowSolver
    m, u, p, fixed = c2
    params = dict(rho=1.0, mu=1e-3, c_vreman=0.07)
    fs = FlowSolver(m, FlowParams(**params), p_fixed=fixed, windows=True, reorder="sfc")
    fs.set_state(u, p)
    fs.step(1e-3, cg_iters=50, graph=True)
    torch.cuda.synchronize()
    assert fs.pcg.resident
    ora = fem.FlowOracle(m, **params, p_fixed=fixed)
    st = ora.step(ora.init_state(u, p), 1e-3, cg_iters=50)
    assert rel_l2(fs.u.cpu().numpy(), st["u"]) <= TOL_STATE
    assert rel_l2(fs.p.cpu().numpy(), st["p"]) <= TOL_STATE


def test_c1_exact_config():
    """BASELINE configs[0] as stated: TGV, 32^3 periodic HEX08, fp64, 10 RK
    time steps (dt = 1e-2, mu = 1/1600), CG converged to 1e-10 each step."""
    from paper_2005_05899_b200.timestep import FlowParams, FlowSolver
    m = meshgen.c1_mesh(32)
    assert m.n_elements == 32 ** 3 and m.n_nodes == 32 ** 3
    u, p = fem.tgv_initial(m.coords)
    pf = np.zeros(m.n_nodes, bool)
    pf[0] = True
    params = dict(rho=1.0, mu=1.0 / 1600, c_vreman=0.0)
    ora = fem.FlowOracle(m, **params, p_fixed=pf)
    st = ora.init_state(u, p)
    fs = FlowSolver(m, FlowParams(**params), p_fixed=pf)
    fs.set_state(u, p)
    its = []
    for _ in range(10):
        st = ora.step(st, 1e-2, cg_iters=2000, cg_tol=1e-10)
        fs.step(1e-2, cg_iters=2000, cg_tol=1e-10)
        its.append((fs.last_cg_iters, st["cg_iters"]))
    torch.cuda.synchronize()
    assert all(abs(a - b) <= 1 for a, b in its), its
    assert rel_l2(fs.u.cpu().numpy(), st["u"]) <= TOL_STATE
    assert rel_l2(fs.p.cpu().numpy(), st["p"]) <= TOL_STATE


def test_mixed_mesh_step_at_scale():
    """A full Algorithm-1 step (element + wall-model boundary assembly) on a
    2.2M-element mixed mesh (c3_mesh(0.42): tet, prism, pyramid, hex windows),
    CUDA graph, vs the oracle."""
    from paper_2005_05899_b200.timestep import FlowParams, FlowSolver
    m = meshgen.c3_mesh(0.42)
    assert m.n_elements > 2_000_000 and len(m.conn) == 4
    bc, wall = meshgen.wall_model_bcs(m)
    x = m.coords
    u = np.stack([np.ones(len(x)) + 0.1 * np.sin(9 * x[:, 1]), 0.05 * np.cos(7 * x[:, 0]),
                  0.02 * np.sin(5 * x[:, 2])], axis=1)
    p = np.zeros(len(x))
    params = dict(rho=1.0, mu=1e-3, c_vreman=0.07)
    fs = FlowSolver(m, FlowParams(**params), **bc, wall=wall, windows=True, reorder="sfc")
    fs.set_state(u, p)
    fs.step(1e-3, cg_iters=50, graph=True)
    torch.cuda.synchronize()
    ora = fem.FlowOracle(m, **params, **bc, wall=wall)
    st = ora.step(ora.init_state(u, p), 1e-3, cg_iters=50)
    assert rel_l2(fs.u.cpu().numpy(), st["u"]) <= TOL_STATE
    assert rel_l2(fs.p.cpu().numpy(), st["p"]) <= TOL_STATE


def test_chunked_setup_paths_equal_unchunked():
    """The chunked setup paths that only activate at C3/C4 sizes (CSR
    pattern: 1<<23 elements per chunk; tet node-order tuning: 1<<22) give
    the same result as one chunk, exercised here with small chunks."""
    from paper_2005_05899_b200.device import DeviceMesh
    from paper_2005_05899_b200.solver import csr_pattern
    m = meshgen.c3_mesh(0.3)
    dm = DeviceMesh(m, reorder="sfc")
    rp0, c0 = csr_pattern(dm, chunk=1 << 30)
    rp1, c1 = csr_pattern(dm, chunk=1 << 16)  # > 8 partial keys: the merge path too
    assert torch.equal(rp0, rp1) and torch.equal(c0, c1)
    a = DeviceMesh(m, reorder="sfc")
    b = DeviceMesh(m, reorder="sfc")
    a.tune_tet_node_order(chunk=1 << 30)
    b.tune_tet_node_order(chunk=1 << 14)
    for ca, cb in zip(a.conn, b.conn):
        assert torch.equal(ca, cb)



"""GPU parity of the Navier-Stokes time-step path against the frozen numpy
oracle (oracle/fem.py; parity unpinned by the reference).

Tolerances (BASELINE.json north star): assembled fp64 vectors rel L2 <= 1e-10;
velocity and pressure after N steps rel L2 <= 1e-8."""

import numpy as np
import pytest
import torch

from conftest import rel_l2
from oracle import fem
from paper_2005_05899_b200 import meshgen

pytestmark = pytest.mark.gpu

TOL_RHS = 1e-10
TOL_STATE = 1e-8


def _meshes():
    return {
        "tet": meshgen.box_tets(6, 5, 4, jitter=0.2, seed=3),
        "hex_periodic": meshgen.c1_mesh(6),
        "mixed": meshgen.c3_mesh(0.05),
        "hex": meshgen.box_hexes(4, 3, 5, lengths=(1.0, 0.7, 1.3)),
    }


MESHES = _meshes()


def _field(m, seed=0):
    rng = np.random.default_rng(seed)
    x = m.coords
    u = np.stack([np.sin(3 * x[:, 0]) * np.cos(2 * x[:, 1]), np.cos(x[:, 2]) * x[:, 0], x[:, 1] ** 2], axis=1)
    return u + 0.1 * rng.standard_normal(u.shape), np.cos(2 * x[:, 0] + x[:, 1]) + rng.standard_normal(len(x)) * 0.1


SCATTER = ["direct", "window", "pipelined"]


def _dm(m, mode):
    from paper_2005_05899_b200.device import DeviceMesh
    return DeviceMesh(m, reorder=None if mode == "direct" else "sfc", windows=mode != "direct",
                      pipelined=mode == "pipelined")


@pytest.mark.parametrize("name", list(MESHES))
@pytest.mark.parametrize("mode", SCATTER)
@pytest.mark.parametrize("c_vreman", [0.0, 0.07])
def test_momentum_rhs(name, mode, c_vreman):
    from paper_2005_05899_b200.ops import assemble_momentum
    from paper_2005_05899_b200.timestep import FlowParams
    m = MESHES[name]
    u, _ = _field(m)
    ref = fem.momentum_rhs(m, u, rho=1.3, mu=0.01, c_vreman=c_vreman)
    dm = _dm(m, mode)
    got = assemble_momentum(dm, u, FlowParams(rho=1.3, mu=0.01, c_vreman=c_vreman)).cpu().numpy()
    assert rel_l2(got, ref) <= TOL_RHS


@pytest.mark.parametrize("name", list(MESHES))
@pytest.mark.parametrize("mode", SCATTER)
def test_divergence_gradient(name, mode):
    from paper_2005_05899_b200.ops import assemble_divergence, assemble_gradient
    m = MESHES[name]
    u, p = _field(m, 1)
    dm = _dm(m, mode)
    assert rel_l2(assemble_divergence(dm, u, 2.0).cpu().numpy(), 2.0 * fem.divergence(m, u)) <= TOL_RHS
    assert rel_l2(assemble_gradient(dm, p).cpu().numpy(), fem.gradient(m, p)) <= TOL_RHS


@pytest.mark.parametrize("name", list(MESHES))
def test_gradient_operator(name):
    """K4/K6 as sparse products with B_ab = int N_a grad N_b (ab_gradop_*) vs the oracle."""
    from paper_2005_05899_b200.device import DeviceMesh, nodes_as4
    from paper_2005_05899_b200.solver import assemble_gradient_operator
    m = MESHES[name]
    u, p = _field(m, 1)
    dm = DeviceMesh(m)
    B = assemble_gradient_operator(dm)
    u4 = nodes_as4(torch.from_numpy(u).cuda())
    out = torch.full((m.n_nodes,), 0.5, dtype=torch.float64, device="cuda")
    B.div(u4, 2.0, out)  # accumulates
    assert rel_l2(out.cpu().numpy() - 0.5, 2.0 * fem.divergence(m, u)) <= TOL_RHS
    g4 = torch.zeros((m.n_nodes, 4), dtype=torch.float64, device="cuda")
    B.grad(torch.from_numpy(p).cuda(), 1.0, g4)
    assert rel_l2(g4[:, :3].cpu().numpy(), fem.gradient(m, p)) <= TOL_RHS
    assert float(g4[:, 3].abs().max()) == 0.0


def test_wall_traction_matches_oracle():
    """K8 (ab_wall_traction) vs oracle/fem.py:wall_traction on the mixed mesh."""
    from paper_2005_05899_b200.timestep import FlowParams
    from paper_2005_05899_b200.wall import assemble_wall_traction
    m = MESHES["mixed"]
    _, (F, O) = meshgen.wall_model_bcs(m)
    u, _ = _field(m, 5)
    ref = fem.wall_traction(m, F, O, u, 1.3, 2e-3)
    got = assemble_wall_traction(m, F, O, u, FlowParams(rho=1.3, mu=2e-3)).cpu().numpy()
    assert np.abs(ref).max() > 0
    assert rel_l2(got, ref) <= TOL_RHS


@pytest.mark.parametrize("graph", [False, True])
def test_time_steps_with_wall_model(graph):
    """Full Algorithm 1 step (element + boundary assembly) vs the oracle."""
    from paper_2005_05899_b200.timestep import FlowParams, FlowSolver
    m = MESHES["mixed"]
    bc, wall = meshgen.wall_model_bcs(m)
    u, p = _field(m, 6)
    params = dict(rho=1.0, mu=0.01, c_vreman=0.07)
    ora = fem.FlowOracle(m, **params, **bc, wall=wall)
    st = ora.init_state(u, p)
    fs = FlowSolver(m, FlowParams(**params), **bc, wall=wall)
    assert fs.wall is not None and fs.wall.n_faces == wall[0].shape[0]
    fs.set_state(u, p)
    for _ in range(3):
        st = ora.step(st, 2e-3, cg_iters=40)
        fs.step(2e-3, cg_iters=40, graph=graph)
    torch.cuda.synchronize()
    assert rel_l2(fs.u.cpu().numpy(), st["u"]) <= TOL_STATE
    assert rel_l2(fs.p.cpu().numpy(), st["p"]) <= TOL_STATE


@pytest.mark.parametrize("name", list(MESHES))
def test_laplacian_and_spmv(name):
    from paper_2005_05899_b200.solver import assemble_laplacian
    m = MESHES[name]
    fixed = meshgen.boundary_nodes(m) if name != "hex_periodic" else np.arange(m.n_nodes) == 0
    L_ref = fem.laplacian(m, fixed)
    A = assemble_laplacian(m, torch.from_numpy(fixed))
    rp, cols, vals = (t.cpu().numpy() for t in A.csr)
    assert np.array_equal(rp, L_ref.indptr) and np.array_equal(cols, L_ref.indices)
    assert rel_l2(vals, L_ref.data) <= 1e-12
    assert rel_l2(A.diag.cpu().numpy(), L_ref.diagonal()) <= 1e-12
    x = np.random.default_rng(0).standard_normal(m.n_nodes)
    y = A.matvec(torch.from_numpy(x).cuda()).cpu().numpy()
    assert rel_l2(y, L_ref @ x) <= 1e-12


CG_VARIANTS = {
    "local-sfc": dict(order=True),          # ab_cg_resident_local, SFC row order, z gathers from shared memory
    "local": dict(),                        # local column map, node order
    "two-kernel": dict(resident=False),     # k_cg_spmv + k_cg_update per iteration
    "two-kernel-sfc": dict(order=True, resident=False, tile_rows=0),  # two kernels on D^-1/2 P A P^T D^-1/2 (SFC)
    "two-kernel-sfc-tile": dict(order=True, resident=False, tile_rows=64),  # tiled SpMV, z in shared memory
    "two-kernel-sfc-single": dict(order=True, resident=False, tile_rows=1024),  # tiled single pass (default form)
    "two-kernel-sfc-jacobi": dict(order=True, resident=False, scaled=False),  # z = D^-1 r form
    "two-kernel-sfc-diag": dict(order=True, resident=False, unit_diag=False),  # scaled, diagonal stored
}


@pytest.mark.parametrize("name", ["tet", "mixed"])
@pytest.mark.parametrize("variant", list(CG_VARIANTS))
def test_pcg_fixed_iterations_and_convergence(name, variant):
    from paper_2005_05899_b200.device import DeviceMesh
    from paper_2005_05899_b200.solver import PCG, assemble_laplacian
    import scipy.sparse.linalg as spla
    m = MESHES[name]
    fixed = meshgen.boundary_nodes(m)
    L = fem.laplacian(m, fixed)
    b = np.random.default_rng(2).standard_normal(m.n_nodes)
    b[fixed] = 0.0
    dm = DeviceMesh(m)
    A = assemble_laplacian(dm, torch.from_numpy(fixed))
    dinv = 1.0 / A.diag
    kw = dict(CG_VARIANTS[variant])
    if kw.pop("order", False):
        kw["order"] = dm.node_order()
    # fixed iteration count: same iterate as the oracle
    pcg = PCG(A, dinv, fixed=torch.from_numpy(fixed), **kw)
    assert pcg.resident == (not variant.startswith("two-kernel"))
    assert (pcg.perm2 is not None) == variant.startswith("two-kernel-sfc")
    if variant in ("local-sfc", "local"):
        assert pcg.local is not None
    if pcg.perm2 is not None:
        assert (pcg.perm2["tile"] is not None) == (variant in ("two-kernel-sfc-tile", "two-kernel-sfc-single"))
        assert pcg.perm2["single"] == (variant == "two-kernel-sfc-single")
    bt = torch.from_numpy(b).cuda()
    x, it = pcg.solve(bt.clone(), 7)
    xr, itr, _ = fem.pcg(L, b, 1.0 / L.diagonal(), 7)
    assert it == itr == 7
    assert rel_l2(x.cpu().numpy(), xr) <= 1e-10
    # to convergence (tested on the device for the resident kernels): matches a direct solve
    pcg2 = PCG(A, dinv, fixed=torch.from_numpy(fixed), **kw)
    x, it = pcg2.solve(bt.clone(), 2000, tol=1e-12, zero_b=False)
    res = pcg2.residual()
    xr2, itr2, _ = fem.pcg(L, b, 1.0 / L.diagonal(), 2000, tol=1e-12)
    assert abs(it - itr2) <= 1  # row order changes the rounding of the dots
    assert res <= 1e-12
    assert rel_l2(x.cpu().numpy(), spla.spsolve(L.tocsc(), b)) <= 1e-9
    # the solve leaves b untouched when zero_b=False and x is in node order
    assert torch.equal(bt, torch.from_numpy(b).cuda())


def _bcs(name, m):
    n = m.n_nodes
    if name == "hex_periodic":
        pf = np.zeros(n, bool)
        pf[0] = True
        return dict(p_fixed=pf)
    x = m.coords
    bnd = meshgen.boundary_nodes(m)
    if name == "mixed":
        uf = np.zeros((n, 3), bool)
        uv = np.zeros((n, 3))
        inflow = np.abs(x[:, 0] - x[:, 0].min()) < 1e-12
        wall = np.abs(x[:, 2] - x[:, 2].min()) < 1e-12
        uf[inflow] = True
        uv[inflow] = (1.0, 0.0, 0.0)
        uf[wall] = True
        uv[wall] = 0.0
        pf = np.abs(x[:, 0] - x[:, 0].max()) < 1e-12
        return dict(p_fixed=pf, u_fixed=uf, u_fixed_values=uv)
    return dict(p_fixed=bnd)


@pytest.mark.parametrize("name", ["tet", "hex_periodic", "mixed"])
@pytest.mark.parametrize("graph", [False, True])
@pytest.mark.parametrize("ops", ["spmv", "element"])
def test_time_steps_match_oracle(name, graph, ops):
    from paper_2005_05899_b200.timestep import FlowParams, FlowSolver
    m = MESHES[name]
    bc = _bcs(name, m)
    if name == "hex_periodic":
        u, p = fem.tgv_initial(m.coords)
        params = dict(rho=1.0, mu=1.0 / 1600, c_vreman=0.0)
    else:
        u, p = _field(m, 4)
        params = dict(rho=1.0, mu=0.01, c_vreman=0.07)
    dt, steps, iters = 2e-3, 3, 40
    ora = fem.FlowOracle(m, **params, **bc)
    st = ora.init_state(u, p)
    fs = FlowSolver(m, FlowParams(**params), **bc, windows=True, reorder="sfc", ops=ops)
    fs.set_state(u, p)
    for _ in range(steps):
        st = ora.step(st, dt, cg_iters=iters)
        fs.step(dt, cg_iters=iters, graph=graph)
    torch.cuda.synchronize()
    assert rel_l2(fs.u.cpu().numpy(), st["u"]) <= TOL_STATE
    assert rel_l2(fs.p.cpu().numpy(), st["p"]) <= TOL_STATE


def test_tgv_converged_cg_and_energy_decay():
    """C1 (TGV 32^3 HEX08, 10 steps) with converged CG, vs the oracle."""
    from paper_2005_05899_b200.timestep import FlowParams, FlowSolver
    m = meshgen.c1_mesh(16)
    u, p = fem.tgv_initial(m.coords)
    pf = np.zeros(m.n_nodes, bool)
    pf[0] = True
    ora = fem.FlowOracle(m, 1.0, 1 / 1600, 0.0, p_fixed=pf)
    st = ora.init_state(u, p)
    fs = FlowSolver(m, FlowParams(1.0, 1 / 1600, 0.0), p_fixed=pf)
    fs.set_state(u, p)
    ke = []
    for _ in range(4):
        st = ora.step(st, 1e-2, cg_iters=500, cg_tol=1e-10)
        fs.step(1e-2, cg_iters=500, cg_tol=1e-10)
        ke.append(float((ora.ml[:, None] * fs.u.cpu().numpy() ** 2).sum()))
    assert rel_l2(fs.u.cpu().numpy(), st["u"]) <= TOL_STATE
    assert rel_l2(fs.p.cpu().numpy(), st["p"]) <= TOL_STATE
    assert all(b < a for a, b in zip(ke, ke[1:]))


def test_full_size_c2_properties():
    """Size-independent properties at BASELINE configs[1] size (4.09M tets)."""
    from paper_2005_05899_b200.device import DeviceMesh
    from paper_2005_05899_b200.ops import assemble_divergence, assemble_gradient
    from paper_2005_05899_b200.assembly import lumped_mass
    m = meshgen.c2_mesh()
    dm = DeviceMesh(m, reorder="sfc", windows=True)
    ml = lumped_mass(dm)
    assert abs(ml.sum() - 1.0) <= 1e-12
    x = torch.from_numpy(m.coords).cuda()
    # (K2 at this size is compared with the oracle in test_gpu_production.py)
    # linear fields are reproduced exactly: D u = div(u) M_L, G p = grad(p) M_L
    inner = ~torch.from_numpy(meshgen.boundary_nodes(m)).cuda()
    u = torch.stack([2 * x[:, 0] + x[:, 1], -x[:, 1] + 0.5 * x[:, 2], 3 * x[:, 2]], dim=1)
    D = assemble_divergence(dm, u)
    mlt = torch.from_numpy(ml).cuda()
    assert float((D - 4.0 * mlt)[inner].abs().max() / mlt.max()) <= 1e-9
    G = assemble_gradient(dm, x[:, 0] - 2 * x[:, 2])
    want = torch.tensor([1.0, 0.0, -2.0], dtype=torch.float64, device="cuda")
    assert float((G - mlt[:, None] * want)[inner].abs().max() / mlt.max()) <= 1e-9


def test_halo_pack_unpack_kernels():
    from paper_2005_05899_b200.halo import cuda_pack, cuda_unpack_add
    rng = np.random.default_rng(0)
    f = rng.standard_normal((50, 4))
    idx = np.array([3, 7, 7, 11, 49], dtype=np.int32)
    ft = torch.from_numpy(f).cuda()
    it = torch.from_numpy(idx).cuda()
    buf = torch.zeros(idx.size * 3, dtype=torch.float64, device="cuda")
    cuda_pack(it, ft, 4, 3, buf)
    assert np.array_equal(buf.cpu().numpy().reshape(-1, 3), f[idx, :3])
    cuda_unpack_add(it, buf, 4, 3, ft)
    want = f.copy()
    np.add.at(want[:, :3], idx, f[idx, :3])
    assert np.allclose(ft.cpu().numpy(), want, rtol=0, atol=1e-15)


@pytest.mark.parametrize("graph,overlap", [(False, False), (True, False), (False, True)])
def test_step_host_matches_oracle(graph, overlap):
    """The end-to-end entry point (pinned host u, p in; step; host u, p out)
    against the oracle over 3 steps, with the host state perturbed between
    steps so the uploaded p differs from the device's.  overlap: p's upload +
    G p^n under the first momentum assembly and p^{n+1}'s download under
    K6 + K7 (side stream); otherwise G p^n while u uploads, then the step."""
    from paper_2005_05899_b200.timestep import FlowParams, FlowSolver
    m = meshgen.box_tets(7, 6, 5, jitter=0.2, seed=5)
    u, p = _field(m, seed=4)
    bc = dict(p_fixed=meshgen.boundary_nodes(m))
    params = dict(rho=1.0, mu=1e-2, c_vreman=0.07)
    ora = fem.FlowOracle(m, **params, **bc)
    fs = FlowSolver(m, FlowParams(**params), **bc)
    fs.set_state(u, p)
    u_h = torch.from_numpy(np.ascontiguousarray(u)).pin_memory()
    p_h = torch.from_numpy(np.ascontiguousarray(p)).pin_memory()
    for k in range(3):
        st = ora.init_state(u_h.numpy().copy(), p_h.numpy().copy())
        st = ora.step(st, 1e-3, cg_iters=30)
        fs.step_host(u_h, p_h, 1e-3, cg_iters=30, graph=graph, overlap=overlap)
        torch.cuda.synchronize()
        assert rel_l2(u_h.numpy(), st["u"]) <= TOL_STATE, k
        assert rel_l2(p_h.numpy(), st["p"]) <= TOL_STATE, k
        p_h += 0.01 * (k + 1)  # the next upload is not the device's p


@pytest.mark.parametrize("name", ["tet", "mixed", "hex_periodic"])
def test_precomputed_filter_width(name):
    """K2 with the per-element Vreman filter width computed once at setup
    (ab_filter_width) equals K2 evaluating V_e^(2/3) itself (to the rounding
    of the unordered fp64 reductions of the scatter), and the widths equal
    the oracle's cbrt(V_e)^2."""
    from paper_2005_05899_b200.ops import assemble_momentum
    from paper_2005_05899_b200.timestep import FlowParams
    m = MESHES[name]
    u, _ = _field(m, seed=2)
    dm = _dm(m, "pipelined")
    ph = FlowParams(rho=1.1, mu=0.02, c_vreman=0.1)
    assert all(d.numel() == c.shape[0] for d, c in zip(dm._d2, dm.conn))
    for k, rule in enumerate(dm.rules):
        X = fem.element_coords(m.coords, dm.conn[k].cpu().numpy(), m.period)
        vol = (fem.jacobian_dets(X, rule) * fem.rule_points_weights(rule)[1][None, :]).sum(axis=1)
        assert rel_l2(dm._d2[k].cpu().numpy(), np.cbrt(vol) ** 2) <= 1e-14
    a = assemble_momentum(dm, u, ph).cpu().numpy()
    dm.clear_filter_width()
    b = assemble_momentum(dm, u, ph).cpu().numpy()
    assert rel_l2(a, b) <= 1e-14


@pytest.mark.parametrize("name", ["tet", "mixed"])
def test_window_tuning_changes_only_rounding(name, monkeypatch):
    """The bank-aware tet node order (tune_tet_node_order) and the bank-spread
    reference order inside window runs (_spread_slot_banks) only reorder
    floating-point sums: K2 with and without them agrees to rounding."""
    from paper_2005_05899_b200.device import DeviceMesh
    from paper_2005_05899_b200.ops import assemble_momentum
    from paper_2005_05899_b200.timestep import FlowParams
    m = MESHES[name]
    u, _ = _field(m, seed=6)
    ph = FlowParams(rho=1.0, mu=0.01, c_vreman=0.07)
    tuned = assemble_momentum(DeviceMesh(m, reorder="sfc", windows=True), u, ph).cpu().numpy()
    monkeypatch.setenv("AB_NO_TET_TUNE", "1")
    monkeypatch.setenv("AB_NO_SLOT_SPREAD", "1")
    plain = assemble_momentum(DeviceMesh(m, reorder="sfc", windows=True), u, ph).cpu().numpy()
    assert rel_l2(tuned, plain) <= 1e-13
    assert rel_l2(tuned, fem.momentum_rhs(m, u, rho=1.0, mu=0.01, c_vreman=0.07)) <= TOL_RHS

"""The C + OpenMP restatement of the time step (oracle/fem_c.c, the CPU
baseline bench.py times) against the numpy oracle (oracle/fem.py): element
operators within 1e-12 relative, 3 full steps (incl. wall model, velocity
Dirichlet values, periodic hexes) within 1e-10.  CPU only."""

import numpy as np
import pytest

from conftest import rel_l2
from oracle import fem, femc
from paper_2005_05899_b200 import meshgen


def _field(m, seed=0):
    rng = np.random.default_rng(seed)
    x = m.coords
    u = np.stack([np.sin(3 * x[:, 0]) * np.cos(2 * x[:, 1]), np.cos(x[:, 2]) * x[:, 0], x[:, 1] ** 2], axis=1)
    return u + 0.1 * rng.standard_normal(u.shape), np.cos(2 * x[:, 0] + x[:, 1]) + 0.1 * rng.standard_normal(len(x))


MESHES = {
    "tet": lambda: meshgen.box_tets(6, 5, 4, jitter=0.2, seed=3),
    "hex_periodic": lambda: meshgen.c1_mesh(5),
    "mixed": lambda: meshgen.c3_mesh(0.06),
}


@pytest.fixture(scope="module", autouse=True)
def _build():
    femc.build()


@pytest.mark.parametrize("name", list(MESHES))
@pytest.mark.parametrize("threads", [1, 3])
def test_element_operators(name, threads):
    m = MESHES[name]()
    u, p = _field(m)
    cm = femc.CMesh(m, threads)
    assert rel_l2(cm.momentum(u, 1.3, 0.01, 0.07), fem.momentum_rhs(m, u, 1.3, 0.01, 0.07)) <= 1e-12
    assert rel_l2(cm.momentum(u, 1.3, 0.01, 0.0), fem.momentum_rhs(m, u, 1.3, 0.01, 0.0)) <= 1e-12
    assert rel_l2(cm.divergence(u, -2.0), -2.0 * fem.divergence(m, u)) <= 1e-12
    assert rel_l2(cm.gradient(p), fem.gradient(m, p)) <= 1e-12


@pytest.mark.parametrize("name", list(MESHES))
def test_steps_match_numpy_oracle(name):
    m = MESHES[name]()
    wall = None
    if name == "hex_periodic":
        u, p = fem.tgv_initial(m.coords)
        pin = np.zeros(m.n_nodes, bool)
        pin[0] = True  # periodic: the pressure is fixed at one node
        bc, params = dict(p_fixed=pin), dict(rho=1.0, mu=1.0 / 1600, c_vreman=0.0)
    elif name == "mixed":
        bc, wall = meshgen.wall_model_bcs(m)
        u, p = _field(m, 2)
        u[:, 0] += 1.0
        params = dict(rho=1.0, mu=2e-3, c_vreman=0.07)
    else:
        bc = dict(p_fixed=meshgen.boundary_nodes(m))
        u, p = _field(m, 1)
        params = dict(rho=1.0, mu=0.01, c_vreman=0.07)
    a = fem.FlowOracle(m, **params, **bc, wall=wall)
    c = femc.CFlowOracle(m, **params, **bc, wall=wall, threads=2)
    sa, sc = a.init_state(u, p), c.init_state(u, p)
    for _ in range(3):
        sa = a.step(sa, 2e-3, cg_iters=30)
        sc = c.step(sc, 2e-3, cg_iters=30)
    assert rel_l2(sc["u"], sa["u"]) <= 1e-10
    assert rel_l2(sc["p"], sa["p"]) <= 1e-10


def test_threads_reported():
    m = MESHES["tet"]()
    assert femc.CMesh(m, 2).threads == 2

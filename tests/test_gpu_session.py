"""The C-ABI session (ab_ctx_create / ab_mesh_upload / ab_state_set /
ab_step / ab_state_get) driven through ctypes only - no torch tensors, no
Python setup: host numpy arrays in, host arrays out - against the oracle
(north-star tolerance: u, p rel L2 <= 1e-8 after N steps)."""

import ctypes as C

import numpy as np
import pytest

from conftest import rel_l2
from oracle import fem
from paper_2005_05899_b200 import meshgen

pytestmark = pytest.mark.gpu


def _run(m, bc, params, u, p, steps, dt, iters, wall=None):
    from paper_2005_05899_b200.session import Session
    from paper_2005_05899_b200.timestep import FlowParams
    s = Session(m, FlowParams(**params), wall=wall, **bc)
    info = s.info()
    assert info["ready"] and info["n_nodes"] == m.n_nodes and sum(info["n_elem"]) == m.n_elements
    s.set_state(u, p)
    for _ in range(steps):
        s.step(dt, iters)  # asynchronous: no host sync between steps
    out = s.get_state()
    s.close()
    ora = fem.FlowOracle(m, **params, **bc, wall=wall)
    st = ora.init_state(u, p)
    for _ in range(steps):
        st = ora.step(st, dt, cg_iters=iters)
    return out, st


def test_session_tet_box_matches_oracle():
    m = meshgen.box_tets(9, 8, 7, jitter=0.2, seed=4)
    u, p = meshgen.c2_initial(m.coords)
    p = np.cos(3 * m.coords[:, 0])
    (uo, po), st = _run(m, dict(p_fixed=meshgen.boundary_nodes(m)), dict(rho=1.0, mu=1e-2, c_vreman=0.07),
                        u, p, 3, 1e-3, 30)
    assert rel_l2(uo, st["u"]) <= 1e-8
    assert rel_l2(po, st["p"]) <= 1e-8


def test_session_several_cg_tiles_matches_oracle():
    """12k nodes: the session's tiled single-pass CG over several 2048-row
    tiles with ghost rows (native tile map), pressure solves converged."""
    m = meshgen.box_tets(24, 22, 20, jitter=0.2, seed=8)
    assert m.n_nodes > 4 * 2048
    u, p = meshgen.c2_initial(m.coords)
    (uo, po), st = _run(m, dict(p_fixed=meshgen.boundary_nodes(m)), dict(rho=1.0, mu=1e-2, c_vreman=0.07),
                        u, p, 2, 1e-3, 400)
    assert rel_l2(uo, st["u"]) <= 1e-8
    assert rel_l2(po, st["p"]) <= 1e-8


def test_session_mixed_wall_model_matches_oracle():
    """All four element kinds, velocity Dirichlet values, wall-model faces.
    The pressure solves run 200 fixed iterations (converged): this system's
    unconverged CG iterate amplifies rounding (40 iterations: ~1e-9..1e-8
    between CG forms of the same algorithm), which is not what this tests."""
    m = meshgen.c3_mesh(0.08)
    bc, wall = meshgen.wall_model_bcs(m)
    x = m.coords
    u = np.stack([np.ones(len(x)) + 0.1 * np.sin(7 * x[:, 1]), 0.05 * np.cos(5 * x[:, 0]),
                  0.02 * np.sin(3 * x[:, 2])], axis=1)
    (uo, po), st = _run(m, bc, dict(rho=1.0, mu=2e-3, c_vreman=0.07), u, np.zeros(len(x)), 2, 1e-3, 200, wall=wall)
    assert rel_l2(uo, st["u"]) <= 1e-8
    assert rel_l2(po, st["p"]) <= 1e-8


def test_session_periodic_hex_tgv():
    m = meshgen.c1_mesh(8)
    u, p = fem.tgv_initial(m.coords)
    pf = np.zeros(m.n_nodes, bool)
    pf[0] = True
    (uo, po), st = _run(m, dict(p_fixed=pf), dict(rho=1.0, mu=1 / 1600, c_vreman=0.0), u, p, 2, 1e-2, 60)
    assert rel_l2(uo, st["u"]) <= 1e-8
    assert rel_l2(po, st["p"]) <= 1e-8


def test_session_errors_are_reported():
    from paper_2005_05899_b200._lib import lib
    L = lib()
    ctx = C.c_void_p()
    assert L.ab_ctx_create(0, C.byref(ctx)) == 0
    assert L.ab_step(ctx, 1e-3, 10, None) == -1
    assert b"no mesh" in L.ab_last_error()
    assert L.ab_ctx_destroy(ctx) == 0
    assert L.ab_ctx_create(10_000, C.byref(ctx)) == -1

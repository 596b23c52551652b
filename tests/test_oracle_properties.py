"""Property checks of the (parity-unpinned) Navier-Stokes oracle: the
register of SURVEY.md Appendix A self-checks.  CPU only."""

import json

import numpy as np
import pytest
import scipy.sparse.linalg as spla

from conftest import GOLDEN
from oracle import fem
from paper_2005_05899_b200 import meshgen


@pytest.mark.parametrize("rule", ["tet1", "tet4", "pyr5", "pri6", "hex8"])
def test_partition_of_unity_and_rule_weights(rule):
    N, dN = fem.shape_tables(rule)
    assert np.allclose(N.sum(axis=0), 1.0, atol=1e-15)
    assert np.allclose(dN.sum(axis=0), 0.0, atol=1e-15)
    _, w = fem.rule_points_weights(rule)
    vol = {"tet": 1 / 6, "pyr": 4 / 3, "pri": 1.0, "hex": 8.0}[fem.RULE_KIND[rule]]
    assert abs(w.sum() - vol) < 1e-15


def test_pyramid_rule_moments():
    """pyr5 integrates 1, z, z^2, x^2, x^2 z exactly on [-1,1]^2 x [0,1]."""
    pts, w = fem.rule_points_weights("pyr5")
    x, z = pts[:, 0], pts[:, 2]
    exact = {"1": 4 / 3, "z": 1 / 3, "z2": 2 / 15, "x2": 4 / 15, "x2z": 2 / 45}
    got = {"1": w.sum(), "z": w @ z, "z2": w @ z ** 2, "x2": w @ x ** 2, "x2z": w @ (x ** 2 * z)}
    for k in exact:
        assert abs(got[k] - exact[k]) < 1e-15, k


def test_mixed_mesh_volume_and_laplacian():
    m = meshgen.c3_mesh(0.05)
    assert abs(fem.lumped_mass(m).sum() - 1.0) < 1e-13
    L = fem.laplacian(m)
    assert abs(L - L.T).max() < 1e-15
    assert np.abs(L @ np.ones(m.n_nodes)).max() < 1e-14
    inner = ~meshgen.boundary_nodes(m)
    for d in range(3):  # linear fields are harmonic
        assert np.abs((L @ m.coords[:, d])[inner]).max() < 1e-14


def test_emac_energy_neutrality_periodic():
    m = meshgen.c1_mesh(8)
    u, _ = fem.tgv_initial(m.coords)
    u = u + 0.05 * np.random.default_rng(0).standard_normal(u.shape)
    R = fem.momentum_rhs(m, u, rho=1.0, mu=0.0, c_vreman=0.0)
    assert abs(np.sum(u * R)) <= 1e-12 * np.linalg.norm(u) * np.linalg.norm(R)


def test_linear_reproduction_of_divergence_and_gradient():
    m = meshgen.box_tets(5, 4, 6, jitter=0.2, seed=2)
    x = m.coords
    inner = ~meshgen.boundary_nodes(m)
    ml = fem.lumped_mass(m)
    u = np.stack([2 * x[:, 0], -x[:, 1] + x[:, 2], 0.5 * x[:, 2]], axis=1)
    assert np.allclose(fem.divergence(m, u)[inner], 1.5 * ml[inner], rtol=0, atol=1e-14)
    g = fem.gradient(m, 3 * x[:, 0] - x[:, 2])
    assert np.allclose(g[inner], ml[inner, None] * np.array([3.0, 0.0, -1.0]), rtol=0, atol=1e-14)


def test_pcg_matches_direct_solve():
    m = meshgen.c3_mesh(0.05)
    fixed = meshgen.boundary_nodes(m)
    L = fem.laplacian(m, fixed)
    b = np.random.default_rng(1).standard_normal(m.n_nodes)
    b[fixed] = 0
    x, it, res = fem.pcg(L, b, 1.0 / L.diagonal(), 1000, tol=1e-12)
    assert res <= 1e-12 and it < 1000
    assert np.linalg.norm(x - spla.spsolve(L.tocsc(), b)) <= 1e-10 * np.linalg.norm(x)


def test_projection_reduces_divergence_and_tgv_decays():
    m = meshgen.c1_mesh(12)
    u, p = fem.tgv_initial(m.coords)
    pf = np.zeros(m.n_nodes, bool)
    pf[0] = True
    o = fem.FlowOracle(m, 1.0, 1 / 1600, 0.0, p_fixed=pf)
    st = o.init_state(u, p)
    ke0 = np.sum(o.ml[:, None] * st["u"] ** 2)
    for _ in range(3):
        st = o.step(st, 1e-2, cg_iters=300, cg_tol=1e-11)
    ke = np.sum(o.ml[:, None] * st["u"] ** 2)
    assert ke < ke0
    assert (ke0 - ke) / ke0 < 1e-2


def test_balance_metrics_match_reference():
    from paper_2005_05899_b200.balance import TimingSample, compute_metrics
    ex = json.loads((GOLDEN / "reference_balance.json").read_text())["examples"]
    for e in ex:
        mt = compute_metrics(TimingSample(1, np.array(e["times"])))
        assert mt.mean == e["mean"] and mt.imbalance == e["imbalance"] and mt.lb == e["lb"]
        assert np.array_equal(mt.per_rank, e["per_rank"]) and np.array_equal(mt.deviations, e["deviations"])
    with pytest.raises(ValueError):
        TimingSample(1, np.array([1.0, 0.0]))


def test_wall_model_oracle_properties():
    """Equilibrium wall model (oracle/fem.py:wall_traction): Reichardt's law is
    solved to rounding, the traction opposes the tangential exchange velocity,
    normal velocity produces none, and the product's face extraction equals
    the oracle's."""
    from paper_2005_05899_b200 import meshgen
    from paper_2005_05899_b200.wall import wall_faces
    ut = np.array([1e-3, 0.1, 1.0, 10.0])
    for y in (1e-4, 1e-2, 0.3):
        utau = fem.reichardt_utau(ut, np.full(4, y), 1e-3)
        up, _ = fem.reichardt_uplus(y * utau / 1e-3)
        assert np.all(np.abs(utau * up - ut) <= 1e-13 * ut)
    m = meshgen.c3_mesh(0.05)
    on = np.abs(m.coords[:, 2] - m.coords[:, 2].min()) < 1e-12
    F, O = fem.wall_faces(m, on)
    Fp, Op = wall_faces(m, on)
    assert np.array_equal(F, Fp) and np.array_equal(O, Op)
    assert F.shape[0] > 0 and np.all(on[F[F >= 0]])
    u = np.zeros((m.n_nodes, 3))
    assert np.abs(fem.wall_traction(m, F, O, u, 1.0, 1e-3)).max() == 0.0
    u[:, 2] = 0.7                                  # normal to the wall: no shear
    assert np.abs(fem.wall_traction(m, F, O, u, 1.0, 1e-3)).max() <= 1e-15
    u[:, 0], u[:, 1] = 1.0, -0.5                   # tangential part (1, -0.5)
    R = fem.wall_traction(m, F, O, u, 1.2, 1e-3)
    assert np.all(R[:, 2] == 0.0)
    f = R.sum(axis=0)
    assert f[0] < 0 and f[1] > 0 and abs(f[0] / f[1] + 2.0) <= 1e-12   # parallel to -(1, -0.5)

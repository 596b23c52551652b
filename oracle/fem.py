"""ORACLE — CPU restatement of the time-step hot path.  TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this module, and only as the checker or
the timed CPU baseline.  The product package never imports it.

Parity status
-------------
* Reference-pinned: reference-element tables for tet1/tet4/hex8, |det J|, the
  packed mass matrix and the lumped mass (row sums of the scattered global
  matrix).  These restate reference pkg/src/coexbal/assembly.py and are pinned
  against golden vectors produced by running the reference itself
  (tests/golden/make_golden.py -> tests/golden/reference_mass.npz).
* PARITY UNPINNED (the reference has no Navier-Stokes code): the
  momentum RHS, divergence/gradient, Laplacian, Jacobi-PCG, the RK3
  fractional step and the equilibrium wall model (boundary assembly,
  Algorithm 1 line 4) below are restated from
  PAPER.md:192-237 with the decisions of SURVEY.md Appendix A fixed in
  DESIGN.md §3.  They are cross-checked by
  property tests (partition of unity, EMAC energy neutrality, SPD Laplacian,
  PCG vs scipy spsolve, TGV energy decay), not by the reference.

Everything is vectorised numpy over elements of one category, processed in
chunks so multi-million-element meshes fit in host memory.
"""

from __future__ import annotations

import math

import numpy as np
import scipy.sparse as sp

CHUNK = 1 << 18

# ---------------------------------------------------------------------------
# Reference-element tables.  tet/hex follow reference assembly.py:33-117
# verbatim in value; pri6/pyr5 are new (absent in the reference).
# ---------------------------------------------------------------------------

_HEX_SIGNS = np.array([[-1, -1, -1], [1, -1, -1], [1, 1, -1], [-1, 1, -1],
                       [-1, -1, 1], [1, -1, 1], [1, 1, 1], [-1, 1, 1]], dtype=np.float64)  # assembly.py:38-50
_TET4_A = (5.0 + 3.0 * math.sqrt(5.0)) / 20.0   # assembly.py:72
_TET4_B = (5.0 - math.sqrt(5.0)) / 20.0         # assembly.py:73
_G3 = 1.0 / math.sqrt(3.0)                      # assembly.py:74
# pyr5: 5-point rule on the pyramid [-1,1]^2 x [0,1] (apex (0,0,1), volume 4/3)
# exact for 1, z, z^2, x^2, y^2, x^2 z and all odd moments.
_PYR_A = math.sqrt(32.0 / 135.0)
_PYR_Z1 = 1.0 / 6.0
_PYR_Z2 = 7.0 / 10.0
_PYR_W1 = 9.0 / 32.0
_PYR_W2 = 5.0 / 24.0

RULE_KIND = {"tet1": "tet", "tet4": "tet", "hex8": "hex", "pri6": "pri", "pyr5": "pyr"}
NNODE = {"tet": 4, "pyr": 5, "pri": 6, "hex": 8}


def rule_points_weights(rule: str):
    if rule == "tet1":                                     # assembly.py:90-95
        return np.array([[0.25, 0.25, 0.25]]), np.array([1.0 / 6.0])
    if rule == "tet4":                                     # assembly.py:96-108
        a, b = _TET4_A, _TET4_B
        return np.array([[a, b, b], [b, a, b], [b, b, a], [b, b, b]]), np.full(4, 1.0 / 24.0)
    if rule == "hex8":                                     # assembly.py:109-116
        return np.array([[sx * _G3, sy * _G3, sz * _G3] for sx, sy, sz in _HEX_SIGNS]), np.ones(8)
    if rule == "pri6":  # 3-point triangle rule x 2-point Gauss line
        tri = [(1.0 / 6.0, 1.0 / 6.0), (2.0 / 3.0, 1.0 / 6.0), (1.0 / 6.0, 2.0 / 3.0)]
        pts = [[x, y, z] for z in (-_G3, _G3) for (x, y) in tri]
        return np.array(pts), np.full(6, 1.0 / 6.0)
    if rule == "pyr5":
        a = _PYR_A
        pts = [[-a, -a, _PYR_Z1], [a, -a, _PYR_Z1], [a, a, _PYR_Z1], [-a, a, _PYR_Z1], [0.0, 0.0, _PYR_Z2]]
        return np.array(pts), np.array([_PYR_W1] * 4 + [_PYR_W2])
    raise KeyError(f"unknown integration rule {rule!r}")


def shape_tables(rule: str):
    """N[a,g] and dN/dxi[a,g,3] of the rule's element kind at its points."""
    pts, _ = rule_points_weights(rule)
    kind = RULE_KIND[rule]
    g = len(pts)
    xi, eta, zeta = pts[:, 0], pts[:, 1], pts[:, 2]
    if kind == "tet":                                      # assembly.py:33-35
        N = np.stack([1.0 - xi - eta - zeta, xi, eta, zeta])
        dN = np.zeros((4, g, 3))
        dN[0] = -1.0
        dN[1, :, 0] = 1.0
        dN[2, :, 1] = 1.0
        dN[3, :, 2] = 1.0
        return N, dN
    if kind == "hex":                                      # assembly.py:53-69
        N = np.empty((8, g))
        dN = np.empty((8, g, 3))
        for i, (sx, sy, sz) in enumerate(_HEX_SIGNS):
            fx, fy, fz = 1 + sx * xi, 1 + sy * eta, 1 + sz * zeta
            N[i] = fx * fy * fz / 8.0
            dN[i, :, 0] = sx * fy * fz / 8.0
            dN[i, :, 1] = fx * sy * fz / 8.0
            dN[i, :, 2] = fx * fy * sz / 8.0
        return N, dN
    if kind == "pri":  # L_a(xi,eta) * (1 -/+ zeta)/2, VTK wedge order
        L = [1.0 - xi - eta, xi, eta]
        dL = [(-1.0, -1.0), (1.0, 0.0), (0.0, 1.0)]
        N = np.empty((6, g))
        dN = np.empty((6, g, 3))
        for half, sz in ((0, -1.0), (1, 1.0)):
            fz = (1.0 + sz * zeta) / 2.0
            for a in range(3):
                i = 3 * half + a
                N[i] = L[a] * fz
                dN[i, :, 0] = dL[a][0] * fz
                dN[i, :, 1] = dL[a][1] * fz
                dN[i, :, 2] = L[a] * sz / 2.0
        return N, dN
    if kind == "pyr":  # rational basis, base (+-1,+-1,0), apex (0,0,1)
        s = 1.0 - zeta
        N = np.empty((5, g))
        dN = np.empty((5, g, 3))
        for i, (sx, sy) in enumerate([(-1, -1), (1, -1), (1, 1), (-1, 1)]):
            N[i] = (s + sx * xi) * (s + sy * eta) / (4.0 * s)
            dN[i, :, 0] = sx * (s + sy * eta) / (4.0 * s)
            dN[i, :, 1] = sy * (s + sx * xi) / (4.0 * s)
            dN[i, :, 2] = -0.25 + sx * sy * xi * eta / (4.0 * s * s)
        N[4] = zeta
        dN[4] = 0.0
        dN[4, :, 2] = 1.0
        return N, dN
    raise KeyError(kind)


# ---------------------------------------------------------------------------
# Geometry
# ---------------------------------------------------------------------------

def element_coords(coords, conn, period=None):
    """Gather element node coordinates, unwrapping periodic axes by minimum
    image relative to the element's first node."""
    X = coords[conn]
    if period is not None and np.any(np.asarray(period) > 0):
        for d in range(3):
            L = float(period[d])
            if L > 0:
                rel = X[:, :, d] - X[:, :1, d]
                X[:, :, d] = X[:, :1, d] + rel - L * np.rint(rel / L)
    return X


def det3(m):
    """Cofactor determinant of (...,3,3) (as reference assembly.py:268-273)."""
    return (m[..., 0, 0] * (m[..., 1, 1] * m[..., 2, 2] - m[..., 1, 2] * m[..., 2, 1])
            - m[..., 0, 1] * (m[..., 1, 0] * m[..., 2, 2] - m[..., 1, 2] * m[..., 2, 0])
            + m[..., 0, 2] * (m[..., 1, 0] * m[..., 2, 1] - m[..., 1, 1] * m[..., 2, 0]))


def inv3(m):
    det = det3(m)
    adj = np.empty_like(m)
    adj[..., 0, 0] = m[..., 1, 1] * m[..., 2, 2] - m[..., 1, 2] * m[..., 2, 1]
    adj[..., 0, 1] = m[..., 0, 2] * m[..., 2, 1] - m[..., 0, 1] * m[..., 2, 2]
    adj[..., 0, 2] = m[..., 0, 1] * m[..., 1, 2] - m[..., 0, 2] * m[..., 1, 1]
    adj[..., 1, 0] = m[..., 1, 2] * m[..., 2, 0] - m[..., 1, 0] * m[..., 2, 2]
    adj[..., 1, 1] = m[..., 0, 0] * m[..., 2, 2] - m[..., 0, 2] * m[..., 2, 0]
    adj[..., 1, 2] = m[..., 0, 2] * m[..., 1, 0] - m[..., 0, 0] * m[..., 1, 2]
    adj[..., 2, 0] = m[..., 1, 0] * m[..., 2, 1] - m[..., 1, 1] * m[..., 2, 0]
    adj[..., 2, 1] = m[..., 0, 1] * m[..., 2, 0] - m[..., 0, 0] * m[..., 2, 1]
    adj[..., 2, 2] = m[..., 0, 0] * m[..., 1, 1] - m[..., 0, 1] * m[..., 1, 0]
    return adj / det[..., None, None], det


def geometry(X, rule):
    """Per Gauss point: |det J| (E,g), dV = |det J| w (E,g), dN/dx (E,g,n,3).

    J[i,j] = dx_i/dxi_j = sum_a x_a,i dN_a/dxi_j  (reference assembly.py:138).
    """
    N, dN = shape_tables(rule)
    _, w = rule_points_weights(rule)
    J = np.einsum("eai,agj->egij", X, dN)
    invJ, det = inv3(J)
    adet = np.abs(det)
    dNdx = np.einsum("agj,egjk->egak", dN, invJ)
    return adet, adet * w[None, :], dNdx


def jacobian_dets(X, rule):
    """|det J| at every Gauss point; tets use the edge matrix (assembly.py:131-133)."""
    kind = RULE_KIND[rule]
    _, w = rule_points_weights(rule)
    if kind == "tet":
        e = X[:, 1:] - X[:, :1]
        d = np.abs(det3(e))
        return np.repeat(d[:, None], len(w), axis=1)
    adet, _, _ = geometry(X, rule)
    return adet


def element_mass(X, rule):
    """Ae[e,i,j] = sum_g J[e,g] w[g] N[i,g] N[j,g], Gauss ascending
    (reference assembly.py:227-244 / :247-263)."""
    N, _ = shape_tables(rule)
    _, w = rule_points_weights(rule)
    J = jacobian_dets(X, rule)
    n = N.shape[0]
    ae = np.zeros((X.shape[0], n, n))
    for g in range(len(w)):
        outer = N[:, g][:, None] * N[:, g][None, :]
        ae += (J[:, g] * w[g])[:, None, None] * outer[None]
    return ae, J


def _chunks(n):
    for s in range(0, n, CHUNK):
        yield s, min(n, s + CHUNK)


def lumped_mass(mesh):
    """M_L = row sums of the scattered consistent mass matrix
    (reference assembly.py:306-309 applied to scatter_global :317-333)."""
    ml = np.zeros(mesh.n_nodes)
    for _tag, rule, conn, _ids in mesh.categories():
        for s, e in _chunks(conn.shape[0]):
            ae, _ = element_mass(element_coords(mesh.coords, conn[s:e], mesh.period), rule)
            np.add.at(ml, conn[s:e].ravel(), ae.sum(axis=2).ravel())
    return ml


def scatter_coo(mesh, mats):
    """Global COO (rows, cols, vals) summed, sorted row-major (assembly.py:317-333)."""
    rows, cols, vals = [], [], []
    for (tag, rule, conn, ids) in mesh.categories():
        ae = mats[rule]
        n = conn.shape[1]
        rows.append(np.repeat(conn, n, axis=1).ravel())
        cols.append(np.tile(conn, (1, n)).ravel())
        vals.append(ae.reshape(ae.shape[0], -1).ravel())
    A = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(mesh.n_nodes, mesh.n_nodes)).tocsr()
    A.sum_duplicates()
    A.sort_indices()
    return A


# ---------------------------------------------------------------------------
# Navier-Stokes operators (PARITY UNPINNED)
# ---------------------------------------------------------------------------

def _scatter(out, conn, contrib):
    """out[conn[e,a]] += contrib[e,a,...]"""
    flat = contrib.reshape(conn.size, -1) if contrib.ndim > 2 else contrib.ravel()
    np.add.at(out, conn.ravel(), flat)


def momentum_rhs(mesh, u, rho=1.0, mu=1.0, c_vreman=0.0):
    """R_a = -sum_e int N_a rho [2 eps(u) u + (div u) u] dV
             -sum_e int 2 (mu + mu_t) eps(u) : grad N_a dV

    EMAC convective form with the modified pressure (PAPER.md:195-211,
    SURVEY Appendix A option (A)); Vreman mu_t = rho c sqrt(B_beta / a:a),
    Delta = V_e^(1/3).  Returns (N,3).
    """
    R = np.zeros((mesh.n_nodes, 3))
    for _tag, rule, conn, _ids in mesh.categories():
        N, _ = shape_tables(rule)
        for s, e in _chunks(conn.shape[0]):
            c = conn[s:e]
            X = element_coords(mesh.coords, c, mesh.period)
            U = u[c]                                               # (E,n,3)
            _, dV, dNdx = geometry(X, rule)
            ug = np.einsum("ag,eai->egi", N, U)                    # (E,g,3)
            G = np.einsum("eai,egaj->egij", U, dNdx)               # G_ij = du_i/dx_j
            div = np.trace(G, axis1=2, axis2=3)
            eps = 0.5 * (G + np.swapaxes(G, 2, 3))
            conv = 2.0 * np.einsum("egij,egj->egi", eps, ug) + div[..., None] * ug
            mu_eff = mu + (vreman(G, dV.sum(axis=1), rho, c_vreman) if c_vreman > 0 else 0.0)
            sig = 2.0 * mu_eff[..., None, None] * eps if np.ndim(mu_eff) else 2.0 * mu_eff * eps
            contrib = -(rho * np.einsum("ag,eg,egi->eai", N, dV, conv)
                        + np.einsum("eg,egij,egaj->eai", dV, sig, dNdx))
            _scatter(R, c, contrib)
    return R


def vreman(G, vol, rho, c):
    """mu_t per Gauss point (E,g) from G (E,g,3,3) and element volume (E,)."""
    alpha = np.swapaxes(G, 2, 3)                    # alpha_ij = du_j/dx_i
    delta2 = np.cbrt(vol) ** 2
    beta = delta2[:, None, None, None] * np.einsum("egmi,egmj->egij", alpha, alpha)
    B = (beta[..., 0, 0] * beta[..., 1, 1] - beta[..., 0, 1] ** 2
         + beta[..., 0, 0] * beta[..., 2, 2] - beta[..., 0, 2] ** 2
         + beta[..., 1, 1] * beta[..., 2, 2] - beta[..., 1, 2] ** 2)
    aa = np.einsum("egij,egij->eg", alpha, alpha)
    B = np.maximum(B, 0.0)
    with np.errstate(divide="ignore", invalid="ignore"):
        mt = np.where(aa > 1e-30, rho * c * np.sqrt(B / np.where(aa > 1e-30, aa, 1.0)), 0.0)
    return mt


def divergence(mesh, u):
    """(D u)_a = sum_e int N_a div(u) dV."""
    out = np.zeros(mesh.n_nodes)
    for _tag, rule, conn, _ids in mesh.categories():
        N, _ = shape_tables(rule)
        for s, e in _chunks(conn.shape[0]):
            c = conn[s:e]
            _, dV, dNdx = geometry(element_coords(mesh.coords, c, mesh.period), rule)
            div = np.einsum("eai,egai->eg", u[c], dNdx)
            _scatter(out, c, np.einsum("ag,eg,eg->ea", N, dV, div))
    return out


def gradient(mesh, p):
    """(G p)_a = sum_e int N_a grad(p) dV, (N,3)."""
    out = np.zeros((mesh.n_nodes, 3))
    for _tag, rule, conn, _ids in mesh.categories():
        N, _ = shape_tables(rule)
        for s, e in _chunks(conn.shape[0]):
            c = conn[s:e]
            _, dV, dNdx = geometry(element_coords(mesh.coords, c, mesh.period), rule)
            gp = np.einsum("ea,egai->egi", p[c], dNdx)
            _scatter(out, c, np.einsum("ag,eg,egi->eai", N, dV, gp))
    return out


def laplacian(mesh, fixed=None):
    """L_ab = sum_e int grad N_a . grad N_b dV, scipy CSR.
    Rows/cols of ``fixed`` nodes are replaced by identity (Dirichlet)."""
    rows, cols, vals = [], [], []
    for _tag, rule, conn, _ids in mesh.categories():
        n = conn.shape[1]
        for s, e in _chunks(conn.shape[0]):
            c = conn[s:e]
            _, dV, dNdx = geometry(element_coords(mesh.coords, c, mesh.period), rule)
            le = np.einsum("eg,egak,egbk->eab", dV, dNdx, dNdx)
            rows.append(np.repeat(c, n, axis=1).ravel())
            cols.append(np.tile(c, (1, n)).ravel())
            vals.append(le.ravel())
    A = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(mesh.n_nodes, mesh.n_nodes)).tocsr()
    A.sum_duplicates()
    A.sort_indices()
    if fixed is not None and np.any(fixed):
        A = apply_dirichlet(A, fixed)
    return A


def apply_dirichlet(A, fixed):
    """Zero rows and columns of fixed nodes (pattern kept), unit diagonal."""
    A = A.tocsr(copy=True)
    fixed = np.asarray(fixed, dtype=bool)
    row_of = np.repeat(np.arange(A.shape[0]), np.diff(A.indptr))
    kill = fixed[row_of] | fixed[A.indices]
    A.data[kill] = 0.0
    diag_pos = kill & (row_of == A.indices)
    A.data[diag_pos] = 1.0
    return A


def pcg(A, b, dinv, maxit, tol=0.0, x0=None):
    """Jacobi-preconditioned CG in the exact operation
    order of the fused GPU kernels: the direction update
    p = z + beta p is evaluated at the start of the next SpMV, and the SpMV
    is applied to the preconditioned residual, q = A p = A z + beta q_old
    (the recursive form of A p, so only z is gathered by the SpMV).

    Stops after ``maxit`` iterations or when ||r||/||b|| <= tol (tol > 0).
    Returns (x, iterations, ||r||/||b||).
    """
    x = np.zeros_like(b) if x0 is None else x0.copy()
    r = b - A @ x if x0 is not None else b.copy()
    z = dinv * r
    rz = float(r @ z)
    bb = float(b @ b)
    rr = float(r @ r)
    p = np.zeros_like(b)
    q = np.zeros_like(b)
    beta = 0.0
    it = 0
    while it < maxit:
        if tol > 0 and bb > 0 and math.sqrt(rr / bb) <= tol:
            break
        p = z + beta * p
        q = A @ z + beta * q
        pq = float(p @ q)
        alpha = rz / pq if pq != 0.0 else 0.0
        x += alpha * p
        r -= alpha * q
        z = dinv * r
        rz_new = float(r @ z)
        rr = float(r @ r)
        beta = rz_new / rz if rz != 0.0 else 0.0
        rz = rz_new
        it += 1
    res = math.sqrt(rr / bb) if bb > 0 else 0.0
    return x, it, res


# ---------------------------------------------------------------------------
# Fractional-step explicit RK3 time step (Algorithm 1)
# ---------------------------------------------------------------------------

# SSP-RK3 (Shu-Osher) in stage form u_s = a_s u^n + b_s (u_{s-1} + dt F(u_{s-1}))
RK3_A = (0.0, 0.75, 1.0 / 3.0)
RK3_B = (1.0, 0.25, 2.0 / 3.0)


# ---------------------------------------------------------------------------
# Boundary assembly: equilibrium wall model (Algorithm 1 line 4, PAPER.md:214,
# :228, :256-257).  The cited wall-law paper is not in /root/reference: the
# law (Reichardt), exchange location and face integration are the decisions
# of DESIGN.md §3.
# ---------------------------------------------------------------------------
# local faces per kind, VTK node order, quads listed around their perimeter
FACES = {
    "tet": [(0, 1, 2), (0, 1, 3), (1, 2, 3), (0, 2, 3)],
    "pyr": [(0, 1, 2, 3), (0, 1, 4), (1, 2, 4), (2, 3, 4), (3, 0, 4)],
    "pri": [(0, 1, 2), (3, 4, 5), (0, 1, 4, 3), (1, 2, 5, 4), (2, 0, 3, 5)],
    "hex": [(0, 1, 2, 3), (4, 5, 6, 7), (0, 1, 5, 4), (1, 2, 6, 5), (2, 3, 7, 6), (3, 0, 4, 7)],
}
KAPPA = 0.41
REICHARDT_ITERS = 12


def wall_faces(mesh, on_wall):
    """Boundary faces whose nodes all satisfy ``on_wall`` (bool per node):
    (face nodes (F,4), -1 padded for triangles; off-face nodes of the owning
    element (F,4), -1 padded), ordered by (category, element, local face)."""
    on_wall = np.asarray(on_wall, bool)
    fn, off = [], []
    for _tag, rule, conn, _ids in mesh.categories():
        kind = RULE_KIND[rule]
        nn = NNODE[kind]
        for f in FACES[kind]:
            hit = on_wall[conn[:, list(f)]].all(axis=1)
            if not hit.any():
                continue
            rest = [a for a in range(nn) if a not in f]
            F = np.full((int(hit.sum()), 4), -1, np.int64)
            F[:, :len(f)] = conn[hit][:, list(f)]
            O = np.full((int(hit.sum()), 4), -1, np.int64)
            O[:, :len(rest)] = conn[hit][:, rest[:4]] if len(rest) <= 4 else conn[hit][:, rest[:4]]
            fn.append((conn[hit].shape[0], F, O, np.nonzero(hit)[0], kind, f))
    if not fn:
        return np.zeros((0, 4), np.int64), np.zeros((0, 4), np.int64)
    return np.concatenate([x[1] for x in fn]), np.concatenate([x[2] for x in fn])


def reichardt_uplus(yp):
    """Reichardt's law u+ (y+) and its derivative."""
    e11, e3 = np.exp(-yp / 11.0), np.exp(-yp / 3.0)
    up = np.log1p(KAPPA * yp) / KAPPA + 7.8 * (1.0 - e11 - (yp / 11.0) * e3)
    dup = 1.0 / (1.0 + KAPPA * yp) + 7.8 * (e11 / 11.0 - e3 / 11.0 + (yp / 33.0) * e3)
    return up, dup


def reichardt_utau(ut, y, nu, iters=REICHARDT_ITERS):
    """u_tau with ut = u_tau u+(y u_tau / nu): Newton from the viscous-
    sublayer guess sqrt(nu ut / y), a fixed number of iterations."""
    ut = np.asarray(ut, float)
    live = ut > 0.0                     # no tangential velocity: no shear
    ut_l = np.where(live, ut, 1.0)
    utau = np.sqrt(nu * ut_l / y)
    for _ in range(iters):
        yp = y * utau / nu
        up, dup = reichardt_uplus(yp)
        f = utau * up - ut_l
        df = up + yp * dup
        utau = np.maximum(utau - f / df, 0.0)
    return np.where(live, utau, 0.0)


def wall_traction(mesh, faces, off, u, rho=1.0, mu=1.0):
    """Boundary assembly of the wall model: per wall face, the exchange point
    is the mean of the owning element's off-face nodes (velocity u_e, wall
    distance y to the face plane); tau_w = rho u_tau^2 from Reichardt's law
    on |u_t|, u_t = u_e - (u_e.n) n; every face node receives
    -tau_w u_t/|u_t| * A_face / n_face_nodes.  Returns (N,3)."""
    R = np.zeros((mesh.n_nodes, 3))
    if faces.shape[0] == 0:
        return R
    X = mesh.coords
    nf = (faces >= 0).sum(axis=1)
    no = (off >= 0).sum(axis=1)
    fx = np.where((faces >= 0)[..., None], X[np.maximum(faces, 0)], 0.0)           # (F,4,3)
    xc = fx.sum(axis=1) / nf[:, None]
    ox = np.where((off >= 0)[..., None], X[np.maximum(off, 0)], 0.0)
    xe = ox.sum(axis=1) / no[:, None]
    ue = np.where((off >= 0)[..., None], u[np.maximum(off, 0)], 0.0).sum(axis=1) / no[:, None]
    a = np.cross(fx[:, 1] - fx[:, 0], fx[:, 2] - fx[:, 0])
    quad = nf == 4
    b = np.cross(fx[:, 2] - fx[:, 0], fx[:, 3] - fx[:, 0])
    area = 0.5 * np.linalg.norm(a, axis=1) + np.where(quad, 0.5 * np.linalg.norm(b, axis=1), 0.0)
    nv = a + np.where(quad[:, None], b, 0.0)
    nv = nv / np.linalg.norm(nv, axis=1)[:, None]
    nv = np.where((np.einsum("fi,fi->f", nv, xc - xe) < 0.0)[:, None], -nv, nv)    # outward
    y = np.abs(np.einsum("fi,fi->f", xe - xc, nv))
    un = np.einsum("fi,fi->f", ue, nv)
    utv = ue - un[:, None] * nv
    utm = np.linalg.norm(utv, axis=1)
    utau = reichardt_utau(utm, y, mu / rho)
    coef = np.where(utm > 0.0, -rho * utau * utau / np.where(utm > 0.0, utm, 1.0) * area / nf, 0.0)
    contrib = coef[:, None] * utv                                                   # per face node
    for k in range(4):
        m = faces[:, k] >= 0
        np.add.at(R, faces[m, k], contrib[m])
    return R


class FlowOracle:
    """Incremental-projection fractional step with SSP-RK3 momentum stages.

    Per step:
      for s in 1..3:  R_s = R(u_{s-1});  u_s = a_s u^n + b_s (u_{s-1} + dt/rho M_L^-1 (R_s - Gp))
                      velocity Dirichlet values re-imposed
      b  = -(rho/dt) D u_3, b = 0 on pressure-Dirichlet nodes
      L' dp = b by Jacobi-PCG (x0 = 0)
      Gd = G dp;  u^{n+1} = u_3 - dt/rho M_L^-1 Gd;  p += dp;  Gp += Gd
    """

    def __init__(self, mesh, rho=1.0, mu=1.0, c_vreman=0.0, p_fixed=None,
                 u_fixed=None, u_fixed_values=None, wall=None):
        self.mesh = mesh
        self.wall = wall  # (faces, off) of wall_faces(): boundary assembly per stage
        self.rho, self.mu, self.c_vreman = rho, mu, c_vreman
        n = mesh.n_nodes
        self.p_fixed = np.zeros(n, bool) if p_fixed is None else np.asarray(p_fixed, bool)
        self.u_fixed = np.zeros((n, 3), bool) if u_fixed is None else np.asarray(u_fixed, bool)
        self.u_fixed_values = np.zeros((n, 3)) if u_fixed_values is None else np.asarray(u_fixed_values, float)
        self.ml = lumped_mass(mesh)
        self.minv = 1.0 / self.ml
        self.L = laplacian(mesh, self.p_fixed)
        self.dinv = 1.0 / self.L.diagonal()

    def init_state(self, u, p):
        u = np.array(u, dtype=np.float64)
        p = np.array(p, dtype=np.float64)
        u[self.u_fixed] = self.u_fixed_values[self.u_fixed]
        return {"u": u, "p": p, "gp": gradient(self.mesh, p)}

    def step(self, st, dt, cg_iters=50, cg_tol=0.0):
        u0 = st["u"]
        u = u0
        k = dt / self.rho
        for s in range(3):
            R = momentum_rhs(self.mesh, u, self.rho, self.mu, self.c_vreman)
            if self.wall is not None:
                R = R + wall_traction(self.mesh, *self.wall, u, self.rho, self.mu)
            u = RK3_A[s] * u0 + RK3_B[s] * (u + k * self.minv[:, None] * (R - st["gp"]))
            u[self.u_fixed] = self.u_fixed_values[self.u_fixed]
        b = -(self.rho / dt) * divergence(self.mesh, u)
        b[self.p_fixed] = 0.0
        dp, iters, res = pcg(self.L, b, self.dinv, cg_iters, cg_tol)
        gd = gradient(self.mesh, dp)
        u = u - k * self.minv[:, None] * gd
        u[self.u_fixed] = self.u_fixed_values[self.u_fixed]
        return {"u": u, "p": st["p"] + dp, "gp": st["gp"] + gd, "cg_iters": iters, "cg_res": res}


def tgv_initial(coords, V0=1.0):
    """Taylor-Green vortex on [0,2pi]^3."""
    x, y, z = coords[:, 0], coords[:, 1], coords[:, 2]
    u = np.stack([V0 * np.sin(x) * np.cos(y) * np.cos(z),
                  -V0 * np.cos(x) * np.sin(y) * np.cos(z),
                  np.zeros_like(x)], axis=1)
    p = (V0 ** 2 / 16.0) * (np.cos(2 * x) + np.cos(2 * y)) * (np.cos(2 * z) + 2.0)
    return u, p


def c2_initial(coords, seed=20200131, noise=0.01):
    """C2 velocity: TGV-like field on the unit cube + N(0, noise^2)."""
    x, y, z = (2 * np.pi * coords[:, i] for i in range(3))
    u = np.stack([np.sin(x) * np.cos(y) * np.cos(z), -np.cos(x) * np.sin(y) * np.cos(z),
                  np.zeros_like(x)], axis=1)
    rng = np.random.default_rng(seed)
    return u + rng.normal(0.0, noise, size=u.shape), np.zeros(coords.shape[0])

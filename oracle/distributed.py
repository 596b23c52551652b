"""ORACLE — the decomposed-domain time step on the CPU.  TEST INFRASTRUCTURE ONLY.

Mirrors paper_2005_05899_b200.timestep.FlowSolver with a halo exchanger:
every rank assembles its own elements (no halo elements), sums
duplicated interface-node values with its neighbours after each assembly and
SpMV, and all-reduces ownership-weighted dot
products.  Run under torch.distributed (gloo) with the
product's decomposition (decompose.py) and exchange protocol (halo.py), it
checks that the multi-GPU algorithm reproduces the single-domain oracle
(tests/test_halo_gloo.py).  Pack/unpack here are numpy, standing in for the
CUDA kernels ab_halo_pack / ab_halo_unpack_add.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import fem


def np_pack(idx, field, stride, ncomp, out):
    f = field.numpy().reshape(-1, stride) if stride > 1 else field.numpy().reshape(-1, 1)
    out.numpy()[: idx.numel() * ncomp] = f[idx.numpy(), :ncomp].ravel()


def np_unpack_add(idx, buf, stride, ncomp, field):
    f = field.numpy().reshape(-1, stride) if stride > 1 else field.numpy().reshape(-1, 1)
    np.add.at(f[:, :ncomp], idx.numpy(), buf.numpy()[: idx.numel() * ncomp].reshape(-1, ncomp))


class DistFlowOracle:
    def __init__(self, sub, halo, rho, mu, c_vreman, p_fixed_local, u_fixed=None, u_fixed_values=None,
                 wall=None):
        self.m, self.halo = sub, halo
        self.wall = wall  # (faces, off) of this rank's wall faces (each face belongs to one element)
        self.uf = None if u_fixed is None else np.asarray(u_fixed, bool)
        self.uv = None if u_fixed_values is None else np.asarray(u_fixed_values, float)
        self.rho, self.mu, self.cv = rho, mu, c_vreman
        n = sub.n_nodes
        self.own = halo.own.numpy()
        ml = torch.from_numpy(fem.lumped_mass(sub))
        halo.sum_(ml, 1, 1)
        self.ml = ml.numpy()
        self.minv = 1.0 / self.ml
        self.pf = np.asarray(p_fixed_local, bool)
        self.L = fem.laplacian(sub, self.pf)
        diag = torch.from_numpy(self.L.diagonal().copy())
        halo.sum_(diag, 1, 1)
        d = diag.numpy()
        d[self.pf] = 1.0
        self.dinv = 1.0 / d
        self.n = n

    def _sum3(self, a):
        t = torch.from_numpy(np.ascontiguousarray(a))
        self.halo.sum_(t, 3, 3)
        return t.numpy()

    def _sum1(self, a):
        t = torch.from_numpy(np.ascontiguousarray(a))
        self.halo.sum_(t, 1, 1)
        return t.numpy()

    def _allsum(self, vals):
        t = torch.tensor(vals, dtype=torch.float64)
        self.halo.allreduce_(t)
        return t.tolist()

    def _bc(self, u):
        if self.uf is not None:
            u[self.uf] = self.uv[self.uf]
        return u

    def init_state(self, u, p):
        return {"u": self._bc(np.array(u, float)), "p": np.array(p, float),
                "gp": self._sum3(fem.gradient(self.m, p))}

    def pcg(self, b, maxit):
        own = self.own
        r = np.where(self.pf, 0.0, b)
        z = self.dinv * r
        x = np.zeros_like(b)
        rz, rr = self._allsum([float(own @ (r * z)), float(own @ (r * r))])
        p = np.zeros_like(b)
        q = np.zeros_like(b)
        beta = 0.0
        for _ in range(maxit):
            p = z + beta * p
            q = self._sum1(self.L @ z) + beta * q
            pq = self._allsum([float(own @ (p * q))])[0]
            alpha = rz / pq if pq != 0.0 else 0.0
            x += alpha * p
            r -= alpha * q
            z = self.dinv * r
            rz_new, rr = self._allsum([float(own @ (r * z)), float(own @ (r * r))])
            beta = rz_new / rz if rz != 0.0 else 0.0
            rz = rz_new
        return x

    def step(self, st, dt, cg_iters):
        u0 = st["u"]
        u = u0
        k = dt / self.rho
        for s in range(3):
            R = fem.momentum_rhs(self.m, u, self.rho, self.mu, self.cv)
            if self.wall is not None:
                R = R + fem.wall_traction(self.m, *self.wall, u, self.rho, self.mu)
            R = self._sum3(R)
            u = fem.RK3_A[s] * u0 + fem.RK3_B[s] * (u + k * self.minv[:, None] * (R - st["gp"]))
            u = self._bc(u)
        b = self._sum1(-(self.rho / dt) * fem.divergence(self.m, u))
        dp = self.pcg(b, cg_iters)
        gd = self._sum3(fem.gradient(self.m, dp))
        u = self._bc(u - k * self.minv[:, None] * gd)
        return {"u": u, "p": st["p"] + dp, "gp": st["gp"] + gd}


def residual_norm(vals) -> float:
    return math.sqrt(sum(v * v for v in vals))

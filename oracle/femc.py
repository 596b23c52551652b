"""ORACLE (C restatement, oracle/fem_c.c) — TEST INFRASTRUCTURE AND CPU BASELINE ONLY.

``CFlowOracle`` is ``fem.FlowOracle`` with the per-step work (momentum RHS,
wall model, RK stages, divergence, Jacobi-PCG, gradient correction) in C +
OpenMP on all host cores; setup (lumped mass, Laplacian, Jacobi diagonal) and
the reference-element tables come from the numpy oracle, so both restatements
share every number.  bench.py's cpu_baseline and ``--impl reference`` legs
time it; tests/test_oracle_c.py checks it against ``fem.FlowOracle``.  The
product package never imports it.  PARITY UNPINNED by the reference (it has no
Navier-Stokes code).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

from . import fem

HERE = Path(__file__).resolve().parent
SRC = HERE / "fem_c.c"
LIB = HERE / "libfemc.so"
CFLAGS = ["-O3", "-march=x86-64-v3", "-fopenmp", "-fPIC", "-shared"]


def build(force: bool = False) -> Path:
    """gcc the restatement into oracle/libfemc.so (x86-64-v3: AVX2 + FMA, so
    the object built here runs on the GPU box's host CPU)."""
    if force or not LIB.exists() or LIB.stat().st_mtime < SRC.stat().st_mtime:
        tmp = LIB.with_suffix(".so.tmp")
        subprocess.run(["gcc", *CFLAGS, "-o", str(tmp), str(SRC), "-lm"], check=True)
        os.replace(tmp, LIB)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        L = C.CDLL(str(LIB))
        vp, i64, i32, f64 = C.c_void_p, C.c_int64, C.c_int, C.c_double
        L.fc_mesh_create.argtypes = [i64, vp, vp, i32]
        L.fc_mesh_create.restype = vp
        L.fc_nthreads.argtypes = [vp]
        L.fc_add_category.argtypes = [vp, i32, i32, i32, i64, vp, vp, vp, vp]
        L.fc_mesh_destroy.argtypes = [vp]
        L.fc_momentum.argtypes = [vp, vp, f64, f64, f64, vp]
        L.fc_divergence.argtypes = [vp, vp, f64, vp]
        L.fc_gradient.argtypes = [vp, vp, vp]
        L.fc_wall.argtypes = [vp, i64, vp, vp, vp, f64, f64, vp]
        L.fc_pcg.argtypes = [i64, vp, vp, vp, vp, vp, i32, f64, vp, vp]
        L.fc_step.argtypes = [vp, f64, f64, f64, f64, i32, f64, vp, vp, vp, vp, vp, vp, vp, i64, vp, vp, vp, vp, vp,
                              vp, vp]
        L.fc_step.restype = i32
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data if a is not None else None


class CMesh:
    """fc_mesh of a meshgen.MeshArrays (keeps the arrays it points to alive)."""

    def __init__(self, mesh, threads: int = 0):
        L = lib()
        self.n = mesh.n_nodes
        self._x = np.ascontiguousarray(mesh.coords, dtype=np.float64)
        self._per = np.ascontiguousarray(np.asarray(mesh.period, dtype=np.float64).reshape(3))
        self.h = L.fc_mesh_create(self.n, _p(self._x), _p(self._per), int(threads))
        self.threads = L.fc_nthreads(self.h)
        self._keep = []
        for _tag, rule, conn, _ids in mesh.categories():
            N, dN = fem.shape_tables(rule)             # N[a,g], dN[a,g,3]
            _, w = fem.rule_points_weights(rule)
            Ng = np.ascontiguousarray(N.T)             # [g][a]
            dNg = np.ascontiguousarray(np.transpose(dN, (1, 0, 2)))  # [g][a][3]
            w = np.ascontiguousarray(w, dtype=np.float64)
            cn = np.ascontiguousarray(conn, dtype=np.int32)
            self._keep += [Ng, dNg, w, cn]
            rc = L.fc_add_category(self.h, N.shape[0], N.shape[1], int(fem.RULE_KIND[rule] == "tet"), cn.shape[0],
                                   _p(cn), _p(Ng), _p(dNg), _p(w))
            assert rc == 0

    def momentum(self, u, rho=1.0, mu=1.0, c_vreman=0.0):
        u = np.ascontiguousarray(u, dtype=np.float64)
        out = np.empty((self.n, 3))
        lib().fc_momentum(self.h, _p(u), rho, mu, c_vreman, _p(out))
        return out

    def divergence(self, u, scale=1.0):
        u = np.ascontiguousarray(u, dtype=np.float64)
        out = np.empty(self.n)
        lib().fc_divergence(self.h, _p(u), scale, _p(out))
        return out

    def gradient(self, p):
        p = np.ascontiguousarray(p, dtype=np.float64)
        out = np.empty((self.n, 3))
        lib().fc_gradient(self.h, _p(p), _p(out))
        return out

    def __del__(self):
        try:
            lib().fc_mesh_destroy(self.h)
        except Exception:
            pass


class CFlowOracle(fem.FlowOracle):
    """fem.FlowOracle with the time step in C + OpenMP (``threads`` 0 = all cores)."""

    def __init__(self, mesh, rho=1.0, mu=1.0, c_vreman=0.0, p_fixed=None, u_fixed=None, u_fixed_values=None,
                 wall=None, threads: int = 0):
        super().__init__(mesh, rho, mu, c_vreman, p_fixed, u_fixed, u_fixed_values, wall)
        self.cm = CMesh(mesh, threads)
        n = mesh.n_nodes
        L = self.L.tocsr()
        self._rp = np.ascontiguousarray(L.indptr, dtype=np.int64)
        self._ci = np.ascontiguousarray(L.indices, dtype=np.int32)
        self._av = np.ascontiguousarray(L.data, dtype=np.float64)
        self._dinv = np.ascontiguousarray(self.dinv, dtype=np.float64)
        self._minv = np.ascontiguousarray(self.minv, dtype=np.float64)
        self._pfix = np.ascontiguousarray(self.p_fixed, dtype=np.uint8)
        self._ufix = np.ascontiguousarray(self.u_fixed, dtype=np.uint8).reshape(n, 3)
        self._ufv = np.ascontiguousarray(self.u_fixed_values, dtype=np.float64).reshape(n, 3)
        if wall is not None and len(wall[0]):
            self._face = np.ascontiguousarray(wall[0], dtype=np.int32)
            self._off = np.ascontiguousarray(wall[1], dtype=np.int32)
        else:
            self._face = self._off = None
        self._work = np.empty(11 * n)

    @property
    def threads(self) -> int:
        return self.cm.threads

    def step(self, st, dt, cg_iters=50, cg_tol=0.0):
        u = np.array(st["u"], dtype=np.float64, order="C")
        p = np.array(st["p"], dtype=np.float64, order="C")
        gp = np.array(st["gp"], dtype=np.float64, order="C")
        nf = 0 if self._face is None else self._face.shape[0]
        it = lib().fc_step(self.cm.h, self.rho, self.mu, self.c_vreman, dt, int(cg_iters), float(cg_tol), _p(u),
                           _p(p), _p(gp), _p(self._minv), _p(self._ufix), _p(self._ufv), _p(self._pfix), nf,
                           _p(self._face), _p(self._off), _p(self._rp), _p(self._ci), _p(self._av), _p(self._dinv),
                           _p(self._work))
        return {"u": u, "p": p, "gp": gp, "cg_iters": it}

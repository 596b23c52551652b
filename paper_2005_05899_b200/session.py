"""The C-ABI session from Python (include/alyab200.h "Session"): one call
per time step, every setup structure built by the native library.  This is
what a C/C++/FFI caller of libalyab200.so sees; the
Python FlowSolver is the same step with the setup done in torch.

    s = Session(mesh_arrays, params, p_fixed=..., u_fixed=..., u_fixed_values=..., wall=(faces, off))
    s.set_state(u, p); s.step(dt, cg_iters); u, p = s.get_state()
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import RULE_ID, AbCategory, AbCtxInfo, AbMeshDesc, AbPhys, call, lib


class Session:
    def __init__(self, mesh, params=None, p_fixed=None, u_fixed=None, u_fixed_values=None, wall=None,
                 device: int = 0):
        from .timestep import FlowParams
        ph = params or FlowParams()
        self.n = mesh.n_nodes
        keep = []  # host arrays referenced by the descriptor until the upload returns

        def host(a, dtype):
            a = np.ascontiguousarray(a, dtype=dtype)
            keep.append(a)
            return a.ctypes.data

        d = AbMeshDesc(n_nodes=self.n, coords=host(mesh.coords, np.float64))
        for k in range(3):
            d.period[k] = float(np.asarray(mesh.period)[k])
        cats = list(mesh.categories())
        d.n_cat = len(cats)
        for k, (_tag, rule, conn, _ids) in enumerate(cats):
            d.cat[k] = AbCategory(rule=RULE_ID[rule], pad_=0, n_elem=conn.shape[0], conn=host(conn, np.int32))
        if p_fixed is not None:
            d.p_fixed = host(np.asarray(p_fixed, bool).astype(np.uint8), np.uint8)
        if u_fixed is not None:
            uf = np.asarray(u_fixed, bool).reshape(self.n, 3)
            d.u_fixed = host(uf[:, 0] * 1 + uf[:, 1] * 2 + uf[:, 2] * 4, np.uint8)
            if u_fixed_values is not None:
                d.u_values = host(np.asarray(u_fixed_values, float).reshape(self.n, 3), np.float64)
        if wall is not None and len(wall[0]):
            d.n_wall_faces = len(wall[0])
            d.wall_face = host(wall[0], np.int32)
            d.wall_off = host(wall[1], np.int32)
        d.phys = AbPhys(rho=ph.rho, mu=ph.mu, c_vreman=ph.c_vreman)
        ctx = C.c_void_p()
        call("ab_ctx_create", device, C.byref(ctx))
        self.ctx = ctx
        try:
            call("ab_mesh_upload", self.ctx, C.byref(d))
        except Exception:
            self.close()
            raise
        del keep

    def info(self) -> dict:
        i = AbCtxInfo()
        call("ab_ctx_info", self.ctx, C.byref(i))
        return {"n_nodes": i.n_nodes, "nnz": i.nnz, "n_cat": i.n_cat, "ready": bool(i.ready),
                "n_elem": list(i.n_elem)[: i.n_cat], "n_velocity_bc": i.n_velocity_bc,
                "n_wall_faces": i.n_wall_faces}

    def set_state(self, u, p, stream=None):
        u = np.ascontiguousarray(u, dtype=np.float64)
        p = np.ascontiguousarray(p, dtype=np.float64)
        call("ab_state_set", self.ctx, u.ctypes.data, p.ctypes.data, stream)
        self._sync()

    def step(self, dt: float, cg_iters: int = 50, stream=None):
        call("ab_step", self.ctx, float(dt), int(cg_iters), stream)

    def get_state(self, stream=None):
        u = np.empty((self.n, 3))
        p = np.empty(self.n)
        call("ab_state_get", self.ctx, u.ctypes.data, p.ctypes.data, stream)
        self._sync()
        return u, p

    def _sync(self):
        import torch
        torch.cuda.synchronize()

    def close(self):
        if getattr(self, "ctx", None):
            lib().ab_ctx_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

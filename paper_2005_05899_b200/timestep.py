"""The fractional-step explicit-RK time step (Algorithm 1)
on the GPU — new entry points ``time_step`` / ``run`` in the reference's
functional style, backed by :class:`FlowSolver`.

Per step (the CPU restatement is oracle/fem.py:FlowOracle):

    for s in 1..3 (SSP-RK3 stage form):
        K2  R_s = R(u_{s-1})                          ab_momentum_rhs  (+ interface sum)
        K3  u_s = a_s u^n + b_s (u_{s-1} + dt/rho M_L^-1 (R_s - G p^n))   ab_rk_stage
            velocity Dirichlet values                 ab_apply_velocity_bc
    K4  b = -(rho/dt) D u_3                           ab_divergence    (+ interface sum)
    K5  L' dp = b, Jacobi-PCG                         ab_cg_*          (+ halo / all-reduce)
    K6  G dp                                          ab_gradient      (+ interface sum)
    K7  u^{n+1} = u_3 - dt/rho M_L^-1 G dp; p += dp; Gp += G dp        ab_correct

With a fixed CG iteration count the whole step is free of host
synchronisation and is captured once into a CUDA graph and replayed.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from ._lib import AbPhys, call, ptr, stream_handle
from .device import DeviceMesh, nodes_as4
from .meshgen import MeshArrays
from .solver import PCG, assemble_gradient_operator, assemble_laplacian

RK3_A = (0.0, 0.75, 1.0 / 3.0)
RK3_B = (1.0, 0.25, 2.0 / 3.0)


@dataclass
class FlowParams:
    rho: float = 1.0
    mu: float = 1.0
    c_vreman: float = 0.0

    def struct(self) -> AbPhys:
        return AbPhys(rho=self.rho, mu=self.mu, c_vreman=self.c_vreman)


class FlowSolver:
    """Owns the device state and workspaces of one (sub)domain.

    ``halo`` (optional, :class:`halo.HaloExchanger`) sums interface-node
    values across ranks and all-reduces the CG scalars; ``own`` gives the
    per-node ownership weights for the dots.
    """

    def __init__(self, mesh, params: FlowParams | None = None, p_fixed=None, u_fixed=None, u_fixed_values=None,
                 windows: bool = True, reorder: str | None = "sfc", halo=None, own=None, ops: str = "spmv",
                 fused_cg: bool | None = None, wall=None, scatter: str = "atomic"):
        self.params = params or FlowParams()
        self.phys = self.params.struct()
        self.dm = mesh if isinstance(mesh, DeviceMesh) else DeviceMesh(mesh, reorder=reorder, windows=windows,
                                                                       scatter=scatter)
        dm = self.dm
        # boundary assembly (Algorithm 1 line 4): wall model faces, (faces, off) or a WallModel
        if wall is not None and not hasattr(wall, "add_traction"):
            from .wall import WallModel
            wall = WallModel(*wall, device=dm.device)
        self.wall = wall if (wall is not None and wall.n_faces > 0) else None
        n = dm.n_nodes
        dev = dm.device
        self.n = n
        self.halo = halo
        s = stream_handle()
        # lumped mass (K1, ml only) and its inverse
        self.ml = torch.zeros(n, dtype=torch.float64, device=dev)
        for k in range(len(dm.rules)):
            call("ab_mass", ctypes.byref(dm.struct), k, None, None, ptr(self.ml), 128, s)
        if halo is not None:
            halo.sum_(self.ml, 1, 1)
        self.minv = torch.empty_like(self.ml)
        call("ab_reciprocal", n, ptr(self.ml), ptr(self.minv), s)
        # pressure Laplacian with Dirichlet rows, Jacobi diagonal
        pf = np.zeros(n, bool) if p_fixed is None else np.asarray(p_fixed, bool)
        self.p_fixed = torch.from_numpy(pf.astype(np.uint8)).to(dev)
        self.L = assemble_laplacian(dm, self.p_fixed if pf.any() else None)
        diag = self.L.diag.clone()
        if halo is not None:
            halo.sum_(diag, 1, 1)
            if pf.any():  # fixed rows are identity on every rank
                diag[self.p_fixed.bool()] = 1.0
        self.dinv = torch.empty_like(diag)
        call("ab_reciprocal", n, ptr(diag), ptr(self.dinv), s)
        self.own = own
        # K4/K6: sparse products with the assembled gradient operator
        # ("spmv", default) or the element loops ("element")
        if ops not in ("spmv", "element"):
            raise ValueError(f"ops must be 'spmv' or 'element', not {ops!r}")
        self.ops = ops
        self.Bop = assemble_gradient_operator(dm, pattern=self.L.csr[:2]) if ops == "spmv" else None
        self.pcg = PCG(self.L, self.dinv, fixed=self.p_fixed if pf.any() else None, own=own, halo=halo,
                       order=dm.node_order() if halo is None else None)
        # velocity Dirichlet nodes (sparse list)
        if u_fixed is not None and np.any(u_fixed):
            uf = np.asarray(u_fixed, bool).reshape(n, 3)
            idx = np.nonzero(uf.any(axis=1))[0]
            mask = (uf[idx, 0] * 1 + uf[idx, 1] * 2 + uf[idx, 2] * 4).astype(np.uint8)
            vals = np.zeros((n, 3)) if u_fixed_values is None else np.asarray(u_fixed_values, float).reshape(n, 3)
            self.bc_idx = torch.from_numpy(idx.astype(np.int32)).to(dev)
            self.bc_mask = torch.from_numpy(mask).to(dev)
            self.bc_vals = torch.from_numpy(np.ascontiguousarray(vals[idx])).to(dev)
        else:
            self.bc_idx = None
        z4 = lambda: torch.zeros((n, 4), dtype=torch.float64, device=dev)  # noqa: E731
        self.U0, self.U, self.R, self.GP, self.GD = z4(), z4(), z4(), z4(), z4()
        self.P = torch.zeros(n, dtype=torch.float64, device=dev)
        self.B = torch.zeros(n, dtype=torch.float64, device=dev)
        # decomposed domains on NCCL (one GPU per rank): the pressure solve runs
        # as one kernel per rank fused with its interface exchange over peer
        # memory (ddcg.FusedDDSolver), validated once against the NCCL-driven
        # two-kernel solve; fused_cg=False keeps the latter
        self.ddcg = None
        self.ddcg_kind = None
        self._force_dd2 = fused_cg == "two-kernel"  # tests: skip the on-chip form
        # (fused_cg=True also forces it on other backends, e.g. gloo ranks sharing one GPU in tests)
        if halo is not None and (fused_cg in (True, "two-kernel")
                                 or (fused_cg is None and (self._nccl(halo) or getattr(halo, "graph_safe", False)))):
            self.ddcg = self._fused_solver(dm, pf, fused_cg)
        self.graph = None
        self._side = None  # step_host: G p^n while u uploads
        self.graph_key = None
        self.last_cg_iters = 0
        self.timeline = None  # list of (name, start, end) CUDA events when profiling

    @staticmethod
    def _nccl(halo) -> bool:
        import torch.distributed as dist
        return dist.is_initialized() and dist.get_backend(halo.group) == "nccl"

    def _fused_solver(self, dm, pf, required):
        """The pressure solve fused with its interface exchange over peer
        memory: the on-chip solver (ddcg.FusedDDSolver, one cooperative
        kernel per solve) when the rank's rows fit on chip, else the
        two-kernel form (peer.FusedDD2Solver).  Each is validated once
        against the NCCL-driven solve (8 iterations, max-norm 1e-10).
        Every branch is collective: all ranks take the same one."""
        import torch.distributed as dist
        from .ddcg import FusedDDSolver
        from .peer import FusedDD2Solver
        plan = self.halo.plan
        fixed = self.p_fixed if pf.any() else None

        def consensus(ok: bool) -> bool:  # every rank takes the same branch
            t = torch.tensor([1 if ok else 0], dtype=torch.int32, device=self.B.device)
            dist.all_reduce(t, op=dist.ReduceOp.MIN, group=self.halo.group)
            return bool(int(t.item()))

        errs = []
        for kind, cls in (("resident", FusedDDSolver), ("two-kernel", FusedDD2Solver)):
            if kind == "resident" and getattr(self, "_force_dd2", False):
                continue
            try:
                dd = cls(dm, self.L, self.dinv, fixed, plan, self.B, group=self.halo.group)
            except Exception as e:  # the constructors' own checks are collective
                errs.append(f"{kind}: {e}")
                continue
            # validation solve: same iterate as the NCCL-driven kernels
            g = torch.Generator(device="cpu").manual_seed(1234)
            bh = torch.randn(len(plan.l2g), generator=g, dtype=torch.float64).to(self.B.device)
            self.B.copy_(bh)
            self.halo.sum_(self.B, 1, 1)
            b0 = self.B.clone()
            ok = True
            try:
                x_dd, it = dd.solve(self.B, 8)
                x_dd = x_dd.clone()
                dd.check()
            except Exception as e:
                ok = False
                errs.append(f"{kind}: {e}")
            if consensus(ok):
                self.B.copy_(b0)
                x_ref, _ = self.pcg.solve(self.B, 8)
                d = torch.tensor([float((x_dd - x_ref).abs().max() / x_ref.abs().max().clamp_min(1e-300))],
                                 dtype=torch.float64, device=self.B.device)
                dist.all_reduce(d, op=dist.ReduceOp.MAX, group=self.halo.group)
                self.B.zero_()
                if float(d.item()) <= 1e-10:
                    self.ddcg_kind = kind
                    return dd
                errs.append(f"{kind}: disagrees with the NCCL-driven solve ({float(d.item()):.2e})")
            self.B.zero_()
        if required:
            raise RuntimeError(f"fused decomposed CG unavailable: {'; '.join(errs)}")
        import warnings
        warnings.warn(f"fused decomposed CG unavailable, using the NCCL-driven solve: {'; '.join(errs)}")
        return None

    def _grad(self, p, out4, scale: float = 1.0):
        if self.Bop is not None:
            self.Bop.grad(p, scale, out4)
        else:
            call("ab_gradient", ctypes.byref(self.dm.struct), ptr(p), scale, ptr(out4), stream_handle())

    # -- state ----------------------------------------------------------------
    def set_state(self, u, p):
        u = torch.as_tensor(u, dtype=torch.float64, device=self.dm.device)
        self.U0.copy_(nodes_as4(u))
        self.P.copy_(torch.as_tensor(p, dtype=torch.float64, device=self.dm.device))
        self._bc(self.U0)
        self.GP.zero_()
        self._grad(self.P, self.GP)
        if self.halo is not None:
            self.halo.sum_(self.GP, 3, 4)

    @property
    def u(self) -> torch.Tensor:
        return self.U0[:, :3]

    @property
    def p(self) -> torch.Tensor:
        return self.P

    def _bc(self, u4):
        if self.bc_idx is not None:
            call("ab_apply_velocity_bc", self.bc_idx.numel(), ptr(self.bc_idx), ptr(self.bc_mask), ptr(self.bc_vals),
                 ptr(u4), stream_handle())

    # -- operators ------------------------------------------------------------
    def momentum(self, u4, out4):
        call("ab_momentum_rhs", ctypes.byref(self.dm.struct), ctypes.byref(self.phys), ptr(u4), ptr(out4),
             stream_handle())
        if self.halo is not None:
            self.halo.sum_(out4, 3, 4)

    # -- one time step ----------------------------------------------------------
    def _mark(self, name):
        """Context manager recording CUDA events around a launch when
        ``self.timeline`` is a list (bench.py's per-kernel breakdown)."""
        solver = self

        class _M:
            def __enter__(self_inner):
                if solver.timeline is not None:
                    self_inner.a = torch.cuda.Event(enable_timing=True)
                    self_inner.a.record()

            def __exit__(self_inner, *exc):
                if solver.timeline is not None:
                    b = torch.cuda.Event(enable_timing=True)
                    b.record()
                    solver.timeline.append((name, self_inner.a, b))
        return _M()

    def _step_body(self, dt: float, cg_iters: int, cg_tol: float, before_k3=None, after_cg=None):
        """One fractional step on the current stream.  Hooks (end-to-end
        overlap, step_host): ``before_k3()`` runs after the first stage's
        right-hand side (K2, K8) and before its K3 (the first use of G p^n);
        ``after_cg(x)`` runs after the pressure solve, before K6 + K7."""
        s = stream_handle()
        dm = self.dm
        rho = self.params.rho
        k = dt / rho
        for st in range(3):
            uin = self.U0 if st == 0 else self.U
            with self._mark("K2_momentum"):
                call("ab_momentum_rhs", ctypes.byref(dm.struct), ctypes.byref(self.phys), ptr(uin), ptr(self.R), s)
            if self.wall is not None:
                with self._mark("K8_wall"):
                    self.wall.add_traction(self.phys, dm.coords4, uin, self.R)
            if self.halo is not None:
                with self._mark("X_halo_sum"):
                    self.halo.sum_(self.R, 3, 4)
            if st == 0 and before_k3 is not None:
                before_k3()
            with self._mark("K3_rk_stage"):
                call("ab_rk_stage", self.n, RK3_A[st], RK3_B[st], k, ptr(self.U0), ptr(uin), ptr(self.R),
                     ptr(self.GP), ptr(self.minv), ptr(self.U), s)
            self._bc(self.U)
        with self._mark("K4_divergence"):
            if self.Bop is not None:
                self.Bop.div(self.U, -rho / dt, self.B)
            else:
                call("ab_divergence", ctypes.byref(dm.struct), ptr(self.U), -rho / dt, ptr(self.B), s)
        if self.halo is not None:
            with self._mark("X_halo_sum"):
                self.halo.sum_(self.B, 1, 1)
        self.pcg.mark = self._mark
        if self.ddcg is not None:
            with self._mark("K5_cg_fused_dd"):
                x, it = self.ddcg.solve(self.B, cg_iters, tol=cg_tol)
        else:
            x, it = self.pcg.solve(self.B, cg_iters, tol=cg_tol)
        self.last_cg_iters = it
        if after_cg is not None:
            after_cg(x)
        if self.Bop is not None and self.halo is None:
            # K6 + K7 fused: u = u_3 - dt/rho M^-1 B dp; p += dp; Gp += B dp
            with self._mark("K67_grad_correct"):
                call("ab_gradop_correct", ctypes.byref(self.Bop.struct), ptr(x), k, ptr(self.U), ptr(self.U0),
                     ptr(self.minv), ptr(self.P), ptr(self.GP), s)
        else:
            with self._mark("K6_gradient"):
                self._grad(x, self.GD)
            if self.halo is not None:
                with self._mark("X_halo_sum"):
                    self.halo.sum_(self.GD, 3, 4)
            with self._mark("K7_correct"):
                call("ab_correct", self.n, k, ptr(self.U), ptr(self.U0), ptr(self.GD), ptr(self.minv), ptr(self.P),
                     ptr(x), ptr(self.GP), s)
        self._bc(self.U0)

    def step_host(self, u_host: torch.Tensor, p_host: torch.Tensor, dt: float, cg_iters: int = 50,
                  graph: bool = True, overlap: bool = True):
        """End-to-end call with HOST buffers (pinned for async copies): upload
        (u, p), advance one step, download (u, p) in place.  Returns after the
        downloads have completed (u_host, p_host are valid).

        Single domain (``overlap``): u goes up first and the step starts as
        soon as it is there; p's upload and G p^n run on a side stream under
        the first momentum assembly, and p^{n+1} = p^n + dp is formed and
        downloaded on the side stream while K6 + K7 run (the step is then
        launched eagerly: the hooks sit inside it).  Otherwise: p first, G p^n
        on a side stream while u uploads, then the (graph) step."""
        main = torch.cuda.current_stream()
        if self._side is None:
            self._side = torch.cuda.Stream()
        if overlap and self.halo is None:
            self._step_host_overlap(u_host, p_host, dt, cg_iters, main)
            return
        self.P.copy_(p_host, non_blocking=True)
        self._side.wait_stream(main)
        with torch.cuda.stream(self._side):
            self.GP.zero_()
            self._grad(self.P, self.GP)
            if self.halo is not None:
                self.halo.sum_(self.GP, 3, 4)
        self.U0[:, :3].copy_(u_host, non_blocking=True)
        main.wait_stream(self._side)
        self.step(dt, cg_iters, graph=graph)
        u_host.copy_(self.U0[:, :3], non_blocking=True)
        p_host.copy_(self.P, non_blocking=True)
        # the host buffers are read by the caller on return
        main.synchronize()
        self.check_health()

    def _step_host_overlap(self, u_host, p_host, dt, cg_iters, main):
        side = self._side
        self.U0[:, :3].copy_(u_host, non_blocking=True)  # the first kernel's input: up first
        side.wait_stream(main)  # (previous step's work on the device buffers is ordered before)
        ev_gp = torch.cuda.Event()
        with torch.cuda.stream(side):
            self.P.copy_(p_host, non_blocking=True)
            self.GP.zero_()
            self._grad(self.P, self.GP)
            ev_gp.record(side)
        if getattr(self, "_P_next", None) is None or self._P_next.shape != self.P.shape:
            self._P_next = torch.empty_like(self.P)

        def before_k3():
            main.wait_event(ev_gp)

        def after_cg(x):
            ev_x = torch.cuda.Event()
            ev_x.record(main)
            ev_read = torch.cuda.Event()
            with torch.cuda.stream(side):
                side.wait_event(ev_x)
                torch.add(self.P, x, out=self._P_next)  # = K7's p + dp, bitwise
                ev_read.record(side)
                p_host.copy_(self._P_next, non_blocking=True)
            main.wait_event(ev_read)  # K6 + K7 update P in place after the side stream read it

        self._step_body(dt, cg_iters, 0.0, before_k3=before_k3, after_cg=after_cg)
        self.last_cg_iters = cg_iters
        u_host.copy_(self.U0[:, :3], non_blocking=True)
        main.wait_stream(side)
        main.synchronize()
        self.check_health()

    def check_health(self):
        """Raise if a fused decomposed pressure solve failed since the last
        check (device-side sticky flag; a host read, so call it outside
        timed loops or where the step synchronises anyway)."""
        if self.ddcg is not None:
            self.ddcg.check()

    @property
    def graph_safe(self) -> bool:
        """A fixed-iteration step can be captured: single domain, or a
        decomposed one whose exchanges are peer-memory kernels (no NCCL call,
        no host sync) and whose pressure solve is fused (no NCCL scalars)."""
        return self.halo is None or (getattr(self.halo, "graph_safe", False) and self.ddcg is not None)

    def step(self, dt: float, cg_iters: int = 50, cg_tol: float = 0.0, graph: bool = False):
        """Advance one step.  ``graph=True`` (fixed iterations) captures the
        step once and replays the CUDA graph afterwards when graph_safe."""
        if graph and cg_tol == 0.0 and self.graph_safe:
            key = (dt, cg_iters)
            if self.graph is None or self.graph_key != key:
                self.capture(dt, cg_iters)
            self.graph.replay()
            self.last_cg_iters = cg_iters
            return
        self._step_body(dt, cg_iters, cg_tol)

    def capture(self, dt: float, cg_iters: int):
        import gc
        # destroy unreachable graphs now: a CUDAGraph freed by the garbage
        # collector in the middle of another capture invalidates that capture
        self.graph = None
        gc.collect()
        torch.cuda.synchronize()
        # snapshot the state: capture runs the body once on a side stream
        saved = [t.clone() for t in (self.U0, self.P, self.GP)]
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            self._step_body(dt, cg_iters, 0.0)  # warm-up outside capture
        torch.cuda.current_stream().wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self._step_body(dt, cg_iters, 0.0)
        for t, v in zip((self.U0, self.P, self.GP), saved):
            t.copy_(v)
        self.graph = g
        self.graph_key = (dt, cg_iters)

    def launches_per_step(self, cg_iters: int) -> int:
        """Kernels of this library launched by one step (no halo)."""
        ncat = len(self.dm.rules) + (1 if self.wall is not None else 0)
        bc = 1 if self.bc_idx is not None else 0
        cg = 1 if self.pcg.resident else 2 + 2 * cg_iters
        if self.Bop is not None:
            return 3 * (ncat + 1 + bc) + 1 + cg + 1 + bc
        return 3 * (ncat + 1 + bc) + ncat + cg + ncat + 1 + bc


def time_step(solver: FlowSolver, dt: float, cg_iters: int = 50, cg_tol: float = 0.0):
    """One fractional step; returns (u, p) views of the device state."""
    solver.step(dt, cg_iters, cg_tol)
    return solver.u, solver.p


def run(mesh, u0, p0, n_steps: int, dt: float, params: FlowParams | None = None, cg_iters: int = 50,
        cg_tol: float = 0.0, **kw):
    """Build a solver for ``mesh``, set (u0, p0) and advance ``n_steps``."""
    solver = mesh if isinstance(mesh, FlowSolver) else FlowSolver(mesh, params, **kw)
    solver.set_state(u0, p0)
    for _ in range(n_steps):
        solver.step(dt, cg_iters, cg_tol)
    return solver

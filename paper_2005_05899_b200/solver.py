"""Pressure Laplacian and Jacobi-PCG — new entry points in the reference's
style: ``assemble_laplacian(mesh) -> SellMatrix`` and
``pcg_solve(A, b, x0, tol, max_it) -> (x, iters, res)``.

The Laplacian L_ab = sum_e int grad N_a . grad N_b is assembled once
(Algorithm 1 line 1): the CSR pattern comes from a GPU sort of
the element (row, col) pairs, values from ``ab_laplacian_csr``, Dirichlet rows
and columns become identity (``ab_csr_dirichlet``), and the matrix is stored
as SELL-32 for the solver (``ab_csr_to_sell``).  The CG (PAPER.md:219,
:329-330) keeps all scalars on the device: one cooperative kernel per solve
when the system fits on chip (``ab_cg_resident_local``), else the tiled
single pass on the symmetrically scaled, SFC-ordered system (one
``ab_cg_tile_iter`` per iteration), with the two-kernel forms as options; in
a decomposed domain driven over NCCL the SpMV result is interface-summed and
the dots all-reduced between the kernels (DESIGN.md §4/§5).
"""

from __future__ import annotations

import ctypes
import ctypes as C
import math
import os
from dataclasses import dataclass

import torch

from ._lib import AbCgLocal, AbSell, AbSell3, call, lib, ptr, stream_handle
from .device import DeviceMesh


@dataclass
class SellMatrix:
    n_rows: int
    slice_ptr: torch.Tensor   # int64 [n_slices+1]
    cols: torch.Tensor        # int32
    vals: torch.Tensor        # f64
    diag: torch.Tensor        # f64 [n_rows]
    csr: tuple | None = None  # (row_ptr int64, cols int32, vals f64), kept for tests/export

    staged: bool = True       # TMA-staged SpMV (ab_cg_spmv) when every slice fits

    def __post_init__(self):
        w = (self.slice_ptr[1:] - self.slice_ptr[:-1]) // 32
        self.max_width = int(w.max().item()) if w.numel() else 0
        self.struct = AbSell(n_rows=self.n_rows, n_slices=self.slice_ptr.numel() - 1,
                             max_width=self.max_width if self.staged else 0,
                             slice_ptr=ptr(self.slice_ptr), cols=ptr(self.cols), vals=ptr(self.vals))

    @property
    def nnz_stored(self) -> int:
        return int(self.vals.numel())

    @property
    def nnz(self) -> int:
        return int(self.csr[1].numel()) if self.csr is not None else -1

    def matvec(self, x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        y = torch.empty_like(x) if out is None else out
        call("ab_sell_spmv", ctypes.byref(self.struct), ptr(x), ptr(y), stream_handle())
        return y


def csr_pattern(dm: DeviceMesh, chunk: int = 1 << 23):
    """Unique (row, col) pairs of all element node pairs, row-major sorted.
    Elements are processed in chunks (per-chunk unique first), so the peak
    memory stays ~ chunk * nnode^2 keys even for 250M-element meshes."""
    N = dm.n_nodes
    keys = []
    for conn in dm.conn:
        nn = conn.shape[1]
        for e0 in range(0, conn.shape[0], chunk):
            c = conn[e0:e0 + chunk].to(torch.int64)
            k = (c[:, :, None] * N + c[:, None, :]).reshape(-1)
            keys.append(torch.unique(k))
            del c, k
        if len(keys) > 8:  # keep the list short: merge partial results
            keys = [torch.unique(torch.cat(keys))]
    key = torch.unique(torch.cat(keys))
    del keys
    rows = key // N
    cols = (key % N).to(torch.int32)
    counts = torch.bincount(rows, minlength=N)
    row_ptr = torch.zeros(N + 1, dtype=torch.int64, device=key.device)
    row_ptr[1:] = torch.cumsum(counts, 0)
    return row_ptr, cols.contiguous()


def csr_to_sell(n: int, row_ptr, cols, vals) -> SellMatrix:
    dev = vals.device
    nnz_row = row_ptr[1:] - row_ptr[:-1]
    n_slices = (n + 31) // 32
    padded = torch.zeros(n_slices * 32, dtype=torch.int64, device=dev)
    padded[:n] = nnz_row
    width = padded.view(n_slices, 32).max(dim=1).values
    slice_ptr = torch.zeros(n_slices + 1, dtype=torch.int64, device=dev)
    slice_ptr[1:] = torch.cumsum(width * 32, 0)
    total = int(slice_ptr[-1].item())
    # zero-filled: lanes of the last slice past n_rows stay (col 0, val 0)
    scols = torch.zeros(total, dtype=torch.int32, device=dev)
    svals = torch.zeros(total, dtype=torch.float64, device=dev)
    diag = torch.empty(n, dtype=torch.float64, device=dev)
    call("ab_csr_to_sell", n, ptr(row_ptr), ptr(cols), ptr(vals), ptr(slice_ptr), ptr(scols), ptr(svals),
         ptr(diag), stream_handle())
    return SellMatrix(n_rows=n, slice_ptr=slice_ptr, cols=scols, vals=svals, diag=diag,
                      csr=(row_ptr, cols, vals))


def permute_matrix(A: SellMatrix, perm: torch.Tensor, drop_diag: bool = False) -> SellMatrix:
    """P A P^T as SELL-32: row i of the result is row perm[i] of A (columns
    renumbered the same way, ascending within each row).  ``drop_diag``
    leaves the diagonal entries out (the unit-diagonal scaled solver)."""
    row_ptr, cols, vals = A.csr
    n = A.n_rows
    dev = vals.device
    perm = perm.to(device=dev, dtype=torch.int64)
    iperm = torch.empty_like(perm)
    iperm[perm] = torch.arange(n, device=dev)
    rows = torch.repeat_interleave(torch.arange(n, device=dev), row_ptr[1:] - row_ptr[:-1])
    if drop_diag:
        off = rows != cols.to(torch.int64)
        rows, cols, vals = rows[off], cols[off], vals[off]
    key = iperm[rows] * n + iperm[cols.to(torch.int64)]
    key, order = torch.sort(key)
    new_rows = key // n
    new_cols = (key % n).to(torch.int32).contiguous()
    new_vals = vals[order].contiguous()
    rp = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    rp[1:] = torch.cumsum(torch.bincount(new_rows, minlength=n), 0)
    return csr_to_sell(n, rp, new_cols, new_vals)


def cg_local_map(A: SellMatrix, rows_per_cta: int, n_cta: int):
    """CTA-local column map for ``ab_cg_resident_local`` (include/alyab200.h):
    per CTA the ascending list of remote columns (ghost rows) and, per SELL
    entry, the 16-bit local column (own row: c - row0; ghost g: rows_per_cta
    + g).  Returns None when a CTA's rows + ghosts exceed 16 bits."""
    n = A.n_rows
    dev = A.cols.device
    sp = A.slice_ptr
    counts = sp[1:] - sp[:-1]
    n_sl = counts.numel()
    slice_of = torch.repeat_interleave(torch.arange(n_sl, device=dev), counts)
    cta = slice_of // (rows_per_cta // 32)
    del slice_of
    r0 = cta * rows_per_cta
    c = A.cols.to(torch.int64)
    local = (c >= r0) & (c < r0 + rows_per_cta)
    remote = ~local
    key = cta[remote] * n + c[remote]
    uk, inv = torch.unique(key, return_inverse=True)
    g_cta = uk // n
    ghost = (uk % n).to(torch.int32).contiguous()
    gcount = torch.bincount(g_cta, minlength=n_cta)
    ghost_ptr = torch.zeros(n_cta + 1, dtype=torch.int64, device=dev)
    ghost_ptr[1:] = torch.cumsum(gcount, 0)
    lc = c - r0
    lc[remote] = rows_per_cta + inv - ghost_ptr[cta[remote]]
    max_ghost = int(gcount.max().item()) if gcount.numel() else 0
    if rows_per_cta + max_ghost > 65536:
        return None
    lcols = torch.where(lc >= 32768, lc - 65536, lc).to(torch.int16).contiguous()
    # CTAs owning each CTA's ghost rows (informational)
    owner = (uk % n) // rows_per_cta
    pair = torch.unique(g_cta * n_cta + owner)
    nbr = (pair % n_cta).to(torch.int32).contiguous()
    nbr_ptr = torch.zeros(n_cta + 1, dtype=torch.int64, device=dev)
    nbr_ptr[1:] = torch.cumsum(torch.bincount(pair // n_cta, minlength=n_cta), 0)
    nbr_ptr = nbr_ptr.to(torch.int32).contiguous()
    ghost_ptr = ghost_ptr.to(torch.int32).contiguous()
    if ghost.numel() == 0:  # no remote columns at all: keep a valid (unused) array
        ghost = torch.zeros(1, dtype=torch.int32, device=dev)
    if nbr.numel() == 0:
        nbr = torch.zeros(1, dtype=torch.int32, device=dev)
    struct = AbCgLocal(rows_per_cta=rows_per_cta, n_cta=n_cta, max_ghost=max_ghost, cols=ptr(lcols),
                       ghost_ptr=ptr(ghost_ptr), ghost=ptr(ghost), nbr_ptr=ptr(nbr_ptr), nbr=ptr(nbr))
    return dict(cols=lcols, ghost_ptr=ghost_ptr, ghost=ghost, max_ghost=max_ghost, struct=struct, nbr=nbr,
                nbr_ptr=nbr_ptr)


def assemble_laplacian(mesh, fixed: torch.Tensor | None = None) -> SellMatrix:
    """Assemble L (SPD after Dirichlet rows/cols of ``fixed`` -> identity)."""
    dm = mesh if isinstance(mesh, DeviceMesh) else DeviceMesh(mesh)
    row_ptr, cols = csr_pattern(dm)
    vals = torch.zeros(cols.numel(), dtype=torch.float64, device=dm.device)
    call("ab_laplacian_csr", ctypes.byref(dm.struct), ptr(row_ptr), ptr(cols), ptr(vals), stream_handle())
    if fixed is not None:
        f8 = fixed.to(device=dm.device, dtype=torch.uint8).contiguous()
        call("ab_csr_dirichlet", dm.n_nodes, ptr(row_ptr), ptr(cols), ptr(vals), ptr(f8), stream_handle())
    return csr_to_sell(dm.n_nodes, row_ptr, cols, vals)


@dataclass
class GradOp:
    """Discrete gradient operator B_ab = int N_a grad N_b (3 planes, SELL-32):
    K4 is scale B . u, K6 is B p."""
    n_rows: int
    slice_ptr: torch.Tensor
    cols: torch.Tensor
    vx: torch.Tensor
    vy: torch.Tensor
    vz: torch.Tensor

    def __post_init__(self):
        self.struct = AbSell3(n_rows=self.n_rows, n_slices=self.slice_ptr.numel() - 1, slice_ptr=ptr(self.slice_ptr),
                              cols=ptr(self.cols), vx=ptr(self.vx), vy=ptr(self.vy), vz=ptr(self.vz))

    @property
    def nnz_stored(self) -> int:
        return int(self.cols.numel())

    def div(self, u4: torch.Tensor, scale: float, out: torch.Tensor) -> torch.Tensor:
        call("ab_gradop_div", ctypes.byref(self.struct), ptr(u4), float(scale), ptr(out), stream_handle())
        return out

    def grad(self, p: torch.Tensor, scale: float, out4: torch.Tensor) -> torch.Tensor:
        call("ab_gradop_grad", ctypes.byref(self.struct), ptr(p), float(scale), ptr(out4), stream_handle())
        return out4


def assemble_gradient_operator(mesh, pattern=None) -> GradOp:
    """B_ab = sum_e int N_a grad N_b on the node-adjacency pattern (the
    Laplacian's; pass ``pattern=(row_ptr, cols)`` to reuse it)."""
    dm = mesh if isinstance(mesh, DeviceMesh) else DeviceMesh(mesh)
    row_ptr, cols = pattern if pattern is not None else csr_pattern(dm)
    nnz = cols.numel()
    v = [torch.zeros(nnz, dtype=torch.float64, device=dm.device) for _ in range(3)]
    call("ab_gradop_csr", ctypes.byref(dm.struct), ptr(row_ptr), ptr(cols), ptr(v[0]), ptr(v[1]), ptr(v[2]),
         stream_handle())
    planes = [csr_to_sell(dm.n_nodes, row_ptr, cols, vk) for vk in v]
    return GradOp(n_rows=dm.n_nodes, slice_ptr=planes[0].slice_ptr, cols=planes[0].cols, vx=planes[0].vals,
                  vy=planes[1].vals, vz=planes[2].vals)


class PCG:
    """Jacobi-PCG workspace bound to one matrix (no per-solve allocation).

    ``halo`` (optional) is an interface exchanger with ``sum_(tensor, ncomp,
    stride)`` and ``allreduce_(tensor)``; ``own`` holds per-row ownership
    weights so duplicated interface rows count once in the dots.
    """

    def __init__(self, A: SellMatrix, dinv: torch.Tensor, fixed: torch.Tensor | None = None,
                 own: torch.Tensor | None = None, halo=None, resident: bool = True,
                 order: torch.Tensor | None = None, prefetch_depth: int = 1, force_mode: int = 0,
                 reorder_two_kernel: bool = True, scaled: bool = True,
                 unit_diag: bool | None = None, tile_rows: int = 2048, single_pass: bool = True):
        self.A = A
        n = A.n_rows
        dev = A.vals.device
        self.n = n
        self.dinv = dinv
        self.fixed = None if fixed is None else fixed.to(device=dev, dtype=torch.uint8).contiguous()
        self.own = own
        self.halo = halo
        z = lambda: torch.zeros(n, dtype=torch.float64, device=dev)  # noqa: E731
        self.x, self.r, self.z, self.p, self.q = z(), z(), z(), z(), z()
        self.t = z() if halo is not None else None  # local A z before the interface sum
        nb = (n + 255) // 256 + 1
        ng = (nb + 63) // 64 + 1
        n_cta = C.c_int32(0)
        rb = C.c_int64(0)
        fits = lib().ab_cg_resident_fits(n, C.byref(rb), C.byref(n_cta))
        # (+ 5 replicated [4][nb] partial tables of the resident solver, all_sum_rep)
        self.part = torch.zeros(max(5 * (nb + ng), 12 * n_cta.value + 1, 8 * n_cta.value + 20 * ((n_cta.value + 3) // 4 * 4)) + 8,
                                dtype=torch.float64, device=dev)
        self.red = torch.zeros(8, dtype=torch.float64, device=dev)
        self.sc = torch.zeros(8, dtype=torch.float64, device=dev)
        self.cnt = torch.zeros(ng + 2, dtype=torch.int32, device=dev)
        self.launches_per_iter = 2 if halo is None else 3
        self.mark = None  # optional event recorder (FlowSolver._mark)
        # single-domain solves run as ONE cooperative kernel when every CTA's
        # rows and ghost rows fit on chip (ab_cg_resident_local, z gathers
        # served from shared memory); otherwise two kernels per iteration.
        # ``order`` (node id per solver row, e.g. an SFC order of the nodes)
        # renumbers the system P A P^T so every CTA's rows are compact and its
        # ghost set small; b and x stay in node order.
        self.local = None
        if resident and halo is None and fits:
            Ap, perm = A, None
            if order is not None:
                perm = order.to(device=dev, dtype=torch.int32).contiguous()
                Ap = permute_matrix(A, perm)
            m = cg_local_map(Ap, rb.value, n_cta.value)
            if m is not None and lib().ab_cg_resident_local_fits(rb.value, m["max_ghost"]) > 0:
                m["A"] = Ap
                m["perm"] = perm
                m["struct"].perm = ptr(perm)
                m["struct"].prefetch_depth = int(prefetch_depth)
                m["struct"].force_mode = int(force_mode)
                pl = perm.to(torch.int64) if perm is not None else None
                m["dinv"] = dinv[pl].contiguous() if pl is not None else dinv
                m["fixed"] = (self.fixed[pl].contiguous() if (pl is not None and self.fixed is not None)
                              else self.fixed)
                self.local = m
        self.resident = self.local is not None
        # two-kernel single-domain solves in the ``order`` row numbering (P A P^T;
        # on C3 an SFC order cuts the SELL padding 4.7% and the iteration 7%)
        self.perm2 = None
        if not self.resident and halo is None and order is not None and reorder_two_kernel:
            pl = order.to(device=dev, dtype=torch.int64).contiguous()
            # scaled form: every diagonal entry of D^-1/2 A D^-1/2 is 1, so it is not stored
            unit = bool(scaled) if unit_diag is None else bool(unit_diag and scaled)
            self.perm2 = dict(A=permute_matrix(A, pl, drop_diag=unit), perm=pl,
                              dinv=dinv[pl].contiguous(),
                              fixed=self.fixed[pl].contiguous() if self.fixed is not None else None,
                              x=z(), scaled=bool(scaled), unit=unit)
            if scaled:
                # CG on D^-1/2 P A P^T D^-1/2 (the permuted copy's values are scaled in place)
                self.perm2["s"] = torch.sqrt(self.perm2["dinv"]).contiguous()
                self.perm2["iperm"] = torch.empty_like(pl)
                self.perm2["iperm"][pl] = torch.arange(n, device=dev)
                self.perm2["d"] = (1.0 / self.perm2["dinv"]).contiguous()
                call("ab_sell_symscale", ctypes.byref(self.perm2["A"].struct), ptr(self.perm2["s"]), stream_handle())
            # tiled SpMV (ab_cg_spmv_tile): z of a tile's rows and ghost rows in
            # shared memory, 16-bit tile-local columns
            if os.environ.get("AB_CG_TILE") is not None:  # lab switch
                tile_rows = int(os.environ["AB_CG_TILE"])
            self.perm2["tile"] = None
            if tile_rows and unit:
                if tile_rows % 64:
                    raise ValueError("tile_rows must be a multiple of 64")
                n_t = (n + tile_rows - 1) // tile_rows
                tm = cg_local_map(self.perm2["A"], tile_rows, n_t)
                if tm is not None:
                    self.perm2["tile"] = tm
            # tiled single pass (ab_cg_tile_iter): one kernel per iteration,
            # (x', p) and (r', q) as 16-byte pairs (64 instead of 88 vector
            # bytes per row); needs a 1024/2048/4096-row tile map
            if os.environ.get("AB_CG_SINGLE_PASS") is not None:  # lab switch
                single_pass = os.environ["AB_CG_SINGLE_PASS"] != "0"
            self.perm2["single"] = bool(single_pass and self.perm2["tile"] is not None
                                        and tile_rows in (1024, 2048, 4096))
            if self.perm2["single"]:
                pair = lambda: torch.zeros(n, 2, dtype=torch.float64, device=dev)  # noqa: E731
                self.perm2["xp"], self.perm2["rq"] = pair(), (pair(), pair())

    def _m(self, name):
        import contextlib
        return self.mark(name) if self.mark is not None else contextlib.nullcontext()

    def solve(self, b: torch.Tensor, maxit: int, tol: float = 0.0, check_every: int = 1, zero_b: bool = True):
        """x = A^-1 b (x0 = 0).  With tol == 0 runs exactly ``maxit``
        iterations without host synchronisation (CUDA-graph capturable).
        ``zero_b`` re-zeroes b (it is an accumulation buffer of K4)."""
        s = stream_handle()
        A = ctypes.byref(self.A.struct)
        if self.local is not None:
            lm = self.local
            with self._m("K5_cg_resident"):
                call("ab_cg_resident_local", ctypes.byref(lm["A"].struct), ctypes.byref(lm["struct"]), ptr(b),
                     ptr(b) if zero_b else None, ptr(lm["fixed"]), ptr(lm["dinv"]), ptr(self.x), ptr(self.z),
                     int(maxit), float(tol), ptr(self.red), ptr(self.sc), ptr(self.part), s)
            it = int(self.red[3].item()) if tol > 0 else maxit
            return self.x, it
        if self.perm2 is not None:
            return self._solve_permuted(b, maxit, tol, check_every, zero_b)
        call("ab_cg_init", self.n, ptr(b), ptr(b) if zero_b else None, ptr(self.fixed), ptr(self.dinv),
             ptr(self.x), ptr(self.r), ptr(self.z), ptr(self.p), ptr(self.q), ptr(self.own), ptr(self.red),
             ptr(self.sc), ptr(self.part), ptr(self.cnt), s)
        if self.halo is not None:
            self.halo.allreduce_(self.red[0:2])
        call("ab_cg_set_bb", ptr(self.red), ptr(self.sc), s)
        it = 0
        while it < maxit:
            if tol > 0 and it % check_every == 0:
                rr, bb = float(self.red[1].item()), float(self.sc[1].item())
                if bb == 0.0 or math.sqrt(rr / bb) <= tol:
                    break
            if self.halo is None:
                with self._m("K5_cg_spmv"):
                    call("ab_cg_spmv", A, ptr(self.z), ptr(self.p), ptr(self.q), None, 1, ptr(self.own),
                         ptr(self.red), ptr(self.sc), ptr(self.part), ptr(self.cnt), s)
            else:
                with self._m("K5_cg_spmv"):
                    call("ab_cg_spmv", A, ptr(self.z), ptr(self.p), ptr(self.q), ptr(self.t), 0, ptr(self.own),
                         ptr(self.red), ptr(self.sc), ptr(self.part), ptr(self.cnt), s)
                with self._m("X_halo_sum"):
                    self.halo.sum_(self.t, 1, 1)
                with self._m("K5_cg_dot"):
                    call("ab_cg_dot", self.n, ptr(self.z), ptr(self.t), ptr(self.p), ptr(self.q), ptr(self.own),
                         ptr(self.red), ptr(self.sc), ptr(self.part), ptr(self.cnt), s)
                with self._m("X_allreduce"):
                    self.halo.allreduce_(self.red[2:3])
            with self._m("K5_cg_update"):
                call("ab_cg_update", self.n, ptr(self.p), ptr(self.q), ptr(self.dinv), ptr(self.x), ptr(self.r),
                     ptr(self.z), ptr(self.own), ptr(self.red), ptr(self.sc), ptr(self.part), ptr(self.cnt), s)
            if self.halo is not None:
                with self._m("X_allreduce"):
                    self.halo.allreduce_(self.red[0:2])
            it += 1
        return self.x, it

    def _solve_permuted(self, b: torch.Tensor, maxit: int, tol: float, check_every: int, zero_b: bool):
        """Two kernels per iteration on P A P^T; b in and x out through the
        row permutation (one gather and one scatter per solve)."""
        s = stream_handle()
        pm = self.perm2
        A = ctypes.byref(pm["A"].struct)
        sc_ = pm["scaled"]
        d = pm["d"] if (sc_ and tol > 0) else None  # true ||r|| only when a tolerance is tested
        if pm.get("single"):
            return self._solve_single_pass(b, maxit, tol, check_every, zero_b, d)
        if sc_:
            call("ab_cg_init_scaled", self.n, ptr(pm["perm"]), ptr(b), 1 if zero_b else 0, ptr(pm["fixed"]),
                 ptr(pm["s"]), ptr(d), ptr(self.x), ptr(self.r), ptr(self.p), ptr(self.q), ptr(self.red),
                 ptr(self.sc), ptr(self.part), ptr(self.cnt), s)
        else:
            call("ab_cg_init_perm", self.n, ptr(pm["perm"]), ptr(b), 1 if zero_b else 0, ptr(pm["fixed"]),
                 ptr(pm["dinv"]), ptr(self.x), ptr(self.r), ptr(self.z), ptr(self.p), ptr(self.q), ptr(self.red),
                 ptr(self.sc), ptr(self.part), ptr(self.cnt), s)
        zvec = self.r if sc_ else self.z  # the scaled form gathers r' where Jacobi gathers z
        it = 0
        while it < maxit:
            if tol > 0 and it % check_every == 0:
                rr, bb = float(self.red[1].item()), float(self.sc[1].item())
                if bb == 0.0 or math.sqrt(rr / bb) <= tol:
                    break
            with self._m("K5_cg_spmv"):
                if pm.get("tile") is not None:
                    call("ab_cg_spmv_tile", A, ctypes.byref(pm["tile"]["struct"]), ptr(zvec), ptr(self.p),
                         ptr(self.q), ptr(self.red), ptr(self.sc), ptr(self.part), ptr(self.cnt), s)
                elif pm["unit"]:
                    call("ab_cg_spmv_unit", A, ptr(zvec), ptr(self.p), ptr(self.q), ptr(self.red), ptr(self.sc),
                         ptr(self.part), ptr(self.cnt), s)
                else:
                    call("ab_cg_spmv", A, ptr(zvec), ptr(self.p), ptr(self.q), None, 1, None, ptr(self.red),
                         ptr(self.sc), ptr(self.part), ptr(self.cnt), s)
            with self._m("K5_cg_update_scaled" if sc_ else "K5_cg_update"):
                if sc_:
                    call("ab_cg_update_scaled", self.n, ptr(self.p), ptr(self.q), ptr(self.x), ptr(self.r), ptr(d),
                         ptr(self.red), ptr(self.sc), ptr(self.part), ptr(self.cnt), s)
                else:
                    call("ab_cg_update", self.n, ptr(self.p), ptr(self.q), ptr(pm["dinv"]), ptr(self.x),
                         ptr(self.r), ptr(self.z), None, ptr(self.red), ptr(self.sc), ptr(self.part), ptr(self.cnt), s)
            it += 1
        if sc_:
            call("ab_cg_finish_scaled", self.n, ptr(pm["iperm"]), ptr(pm["s"]), ptr(self.x), ptr(pm["x"]), s)
        else:
            call("ab_perm_scatter", self.n, ptr(pm["perm"]), ptr(self.x), ptr(pm["x"]), s)
        return pm["x"], it

    def _solve_single_pass(self, b, maxit: int, tol: float, check_every: int, zero_b: bool, d):
        """One kernel per iteration (ab_cg_tile_iter): iteration k forms x'_k,
        r'_k, p_k and q_k; the finish adds the last alpha p when all ``maxit``
        iterations ran (the same SpMV count as the two-kernel loop)."""
        s = stream_handle()
        pm = self.perm2
        A = ctypes.byref(pm["A"].struct)
        tm = ctypes.byref(pm["tile"]["struct"])
        xp, rq = pm["xp"], pm["rq"]
        call("ab_cg_tile_init", self.n, ptr(pm["perm"]), ptr(b), 1 if zero_b else 0, ptr(pm["fixed"]),
             ptr(pm["s"]), ptr(d), ptr(xp), ptr(rq[0]), ptr(self.red), ptr(self.sc), ptr(self.part), ptr(self.cnt), s)
        it, apply = 0, 1 if maxit > 0 else 0
        while it < maxit:
            # kernel `it` forms r'_it (and x'_it), then the SpMV of iteration it
            with self._m("K5_cg_tile_iter"):
                call("ab_cg_tile_iter", A, tm, ptr(rq[it & 1]), ptr(rq[(it + 1) & 1]), ptr(xp), ptr(d),
                     ptr(self.red), ptr(self.part), ptr(self.cnt), s)
            if tol > 0 and it % check_every == 0:
                rr, bb = float(self.red[1].item()), float(self.sc[1].item())
                if bb == 0.0 or math.sqrt(rr / bb) <= tol:
                    apply = 0  # r'_it converged: x'_it is the answer
                    break
            it += 1
        call("ab_cg_tile_finish", self.n, ptr(pm["iperm"]), ptr(pm["s"]), ptr(xp), ptr(self.red), apply,
             ptr(pm["x"]), s)
        return pm["x"], it

    def residual(self) -> float:
        rr, bb = float(self.red[1].item()), float(self.sc[1].item())
        return math.sqrt(rr / bb) if bb > 0 else 0.0


def pcg_solve(A: SellMatrix, b: torch.Tensor, x0=None, tol: float = 1e-10, max_it: int = 1000,
              fixed: torch.Tensor | None = None):
    """Drop-in style solve: returns (x, iterations, ||r||/||b||)."""
    dinv = 1.0 / A.diag
    solver = PCG(A, dinv, fixed=fixed)
    rhs = b.clone()
    if x0 is not None:
        rhs = rhs - A.matvec(x0)
    x, it = solver.solve(rhs, max_it, tol=tol, zero_b=False)
    x = x.clone()
    if x0 is not None:
        x = x + x0
    return x, it, solver.residual()

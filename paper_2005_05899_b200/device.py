"""Device-resident mesh: the HBM layout every kernel reads.

* ``coords4``: f64 [N][4] (x, y, z, 0) — one 256-bit load per node;
* per category: int32 connectivity [E_k][n_k] (reference VTK node order) and
  the int64 global element ids of its rows;
* optional SFC reordering of the elements of each category (Hilbert order of
  the centroids), which makes consecutive elements spatially compact so
  node gathers hit L2 and the node windows of the windowed scatter are small;
* optional node windows (``ab_set_windows``) per category, built once on the
  GPU with a stable sort of (block, node) keys.
"""

from __future__ import annotations

import os

import numpy as np
import torch

from . import _lib
from ._lib import AbMesh, AbCategory, RULE_ID, call, ptr, stream_handle
from .meshgen import MeshArrays, NODE_COUNT, RULE_KIND

WINDOW_BLOCK = 128


class DeviceMesh:
    def __init__(self, mesh: MeshArrays, device="cuda", reorder: str | None = None, windows: bool = False,
                 pipelined: bool = True, scatter: str = "atomic"):
        if not torch.cuda.is_available():
            raise RuntimeError("DeviceMesh needs a CUDA device (there is no CPU fallback)")
        self.device = torch.device(device)
        self.host = mesh
        self.n_nodes = mesh.n_nodes
        c4 = np.zeros((mesh.n_nodes, 4), dtype=np.float64)
        c4[:, :3] = mesh.coords
        self.coords4 = torch.from_numpy(c4).to(self.device)
        self.period = np.asarray(mesh.period, dtype=np.float64)
        self.rules, self.conn, self.ids = [], [], []
        for _tag, rule, conn, ids in mesh.categories():
            self.rules.append(rule)
            self.conn.append(torch.from_numpy(np.ascontiguousarray(conn, dtype=np.int32)).to(self.device))
            self.ids.append(torch.from_numpy(np.asarray(ids, dtype=np.int64)).to(self.device))
        self._win = []
        self._col = []
        self.pipelined = pipelined
        if scatter not in ("atomic", "colour"):
            raise ValueError(f"scatter must be 'atomic' or 'colour', not {scatter!r}")
        if scatter == "colour" and not (windows and pipelined):
            raise ValueError("scatter='colour' needs the pipelined node windows (windows=True, pipelined=True)")
        self.scatter = scatter
        self._build_struct()
        if reorder == "sfc":
            self.reorder_sfc()
        if windows and pipelined and os.environ.get("AB_NO_TET_TUNE", "0") != "1":
            self.tune_tet_node_order()
        if windows:
            self.build_windows()
        self._d2 = []
        if os.environ.get("AB_NO_FILTER_WIDTH", "0") != "1":
            self.build_filter_width()

    # -- C struct -------------------------------------------------------------
    def _build_struct(self):
        m = AbMesh()
        m.n_nodes = self.n_nodes
        m.coords = ptr(self.coords4)
        for d in range(3):
            m.period[d] = float(self.period[d])
        m.n_cat = len(self.rules)
        for k, (rule, conn) in enumerate(zip(self.rules, self.conn)):
            m.cat[k] = AbCategory(rule=RULE_ID[rule], pad_=0, n_elem=conn.shape[0], conn=ptr(conn))
        self.struct = m

    @property
    def n_elements(self) -> int:
        return int(sum(c.shape[0] for c in self.conn))

    def element_counts(self):
        return {r: int(c.shape[0]) for r, c in zip(self.rules, self.conn)}

    def sub(self, k: int) -> AbMesh:
        """ab_mesh restricted to category k (for per-category launches)."""
        m = AbMesh()
        m.n_nodes = self.n_nodes
        m.coords = ptr(self.coords4)
        for d in range(3):
            m.period[d] = float(self.period[d])
        m.n_cat = 1
        m.cat[0] = self.struct.cat[k]
        return m

    # -- SFC ordering ---------------------------------------------------------
    def centroids(self, k: int) -> torch.Tensor:
        out = torch.empty((self.conn[k].shape[0], 3), dtype=torch.float64, device=self.device)
        call("ab_centroids", C_ref(self.struct), k, ptr(out), stream_handle())
        return out

    def reorder_sfc(self, level: int = 10):
        """Sort the elements of each category by the Hilbert key of their
        centroid (stable, so ties keep generator order)."""
        self.clear_windows()
        had_d2 = bool(getattr(self, "_d2", []))
        self.clear_filter_width()
        cents = [self.centroids(k) for k in range(len(self.rules))]
        allc = torch.cat(cents)
        lo = allc.min(dim=0).values
        hi = allc.max(dim=0).values
        span = torch.clamp(hi - lo, min=1e-300) * (1 + 1e-12)
        for k, c in enumerate(cents):
            keys = torch.empty(c.shape[0], dtype=torch.int64, device=self.device)
            call("ab_hilbert_keys", c.shape[0], ptr(c), ptr(lo), ptr(span), level, ptr(keys), stream_handle())
            order = torch.sort(keys, stable=True).indices
            self.conn[k] = self.conn[k][order].contiguous()
            self.ids[k] = self.ids[k][order].contiguous()
        self._build_struct()
        if had_d2:
            self.build_filter_width()

    def node_order(self, level: int = 10) -> torch.Tensor:
        """Node ids sorted by the Hilbert key of their coordinates (stable):
        the solver-row numbering of the resident CG (compact per-CTA row
        ranges)."""
        c = self.coords4[:, :3].contiguous()
        lo = c.min(dim=0).values
        hi = c.max(dim=0).values
        span = torch.clamp(hi - lo, min=1e-300) * (1 + 1e-12)
        keys = torch.empty(c.shape[0], dtype=torch.int64, device=self.device)
        call("ab_hilbert_keys", c.shape[0], ptr(c), ptr(lo), ptr(span), level, ptr(keys), stream_handle())
        return torch.sort(keys, stable=True).indices.to(torch.int32)

    # -- node windows ---------------------------------------------------------
    def tune_tet_node_order(self, block: int = WINDOW_BLOCK, chunk: int = 1 << 22):
        """Permute the 4 nodes of every tetrahedron (all tet kernels use |det J|
        and are symmetric in the node order, so results change only by
        rounding) so that the window gathers of K2 — instruction a reads node a
        of 32 consecutive elements, 8 lanes per shared-memory phase, 16-byte
        words — hit distinct banks: greedy per group of 8 elements, choosing
        for each element the permutation with the fewest same-bank, different-
        address partners among the group's earlier elements.  Window-local
        indices do not depend on the node order, so they are computed first.
        Processed in chunks of whole blocks (``chunk`` elements) to bound the
        memory on 250M-element meshes."""
        import itertools
        perms = torch.tensor(list(itertools.permutations(range(4))), dtype=torch.int64, device=self.device)
        N = self.n_nodes
        chunk = max(block, chunk // block * block)
        gs = int(os.environ.get("AB_TET_TUNE_GROUP", "8"))  # lanes per modelled shared-memory phase
        for k, (rule, conn) in enumerate(zip(self.rules, self.conn)):
            E = conn.shape[0]
            if not rule.startswith("tet") or E < gs:
                continue
            E8 = E // gs * gs
            conn = conn.clone()
            for e0 in range(0, E8, chunk):
                e1 = min(E8, e0 + chunk)
                n = e1 - e0
                c = conn[e0:e1].to(torch.int64)
                blk = (torch.arange(n, device=self.device, dtype=torch.int64) // block).repeat_interleave(4)
                _, inv = torch.unique(blk * N + c.reshape(-1), return_inverse=True)  # (block, node) ascending
                first = torch.zeros(int(blk[-1].item()) + 1, dtype=inv.dtype, device=self.device)
                first.scatter_reduce_(0, blk, inv, reduce="amin", include_self=False)
                loc = (inv - first[blk]).view(-1, gs, 4)  # (G, gs, 4) window indices
                del inv, blk
                G = loc.shape[0]
                rows = torch.arange(G, device=self.device)
                chosen = torch.empty((G, gs, 4), dtype=torch.int64, device=self.device)
                best_all = torch.empty((G, gs), dtype=torch.int64, device=self.device)
                for j in range(gs):
                    cand = loc[:, j, :][:, perms]  # (G, 24, 4): the value placed in slot a
                    if j == 0:
                        best = torch.zeros(G, dtype=torch.int64, device=self.device)
                    else:
                        cv = cand[:, :, None, :]
                        pv = chosen[:, None, :j, :]
                        cost = (((cv - pv) % 8 == 0) & (cv != pv)).sum(dim=(2, 3))
                        best = torch.argmin(cost, dim=1)  # first minimum
                    best_all[:, j] = best
                    chosen[:, j, :] = cand[rows, best]
                # refinement sweeps: re-choose each element against all the
                # others of its group (never worse than the current choice,
                # which is candidate best_all[:, j] with the same cost model)
                for _ in range(int(os.environ.get("AB_TET_TUNE_SWEEPS", "1"))):
                    for j in range(gs):
                        cand = loc[:, j, :][:, perms]
                        others = torch.cat([chosen[:, :j, :], chosen[:, j + 1:, :]], dim=1)
                        cv = cand[:, :, None, :]
                        pv = others[:, None, :, :]
                        cost = (((cv - pv) % 8 == 0) & (cv != pv)).sum(dim=(2, 3))
                        cur = cost[rows, best_all[:, j]]
                        best = torch.argmin(cost, dim=1)
                        best = torch.where(cost[rows, best] < cur, best, best_all[:, j])
                        best_all[:, j] = best
                        chosen[:, j, :] = cand[rows, best]
                pidx = perms[best_all.view(-1)]
                conn[e0:e1] = torch.gather(c, 1, pidx).to(torch.int32)
                del loc, chosen, c
            self.conn[k] = conn.contiguous()
        self._build_struct()

    def build_windows(self):
        self.clear_windows()
        for conn in self.conn:
            if conn.shape[0] == 0:
                self._win.append(None)
                continue
            w = window_arrays(conn, self.n_nodes, WINDOW_BLOCK,
                              spread=self.pipelined and os.environ.get("AB_NO_SLOT_SPREAD", "0") != "1")
            blk_ptr, wnode, wptr, wslot, loc, wmax, desc, wref = w
            self._win.append(w)
            call("ab_set_windows", ptr(conn), WINDOW_BLOCK, ptr(blk_ptr), ptr(wnode), ptr(wptr), ptr(wslot),
                 ptr(loc), ptr(desc) if self.pipelined else None, wmax)
            call("ab_set_window_refs", ptr(conn), ptr(wref))
        self.windows = True
        if self.scatter == "colour":
            self.build_colours()

    def build_colours(self):
        """Colour the window blocks of every category (two blocks conflict
        when they share a window node; Jones-Plassmann on the GPU,
        ``ab_colour_blocks``) and register the colour mode: the pipelined
        kernels then process the blocks colour by colour and update each node
        with one plain read-add-write in a fixed order (bitwise reproducible
        K2/K4/K6, the north star's "mesh colouring" scatter)."""
        self.clear_colours()
        dev = self.device
        N = self.n_nodes
        for conn, w in zip(self.conn, self._win):
            if w is None:
                self._col.append(None)
                continue
            blk_ptr, wnode = w[0], w[1]
            nb = blk_ptr.numel() - 1
            nw = int(blk_ptr[-1].item())
            counts = blk_ptr[1:] - blk_ptr[:-1]
            wblk = torch.repeat_interleave(torch.arange(nb, device=dev, dtype=torch.int32), counts)
            wn = wnode[:nw].to(torch.int64)
            order = torch.sort(wn, stable=True).indices
            nblk = wblk[order].contiguous()
            del wblk, order
            nptr = torch.zeros(N + 1, dtype=torch.int64, device=dev)
            nptr[1:] = torch.cumsum(torch.bincount(wn, minlength=N), 0)
            del wn
            colour = torch.empty(nb, dtype=torch.int32, device=dev)
            flags = torch.zeros(2, dtype=torch.int32, device=dev)
            call("ab_colour_blocks", nb, ptr(blk_ptr), ptr(wnode), ptr(nptr), ptr(nblk), ptr(colour), ptr(flags),
                 stream_handle())
            del nptr, nblk
            ncol = int(colour.max().item()) + 1
            corder = torch.sort(colour, stable=True).indices.to(torch.int32).contiguous()
            cptr = torch.zeros(ncol + 1, dtype=torch.int64, device=dev)
            cptr[1:] = torch.cumsum(torch.bincount(colour.to(torch.int64), minlength=ncol), 0)
            gbar = torch.zeros(max(ncol, 1), dtype=torch.int32, device=dev)  # one barrier counter per colour
            call("ab_set_window_colours", ptr(conn), ncol, ptr(corder), ptr(cptr), ptr(gbar))
            self._col.append((corder, cptr, gbar, ncol, colour))

    def clear_colours(self):
        for conn, c in zip(self.conn, self._col):
            if c is not None:
                call("ab_set_window_colours", ptr(conn), 0, None, None, None)
        self._col = []

    def colour_stats(self):
        """Per category: number of colours and blocks per colour."""
        out = {}
        for rule, c in zip(self.rules, self._col):
            if c is not None:
                out[rule] = {"colours": c[3], "blocks": [int(v) for v in (c[1][1:] - c[1][:-1]).tolist()]}
        return out

    def build_filter_width(self):
        """Vreman filter width Delta^2 = V_e^(2/3) of every element (geometry
        only), registered for K2 (ab_set_filter_width)."""
        self.clear_filter_width()
        for k, conn in enumerate(self.conn):
            d2 = torch.empty(conn.shape[0], dtype=torch.float64, device=self.device)
            if conn.shape[0]:
                call("ab_filter_width", C_ref(self.struct), k, ptr(d2), stream_handle())
                call("ab_set_filter_width", ptr(conn), conn.shape[0], ptr(d2))
            self._d2.append(d2)

    def clear_filter_width(self):
        for conn, d2 in zip(self.conn, getattr(self, "_d2", [])):
            if d2.numel():
                call("ab_set_filter_width", ptr(conn), 0, None)
        self._d2 = []

    def window_stats(self):
        out = {}
        for rule, conn, w in zip(self.rules, self.conn, self._win):
            if w is None:
                continue
            out[rule] = {"refs": int(conn.numel()), "window_nodes": int(w[1].numel()), "wmax": w[5],
                         "reduction": float(conn.numel()) / max(1, int(w[1].numel()))}
        return out

    def clear_windows(self):
        self.clear_colours()
        for conn, w in zip(self.conn, self._win):
            if w is not None:
                call("ab_set_windows", ptr(conn), WINDOW_BLOCK, None, None, None, None, None, None, 0)
        self._win = []
        self.windows = False

    def __del__(self):
        try:
            self.clear_windows()
            self.clear_filter_width()
        except Exception:
            pass


def _spread_slot_banks(order, starts, slot, E, nn, B, chunk_blocks: int = 1 << 17):
    """Reorder the references inside every window node's run (sum order only)
    so that the phase-D slot loads — lane t of a block reads sorted positions
    t*nn .. t*nn+nn-1, instruction k position t*nn+k, 16 lanes per shared-
    memory phase of 8-byte words, bank = slot offset mod 16 — meet few
    same-bank partners: position by position, the run's remaining reference
    with the fewest already placed same-bank references in that phase."""
    dev = order.device
    R = order.numel()
    RB = B * nn
    nblk_full = R // RB
    if nblk_full == 0:
        return order
    run_end = torch.empty(R, dtype=torch.int64, device=dev)
    ends = torch.cat([starts[1:], torch.tensor([R], device=dev)])
    run_end[starts] = ends
    run_end = torch.cummax(torch.where(torch.zeros(R, dtype=torch.bool, device=dev).index_fill_(0, starts, True),
                                       run_end, torch.zeros_like(run_end)), 0).values
    out = order.clone()
    bank_all = slot % 16
    maxrun = int((ends - starts).max().item())
    n_ph = (B // 16) * nn
    for b0 in range(0, nblk_full, chunk_blocks):
        b1 = min(nblk_full, b0 + chunk_blocks)
        nb = b1 - b0
        base = torch.arange(b0, b1, device=dev) * RB
        o = out[b0 * RB:b1 * RB].view(nb, RB).clone()
        re = (run_end[b0 * RB:b1 * RB].view(nb, RB) - base[:, None])  # run end (block-relative) of each position
        cnt = torch.zeros((nb, n_ph, 16), dtype=torch.int32, device=dev)
        rows = torch.arange(nb, device=dev)
        jj = torch.arange(maxrun, device=dev)
        for p_ in range(RB):
            t, k = divmod(p_, nn)
            ph = (t // 16) * nn + k
            cand = p_ + jj[None, :]                                   # (nb, maxrun) positions
            ok = cand < re[:, p_:p_ + 1]
            cand = torch.where(ok, cand, torch.full_like(cand, p_))
            bk = bank_all[o.gather(1, cand)]                          # banks of the candidates
            cost = cnt[rows, ph].gather(1, bk).to(torch.int64) * 4096 + jj[None, :]
            cost = torch.where(ok, cost, torch.full_like(cost, 1 << 40))
            pick = cand[rows, torch.argmin(cost, dim=1)]
            a_ = o[rows, p_].clone()
            o[rows, p_] = o[rows, pick]
            o[rows, pick] = a_
            cnt[rows, ph, bank_all[o[rows, p_]]] += 1
        out[b0 * RB:b1 * RB] = o.view(-1)
    return out


def window_arrays(conn: torch.Tensor, N: int, B: int = WINDOW_BLOCK, spread: bool = True):
    """Node windows of one category (any device): returns (blk_ptr, wnode,
    wptr, wslot, loc, wmax, desc, wref) as registered by ab_set_windows /
    ab_set_window_refs (include/alyab200.h).  Window indices ascend with the
    node id inside each block."""
    dev = conn.device
    E, nn = conn.shape
    e = torch.arange(E, device=dev, dtype=torch.int64)
    blk = (e // B).repeat_interleave(nn)
    # shared-memory slot offset a * B + (e % B) of every (element, node) reference
    slot = (e % B).repeat_interleave(nn) + B * torch.arange(nn, device=dev).repeat(E)
    node = conn.reshape(-1).to(torch.int64)
    key = blk * N + node
    order = torch.sort(key, stable=True).indices
    ks = key[order]
    start = torch.ones_like(ks, dtype=torch.bool)
    start[1:] = ks[1:] != ks[:-1]
    starts = torch.nonzero(start).squeeze(1)
    wnode = (ks[starts] % N).to(torch.int32).contiguous()
    wblk = ks[starts] // N
    wptr = torch.cat([starts, torch.tensor([ks.numel()], device=dev)]).to(torch.int32).contiguous()
    wslot = slot[order].to(torch.int16).contiguous()
    nblk = (E + B - 1) // B
    blk_ptr = torch.searchsorted(wblk, torch.arange(nblk + 1, device=dev, dtype=torch.int64))
    blk_ptr = blk_ptr.to(torch.int64).contiguous()
    if spread and nn * B <= 4096:
        order = _spread_slot_banks(order, starts, slot, E, nn, B)
    # window-local index of every (element, node) reference
    uid = torch.cumsum(start.to(torch.int64), 0) - 1
    local = uid - blk_ptr[blk[order]]
    loc = torch.empty_like(local)
    loc[order] = local
    loc = loc.to(torch.int16).reshape(E, nn).contiguous()
    # sorted references of every block (slot offset | window index << 16), padded to whole blocks
    wref = torch.full((nblk * B * nn,), 0xFFFF << 16, dtype=torch.int64, device=dev)
    wref[:E * nn] = slot[order] | (local << 16)
    wref = torch.where(wref >= 1 << 31, wref - (1 << 32), wref).to(torch.int32).contiguous()
    wmax = int((blk_ptr[1:] - blk_ptr[:-1]).max().item())
    # per-block descriptors for the pipelined kernels
    b0, b1 = blk_ptr[:-1], blk_ptr[1:]
    desc = torch.stack([b0, b1, wptr[b0].to(torch.int64), wptr[b1].to(torch.int64)], dim=1)
    desc = desc.to(torch.int32).contiguous()
    # bulk copies read whole 16-byte granules: pad every array
    wnode, wptr, wslot, loc = (_padded(t) for t in (wnode, wptr, wslot, loc))
    return (blk_ptr, wnode, wptr, wslot, loc, wmax, desc, wref)


def _padded(t: torch.Tensor) -> torch.Tensor:
    """Copy of a 1D/2D tensor with 64 spare bytes behind its data (views keep
    the original shape)."""
    flat = t.reshape(-1)
    extra = max(1, 64 // flat.element_size())
    buf = torch.zeros(flat.numel() + extra, dtype=flat.dtype, device=flat.device)
    buf[: flat.numel()] = flat
    return buf[: flat.numel()].view(t.shape)


def C_ref(struct):
    import ctypes
    return ctypes.byref(struct)


def nodes_as4(x: torch.Tensor) -> torch.Tensor:
    """(N,3) -> contiguous (N,4) f64 with zero pad (no-op for (N,4))."""
    if x.dim() == 2 and x.shape[1] == 4 and x.is_contiguous() and x.dtype == torch.float64:
        return x
    out = torch.zeros((x.shape[0], 4), dtype=torch.float64, device=x.device)
    out[:, :3] = x[:, :3]
    return out

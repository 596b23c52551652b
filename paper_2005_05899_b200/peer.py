"""Peer-memory interface exchange and the decomposed CG for large subdomains
(include/alyab200.h "Peer-memory interface exchange").

One process per GPU.  Every rank allocates the buffers its neighbours write
into - receive slots, arrival counters, reduction records - and the
neighbours map them with CUDA IPC (NVLink/NVSwitch peer stores).  No NCCL
call and no host synchronisation happen per exchange or per CG iteration:
progress state (exchange counts, record epochs, scalars) is device-resident,
so a whole multi-rank time step is captured in one CUDA graph.

* :class:`PeerHalo` - ``sum_(field, ncomp, stride)`` adds the sharers'
  partials of every interface node in global rank order (bitwise identical
  copies on all ranks; drop-in for halo.HaloExchanger).
* :class:`DD2Rank` / :class:`DD2Solver` - Jacobi-PCG of a decomposed domain
  too large for the on-chip solver (ab_cg_dd): SpMV with the interface rows
  first (their partial products travel while the interior rows stream),
  a small interface kernel, and the update; p.q and {r.z, r.r} reduced across
  ranks through {value, epoch} records.

Ranks may also share one process and GPU ("virtual ranks", tests): the peer
pointers are then plain device pointers, and every phase is launched for all
ranks before the next phase (``virtual_halo_sum``, ``DD2Solver`` with
several ranks), so no kernel waits on a launch that has not been issued.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from ._lib import PEER_MAX, AbDdcg2Rank, AbPeerHalo, call, lib, ptr, stream_handle
from .solver import SellMatrix, cg_local_map, permute_matrix


# ---------------------------------------------------------------------------
# mapping helpers
# ---------------------------------------------------------------------------

def _ipc_handle(t: torch.Tensor):
    h = (C.c_ubyte * 64)()
    off = C.c_int64(0)
    call("ab_ipc_get_handle", ptr(t), h, C.byref(off))
    return bytes(h), off.value


def ipc_exchange(tensors: dict, meta: dict, n_ranks: int, rank: int, group=None):
    """All-gather IPC handles of ``tensors`` (+ ``meta``) and map every other
    rank's buffers: returns {q: {"name": device pointer, ..., **meta_q}}."""
    import torch.distributed as dist
    try:
        mine = {k: _ipc_handle(v) for k, v in tensors.items()}
        mine.update(meta)
    except Exception as e:  # take part in the exchange, then fail everywhere
        mine = {"error": str(e)}
    allx = [None] * n_ranks
    dist.all_gather_object(allx, mine, group=group)
    bad = [q for q, x in enumerate(allx) if "error" in x]
    if bad:
        raise RuntimeError(f"CUDA IPC export failed on ranks {bad}: {allx[bad[0]]['error']}")
    out = {}
    opened = []
    for q in range(n_ranks):
        if q == rank:
            continue
        d = {k: v for k, v in allx[q].items() if k not in tensors}
        for k in tensors:
            h, off = allx[q][k]
            p = C.c_void_p()
            call("ab_ipc_open_handle", (C.c_ubyte * 64).from_buffer_copy(h), C.byref(p))
            opened.append(p.value)
            d[k] = p.value + off
        out[q] = d
    return out, opened


# ---------------------------------------------------------------------------
# interface sum
# ---------------------------------------------------------------------------

class PeerHalo:
    """Interface sums over peer memory for one rank (plan: decompose.
    InterfacePlan / dmesh.interface_plan_local).  ``max_shared`` must be the
    same on every rank (the longest shared list of any pair)."""

    graph_safe = True

    def __init__(self, plan, device, max_shared: int):
        self.plan = plan
        self.group = None
        self.device = torch.device(device)
        dev = self.device
        self.rank, self.n_ranks = plan.rank, plan.n_ranks
        self.neighbors = list(plan.neighbors)
        if len(self.neighbors) > PEER_MAX:
            raise ValueError(f"at most {PEER_MAX} neighbours")
        self.own = torch.from_numpy(np.asarray(plan.own, dtype=np.float64)).to(dev)
        # interface nodes, ascending local id; per node its sharers (ascending rank) and slots
        nodes, ranks, slots = [], [], []
        for q in self.neighbors:
            idx = np.asarray(plan.shared[q], dtype=np.int64)
            nodes.append(idx)
            ranks.append(np.full(idx.size, q, np.int64))
            slots.append(np.arange(idx.size, dtype=np.int64))
        if nodes:
            nd, rk, sl = np.concatenate(nodes), np.concatenate(ranks), np.concatenate(slots)
            o = np.lexsort((rk, nd))
            nd, rk, sl = nd[o], rk[o], sl[o]
            if_node, start = np.unique(nd, return_index=True)
            if_ptr = np.append(start, nd.size)
        else:
            if_node = np.zeros(0, np.int64)
            if_ptr = np.zeros(1, np.int64)
            rk = sl = np.zeros(0, np.int64)
        t32 = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).to(dev)  # noqa: E731
        self.if_node, self.if_ptr, self.if_rank, self.if_slot = (t32(if_node), t32(if_ptr), t32(rk), t32(sl))
        self.n_if = int(if_node.size)
        self.M = max(1, int(max_shared))
        self.recv = torch.zeros(2 * self.n_ranks * self.M * 3, dtype=torch.float64, device=dev)
        self.cnt_in = torch.zeros(self.n_ranks, dtype=torch.int64, device=dev)
        self.state = torch.zeros(4, dtype=torch.int64, device=dev)
        self.n_cta = int(lib().ab_peer_halo_grid(self.n_if))
        self._ipc = []
        self.struct = None

    def exports(self) -> dict:
        return {"recv": self.recv, "cnt_in": self.cnt_in}

    def wire(self, peers: dict):
        """peers: q -> {"recv": ptr, "cnt_in": ptr, "n_cta": int} for every neighbour."""
        h = AbPeerHalo(rank=self.rank, n_ranks=self.n_ranks, n_if=self.n_if, n_cta=self.n_cta, max_shared=self.M,
                       n_nbr=len(self.neighbors), if_node=ptr(self.if_node), if_ptr=ptr(self.if_ptr),
                       if_rank=ptr(self.if_rank), if_slot=ptr(self.if_slot), recv=ptr(self.recv),
                       cnt_in=ptr(self.cnt_in), state=ptr(self.state))
        for k, q in enumerate(self.neighbors):
            h.nbr_rank[k] = q
            h.nbr_ncta[k] = int(peers[q]["n_cta"])
            h.nbr_recv[k] = int(peers[q]["recv"])
            h.nbr_cnt[k] = int(peers[q]["cnt_in"]) + 8 * self.rank
        self.struct = h

    @classmethod
    def connect(cls, plan, device, group=None) -> "PeerHalo":
        """Collective over the process group: agree on M, allocate, map the
        neighbours' buffers with CUDA IPC."""
        import torch.distributed as dist
        ms = max([0] + [len(v) for v in plan.shared.values()])
        t = torch.tensor([ms], dtype=torch.int64)
        if dist.get_backend(group) == "nccl":
            t = t.to(device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        h = cls(plan, device, int(t.item()))
        h.group = group
        peers, h._ipc = ipc_exchange(h.exports(), {"n_cta": h.n_cta}, h.n_ranks, h.rank, group)
        h.wire({q: peers[q] for q in h.neighbors})
        return h

    # -- exchange -------------------------------------------------------------
    def put(self, field: torch.Tensor, ncomp: int, stride: int):
        call("ab_peer_halo_put", C.byref(self.struct), ptr(field), ncomp, stride, stream_handle())

    def add(self, field: torch.Tensor, ncomp: int, stride: int):
        call("ab_peer_halo_add", C.byref(self.struct), ptr(field), ncomp, stride, stream_handle())

    def sum_(self, field: torch.Tensor, ncomp: int, stride: int):
        """field[shared] = rank-ordered sum of all sharers' values (one put +
        one add launch; asynchronous, graph-capturable)."""
        self.put(field, ncomp, stride)
        self.add(field, ncomp, stride)

    def allreduce_(self, t: torch.Tensor):
        """Setup-time reductions (not on the step path)."""
        import torch.distributed as dist
        if dist.get_backend(self.group) == "gloo" and t.is_cuda:
            h = t.cpu()
            dist.all_reduce(h, group=self.group)
            t.copy_(h)
        else:
            dist.all_reduce(t, group=self.group)

    def failed(self) -> bool:
        return int(self.state[2].item()) != 0

    def close(self):
        for p in self._ipc:
            try:
                call("ab_ipc_close", p)
            except Exception:
                pass
        self._ipc = []


def virtual_halos(plans: list, device) -> list:
    """PeerHalo objects of several ranks sharing one GPU in this process."""
    ms = max([0] + [len(v) for pl in plans for v in pl.shared.values()])
    hs = [PeerHalo(pl, device, ms) for pl in plans]
    for h in hs:
        h.wire({q: {"recv": ptr(hs[q].recv), "cnt_in": ptr(hs[q].cnt_in), "n_cta": hs[q].n_cta}
                for q in h.neighbors})
    return hs


def virtual_halo_sum(halos: list, fields: list, ncomp: int, stride: int):
    """Interface sum over virtual ranks: every put, then every add."""
    for h, f in zip(halos, fields):
        h.put(f, ncomp, stride)
    for h, f in zip(halos, fields):
        h.add(f, ncomp, stride)


# ---------------------------------------------------------------------------
# decomposed CG, large subdomains
# ---------------------------------------------------------------------------

class DD2Rank:
    """One rank of the two-kernel decomposed CG.

    A: the rank's assembled Laplacian (local node numbering, Dirichlet rows
    identity); dinv: 1/diag of the GLOBAL operator at the local nodes; own:
    ownership weights; shared: neighbour -> local nodes shared with it in
    ascending global id (both sides list the same nodes in the same order);
    order: an SFC order of the local nodes (solver rows = interface nodes
    first, in this order, then the interior nodes in this order)."""

    def __init__(self, rank: int, n_ranks: int, A: SellMatrix, dinv: torch.Tensor, own, shared: dict,
                 order: torch.Tensor, fixed: torch.Tensor | None = None, max_shared: int | None = None,
                 scaled: bool = True, tile_rows: int = 2048, single_pass: bool = True):
        dev = A.vals.device
        n = A.n_rows
        self.rank, self.n_ranks, self.n = rank, n_ranks, n
        self.neighbors = sorted(int(q) for q in shared)
        is_if = torch.zeros(n, dtype=torch.bool, device=dev)
        for q in self.neighbors:
            is_if[torch.as_tensor(np.asarray(shared[q]), device=dev).to(torch.int64)] = True
        order = order.to(device=dev, dtype=torch.int64)
        f = is_if[order]
        perm = torch.cat([order[f], order[~f]])
        self.n_if = int(f.sum().item())
        self.perm = perm.to(torch.int32).contiguous()
        iperm = torch.empty_like(perm)
        iperm[perm] = torch.arange(n, device=dev)
        self.A = permute_matrix(A, self.perm)
        self.dinv = dinv.to(dev)[perm].contiguous()
        # symmetrically scaled form (CG on D^-1/2 A D^-1/2, D the GLOBAL diagonal, so every rank scales its
        # partial rows alike): no z vector and no D^-1 stream per iteration
        self.scaled = bool(scaled)
        self.s = torch.sqrt(self.dinv).contiguous() if scaled else None
        if scaled:
            call("ab_sell_symscale", C.byref(self.A.struct), ptr(self.s), stream_handle())
        self.fixed = fixed.to(device=dev, dtype=torch.uint8)[perm].contiguous() if fixed is not None else None
        self.own = torch.as_tensor(np.asarray(own), dtype=torch.float64, device=dev)[perm].contiguous()
        self.M = int(max_shared if max_shared is not None else max([0] + [len(v) for v in shared.values()]))
        self.M = max(1, self.M)
        self.peers = [q for q in range(n_ranks) if q != rank]
        if len(self.peers) > PEER_MAX:
            raise ValueError(f"at most {PEER_MAX + 1} ranks")
        pidx = {q: k for k, q in enumerate(self.peers)}
        # per interface row: sends (peer index, slot in its recv) and receives (rank, slot in mine)
        rows, sp, so, rr, ro = [], [], [], [], []
        for q in self.neighbors:
            loc = torch.as_tensor(np.asarray(shared[q]), device=dev).to(torch.int64)
            row = iperm[loc]
            k = torch.arange(loc.numel(), device=dev, dtype=torch.int64)
            rows.append(row)
            sp.append(torch.full_like(k, pidx[q]))
            so.append(rank * self.M + k)
            rr.append(torch.full_like(k, q))
            ro.append(q * self.M + k)
        if rows:
            row = torch.cat(rows)
            o = torch.sort(row * (n_ranks + 1) + torch.cat(rr)).indices
            row, sp_, so_, rr_, ro_ = row[o], torch.cat(sp)[o], torch.cat(so)[o], torch.cat(rr)[o], torch.cat(ro)[o]
        else:
            row = sp_ = so_ = rr_ = ro_ = torch.zeros(0, dtype=torch.int64, device=dev)
        assert row.numel() == 0 or int(row.max().item()) < self.n_if
        cnt = torch.bincount(row, minlength=self.n_if)[: self.n_if] if self.n_if else torch.zeros(0, dtype=torch.int64,
                                                                                                  device=dev)
        ptr_ = torch.zeros(self.n_if + 1, dtype=torch.int32, device=dev)
        if self.n_if:
            ptr_[1:] = torch.cumsum(cnt, 0).to(torch.int32)
        i32t = lambda t: (t.to(torch.int32).contiguous() if t.numel()  # noqa: E731
                          else torch.zeros(1, dtype=torch.int32, device=dev))
        self.send_ptr = ptr_
        self.recv_ptr = ptr_.clone()
        self.send_peer, self.send_off = i32t(sp_), i32t(so_)
        self.recv_rank, self.recv_off = i32t(rr_), i32t(ro_)
        z = lambda k, dt=torch.float64: torch.zeros(max(1, k), dtype=dt, device=dev)  # noqa: E731
        self.x, self.r, self.zv, self.p, self.q = z(n), z(n), z(n), z(n), z(n)
        self.tif = z(self.n_if)
        self.recv = z(n_ranks * self.M)
        self.cnt_in = z(n_ranks, torch.int64)
        self.rec = torch.full((2 * n_ranks * 10,), -1.0, dtype=torch.float64, device=dev)
        self.part = z(int(lib().ab_ddcg2_part_size(n)))
        nb = (n + 63) // 64 + 1  # grid-sum counters: blocks of >= 64 rows (ab_ddcg2 kernels), then the interface kernels'
        self.cnt = z((nb + 63) // 64 + 16, torch.int32)
        self.scal = z(24)
        # tiled SpMV (k_d2_spmv_tile): z of a tile's rows and ghost rows in shared
        # memory, 16-bit tile-local columns; signalling blocks are tiles then
        self.tile = None
        if tile_rows:
            if tile_rows % 64:
                raise ValueError("tile_rows must be a multiple of 64")
            self.tile = cg_local_map(self.A, tile_rows, (n + tile_rows - 1) // tile_rows)
        self.tile_rows = tile_rows if self.tile is not None else 0
        blk = self.tile_rows or 256
        self.nsig = (self.n_if + blk - 1) // blk
        # single pass (ab_ddcg2_tile_iter + ab_ddcg2_tile_iface: two launches per
        # iteration, (x', p) and (r', q) as 16-byte pairs): scaled form on tiles
        self.single_pass = bool(single_pass and self.scaled and self.tile is not None)
        if self.single_pass:
            pair = lambda: torch.zeros(max(1, n), 2, dtype=torch.float64, device=dev)  # noqa: E731
            self.xp, self.rq = pair(), (pair(), pair())
        self.x_node = z(n)
        self.peer = {}
        self._ipc = []
        self.struct = None

    def exports(self) -> dict:
        return {"recv": self.recv, "cnt_in": self.cnt_in, "rec": self.rec}

    def wire(self, peers: dict):
        """peers: q -> {"recv", "cnt_in", "rec": pointers, "nsig": int} for every other rank."""
        d = AbDdcg2Rank(n_rows=self.n, n_if=self.n_if, rank=self.rank, n_ranks=self.n_ranks,
                        n_peers=len(self.peers), recv_stride=self.M)
        for name, t in (("slice_ptr", self.A.slice_ptr), ("cols", self.A.cols), ("vals", self.A.vals),
                        ("dinv", self.dinv), ("fixed", self.fixed), ("own", self.own), ("s", self.s),
                        ("perm", self.perm),
                        ("x", self.x), ("r", self.r), ("z", self.zv), ("p", self.p), ("q", self.q),
                        ("tif", self.tif), ("send_ptr", self.send_ptr), ("send_peer", self.send_peer),
                        ("send_off", self.send_off), ("recv_ptr", self.recv_ptr), ("recv_rank", self.recv_rank),
                        ("recv_off", self.recv_off), ("recv", self.recv), ("cnt_in", self.cnt_in),
                        ("rec", self.rec), ("part", self.part), ("cnt", self.cnt), ("scal", self.scal)):
            setattr(d, name, ptr(t))
        d.nsig = self.nsig
        d.scaled = 1 if self.scaled else 0
        if self.tile is not None:
            d.tcols, d.tghost_ptr, d.tghost = ptr(self.tile["cols"]), ptr(self.tile["ghost_ptr"]), ptr(self.tile["ghost"])
            d.tile_rows, d.tmax_ghost = self.tile_rows, int(self.tile["max_ghost"])
        if self.single_pass:
            d.xp, d.rq[0], d.rq[1], d.single_pass = ptr(self.xp), ptr(self.rq[0]), ptr(self.rq[1]), 1
        for k, q in enumerate(self.peers):
            d.peer_rank[k] = q
            d.peer_nsig[k] = int(peers[q]["nsig"]) if q in self.neighbors else 0
            d.peer_recv[k] = int(peers[q]["recv"])
            d.peer_cnt[k] = int(peers[q]["cnt_in"]) + 8 * self.rank
            d.peer_rec[k] = int(peers[q]["rec"])
        self.struct = d

    @property
    def iterations(self) -> int:
        return int(self.scal[0].item())

    def failed(self) -> bool:
        return float(self.scal[12].item()) != 0.0

    def residual(self) -> float:
        rr, bb = float(self.scal[11].item()), float(self.scal[2].item())
        return float(np.sqrt(rr / bb)) if bb > 0 else 0.0


def virtual_dd2(ranks: list) -> list:
    for r in ranks:
        r.wire({q: {"recv": ptr(ranks[q].recv), "cnt_in": ptr(ranks[q].cnt_in), "rec": ptr(ranks[q].rec),
                    "nsig": ranks[q].nsig} for q in r.peers})
    return ranks


class DD2Solver:
    """Drives the two-kernel decomposed CG of the ranks hosted by this
    process: one rank per GPU in a multi-GPU run (IPC-wired by
    :meth:`connect`), or several virtual ranks on one GPU (phase-major
    launches)."""

    def __init__(self, ranks: list, check_every: int = 16):
        self.ranks = ranks
        self.check_every = check_every
        self.mark = None

    @classmethod
    def connect(cls, rank: DD2Rank, group=None) -> "DD2Solver":
        peers, rank._ipc = ipc_exchange(rank.exports(), {"nsig": rank.nsig}, rank.n_ranks, rank.rank, group)
        rank.wire(peers)
        return cls([rank])

    def solve(self, bs, maxit: int, tol: float = 0.0, zero_b: bool = True):
        """x = A^-1 b for every hosted rank (b and x in local node order).
        With tol == 0 exactly ``maxit`` iterations and no host sync
        (graph-capturable); with tol > 0 the device decides convergence and
        the host stops launching once it reads the flag (every
        ``check_every`` iterations)."""
        if isinstance(bs, torch.Tensor):
            bs = [bs]
        s = stream_handle()
        for r, b in zip(self.ranks, bs):
            call("ab_ddcg2_init", C.byref(r.struct), ptr(b), ptr(b) if zero_b else None, float(tol), s)
        for it in range(maxit):
            if tol > 0 and it % self.check_every == 0 and it > 0:
                if float(self.ranks[0].scal[1].item()) != 0.0:
                    break
            fns = (("ab_ddcg2_tile_iter", "ab_ddcg2_tile_iface") if self.ranks[0].single_pass
                   else ("ab_ddcg2_spmv", "ab_ddcg2_iface", "ab_ddcg2_update"))
            for fn in fns:
                for r in self.ranks:
                    call(fn, C.byref(r.struct), s)
        for r in self.ranks:
            call("ab_ddcg2_finish", C.byref(r.struct), ptr(r.x_node), s)
        if tol > 0 or (len(self.ranks) > 1 and not torch.cuda.is_current_stream_capturing()):
            for r in self.ranks:
                if r.failed():
                    raise RuntimeError("decomposed CG: a peer wait timed out (ranks out of step)")
        its = self.ranks[0].iterations if tol > 0 else maxit
        return [r.x_node for r in self.ranks], its

    def check(self):
        for r in self.ranks:
            if r.failed():
                raise RuntimeError("decomposed CG: a peer wait timed out (ranks out of step)")


class FusedDD2Solver:
    """The two-kernel decomposed pressure solve of one rank of a multi-GPU
    run (one process per GPU, buffers IPC-mapped); ``solve(b, maxit, tol)``
    mirrors PCG.solve, b is interface-summed and re-zeroed."""

    def __init__(self, dm, A: SellMatrix, dinv: torch.Tensor, fixed, plan, b: torch.Tensor, group=None):
        import torch.distributed as dist
        dev = dinv.device
        ms = torch.tensor([max([0] + [len(v) for v in plan.shared.values()])], dtype=torch.int64)
        if dist.get_backend(group) == "nccl":
            ms = ms.to(dev)
        dist.all_reduce(ms, op=dist.ReduceOp.MAX, group=group)
        if plan.n_ranks > PEER_MAX + 1:
            raise ValueError(f"at most {PEER_MAX + 1} ranks")
        self.rank = DD2Rank(plan.rank, plan.n_ranks, A, dinv, plan.own, plan.shared, dm.node_order(), fixed=fixed,
                            max_shared=int(ms.item()))
        self.solver = DD2Solver.connect(self.rank, group)
        self.b = b

    @property
    def x(self) -> torch.Tensor:
        return self.rank.x_node

    def solve(self, b: torch.Tensor, maxit: int, tol: float = 0.0):
        assert b.data_ptr() == self.b.data_ptr(), "the fused solver is bound to its right-hand side buffer"
        xs, it = self.solver.solve([b], maxit, tol, zero_b=True)
        return xs[0], it

    def check(self):
        self.solver.check()

"""Decomposed pressure solve fused with its interface exchange (ab_cg_dd).

Each rank (subdomain of the element-disjoint decomposition, decompose.py)
solves its part of the global system in ONE cooperative kernel per solve: the
interface rows' partial products go straight into the neighbours' receive
arrays (peer memory), and both CG reductions are completed across ranks
inside the kernel (include/alyab200.h "K5 across ranks").

Two ways to host the ranks:

* :func:`virtual_ranks` - several ranks in one process on one GPU, one CTA
  group per rank in a single cooperative launch; the peer pointers are plain
  device pointers.  This runs the exchange protocol end to end on one GPU
  (tests/test_gpu_ddcg.py).
* :func:`ipc_ranks` - one rank per process/GPU (torch.distributed): the
  receive/counter/record buffers are exported with CUDA IPC handles and
  mapped by every peer (NVLink over NVSwitch).

Setup is host code (numpy/torch); the solve launches a single kernel.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from ._lib import call, ptr, stream_handle, vp, i32, i64
from .solver import SellMatrix, cg_local_map, permute_matrix

MAX_PEERS = 8


class AbCgDdRank(C.Structure):
    _fields_ = ([("n_rows", i64), ("rows_per_cta", i64), ("cta0", i32), ("n_cta", i32), ("max_ghost", i32),
                 ("rank", i32), ("n_ranks", i32), ("pad0_", i32)]
                + [(nm, vp) for nm in ("slice_ptr", "cols", "vals", "ghost_ptr", "ghost", "perm", "dinv", "fixed",
                                      "own", "b_in", "b_zero", "x_out", "zg", "red", "sc", "part", "bar",
                                      "ifmask", "send_ptr", "send_peer", "send_off", "rrow_ptr", "rrow", "recv_ptr",
                                      "recv_off", "recv", "cnt_in", "red_in", "evbase")]
                + [("n_peers", i32), ("recv_stride", i32), ("peer_rank", i32 * MAX_PEERS), ("peer_ncta", i32 * MAX_PEERS),
                   ("peer_recv", vp * MAX_PEERS), ("peer_cnt", vp * MAX_PEERS), ("peer_red", vp * MAX_PEERS)])


def rows_per_cta(n_rows: int, n_cta: int) -> int:
    return ((n_rows + n_cta - 1) // n_cta + 31) // 32 * 32


class DDRank:
    """One rank's part of the decomposed solve.

    A: the rank's assembled Laplacian (local node numbering, Dirichlet rows
    identity); dinv: 1 / diagonal of the GLOBAL operator at the local nodes;
    own: ownership weights (1 on the lowest sharing rank); shared: neighbour
    rank -> local node ids shared with it, ascending global id (both sides
    list the same nodes in the same order); order: solver-row -> local node
    (an SFC order); n_cta: CTAs working on this rank."""

    def __init__(self, rank: int, n_ranks: int, A: SellMatrix, dinv: torch.Tensor, own, shared: dict,
                 order: torch.Tensor, n_cta: int, fixed: torch.Tensor | None = None, max_shared: int | None = None):
        dev = A.vals.device
        n = A.n_rows
        self.rank, self.n_ranks, self.n, self.n_cta = rank, n_ranks, n, n_cta
        self.rb = rows_per_cta(n, n_cta)
        if (n + self.rb - 1) // self.rb != n_cta:
            self.n_cta = n_cta = (n + self.rb - 1) // self.rb
        perm = order.to(device=dev, dtype=torch.int32).contiguous()
        self.perm = perm
        pl = perm.to(torch.int64)
        iperm = torch.empty_like(pl)
        iperm[pl] = torch.arange(n, device=dev)
        self.A = permute_matrix(A, perm)
        m = cg_local_map(self.A, self.rb, n_cta)
        if m is None:
            raise ValueError("rows + ghosts of a CTA exceed 16-bit local columns")
        self.map = m
        self.dinv = dinv.to(dev)[pl].contiguous()
        self.fixed = fixed.to(device=dev, dtype=torch.uint8)[pl].contiguous() if fixed is not None else None
        self.own = torch.as_tensor(own, dtype=torch.float64, device=dev)[pl].contiguous()
        # ---- interface, in solver-row order
        self.neighbors = sorted(int(q) for q in shared)
        if len(self.neighbors) > MAX_PEERS:
            raise ValueError(f"at most {MAX_PEERS} neighbours")
        rows = {q: iperm[torch.as_tensor(np.asarray(shared[q]), device=dev).to(torch.int64)] for q in self.neighbors}
        self.n_shared = {q: int(rows[q].numel()) for q in self.neighbors}
        self.M = int(max_shared if max_shared is not None else max([0] + list(self.n_shared.values())))
        # peers = every other rank (the reductions); neighbours receive halo data
        self.peers = [q for q in range(n_ranks) if q != rank]
        pidx = {q: k for k, q in enumerate(self.peers)}
        srow, speer, soff, roff = [], [], [], []
        for q in self.neighbors:
            k = torch.arange(self.n_shared[q], device=dev, dtype=torch.int64)
            srow.append(rows[q])
            speer.append(torch.full_like(k, pidx[q]))
            soff.append(rank * self.M + k)      # slot in q's recv array for data from this rank
            roff.append(q * self.M + k)         # slot in this rank's recv array for data from q
        if srow:
            srow_t = torch.cat(srow)
            # entries sorted by (row, peer rank): deterministic add order on the receiving side
            key = srow_t * (n_ranks + 1) + torch.cat([torch.full((self.n_shared[q],), q, device=dev,
                                                                  dtype=torch.int64) for q in self.neighbors])
            o = torch.sort(key).indices
            srow_t, speer_t, soff_t, roff_t = srow_t[o], torch.cat(speer)[o], torch.cat(soff)[o], torch.cat(roff)[o]
        else:
            srow_t = speer_t = soff_t = roff_t = torch.zeros(0, dtype=torch.int64, device=dev)
        cnt = torch.bincount(srow_t, minlength=n)
        self.send_ptr = torch.zeros(n + 1, dtype=torch.int32, device=dev)
        self.send_ptr[1:] = torch.cumsum(cnt, 0).to(torch.int32)
        self.send_peer = speer_t.to(torch.int32).contiguous()
        self.send_off = soff_t.to(torch.int32).contiguous()
        self.rrow = torch.unique(srow_t).to(torch.int32).contiguous()
        rc = cnt[self.rrow.to(torch.int64)] if self.rrow.numel() else torch.zeros(0, dtype=torch.int64, device=dev)
        self.recv_ptr = torch.zeros(self.rrow.numel() + 1, dtype=torch.int32, device=dev)
        if self.rrow.numel():
            self.recv_ptr[1:] = torch.cumsum(rc, 0).to(torch.int32)
        self.recv_off = roff_t.to(torch.int32).contiguous()
        bounds = torch.arange(n_cta + 1, device=dev, dtype=torch.int64) * self.rb
        self.rrow_ptr = torch.searchsorted(self.rrow.to(torch.int64), bounds).to(torch.int32).contiguous()
        nwords = (n_cta * self.rb) // 32
        bits = torch.zeros(nwords * 32, dtype=torch.int64, device=dev)
        if self.rrow.numel():
            bits[self.rrow.to(torch.int64)] = 1
        w = (bits.view(nwords, 32) << torch.arange(32, device=dev, dtype=torch.int64)).sum(1)
        self.ifmask = (w - (w >= 2 ** 31).to(torch.int64) * 2 ** 32).to(torch.int32).contiguous()
        # ---- buffers (peers write recv, cnt_in, red_in)
        z = lambda k, dt=torch.float64: torch.zeros(k, dtype=dt, device=dev)  # noqa: E731
        self.recv = z(max(1, n_ranks * self.M))
        self.cnt_in = z(n_ranks, torch.int64)
        self.red_in = z(3 * n_ranks * 4)
        self.evbase = z(2, torch.int64)
        self.part = z(6 * n_cta + 8)
        self.bar = z(2, torch.int32)
        self.red = z(8)
        self.sc = z(8)
        self.zg = z(n)
        self.x = z(n)
        self.peer_recv, self.peer_cnt, self.peer_red = {}, {}, {}

    # addresses of the buffers the peers write into (same device or IPC-mapped)
    def exports(self) -> dict:
        return {"recv": ptr(self.recv), "cnt_in": ptr(self.cnt_in), "red_in": ptr(self.red_in),
                "n_cta": self.n_cta}

    def connect(self, q: int, recv_ptr: int, cnt_in_ptr: int, red_in_ptr: int, n_cta: int):
        self.peer_recv[q] = recv_ptr
        self.peer_cnt[q] = cnt_in_ptr + 8 * self.rank   # &peer.cnt_in[my rank]
        self.peer_red[q] = red_in_ptr
        self.peer_ncta_ = getattr(self, "peer_ncta_", {})
        self.peer_ncta_[q] = n_cta

    def struct(self, cta0: int, b_in: torch.Tensor, b_zero: torch.Tensor | None) -> AbCgDdRank:
        s = AbCgDdRank()
        s.n_rows, s.rows_per_cta, s.cta0, s.n_cta = self.n, self.rb, cta0, self.n_cta
        s.max_ghost, s.rank, s.n_ranks = self.map["max_ghost"], self.rank, self.n_ranks
        s.slice_ptr, s.cols, s.vals = ptr(self.A.slice_ptr), ptr(self.map["cols"]), ptr(self.A.vals)
        s.ghost_ptr, s.ghost, s.perm = ptr(self.map["ghost_ptr"]), ptr(self.map["ghost"]), ptr(self.perm)
        s.dinv, s.fixed, s.own = ptr(self.dinv), ptr(self.fixed), ptr(self.own)
        s.b_in, s.b_zero, s.x_out, s.zg = ptr(b_in), ptr(b_zero), ptr(self.x), ptr(self.zg)
        s.red, s.sc, s.part, s.bar = ptr(self.red), ptr(self.sc), ptr(self.part), ptr(self.bar)
        s.ifmask, s.send_ptr, s.send_peer, s.send_off = (ptr(self.ifmask), ptr(self.send_ptr), ptr(self.send_peer),
                                                         ptr(self.send_off))
        s.rrow_ptr, s.rrow, s.recv_ptr, s.recv_off = (ptr(self.rrow_ptr), ptr(self.rrow), ptr(self.recv_ptr),
                                                      ptr(self.recv_off))
        s.recv, s.cnt_in, s.red_in, s.evbase = ptr(self.recv), ptr(self.cnt_in), ptr(self.red_in), ptr(self.evbase)
        s.pad0_ = 1 if getattr(self, "same_device", False) else 0
        s.n_peers = len(self.peers)
        s.recv_stride = max(1, self.M)
        for k, q in enumerate(self.peers):
            s.peer_rank[k] = q
            s.peer_ncta[k] = self.peer_ncta_[q]
            s.peer_recv[k] = self.peer_recv[q]
            s.peer_cnt[k] = self.peer_cnt[q]
            s.peer_red[k] = self.peer_red[q]
        return s

    def fits(self) -> bool:
        """Shared memory of ab_cg_dd for this rank (z + ghosts + tables)."""
        dev = self.A.vals.device
        optin = getattr(torch.cuda.get_device_properties(dev), "shared_memory_per_block_optin", 232448)
        rb, mg = self.rb, self.map["max_ghost"]
        need = (4 * rb + mg) * 8 + 2 * (rb // 32 + 1) * 8 + mg * 4 + 16
        return need + 1024 <= optin and rb <= 8192

    @property
    def iterations(self) -> int:
        return int(self.red[3].item())

    def residual(self) -> float:
        rr, bb = float(self.red[1].item()), float(self.sc[1].item())
        return float(np.sqrt(rr / bb)) if bb > 0 else 0.0


class DDSolve:
    """A cooperative launch hosting ``ranks`` (CTA groups); b[k] / x of rank k
    in its local node order."""

    def __init__(self, ranks: list, bs: list, zero_b: bool = True):
        self.ranks = ranks
        cta0 = 0
        structs = []
        for r, b in zip(ranks, bs):
            structs.append(r.struct(cta0, b, b if zero_b else None))
            cta0 += r.n_cta
        self.n_cta = cta0
        raw = b"".join(bytes(s) for s in structs)
        dev = ranks[0].A.vals.device
        self.dev_structs = torch.frombuffer(bytearray(raw), dtype=torch.uint8).to(dev)
        self.max_rb = max(r.rb for r in ranks)
        self.max_ghost = max(r.map["max_ghost"] for r in ranks)

    def run(self, maxit: int, tol: float = 0.0):
        for r in self.ranks:
            r.bar.zero_()
        call("ab_cg_dd", ptr(self.dev_structs), len(self.ranks), self.n_cta, int(maxit), float(tol), self.max_rb,
             self.max_ghost, stream_handle())


class FusedDDSolver:
    """The decomposed pressure solve of one rank of a multi-GPU run (one
    process per GPU): ab_cg_dd with peer buffers mapped through CUDA IPC.
    ``solve(b, maxit, tol)`` mirrors PCG.solve; b is interface-summed."""

    def __init__(self, dm, A: SellMatrix, dinv: torch.Tensor, fixed, plan, b: torch.Tensor, group=None):
        import torch.distributed as dist
        dev = dinv.device
        n_ranks = plan.n_ranks

        def all_ok(ok: bool, what: str):  # collective: every rank takes the same branch
            t = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
            if int(t.item()) == 0:
                raise RuntimeError(f"fused decomposed CG: {what} failed on some rank")

        ms = torch.tensor([max([0] + [len(v) for v in plan.shared.values()])], dtype=torch.int64, device=dev)
        dist.all_reduce(ms, op=dist.ReduceOp.MAX, group=group)
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        try:
            self.rank = DDRank(plan.rank, n_ranks, A, dinv, plan.own, plan.shared, dm.node_order(), sms,
                               fixed=fixed, max_shared=int(ms.item()))
            ok = self.rank.fits()
        except Exception:
            ok = False
        all_ok(ok, "setup")
        try:
            ipc_ranks(self.rank, group)
            ok = True
        except Exception:
            ok = False
        all_ok(ok, "peer mapping (CUDA IPC)")
        self.launch = DDSolve([self.rank], [b], zero_b=True)
        self.b = b

    @property
    def x(self) -> torch.Tensor:
        return self.rank.x

    def solve(self, b: torch.Tensor, maxit: int, tol: float = 0.0):
        """With tol > 0 the iteration count is read back (host sync) and a
        failed solve raises at once; with tol == 0 nothing synchronises and a
        failure stays recorded in the sticky device flag (see check())."""
        assert b.data_ptr() == self.b.data_ptr(), "the fused solver is bound to its right-hand side buffer"
        self.launch.run(maxit, tol)
        if tol > 0:
            it = self.rank.iterations
            if it < 0:
                self.check()
            return self.rank.x, it
        return self.rank.x, maxit

    def check(self):
        """Raise if any solve since the last check timed out waiting for a
        peer (red[AB_RED_FAIL], set by the kernel).  The iterate of such a
        solve is meaningless, and the cross-rank counters are out of step, so
        the fused solver cannot be used again."""
        if float(self.rank.red[5].item()) != 0.0:
            raise RuntimeError("fused decomposed CG: a peer wait timed out (ranks out of step); "
                               "the pressure increment of that step is invalid")


def virtual_ranks(ranks: list):
    """Wire ranks hosted by one process on one GPU (peer pointers = device
    pointers of the other ranks' buffers)."""
    ex = [r.exports() for r in ranks]
    for r in ranks:
        r.same_device = True
        for q in r.peers:
            r.connect(q, ex[q]["recv"], ex[q]["cnt_in"], ex[q]["red_in"], ex[q]["n_cta"])
    return ranks


def ipc_ranks(rank: DDRank, group=None):
    """Wire one rank per process/GPU through CUDA IPC handles exchanged with
    torch.distributed (every rank maps every peer's recv / cnt_in / red_in)."""
    import torch.distributed as dist

    def handle(t):
        h = (C.c_ubyte * 64)()
        off = C.c_int64(0)
        call("ab_ipc_get_handle", ptr(t), h, C.byref(off))
        return bytes(h), off.value

    try:
        mine = {"recv": handle(rank.recv), "cnt_in": handle(rank.cnt_in), "red_in": handle(rank.red_in),
                "n_cta": rank.n_cta}
    except Exception as e:  # still take part in the exchange, then fail
        mine = {"error": str(e)}
    allx = [None] * rank.n_ranks
    dist.all_gather_object(allx, mine, group=group)
    bad = [q for q, x in enumerate(allx) if "error" in x]
    if bad:
        raise RuntimeError(f"CUDA IPC export failed on ranks {bad}")
    rank._ipc = []
    for q in rank.peers:
        ptrs = {}
        for key in ("recv", "cnt_in", "red_in"):
            h, off = allx[q][key]
            p = C.c_void_p()
            call("ab_ipc_open_handle", (C.c_ubyte * 64).from_buffer_copy(h), C.byref(p))
            ptrs[key] = p.value + off
            rank._ipc.append(p.value)
        rank.connect(q, ptrs["recv"], ptrs["cnt_in"], ptrs["red_in"], allx[q]["n_cta"])
    return rank

"""Interface-node exchange over NCCL.

One process per GPU (torch.distributed, backend "nccl" over NVLink /
NVSwitch).  ``sum_`` adds to every duplicated interface node the partial
values its neighbours assembled:

    pack (ab_halo_pack)  ->  grouped send/recv with each neighbour
    (dist.batch_isend_irecv = one ncclGroupStart/End)  ->  unpack-add
    (ab_halo_unpack_add)

and ``allreduce_`` sums the CG reduction slots (ncclAllReduce, fp64).  The
pack/unpack callables are injectable so the exchange protocol itself is
covered by world-size-2 gloo tests on CPU (tests/test_halo_gloo.py); on a
GPU they are always the CUDA kernels — there is no host fallback.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from ._lib import call, ptr, stream_handle
from .decompose import InterfacePlan


def cuda_pack(idx: torch.Tensor, field: torch.Tensor, stride: int, ncomp: int, out: torch.Tensor):
    call("ab_halo_pack", idx.numel(), ptr(idx), ptr(field), stride, ncomp, ptr(out), stream_handle())


def cuda_unpack_add(idx: torch.Tensor, buf: torch.Tensor, stride: int, ncomp: int, field: torch.Tensor):
    call("ab_halo_unpack_add", idx.numel(), ptr(idx), ptr(buf), stride, ncomp, ptr(field), stream_handle())


class HaloExchanger:
    def __init__(self, plan: InterfacePlan, device, group=None, pack=None, unpack=None, max_ncomp: int = 3):
        self.plan = plan
        self.group = group
        self.device = torch.device(device)
        self.neighbors = list(plan.neighbors)
        self.idx = {q: torch.from_numpy(plan.shared[q]).to(self.device) for q in self.neighbors}
        n = sum(int(v.numel()) for v in self.idx.values())
        self.send = torch.zeros(max(1, n * max_ncomp), dtype=torch.float64, device=self.device)
        self.recv = torch.zeros_like(self.send)
        self.pack = pack or cuda_pack
        self.unpack = unpack or cuda_unpack_add
        self.own = torch.from_numpy(plan.own).to(self.device) if plan.own is not None else None
        self.bytes_per_sum = {c: 8 * n * c for c in (1, 3)}

    def _global(self, q: int) -> int:
        return q if self.group is None else dist.get_global_rank(self.group, q)

    def _host_staged(self, t: torch.Tensor) -> bool:
        # gloo cannot move CUDA tensors point to point: stage through the host
        # (used to run several ranks on one GPU in tests; NCCL moves device
        # buffers directly)
        return t.is_cuda and dist.get_backend(self.group) == "gloo"

    def sum_(self, field: torch.Tensor, ncomp: int, stride: int):
        """field[shared] += neighbours' values at the shared nodes."""
        if not self.neighbors:
            return
        off = 0
        views = []
        for q in self.neighbors:
            m = self.idx[q].numel() * ncomp
            s = self.send[off:off + m]
            self.pack(self.idx[q], field, stride, ncomp, s)
            views.append((q, s, self.recv[off:off + m]))
            off += m
        staged = self._host_staged(self.send)
        if staged:
            torch.cuda.current_stream().synchronize()
            views = [(q, s.cpu(), r.cpu(), r) for q, s, r in views]
        else:
            views = [(q, s, r, r) for q, s, r in views]
        ops = []
        for q, s, r, _dev in views:
            ops.append(dist.P2POp(dist.isend, s, self._global(q), group=self.group))
            ops.append(dist.P2POp(dist.irecv, r, self._global(q), group=self.group))
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        for q, _s, r, dev in views:
            if staged:
                dev.copy_(r)
            self.unpack(self.idx[q], dev, stride, ncomp, field)

    def allreduce_(self, t: torch.Tensor):
        if self._host_staged(t):
            h = t.cpu()
            dist.all_reduce(h, op=dist.ReduceOp.SUM, group=self.group)
            t.copy_(h)
        else:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)

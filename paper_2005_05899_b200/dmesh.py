"""Per-rank generation and decomposition of the structured boundary-layer
box (C3/C4/C5) — every rank builds only its own subdomain.

The global path (decompose.py) needs the whole mesh on every rank plus a
global ``np.unique`` over all element-node incidences to find the interface
(~1e9 keys and ~20 GB of host memory per rank at C4).  The paper's model is
that each MPI process owns its element set, and the
reference's partitioner contract is chunk-invariant SFC splitting of weighted
bins (sfc.py:258-307, :326-374).  Here the bins are the structured cells:

1. every cell of the nx x ny x nz box gets its Hilbert key (integer cell
   coordinates, level ceil(log2(max(nx, ny, nz))), so no two cells share a
   key) and its Gauss-point weight (the elements it produces: hex 8, two
   prisms 12, pyramid + 4 tets 21, 6 Kuhn tets 24 - the DD weights of
   mesh.py:66-71);
2. the cells, sorted by key, are split by the reference's closest-boundary
   rule (``partition.split_cuts`` = split_1d's cut rule, optionally with
   throughput coefficients lambda - the DLB analog);
3. a rank generates the elements of its own cells only
   (``meshgen.boundary_layer_blocks``: identical elements, node ids, element
   ids and order as the global generator restricted to those cells);
4. the interface is local: a grid node's sharers are the owners of its (up to
   8) adjacent cells, read from the per-cell owner array, so no rank ever
   touches another rank's elements.

Per-rank host memory is O(cells) bytes for the owner array (44M bytes at C4)
plus the rank's own subdomain.  All steps are array code (torch on the
partition's device, numpy for the element blocks); the Hilbert keys come from
the ``ab_hilbert_cells`` kernel, or from an injected function (the CPU tests
pass the oracle's restatement).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import meshgen
from .decompose import InterfacePlan
from .meshgen import MeshArrays


@dataclass(frozen=True)
class BoxSpec:
    """The boundary-layer box of meshgen.boundary_layer_mesh."""
    nx: int
    ny: int
    nz: int
    layers: int
    hex_fraction: float = 0.25
    lengths: tuple = (1.0, 1.0, 1.0)

    @property
    def n_cells(self) -> int:
        return self.nx * self.ny * self.nz

    @property
    def n_nodes(self) -> int:
        return (self.nx + 1) * (self.ny + 1) * (self.nz + 1)

    @property
    def patch(self) -> tuple:
        return meshgen.patch_extent(self.nx, self.ny, self.hex_fraction)

    def cell_ijk(self, cid):
        k = cid % self.nz
        j = (cid // self.nz) % self.ny
        i = cid // (self.nz * self.ny)
        return i, j, k

    def codes(self, cid):
        i, j, k = self.cell_ijk(cid)
        px, py = self.patch
        return meshgen.cell_codes(i, j, k, self.layers, px, py)

    def global_mesh(self) -> MeshArrays:
        return meshgen.boundary_layer_mesh(self.nx, self.ny, self.nz, self.layers, self.hex_fraction, self.lengths)

    def bounds(self):
        return np.zeros(3), np.asarray(self.lengths, dtype=np.float64)


def c3_spec(scale: float = 1.0) -> BoxSpec:
    nx = max(2, int(round(150 * scale)))
    nz = max(4, int(round(245 * scale)))
    return BoxSpec(nx, nx, nz, max(1, int(round(30 * scale))))


def c4_spec() -> BoxSpec:
    """BASELINE configs[3]: 300 x 300 x 490 cells, 40 prism layers (~249M elements)."""
    return BoxSpec(300, 300, 490, 40)


def c5_spec(n_ranks: int) -> BoxSpec:
    """BASELINE configs[4] weak scaling: 150 x 150 x (237 P + 21) cells, 30
    prism layers -> ~32M elements per rank."""
    return BoxSpec(150, 150, 237 * n_ranks + 21, 30)


def _level(spec: BoxSpec) -> int:
    m = max(spec.nx, spec.ny, spec.nz)
    return max(1, int(np.ceil(np.log2(m))))


def cuda_cell_keys(cells: torch.Tensor, level: int) -> torch.Tensor:
    from ._lib import call, ptr, stream_handle
    keys = torch.empty(cells.shape[0], dtype=torch.int64, device=cells.device)
    call("ab_hilbert_cells", cells.shape[0], ptr(cells.contiguous()), level, ptr(keys), stream_handle())
    return keys


@dataclass
class CellPartition:
    """Owner (0-based rank) of every cell plus the split's cut positions in
    the sorted cell sequence and the subdomain weights (sum of Gauss points)."""
    n_parts: int
    owner: torch.Tensor         # int8 [n_cells], indexed by cell id
    cuts: np.ndarray            # (P-1,) last sorted position of parts 0..P-2
    weights: np.ndarray         # (P,) subdomain weights


def partition_cells(spec: BoxSpec, n_parts: int, coeffs=None, device="cuda", keys_fn=None,
                    chunk: int = 1 << 24) -> CellPartition:
    """SFC split of the cells (deterministic: every rank computes the same)."""
    from .partition import split_cuts
    if n_parts > 127:
        raise ValueError("at most 127 parts")
    dev = torch.device(device)
    if n_parts == 1:  # one subdomain: no curve needed
        w_all = meshgen.CELL_GAUSS[np.asarray(spec.codes(np.arange(spec.n_cells, dtype=np.int64)))]
        return CellPartition(n_parts=1, owner=torch.zeros(spec.n_cells, dtype=torch.int8, device=dev),
                             cuts=np.zeros(0, np.int64), weights=np.array([float(w_all.sum())]))
    keys_fn = keys_fn or cuda_cell_keys
    L = _level(spec)
    nc = spec.n_cells
    keys = torch.empty(nc, dtype=torch.int64, device=dev)
    for c0 in range(0, nc, chunk):
        cid = torch.arange(c0, min(nc, c0 + chunk), dtype=torch.int64, device=dev)
        i, j, k = spec.cell_ijk(cid)
        keys[c0:c0 + cid.numel()] = keys_fn(torch.stack([i, j, k], dim=1).contiguous(), L)
        del cid, i, j, k
    order = torch.sort(keys).indices  # keys are unique: the order is deterministic
    del keys
    code = torch.from_numpy(np.asarray(spec.codes(order.cpu().numpy()), dtype=np.int64))
    w = meshgen.CELL_GAUSS[code.numpy()].astype(np.float64)
    cuts, sub = split_cuts(w, n_parts, coeffs)
    part_sorted = torch.zeros(nc, dtype=torch.int8, device=dev)
    for c in cuts:
        part_sorted[int(c) + 1:] += 1
    owner = torch.empty(nc, dtype=torch.int8, device=dev)
    owner[order] = part_sorted
    return CellPartition(n_parts=n_parts, owner=owner, cuts=cuts, weights=sub)


def local_mesh(spec: BoxSpec, part: CellPartition, rank: int):
    """(submesh with local node numbering, InterfacePlan) of 0-based ``rank``.

    The submesh equals ``decompose.submesh(global mesh, parts, rank + 1)``
    (same elements, element ids, order, coordinates and l2g) and the plan
    equals ``decompose.interface_plan`` of the global mesh, without either
    being built."""
    owner = part.owner
    P = part.n_parts
    mine = torch.nonzero(owner == rank).squeeze(1).cpu().numpy()   # ascending cell id
    i, j, k = spec.cell_ijk(mine)
    px, py = spec.patch
    blocks = meshgen.boundary_layer_blocks(spec.nx, spec.ny, spec.nz, spec.layers, px, py, i, j, k)
    # global element ids: per kind, count the cells of each type before each of mine
    code_all = None
    ids = {}
    if blocks:
        cid_all = np.arange(spec.n_cells, dtype=np.int64)
        code_all = np.asarray(spec.codes(cid_all))
        del cid_all
        n_type = {c: int((code_all == c).sum()) for c in range(4)}
        my_code = code_all[mine]
        # kind order hex < pri < pyr < tet; tets: transition tets first
        start = {"hex": 0}
        start["pri"] = n_type[meshgen.CELL_HEX] * 1
        start["pyr"] = start["pri"] + n_type[meshgen.CELL_PRI] * 2
        start["tet"] = start["pyr"] + n_type[meshgen.CELL_TRANS] * 1
        n_trans_tets = n_type[meshgen.CELL_TRANS] * 4

        def before(c):  # number of type-c cells with smaller cell id, for my type-c cells
            csum = np.cumsum(code_all == c) - (code_all == c)
            return csum[mine[my_code == c]]

        per = {"hex": (meshgen.CELL_HEX, 1), "pri": (meshgen.CELL_PRI, 2), "pyr": (meshgen.CELL_TRANS, 1)}
        for tag, (c, ne) in per.items():
            if tag in blocks:
                b = before(c)
                ids[tag] = (start[tag] + b[:, None] * ne + np.arange(ne)[None, :]).reshape(-1)
        if "tet" in blocks:
            parts_ = []
            if (my_code == meshgen.CELL_TRANS).any():
                b = before(meshgen.CELL_TRANS)
                parts_.append(start["tet"] + (b[:, None] * 4 + np.arange(4)[None, :]).reshape(-1))
            if (my_code == meshgen.CELL_KUHN).any():
                b = before(meshgen.CELL_KUHN)
                parts_.append(start["tet"] + n_trans_tets + (b[:, None] * 6 + np.arange(6)[None, :]).reshape(-1))
            ids["tet"] = np.concatenate(parts_)
        del code_all
    # local nodes = grid nodes touched by my elements, ascending global id
    # (a mark-and-compact over the grid instead of sorting E * n_k ids)
    used = np.zeros(spec.n_nodes, dtype=bool)
    for b in blocks.values():
        used[b.reshape(-1)] = True
    l2g = np.flatnonzero(used).astype(np.int64)
    del used
    g2l = np.full(spec.n_nodes, -1, dtype=np.int32)
    g2l[l2g] = np.arange(l2g.size, dtype=np.int32)
    # coordinates exactly as meshgen._grid_nodes
    nyz = (spec.ny + 1) * (spec.nz + 1)
    gi, gj, gk = l2g // nyz, (l2g // (spec.nz + 1)) % (spec.ny + 1), l2g % (spec.nz + 1)
    xs = np.linspace(0.0, spec.lengths[0], spec.nx + 1)
    ys = np.linspace(0.0, spec.lengths[1], spec.ny + 1)
    zs = np.linspace(0.0, spec.lengths[2], spec.nz + 1)
    sub = MeshArrays(coords=np.ascontiguousarray(np.stack([xs[gi], ys[gj], zs[gk]], axis=1)))
    for tag in meshgen.KIND_TAGS:
        if tag in blocks:
            rule = meshgen.DEFAULT_RULE[tag]
            sub.conn[rule] = np.ascontiguousarray(g2l[blocks[tag]])
            sub.elem_ids[rule] = np.asarray(ids[tag], dtype=np.int64)
            del blocks[tag]
    del g2l
    sub.shape = None
    if P == 1:
        plan = InterfacePlan(rank=0, n_ranks=1, l2g=l2g, own=np.ones(l2g.size))
    else:
        plan = interface_plan_local(spec, owner, rank, P, l2g)
    return sub, plan


def interface_plan_local(spec: BoxSpec, owner: torch.Tensor, rank: int, n_parts: int, l2g: np.ndarray,
                         chunk: int = 1 << 24) -> InterfacePlan:
    """Sharers of every local node from the owners of its adjacent cells:
    bit q of the node's mask is set when a cell of rank q touches it."""
    dev = owner.device
    g = torch.from_numpy(l2g).to(dev)
    nyz = (spec.ny + 1) * (spec.nz + 1)
    mask = torch.zeros(g.numel(), dtype=torch.int64, device=dev)
    for s0 in range(0, g.numel(), chunk):
        gg = g[s0:s0 + chunk]
        gi, gj, gk = gg // nyz, (gg // (spec.nz + 1)) % (spec.ny + 1), gg % (spec.nz + 1)
        m = torch.zeros(gg.numel(), dtype=torch.int64, device=dev)
        for di in (-1, 0):
            for dj in (-1, 0):
                for dk in (-1, 0):
                    ci, cj, ck = gi + di, gj + dj, gk + dk
                    ok = (ci >= 0) & (ci < spec.nx) & (cj >= 0) & (cj < spec.ny) & (ck >= 0) & (ck < spec.nz)
                    cid = (ci.clamp(0, spec.nx - 1) * spec.ny + cj.clamp(0, spec.ny - 1)) * spec.nz \
                        + ck.clamp(0, spec.nz - 1)
                    r = owner[cid].to(torch.int64)
                    m |= torch.where(ok, torch.ones_like(r) << r, torch.zeros_like(r))
        mask[s0:s0 + gg.numel()] = m
    # owner = lowest sharing rank
    low = (mask & -mask)
    own = (low == (1 << rank)).to(torch.float64)
    plan = InterfacePlan(rank=rank, n_ranks=n_parts, l2g=l2g.astype(np.int64), own=own.cpu().numpy())
    for q in range(n_parts):
        if q == rank:
            continue
        idx = torch.nonzero((mask >> q) & 1).squeeze(1)
        if idx.numel():
            plan.neighbors.append(q)
            plan.shared[q] = idx.to(torch.int32).cpu().numpy()
    return plan


def wall_model_bcs_local(sub: MeshArrays, spec: BoxSpec):
    """meshgen.wall_model_bcs with the GLOBAL box bounds (a subdomain's own
    coordinate extent is not the box's)."""
    return meshgen.wall_model_bcs(sub, bounds=spec.bounds())

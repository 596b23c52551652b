"""Packed element assembly — drop-in for reference pkg/src/coexbal/assembly.py.

Same public names, dataclasses, signatures and exceptions:
``Category``/``Pack``/``PackSet`` (assembly.py:149-175), ``build_packs``
(:178-221), ``assemble_packs`` (:227-244), ``assemble_reference``
(:247-263), ``CooMatrix``/``scatter_global`` (:294-333), ``SweepRow``/
``sweep_pack_size``/``sweep_csv`` (:341-380), plus ``lumped_mass``.

What changed (the B200 path):
* the element kernel is K1 (``ab_mass``): one thread per element, one CTA
  per pack (the reference's pack becomes the CTA tile), |det J| computed
  in-kernel instead of being precomputed on the host;
* ``scatter_global`` builds the global COO on the GPU: a stable sort of
  (row, col) keys generated in ascending element id, then the ordered
  segmented sum ``ab_segment_sum`` — the same accumulation order as the
  reference's dict, so values match bit for bit given equal element matrices;
* ``sweep_pack_size`` times the device kernel with CUDA events (build
  excluded, one warm-up, median), sweeping the CTA tile.

``assemble_reference`` keeps its meaning — the classical element-by-element
loop — as the same kernel launched with one element per CTA.
"""

from __future__ import annotations

import ctypes
import statistics
from dataclasses import dataclass

import numpy as np
import torch

from ._lib import call, ptr, stream_handle
from .device import DeviceMesh
from .elements import RULES, shape_values
from .mesh import ElementKind, FullMesh, to_arrays
from .meshgen import MeshArrays, NODE_COUNT, RULE_KIND


@dataclass(frozen=True)
class Category:
    kind: ElementKind
    rule: str
    nnode: int
    ngaus: int


@dataclass(frozen=True)
class Pack:
    category: Category
    pack_size: int
    element_ids: np.ndarray   # (valid_count,) positions in the full mesh
    valid_count: int
    jacobian: np.ndarray      # (pack_size, ngaus), zero in padded lanes
    weights: np.ndarray       # (ngaus,)
    shape: np.ndarray         # (nnode, ngaus)


class PackSet:
    """Packs of one mesh.  The device mesh and per-category |det J| tables
    live on the GPU; ``packs`` materialises the reference's tuple of
    :class:`Pack` views on first access (small meshes / interop)."""

    def __init__(self, dm: DeviceMesh, pack_size: int, jdet: list):
        self.dm = dm
        self.pack_size = pack_size
        self._jdet = jdet
        self._packs = None

    @property
    def n_elements(self) -> int:
        return self.dm.n_elements

    @property
    def categories(self):
        out = []
        for rule in self.dm.rules:
            r = RULES[rule]
            out.append(Category(kind=r.kind, rule=rule, nnode=r.kind.node_count, ngaus=r.ngaus))
        return out

    @property
    def packs(self) -> tuple:
        if self._packs is None:
            packs = []
            for cat, ids, J in zip(self.categories, self.dm.ids, self._jdet):
                rule = RULES[cat.rule]
                ids_h = ids.cpu().numpy()
                J_h = J.cpu().numpy()
                nt = shape_values(rule)
                for s in range(0, ids_h.size, self.pack_size):
                    chunk = ids_h[s:s + self.pack_size]
                    jac = np.zeros((self.pack_size, rule.ngaus))
                    jac[:chunk.size] = J_h[s:s + chunk.size]
                    packs.append(Pack(category=cat, pack_size=self.pack_size, element_ids=chunk.astype(np.int64),
                                      valid_count=int(chunk.size), jacobian=jac, weights=rule.weights, shape=nt))
            self._packs = tuple(packs)
        return self._packs


def _device_mesh(full_mesh) -> DeviceMesh:
    arrays = full_mesh if isinstance(full_mesh, MeshArrays) else to_arrays(full_mesh)
    return DeviceMesh(arrays)


def build_packs(full_mesh, pack_size: int) -> PackSet:
    """Group by (kind, rule) in sorted order, ids ascending within a category
    (assembly.py:187-198); |det J| at the Gauss points computed by K1.

    Raises ValueError for pack_size < 1 and KeyError for unknown or
    mismatched rules, like the reference (assembly.py:185-193)."""
    if pack_size < 1:
        raise ValueError("pack_size must be >= 1")
    dm = _device_mesh(full_mesh)
    s = stream_handle()
    jdet = []
    for k, rule in enumerate(dm.rules):
        J = torch.zeros((dm.conn[k].shape[0], RULES[rule].ngaus), dtype=torch.float64, device=dm.device)
        call("ab_mass", ctypes.byref(dm.struct), k, None, ptr(J), None, 128, s)
        jdet.append(J)
    return PackSet(dm, pack_size, jdet)


def _tile(pack_size: int) -> int:
    return max(1, min(int(pack_size), 1024))


def assemble_packs_device(packs: PackSet, tile: int | None = None, ml: torch.Tensor | None = None):
    """Bulk variant: per-category device tensors Ae[E_k, n_k, n_k]."""
    dm = packs.dm
    s = stream_handle()
    out = []
    t = _tile(packs.pack_size if tile is None else tile)
    for k, rule in enumerate(dm.rules):
        nn = NODE_COUNT[RULE_KIND[rule]]
        ae = torch.empty((dm.conn[k].shape[0], nn, nn), dtype=torch.float64, device=dm.device)
        call("ab_mass", ctypes.byref(dm.struct), k, ptr(ae), None, ptr(ml), t, s)
        out.append(ae)
    return out


def _to_dict(dm: DeviceMesh, mats) -> dict:
    out = {}
    for ids, ae in zip(dm.ids, mats):
        ids_h = ids.cpu().numpy()
        ae_h = ae.cpu().numpy()
        for i, eid in enumerate(ids_h.tolist()):
            out[eid] = ae_h[i]
    return out


def assemble_packs(packs: PackSet) -> dict:
    """Mass matrices Ae[e,i,j] = sum_g J w N_i N_j for all elements (K1),
    keyed by element id (assembly.py:227-244).  Per-element results do not
    depend on the pack size: every lane runs the same Gauss loop."""
    return _to_dict(packs.dm, assemble_packs_device(packs))


def assemble_reference(full_mesh) -> dict:
    """Element-by-element assembly (one element per CTA), assembly.py:247-263."""
    ps = build_packs(full_mesh, 1)
    return _to_dict(ps.dm, assemble_packs_device(ps, tile=1))


@dataclass(frozen=True)
class CooMatrix:
    """Node-by-node sparse matrix in coordinate-list form (assembly.py:294-314)."""

    n_nodes: int
    rows: np.ndarray
    cols: np.ndarray
    values: np.ndarray

    def total(self) -> float:
        return float(self.values.sum())

    def row_sums(self) -> np.ndarray:
        sums = np.zeros(self.n_nodes)
        np.add.at(sums, self.rows, self.values)
        return sums

    def to_dense(self) -> np.ndarray:
        dense = np.zeros((self.n_nodes, self.n_nodes))
        np.add.at(dense, (self.rows, self.cols), self.values)
        return dense


def scatter_global(matrices: dict, full_mesh) -> CooMatrix:
    """Global COO accumulated in ascending element id, entries sorted by
    (row, col) (assembly.py:317-333), built on the GPU."""
    if isinstance(full_mesh, MeshArrays):
        full_mesh = _full_from_arrays(full_mesh)
    n = len(full_mesh.nodes)
    dev = torch.device("cuda")
    ids = sorted(matrices)
    if not ids:
        e = np.zeros(0, dtype=np.int64)
        return CooMatrix(n_nodes=n, rows=e, cols=e.copy(), values=np.zeros(0))
    rows, cols, vals = [], [], []
    for eid in ids:
        conn = np.asarray(full_mesh.elements[eid].conn, dtype=np.int64)
        m = np.asarray(matrices[eid], dtype=np.float64)
        rows.append(np.repeat(conn, conn.size))
        cols.append(np.tile(conn, conn.size))
        vals.append(m.reshape(-1))
    r = torch.from_numpy(np.concatenate(rows)).to(dev)
    c = torch.from_numpy(np.concatenate(cols)).to(dev)
    v = torch.from_numpy(np.concatenate(vals)).to(dev)
    key = r * n + c
    order = torch.sort(key, stable=True).indices
    ks = key[order]
    vs = v[order].contiguous()
    start = torch.ones_like(ks, dtype=torch.bool)
    start[1:] = ks[1:] != ks[:-1]
    starts = torch.nonzero(start).squeeze(1)
    seg = torch.cat([starts, torch.tensor([ks.numel()], device=dev)]).contiguous()
    out = torch.empty(starts.numel(), dtype=torch.float64, device=dev)
    call("ab_segment_sum", starts.numel(), ptr(seg), ptr(vs), ptr(out), stream_handle())
    uk = ks[starts]
    return CooMatrix(n_nodes=n, rows=(uk // n).cpu().numpy(), cols=(uk % n).cpu().numpy(),
                     values=out.cpu().numpy())


def _full_from_arrays(arrays):
    from .mesh import from_arrays
    return from_arrays(arrays)


def lumped_mass(mesh) -> np.ndarray:
    """M_L = row sums of the global mass matrix, fused into K1's scatter."""
    dm = mesh if isinstance(mesh, DeviceMesh) else _device_mesh(mesh)
    ml = torch.zeros(dm.n_nodes, dtype=torch.float64, device=dm.device)
    for k in range(len(dm.rules)):
        call("ab_mass", ctypes.byref(dm.struct), k, None, None, ptr(ml), 128, stream_handle())
    return ml.cpu().numpy()


@dataclass(frozen=True)
class SweepRow:
    pack_size: int
    median_seconds: float
    speedup: float


def sweep_pack_size(full_mesh, sizes, reps: int = 5) -> list:
    """Median K1 device time per pack size (CTA tile), normalised against
    pack size 1; build excluded, one warm-up (assembly.py:348-373)."""
    if reps < 3:
        raise ValueError("reps must be >= 3")
    sizes = sorted(set(int(s) for s in sizes) | {1})
    if any(s < 1 for s in sizes):
        raise ValueError("pack sizes must be >= 1")
    ps = build_packs(full_mesh, 1)
    dm = ps.dm
    ml = torch.zeros(dm.n_nodes, dtype=torch.float64, device=dm.device)
    outs = [torch.empty((c.shape[0], c.shape[1], c.shape[1]), dtype=torch.float64, device=dm.device) for c in dm.conn]
    med = {}
    for size in sizes:
        def launch():
            for k in range(len(dm.rules)):
                call("ab_mass", ctypes.byref(dm.struct), k, ptr(outs[k]), None, ptr(ml), _tile(size), stream_handle())
        launch()  # warm-up
        samples = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            launch()
            b.record()
            b.synchronize()
            samples.append(a.elapsed_time(b) / 1e3)
        med[size] = statistics.median(samples)
    base = med[1]
    return [SweepRow(s, med[s], base / med[s]) for s in sizes]


def sweep_csv(rows) -> str:
    lines = ["pack_size,median_seconds,speedup"]
    for r in rows:
        lines.append(f"{r.pack_size},{r.median_seconds!r},{r.speedup!r}")
    return "\n".join(lines) + "\n"

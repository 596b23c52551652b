"""Space-filling-curve domain decomposition — drop-in for reference
pkg/src/coexbal/sfc.py, array-native on the GPU.

Same names and semantics: ``SfcConfig`` (sfc.py:23-32), ``hilbert_key`` /
``hilbert_decode`` / ``hilbert_keys_batch`` (:45-148), ``Bin`` /
``BinSequence`` (:156-181), ``quantize_cells`` / ``project_to_bins``
(:184-221), ``Partition`` / ``split_1d`` (:229-307), ``partition_chunked``
(:326-374), ``store_partition`` / ``load_partition`` (:385-417).

The key computation (quantise + Hilbert transform) runs in one kernel
(``ab_hilbert_keys``) with the reference's exact float operation order, so
keys, bins, cuts and assignments are identical to the reference's on the
same input (tests/test_partition.py pins this on the reference's own
fixture mesh).  ``sfc_partition`` is the array-native entry point used by the
multi-GPU path: per-element subdomain ids without any per-element Python
objects.
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch

from ._lib import AbMesh, call, ptr, stream_handle
from .mesh import BoundingBox, Mesh, bounding_box_of_points

MAX_LEVEL = 20


@dataclass(frozen=True)
class SfcConfig:
    level: int = 8
    curve: str = "hilbert"

    def __post_init__(self):
        if not 1 <= self.level <= MAX_LEVEL:
            raise ValueError(f"level must be in [1, {MAX_LEVEL}], got {self.level}")
        if self.curve != "hilbert":
            raise ValueError(f"unsupported curve {self.curve!r}")


def _dev():
    if not torch.cuda.is_available():
        raise RuntimeError("the SFC partitioner runs on the GPU (there is no CPU fallback)")
    return torch.device("cuda")


# ---------------------------------------------------------------------------
# Hilbert curve (Skilling transpose form); scalar helpers are host integer
# code, the batch path is the CUDA kernel.
# ---------------------------------------------------------------------------

def hilbert_key(cell, level: int) -> int:
    side = 1 << level
    x = [int(c) for c in cell]
    if len(x) != 3:
        raise ValueError("cell must have 3 coordinates")
    for c in x:
        if not 0 <= c < side:
            raise ValueError(f"cell coordinate {c} outside [0, {side})")
    keys = hilbert_keys_batch(np.array([x], dtype=np.int64), level)
    return int(keys[0])


def hilbert_decode(key: int, level: int) -> tuple:
    """Inverse transform (transpose -> axes), host integer code."""
    if not 0 <= key < 1 << (3 * level):
        raise ValueError(f"key {key} outside [0, 2^{3 * level})")
    x = [0, 0, 0]
    bit = 3 * level - 1
    for j in range(level - 1, -1, -1):   # de-interleave, MSB first
        for i in range(3):
            x[i] |= ((key >> bit) & 1) << j
            bit -= 1
    top = 2 << (level - 1)
    t = x[2] >> 1                         # Gray decode
    x[2] ^= x[1]
    x[1] ^= x[0]
    x[0] ^= t
    q = 2
    while q != top:                       # undo excess work, low to high
        mask = q - 1
        for i in (2, 1, 0):
            if x[i] & q:
                x[0] ^= mask
            else:
                t = (x[0] ^ x[i]) & mask
                x[0] ^= t
                x[i] ^= t
        q <<= 1
    return tuple(x)


def hilbert_keys_batch(cells, level: int) -> np.ndarray:
    cells = np.asarray(cells, dtype=np.int64)
    side = 1 << level
    if cells.ndim != 2 or cells.shape[1] != 3:
        raise ValueError("cells must have shape (n, 3)")
    if (cells < 0).any() or (cells >= side).any():
        raise ValueError("cell coordinate outside grid")
    if not 1 <= level <= MAX_LEVEL:
        raise ValueError(f"level must be in [1, {MAX_LEVEL}]")
    dev = _dev()
    c = torch.from_numpy(np.ascontiguousarray(cells)).to(dev)
    keys = torch.empty(cells.shape[0], dtype=torch.int64, device=dev)
    call("ab_hilbert_cells", cells.shape[0], ptr(c), level, ptr(keys), stream_handle())
    return keys.cpu().numpy()


def keys_from_centroids(cent: torch.Tensor, box: BoundingBox, level: int) -> torch.Tensor:
    """Quantise centroids onto the 2^L grid of ``box`` and key them (GPU)."""
    dev = cent.device
    lo = torch.tensor(box.lo, dtype=torch.float64, device=dev)
    span = torch.tensor(np.array(box.hi) - np.array(box.lo), dtype=torch.float64, device=dev)
    keys = torch.empty(cent.shape[0], dtype=torch.int64, device=dev)
    c = cent.contiguous()
    call("ab_hilbert_keys", c.shape[0], ptr(c), ptr(lo), ptr(span), level, ptr(keys), stream_handle())
    return keys


# ---------------------------------------------------------------------------
# Binning
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Bin:
    key: int
    weight: float
    element_ids: tuple


@dataclass(frozen=True)
class BinSequence:
    """Sparse, key-sorted sequence of occupied grid cells."""

    keys: np.ndarray
    weights: np.ndarray
    element_ids: tuple
    total_weight: float

    @property
    def n_bins(self) -> int:
        return len(self.keys)

    def bin(self, i: int) -> Bin:
        return Bin(key=int(self.keys[i]), weight=float(self.weights[i]),
                   element_ids=tuple(int(e) for e in self.element_ids[i]))


def quantize_cells(mesh: Mesh, cfg: SfcConfig, box: BoundingBox | None = None) -> np.ndarray:
    box = box or mesh.bounding_box
    dev = _dev()
    side = 1 << cfg.level
    lo = torch.tensor(box.lo, dtype=torch.float64, device=dev)
    span = torch.tensor(np.array(box.hi) - np.array(box.lo), dtype=torch.float64, device=dev)
    rel = (torch.from_numpy(mesh.centroid_array()).to(dev) - lo) / span
    cells = torch.floor(rel * side).to(torch.int64)
    return torch.clamp(cells, 0, side - 1).cpu().numpy()


@dataclass
class BinsDevice:
    """Array-native bin sequence: bins sorted by key, elements sorted by
    (key, id); ``elem_bin`` maps every sorted element to its bin."""

    keys: torch.Tensor        # (m,) int64
    weights: torch.Tensor     # (m,) f64
    starts: torch.Tensor      # (m+1,) int64 offsets into the sorted elements
    ids_sorted: torch.Tensor  # (E,) int64


def group_bins_device(keys: torch.Tensor, ids: torch.Tensor, weights: torch.Tensor) -> BinsDevice:
    """lexsort((ids, keys)) then per-bin sums (sfc.py:206-221)."""
    o1 = torch.sort(ids, stable=True).indices
    o2 = torch.sort(keys[o1], stable=True).indices
    order = o1[o2]
    ks, ids_s, w_s = keys[order], ids[order], weights[order]
    start = torch.ones_like(ks, dtype=torch.bool)
    start[1:] = ks[1:] != ks[:-1]
    starts = torch.nonzero(start).squeeze(1)
    bounds = torch.cat([starts, torch.tensor([ks.numel()], device=ks.device)])
    # ordered per-bin sums (weights are Gauss counts -> exact; ordered anyway)
    seg = bounds.contiguous()
    wsum = torch.empty(starts.numel(), dtype=torch.float64, device=ks.device)
    w_c = w_s.to(torch.float64).contiguous()
    call("ab_segment_sum", starts.numel(), ptr(seg), ptr(w_c), ptr(wsum), stream_handle())
    return BinsDevice(keys=ks[starts], weights=wsum, starts=bounds, ids_sorted=ids_s)


def _to_sequence(b: BinsDevice) -> BinSequence:
    st = b.starts.cpu().numpy()
    ids = b.ids_sorted.cpu().numpy()
    w = b.weights.cpu().numpy()
    return BinSequence(keys=b.keys.cpu().numpy(), weights=w,
                       element_ids=tuple(ids[st[i]:st[i + 1]] for i in range(len(st) - 1)),
                       total_weight=float(np.sum(w)))


def project_to_bins(mesh: Mesh, cfg: SfcConfig) -> BinSequence:
    if mesh.n_elements == 0:
        raise ValueError("cannot bin an empty mesh")
    dev = _dev()
    cent = torch.from_numpy(mesh.centroid_array()).to(dev)
    keys = keys_from_centroids(cent, mesh.bounding_box, cfg.level)
    ids = torch.from_numpy(mesh.id_array()).to(dev)
    w = torch.from_numpy(mesh.weight_array()).to(dev)
    return _to_sequence(group_bins_device(keys, ids, w))


# ---------------------------------------------------------------------------
# 1D split
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Partition:
    n_parts: int
    cut_bins: np.ndarray
    assignment: dict
    subdomain_weights: np.ndarray

    def __eq__(self, other) -> bool:
        if not isinstance(other, Partition):
            return NotImplemented
        return (self.n_parts == other.n_parts and np.array_equal(self.cut_bins, other.cut_bins)
                and np.array_equal(self.subdomain_weights, other.subdomain_weights)
                and self.assignment == other.assignment)


def validate_coeffs(coeffs, n_parts: int) -> np.ndarray:
    lam = np.asarray(coeffs, dtype=np.float64)
    if lam.shape != (n_parts,):
        raise ValueError(f"expected {n_parts} coefficients, got shape {lam.shape}")
    if (lam <= 0).any():
        raise ValueError("all correction coefficients must be > 0")
    if abs(lam.sum() - n_parts) > 1e-9 * n_parts:
        raise ValueError(f"coefficients must sum to {n_parts}, got {lam.sum()!r}")
    return lam


def split_cuts(bin_weights: np.ndarray, n_parts: int, coeffs=None):
    """Cut positions and subdomain weights: cut i follows the boundary whose
    prefix weight is closest to the running target lambda-cumsum * W/P (ties
    to the earlier boundary), each part keeping >= 1 bin (sfc.py:258-307)."""
    if n_parts < 1:
        raise ValueError("n_parts must be >= 1")
    m = len(bin_weights)
    if n_parts > m:
        raise ValueError(f"insufficient granularity: {n_parts} parts requested but only {m} bins")
    lam = np.ones(n_parts) if coeffs is None else validate_coeffs(coeffs, n_parts)
    prefix = np.cumsum(bin_weights)
    total = prefix[-1]
    goals = np.cumsum(lam)[:-1] * (total / n_parts)
    cuts = np.empty(n_parts - 1, dtype=np.int64)
    prev = -1
    for i, goal in enumerate(goals, start=1):
        lo, hi = prev + 1, m - 1 - (n_parts - i)
        j = min(int(np.searchsorted(prefix, goal)), m - 1)
        if j > 0 and abs(prefix[j - 1] - goal) <= abs(prefix[j] - goal):
            j -= 1
        j = min(max(j, lo), hi)
        cuts[i - 1] = j
        prev = j
    bounds = np.concatenate([[-1], cuts, [m - 1]])
    sub = np.empty(n_parts)
    for s in range(n_parts):
        left = prefix[bounds[s]] if bounds[s] >= 0 else 0.0
        sub[s] = prefix[bounds[s + 1]] - left
    return cuts, sub


def split_1d(seq: BinSequence, n_parts: int, coeffs=None) -> Partition:
    cuts, sub = split_cuts(seq.weights, n_parts, coeffs)
    bounds = np.concatenate([[-1], cuts, [seq.n_bins - 1]])
    assignment: dict = {}
    for s in range(n_parts):
        for b in range(bounds[s] + 1, bounds[s + 1] + 1):
            for eid in seq.element_ids[b]:
                assignment[int(eid)] = s + 1
    return Partition(n_parts=n_parts, cut_bins=cuts, assignment=assignment, subdomain_weights=sub)


def partition_chunked(mesh: Mesh, cfg: SfcConfig, n_parts: int, coeffs=None, n_chunks: int = 1) -> Partition:
    """Key-range chunks binned independently and concatenated; since chunks
    are contiguous in key space the result is chunk-count invariant
    (sfc.py:326-374)."""
    if n_chunks < 1:
        raise ValueError("n_chunks must be >= 1")
    if mesh.n_elements == 0:
        raise ValueError("cannot partition an empty mesh")
    dev = _dev()
    cent = torch.from_numpy(mesh.centroid_array()).to(dev)
    keys = keys_from_centroids(cent, mesh.bounding_box, cfg.level)
    ids = torch.from_numpy(mesh.id_array()).to(dev)
    w = torch.from_numpy(mesh.weight_array()).to(dev)
    space = 1 << (3 * cfg.level)
    n_chunks = min(n_chunks, space)
    edges = [space * c // n_chunks for c in range(n_chunks + 1)]
    pieces = []
    for c in range(n_chunks):
        sel = (keys >= edges[c]) & (keys < edges[c + 1])
        if bool(sel.any()):
            pieces.append(_to_sequence(group_bins_device(keys[sel], ids[sel], w[sel])))
    merged = BinSequence(keys=np.concatenate([p.keys for p in pieces]),
                         weights=np.concatenate([p.weights for p in pieces]),
                         element_ids=tuple(e for p in pieces for e in p.element_ids),
                         total_weight=float(np.sum(np.concatenate([p.weights for p in pieces]))))
    return split_1d(merged, n_parts, coeffs)


def store_partition(part: Partition, path) -> None:
    lines = [f"part 1 {part.n_parts} {len(part.assignment)}"]
    for eid in sorted(part.assignment):
        lines.append(f"{eid} {part.assignment[eid]}")
    Path(path).write_text("\n".join(lines) + "\n", encoding="utf-8")
    side = {"cut_bins": [int(c) for c in part.cut_bins],
            "subdomain_weights": [float(w) for w in part.subdomain_weights]}
    Path(str(path) + ".json").write_text(json.dumps(side), encoding="utf-8")


def load_partition(path) -> Partition:
    lines = Path(path).read_text(encoding="utf-8").splitlines()
    head = lines[0].split()
    if len(head) != 4 or head[0] != "part" or head[1] != "1":
        raise ValueError(f"{path}:1: bad partition header {lines[0]!r}")
    n_parts, n_elem = int(head[2]), int(head[3])
    assignment = {}
    for ln in lines[1:]:
        if ln.strip():
            eid, sub = ln.split()
            assignment[int(eid)] = int(sub)
    if len(assignment) != n_elem:
        raise ValueError(f"{path}: expected {n_elem} assignments, got {len(assignment)}")
    side = json.loads(Path(str(path) + ".json").read_text(encoding="utf-8"))
    return Partition(n_parts=n_parts, cut_bins=np.array(side["cut_bins"], dtype=np.int64), assignment=assignment,
                     subdomain_weights=np.array(side["subdomain_weights"], dtype=np.float64))


# ---------------------------------------------------------------------------
# Array-native path for the multi-GPU decomposition
# ---------------------------------------------------------------------------

def element_centroids_device(arrays) -> tuple:
    """(centroids (E,3) f64, ids (E,), gauss weights (E,)) on the GPU, in
    category order; centroids match reference mesh.py:375 bit for bit."""
    from .device import DeviceMesh
    from .meshgen import GAUSS_COUNT, RULE_KIND
    from .mesh import ElementKind
    dm = DeviceMesh(arrays)
    cents, ids, ws = [], [], []
    for k, rule in enumerate(dm.rules):
        cents.append(dm.centroids(k))
        ids.append(dm.ids[k])
        kind = ElementKind(RULE_KIND[rule])
        ws.append(torch.full((dm.conn[k].shape[0],), float(kind.default_gauss_count), dtype=torch.float64,
                             device=dm.device))
    return torch.cat(cents), torch.cat(ids), torch.cat(ws)


def element_centroids(arrays) -> np.ndarray:
    cent, ids, _ = element_centroids_device(arrays)
    out = torch.empty_like(cent)
    out[ids] = cent
    return out.cpu().numpy()


def sfc_partition(arrays, n_parts: int, coeffs=None, level: int = 8):
    """Per-element subdomain (1..P, indexed by global element id), cut bins
    and subdomain weights — identical to partition_mesh_from_full ->
    project_to_bins -> split_1d of the reference, without Python objects."""
    cent, ids, w = element_centroids_device(arrays)
    box = bounding_box_of_points(_minmax_points(cent))
    keys = keys_from_centroids(cent, box, level)
    bins = group_bins_device(keys, ids, w)
    cuts, sub = split_cuts(bins.weights.cpu().numpy(), n_parts, coeffs)
    # bin -> part, then sorted element -> part
    m = bins.keys.numel()
    part_of_bin = torch.ones(m, dtype=torch.int32, device=cent.device)
    for c in cuts:
        part_of_bin[int(c) + 1:] += 1
    counts = bins.starts[1:] - bins.starts[:-1]
    part_sorted = torch.repeat_interleave(part_of_bin, counts)
    parts = torch.empty(ids.numel(), dtype=torch.int32, device=cent.device)
    parts[bins.ids_sorted] = part_sorted
    return parts.cpu().numpy(), cuts, sub


def _minmax_points(cent: torch.Tensor) -> np.ndarray:
    """Two points carrying the exact per-axis min and max (box computation)."""
    return torch.stack([cent.min(dim=0).values, cent.max(dim=0).values]).cpu().numpy()


# ---------------------------------------------------------------------------
# Array-native `part 1` I/O: the same files as
# store_partition / load_partition (reference sfc.py:385-417) from / into a
# dense per-element subdomain array, formatted and parsed by the native
# library (ab_format_partition / ab_parse_partition), for decompositions too
# large for an assignment dict.
# ---------------------------------------------------------------------------

def _host_io(name, *args) -> int:
    from ._lib import lib
    rc = int(getattr(lib(), name)(*args))
    if rc < 0:
        raise ValueError(f"{name}: {lib().ab_last_error().decode(errors='replace')}")
    return rc


def store_partition_parts(parts, n_parts: int, cut_bins, subdomain_weights, path, chunk: int = 1 << 22) -> None:
    """``parts[i]`` = subdomain (1..P) of element i (the output of
    :func:`sfc_partition`); writes byte-identical files to
    ``store_partition(Partition(...))``."""
    a = np.ascontiguousarray(np.asarray(parts), dtype=np.int32)
    if a.ndim != 1:
        raise ValueError("parts must be a 1D array")
    if a.size and (int(a.min()) < 1 or int(a.max()) > n_parts):
        raise ValueError(f"subdomain ids must lie in 1..{n_parts}")
    buf = np.empty(chunk * 24 + 64, dtype=np.uint8)
    with open(path, "wb") as f:
        f.write(f"part 1 {n_parts} {a.size}\n".encode())
        for s in range(0, a.size, chunk):
            n = min(chunk, a.size - s)
            w = _host_io("ab_format_partition", a[s:].ctypes.data, s, n, buf.ctypes.data, buf.size)
            f.write(buf[:w].tobytes())
    side = {"cut_bins": [int(c) for c in cut_bins], "subdomain_weights": [float(x) for x in subdomain_weights]}
    Path(str(path) + ".json").write_text(json.dumps(side), encoding="utf-8")


def load_partition_parts(path):
    """(parts int32 [E], n_parts, cut_bins, subdomain_weights) of a `part 1`
    file whose element ids are 0..E-1; the same validation as
    :func:`load_partition` (header, count, no duplicates)."""
    raw = Path(path).read_bytes()
    nl = raw.find(b"\n")
    head = (raw if nl < 0 else raw[:nl]).decode("utf-8").split()
    if len(head) != 4 or head[0] != "part" or head[1] != "1":
        raise ValueError(f"{path}:1: bad partition header {head!r}")
    n_parts, n_elem = int(head[2]), int(head[3])
    body = np.frombuffer(raw, dtype=np.uint8, offset=nl + 1 if nl >= 0 else len(raw))
    parts = np.zeros(n_elem, dtype=np.int32)
    seen = np.empty(max(n_elem, 1), dtype=np.uint8)
    got = _host_io("ab_parse_partition", body.ctypes.data if body.size else None, body.size, parts.ctypes.data,
                   n_elem, seen.ctypes.data)
    if got != n_elem:
        raise ValueError(f"{path}: expected {n_elem} assignments, got {got}")
    side = json.loads(Path(str(path) + ".json").read_text(encoding="utf-8"))
    return (parts, n_parts, np.array(side["cut_bins"], dtype=np.int64),
            np.array(side["subdomain_weights"], dtype=np.float64))

"""ORACLE — numpy restatement of the reference's SFC partitioner.  TEST
INFRASTRUCTURE ONLY (see oracle/fem.py header for the import rule).

Restates reference pkg/src/coexbal/sfc.py: Hilbert keys (transpose form,
:114-148), quantisation (:184-192), binning (:206-221) and the 1D split
(:258-307).  Pinned bit-exactly against tests/golden/reference_sfc.npz,
produced by the reference itself.
"""

from __future__ import annotations

import numpy as np


def hilbert_keys(cells: np.ndarray, level: int) -> np.ndarray:
    """Vectorised Skilling transpose + MSB-first interleave (sfc.py:114-148)."""
    x = [cells[:, i].astype(np.int64).copy() for i in range(3)]
    q = np.int64(1) << (level - 1)
    while q > 1:
        p = q - 1
        for i in range(3):
            hit = (x[i] & q) != 0
            x[0] = np.where(hit, x[0] ^ p, x[0])
            t = np.where(hit, 0, (x[0] ^ x[i]) & p)
            x[0] ^= t
            x[i] ^= t
        q >>= 1
    x[1] ^= x[0]
    x[2] ^= x[1]
    t = np.zeros(len(cells), dtype=np.int64)
    q = np.int64(1) << (level - 1)
    while q > 1:
        t = np.where((x[2] & q) != 0, t ^ (q - 1), t)
        q >>= 1
    for i in range(3):
        x[i] ^= t
    key = np.zeros(len(cells), dtype=np.int64)
    for j in range(level - 1, -1, -1):
        for i in range(3):
            key |= ((x[i] >> j) & 1) << (3 * j + 2 - i)
    return key


def bounding_box(points: np.ndarray, margin: float = 1e-9):
    """Centroid box grown by ``margin`` (reference mesh.py:139-146)."""
    lo, hi = points.min(axis=0), points.max(axis=0)
    ext = hi - lo
    pad = np.maximum(margin * np.maximum(ext, float(ext.max())), margin)
    return lo - pad, hi + pad


def quantize(cent: np.ndarray, lo, hi, level: int) -> np.ndarray:
    side = 1 << level
    rel = (cent - np.asarray(lo)) / (np.asarray(hi) - np.asarray(lo))
    return np.clip(np.floor(rel * side).astype(np.int64), 0, side - 1)


def group_bins(keys, ids, weights):
    order = np.lexsort((ids, keys))
    k, i, w = keys[order], ids[order], weights[order]
    starts = np.flatnonzero(np.concatenate([[True], k[1:] != k[:-1]]))
    return k[starts], np.add.reduceat(w, starts), starts, i


def split(bin_weights, n_parts, lam=None):
    """Closest-to-target cuts, ties to the earlier boundary, >= 1 bin/part."""
    m = len(bin_weights)
    lam = np.ones(n_parts) if lam is None else np.asarray(lam, float)
    prefix = np.cumsum(bin_weights)
    goals = np.cumsum(lam)[:-1] * (prefix[-1] / n_parts)
    cuts = []
    prev = -1
    for i, goal in enumerate(goals, start=1):
        j = min(int(np.searchsorted(prefix, goal)), m - 1)
        if j > 0 and abs(prefix[j - 1] - goal) <= abs(prefix[j] - goal):
            j -= 1
        j = min(max(j, prev + 1), m - 1 - (n_parts - i))
        cuts.append(j)
        prev = j
    cuts = np.array(cuts, dtype=np.int64)
    bounds = np.concatenate([[-1], cuts, [m - 1]])
    sub = np.array([prefix[bounds[s + 1]] - (prefix[bounds[s]] if bounds[s] >= 0 else 0.0)
                    for s in range(n_parts)])
    return cuts, sub


def partition(cent, ids, weights, n_parts, level=8, lam=None):
    """Per-element part (1-based, indexed like ``ids``), cuts, sub weights."""
    lo, hi = bounding_box(cent)
    keys = hilbert_keys(quantize(cent, lo, hi, level), level)
    bkeys, bw, starts, ids_sorted = group_bins(keys, ids, weights)
    cuts, sub = split(bw, n_parts, lam)
    part_of_bin = np.ones(len(bkeys), dtype=np.int64)
    for c in cuts:
        part_of_bin[c + 1:] += 1
    counts = np.diff(np.concatenate([starts, [len(ids_sorted)]]))
    parts_sorted = np.repeat(part_of_bin, counts)
    out = np.empty(len(ids), dtype=np.int64)
    pos = np.empty(int(ids.max()) + 1, dtype=np.int64)
    pos[ids] = np.arange(len(ids))
    out[pos[ids_sorted]] = parts_sorted
    return out, cuts, sub


def centroids(coords, conn):
    """Node mean in node order (reference mesh.py:375)."""
    s = np.zeros((conn.shape[0], 3))
    for a in range(conn.shape[1]):
        s = s + coords[conn[:, a]]
    return s / conn.shape[1]

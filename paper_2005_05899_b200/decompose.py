"""Element-disjoint subdomains with duplicated interface nodes.

Given a per-element subdomain assignment (from :func:`partition.sfc_partition`,
optionally steered by throughput-weighted coefficients), every rank builds:

* its submesh: the elements assigned to it and the nodes they touch, with a
  local node numbering that preserves global order (``l2g`` sorted);
* its interface plan: for every neighbouring rank q the local indices of the
  nodes shared with q, sorted by global id on both sides so the exchanged
  buffers line up element for element;
* ownership weights: an interface node counts once in global dot products,
  on the lowest rank that holds it.

This is setup-time host code (numpy); the per-step exchange is halo.py.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .meshgen import MeshArrays


@dataclass
class InterfacePlan:
    rank: int                      # 0-based
    n_ranks: int
    neighbors: list = field(default_factory=list)     # 0-based ranks, ascending
    shared: dict = field(default_factory=dict)        # q -> local node indices (int32, global-id order)
    own: np.ndarray | None = None                     # (n_local,) f64 ownership weights
    l2g: np.ndarray | None = None                     # (n_local,) global node ids

    @property
    def n_interface(self) -> int:
        if not self.shared:
            return 0
        return int(np.unique(np.concatenate(list(self.shared.values()))).size)


def submesh(arrays: MeshArrays, parts: np.ndarray, part: int):
    """Elements with ``parts[global_id] == part`` (1-based) and their nodes."""
    parts = np.asarray(parts)
    sel = {}
    used = []
    for _tag, rule, conn, ids in arrays.categories():
        m = parts[ids] == part
        sel[rule] = (conn[m], ids[m])
        used.append(conn[m].ravel())
    l2g = np.unique(np.concatenate(used)) if used else np.zeros(0, np.int64)
    sub = MeshArrays(coords=np.ascontiguousarray(arrays.coords[l2g]))
    for rule, (c, ids) in sel.items():
        sub.conn[rule] = np.searchsorted(l2g, c).astype(np.int32)
        sub.elem_ids[rule] = ids.astype(np.int64)
    sub.period = np.asarray(arrays.period, dtype=np.float64).copy()
    return sub, l2g.astype(np.int64)


def node_sharers(arrays: MeshArrays, parts: np.ndarray, n_parts: int):
    """Unique (node, part) incidences as sorted keys node * P + (part - 1)."""
    keys = []
    for _tag, _rule, conn, ids in arrays.categories():
        p = (np.asarray(parts)[ids] - 1).astype(np.int64)
        keys.append(np.unique((conn.astype(np.int64) * n_parts + p[:, None]).ravel()))
    return np.unique(np.concatenate(keys))


def interface_plan(arrays: MeshArrays, parts: np.ndarray, n_parts: int, rank: int, l2g: np.ndarray,
                   sharers: np.ndarray | None = None) -> InterfacePlan:
    """Interface plan of 0-based ``rank`` whose local nodes are ``l2g``."""
    keys = node_sharers(arrays, parts, n_parts) if sharers is None else sharers
    node = keys // n_parts
    prt = keys % n_parts
    # owner = lowest part touching the node (keys sorted -> first per node)
    first = np.ones(node.size, dtype=bool)
    first[1:] = node[1:] != node[:-1]
    owner_nodes, owner = node[first], prt[first]
    own_full = owner[np.searchsorted(owner_nodes, l2g)]
    plan = InterfacePlan(rank=rank, n_ranks=n_parts, l2g=l2g, own=(own_full == rank).astype(np.float64))
    mine = np.unique(node[prt == rank])
    for q in range(n_parts):
        if q == rank:
            continue
        theirs = node[prt == q]
        common = np.intersect1d(mine, theirs, assume_unique=False)
        if common.size:
            plan.neighbors.append(q)
            plan.shared[q] = np.searchsorted(l2g, common).astype(np.int32)
    return plan


def decompose(arrays: MeshArrays, parts: np.ndarray, n_parts: int, rank: int):
    """(submesh, plan) of 0-based ``rank``."""
    sub, l2g = submesh(arrays, parts, rank + 1)
    plan = interface_plan(arrays, parts, n_parts, rank, l2g)
    return sub, plan

"""Boundary assembly of the equilibrium wall model (Algorithm 1 line 4,
PAPER.md:214, :228): the wall faces of a mesh and the K8 launch
(``ab_wall_traction``).  The scheme (Reichardt's law at an exchange point
one element above the face, lumped face integration) is DESIGN.md §3.

Face extraction is setup-time host code (numpy); the per-stage traction is
one CUDA kernel over the faces.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from ._lib import AbWall, call, ptr, stream_handle
from .meshgen import RULE_KIND, NODE_COUNT

# local faces per element kind, VTK node order, quads around their perimeter
FACES = {
    "tet": [(0, 1, 2), (0, 1, 3), (1, 2, 3), (0, 2, 3)],
    "pyr": [(0, 1, 2, 3), (0, 1, 4), (1, 2, 4), (2, 3, 4), (3, 0, 4)],
    "pri": [(0, 1, 2), (3, 4, 5), (0, 1, 4, 3), (1, 2, 5, 4), (2, 0, 3, 5)],
    "hex": [(0, 1, 2, 3), (4, 5, 6, 7), (0, 1, 5, 4), (1, 2, 6, 5), (2, 3, 7, 6), (3, 0, 4, 7)],
}


def wall_faces(mesh, on_wall) -> tuple[np.ndarray, np.ndarray]:
    """Faces whose nodes all satisfy ``on_wall``: (face nodes (F,4) int32,
    -1 in slot 3 for triangles; the owning element's off-face nodes (F,4),
    -1 padded), ordered by (category, local face, element)."""
    on_wall = np.asarray(on_wall, bool)
    faces, offs = [], []
    for _tag, rule, conn, _ids in mesh.categories():
        kind = RULE_KIND[rule]
        nn = NODE_COUNT[kind]
        for f in FACES[kind]:
            hit = on_wall[conn[:, list(f)]].all(axis=1)
            if not hit.any():
                continue
            rest = [a for a in range(nn) if a not in f][:4]
            c = conn[hit]
            F = np.full((c.shape[0], 4), -1, np.int32)
            F[:, :len(f)] = c[:, list(f)]
            O = np.full((c.shape[0], 4), -1, np.int32)
            O[:, :len(rest)] = c[:, rest]
            faces.append(F)
            offs.append(O)
    if not faces:
        return np.zeros((0, 4), np.int32), np.zeros((0, 4), np.int32)
    return np.concatenate(faces), np.concatenate(offs)


class WallModel:
    """Device face lists + the K8 launch: rhs4 += wall traction of u4."""

    def __init__(self, faces: np.ndarray, off: np.ndarray, device="cuda", ordered: bool = True):
        """``ordered``: the face tractions are summed per wall node in
        ascending face order (second small kernel, bitwise reproducible);
        False keeps the fp64 reductions per face node."""
        self.face = torch.from_numpy(np.ascontiguousarray(faces, dtype=np.int32)).to(device)
        self.off = torch.from_numpy(np.ascontiguousarray(off, dtype=np.int32)).to(device)
        self.struct = AbWall(n_faces=int(self.face.shape[0]), face=ptr(self.face), off=ptr(self.off))
        self.ordered = bool(ordered and self.face.shape[0] > 0)
        if self.ordered:
            f = self.face.to(torch.int64)
            nf = f.shape[0]
            fid = torch.arange(nf, device=f.device, dtype=torch.int64)[:, None].expand(nf, 4).reshape(-1)
            nd = f.reshape(-1)
            keep = nd >= 0
            nd, fid = nd[keep], fid[keep]
            order = torch.sort(nd * nf + fid).indices  # by node, then ascending face id
            nd, fid = nd[order], fid[order]
            self.wnode, counts = torch.unique_consecutive(nd, return_counts=True)
            self.wnode = self.wnode.to(torch.int32).contiguous()
            self.wptr = torch.zeros(self.wnode.numel() + 1, dtype=torch.int64, device=f.device)
            self.wptr[1:] = torch.cumsum(counts, 0)
            self.fref = fid.to(torch.int32).contiguous()
            self.ftrac = torch.zeros((nf, 3), dtype=torch.float64, device=f.device)
            s = self.struct
            s.n_nodes = int(self.wnode.numel())
            s.node, s.ptr, s.fref, s.ftrac = ptr(self.wnode), ptr(self.wptr), ptr(self.fref), ptr(self.ftrac)

    @property
    def n_faces(self) -> int:
        return int(self.face.shape[0])

    def add_traction(self, phys, coords4: torch.Tensor, u4: torch.Tensor, rhs4: torch.Tensor):
        call("ab_wall_traction", ctypes.byref(self.struct), ctypes.byref(phys), ptr(coords4), ptr(u4), ptr(rhs4),
             stream_handle())


def assemble_wall_traction(mesh, faces, off, u, params=None) -> torch.Tensor:
    """Functional form (N,3): the wall-model contribution to the momentum RHS."""
    from .device import DeviceMesh, nodes_as4
    from .timestep import FlowParams
    dm = mesh if isinstance(mesh, DeviceMesh) else DeviceMesh(mesh, windows=False)
    ph = (params or FlowParams()).struct()
    u4 = nodes_as4(torch.as_tensor(u, dtype=torch.float64, device=dm.device))
    out = torch.zeros((dm.n_nodes, 4), dtype=torch.float64, device=dm.device)
    WallModel(faces, off, dm.device).add_traction(ph, dm.coords4, u4, out)
    return out[:, :3]

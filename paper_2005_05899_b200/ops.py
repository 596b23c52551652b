"""Functional element-operator entry points:
``assemble_momentum(mesh, u, params) -> rhs``, ``assemble_divergence``,
``assemble_gradient``.  Thin wrappers over K2/K4/K6 that accept an
array-native mesh or a DeviceMesh and (N,3)/(N,) tensors or arrays."""

from __future__ import annotations

import ctypes

import torch

from ._lib import call, ptr, stream_handle
from .device import DeviceMesh, nodes_as4


def _dm(mesh, **kw) -> DeviceMesh:
    return mesh if isinstance(mesh, DeviceMesh) else DeviceMesh(mesh, **kw)


def _t(x, dm):
    return torch.as_tensor(x, dtype=torch.float64, device=dm.device)


def assemble_momentum(mesh, u, params=None, windows: bool = False) -> torch.Tensor:
    """R(u) (N,3): EMAC convection + viscous + Vreman (K2)."""
    from .timestep import FlowParams
    dm = _dm(mesh, windows=windows)
    ph = (params or FlowParams()).struct()
    u4 = nodes_as4(_t(u, dm))
    out = torch.zeros((dm.n_nodes, 4), dtype=torch.float64, device=dm.device)
    call("ab_momentum_rhs", ctypes.byref(dm.struct), ctypes.byref(ph), ptr(u4), ptr(out), stream_handle())
    return out[:, :3]


def assemble_divergence(mesh, u, scale: float = 1.0, windows: bool = False) -> torch.Tensor:
    """scale * (D u)_a = scale * sum_e int N_a div(u) (K4)."""
    dm = _dm(mesh, windows=windows)
    u4 = nodes_as4(_t(u, dm))
    out = torch.zeros(dm.n_nodes, dtype=torch.float64, device=dm.device)
    call("ab_divergence", ctypes.byref(dm.struct), ptr(u4), scale, ptr(out), stream_handle())
    return out


def assemble_gradient(mesh, p, scale: float = 1.0, windows: bool = False) -> torch.Tensor:
    """scale * (G p)_a = scale * sum_e int N_a grad(p) (K6), (N,3)."""
    dm = _dm(mesh, windows=windows)
    pt = _t(p, dm).contiguous()
    out = torch.zeros((dm.n_nodes, 4), dtype=torch.float64, device=dm.device)
    call("ab_gradient", ctypes.byref(dm.struct), ptr(pt), scale, ptr(out), stream_handle())
    return out[:, :3]

"""Load-balance plumbing on the hot path — the reference's workload-plugin
interface (reference pkg/src/coexbal/balance.py).

Kept verbatim in meaning: ``Phase`` (balance.py:39-42), ``TimingSample``
(:50-66), ``BalanceMetrics`` / ``compute_metrics`` (:69-92) and the plugin
type ``Timer = Callable[[Partition], TimingSample]`` (:241).  The reference's
real Timer (cli._make_bench_timer, cli.py:171-187) times the CPU assembly of
each subdomain one after another; :func:`gpu_timer` times K2 (the momentum
element assembly, ``Phase.ELEMENT_ASSEMBLY``) of each subdomain on the GPU
with CUDA events, and :func:`distributed_timer` does it on every rank at once
and all-gathers the times.

The regression balancer (SLR/WLR, balance.py:136-346) is out of scope
(SURVEY.md §8(e), F8-ii); the north star's DLB analog is the one-shot
throughput-weighted coefficients of :func:`throughput_coefficients`,
lambda_i = P theta_i / sum(theta), theta_i = W_i / t_i — the analytic fixed
point of the reference's linear model.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum
from typing import Callable

import numpy as np


class Phase(Enum):
    ELEMENT_ASSEMBLY = "element_assembly"
    BOUNDARY_ASSEMBLY = "boundary_assembly"
    SOLVER = "solver"


@dataclass(frozen=True)
class TimingSample:
    iteration: int
    times: np.ndarray
    phase: Phase = Phase.ELEMENT_ASSEMBLY

    def __post_init__(self):
        t = np.asarray(self.times, dtype=np.float64)
        object.__setattr__(self, "times", t)
        if t.ndim != 1 or len(t) == 0:
            raise ValueError("times must be a non-empty 1D array")
        if (t <= 0).any():
            raise ValueError("all times must be > 0")

    @property
    def n_ranks(self) -> int:
        return len(self.times)


@dataclass(frozen=True)
class BalanceMetrics:
    mean: float
    imbalance: float
    per_rank: np.ndarray
    deviations: np.ndarray
    lb: float

    @property
    def max_deviation(self) -> float:
        return float(self.deviations.max())


def compute_metrics(sample: TimingSample) -> BalanceMetrics:
    """I = max/mean, LB = mean/max, per-rank t/mean, |t - mean|."""
    t = sample.times
    mean = float(t.sum() / len(t))
    tmax = float(t.max())
    return BalanceMetrics(mean=mean, imbalance=tmax / mean, per_rank=t / mean, deviations=np.abs(t - mean),
                          lb=mean / tmax)


Timer = Callable[["object"], TimingSample]


def throughput_coefficients(times, loads) -> np.ndarray:
    """lambda_i = P theta_i / sum(theta), theta_i = load_i / t_i: the
    coefficients that equalise t_i under a linear cost model (one shot)."""
    t = np.asarray(times, dtype=np.float64)
    w = np.asarray(loads, dtype=np.float64)
    if t.shape != w.shape or t.ndim != 1 or (t <= 0).any() or (w <= 0).any():
        raise ValueError("times and loads must be positive 1D arrays of equal length")
    theta = w / t
    return len(t) * theta / theta.sum()


def _time_momentum(dm, reps: int = 5) -> float:
    """Median CUDA-event time of one K2 launch over ``dm`` (seconds)."""
    import ctypes
    import torch
    from ._lib import call, ptr, stream_handle
    from .timestep import FlowParams
    phys = FlowParams().struct()
    u = torch.zeros((dm.n_nodes, 4), dtype=torch.float64, device=dm.device)
    r = torch.zeros_like(u)
    call("ab_momentum_rhs", ctypes.byref(dm.struct), ctypes.byref(phys), ptr(u), ptr(r), stream_handle())
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        call("ab_momentum_rhs", ctypes.byref(dm.struct), ctypes.byref(phys), ptr(u), ptr(r), stream_handle())
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) / 1e3)
    return float(np.median(ts))


def gpu_timer(arrays, reps: int = 5, iteration_start: int = 1) -> Timer:
    """Timer plugin: for a Partition (assignment dict or per-element part
    array), time K2 over each subdomain's elements on this GPU in turn —
    the device analog of cli._make_bench_timer (cli.py:171-187)."""
    from .decompose import submesh
    from .device import DeviceMesh
    state = {"it": iteration_start}

    def timer(part) -> TimingSample:
        parts = _parts_array(part, arrays.n_elements)
        n_parts = int(parts.max())
        times = []
        for r in range(1, n_parts + 1):
            sub, _ = submesh(arrays, parts, r)
            times.append(_time_momentum(DeviceMesh(sub, reorder="sfc", windows=True), reps))
        s = TimingSample(iteration=state["it"], times=np.array(times), phase=Phase.ELEMENT_ASSEMBLY)
        state["it"] += 1
        return s

    return timer


def distributed_timer(solver, group=None, reps: int = 5):
    """Every rank times K2 on its own subdomain; times are all-gathered."""
    import torch
    import torch.distributed as dist
    t = _time_momentum(solver.dm, reps)
    dev = solver.dm.device if dist.get_backend(group) == "nccl" else torch.device("cpu")
    buf = torch.tensor([t], dtype=torch.float64, device=dev)
    out = [torch.zeros_like(buf) for _ in range(dist.get_world_size(group))]
    dist.all_gather(out, buf, group=group)
    return TimingSample(iteration=1, times=np.array([float(x.item()) for x in out]))


def _parts_array(part, n_elements: int) -> np.ndarray:
    if isinstance(part, np.ndarray):
        return part.astype(np.int64)
    arr = np.zeros(n_elements, dtype=np.int64)
    for eid, s in part.assignment.items():
        arr[eid] = s
    return arr

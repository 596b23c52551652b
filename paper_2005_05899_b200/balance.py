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

The north star's DLB analog is the one-shot throughput-weighted
coefficients of :func:`throughput_coefficients`, lambda_i = P theta_i /
sum(theta), theta_i = W_i / t_i — the analytic fixed point of the
reference's linear model.

The paper's own regression balancer (reference
balance.py:95-346) is restated below with the same types
and update rule, so :func:`run_balancing_loop` driven by the same Timer gives
the reference's coefficient sequence (tests/test_dlb.py pins it against
golden runs of the reference).  ``stabilised=True`` swaps the per-splitting-
point regression, whose mean-normalised observations drift when devices are
heterogeneous (I = 1.097 -> 2.62 on the hetero_s20 plan), for a
per-rank weighted regression of the affine cost model t_k = c_k + s_k W_k
(the same anchored SLR/WLR fit, on absolute times and loads) and picks the
loads that equalise the predicted times.
"""

from __future__ import annotations

import csv
import io
import math
from dataclasses import dataclass
from enum import Enum
from typing import Callable

import numpy as np

# Constants of the regression update (reference balance.py:29-36): keep every
# cumulative splitting point DELTA_MIN above its predecessor, treat slopes
# <= BETA_MIN as unusable, and weigh WLR observation k by growth**(k-1).
DELTA_MIN = 0.01
BETA_MIN = 1e-9
DEFAULT_WLR_GROWTH = 1.5


class RegressionMode(Enum):
    SLR = "slr"
    WLR = "wlr"


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


# ---------------------------------------------------------------------------
# Regression DLB (reference balance.py:95-346)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class CorrectionState:
    """Coefficients lambda (P,) and, per splitting point i = 1..P-1, the
    history of (cumulative coefficient, mean-normalised cumulative time)
    pairs (reference balance.py:101-133)."""

    n_parts: int
    lam: np.ndarray
    history: tuple
    mode: RegressionMode = RegressionMode.WLR
    wlr_growth: float = DEFAULT_WLR_GROWTH

    @classmethod
    def initial(cls, n_parts: int, mode: RegressionMode = RegressionMode.WLR,
                wlr_growth: float = DEFAULT_WLR_GROWTH) -> "CorrectionState":
        if n_parts < 1:
            raise ValueError("n_parts must be >= 1")
        return cls(n_parts, np.ones(n_parts), ((),) * (n_parts - 1), mode, wlr_growth)

    def cumulative(self) -> np.ndarray:
        """[0, lam_1, lam_1 + lam_2, ..., P] with both ends pinned."""
        out = np.concatenate(([0.0], np.cumsum(self.lam)))
        out[-1] = float(self.n_parts)
        return out


def observe(state: CorrectionState, sample: TimingSample) -> CorrectionState:
    """Record (Lambda_i, Upsilon_i) for every splitting point, Upsilon_i =
    sum_{k<=i} t_k / mean(t) (reference balance.py:136-156)."""
    p = state.n_parts
    if sample.n_ranks != p:
        raise ValueError(f"sample has {sample.n_ranks} ranks, state expects {p}")
    ups = np.cumsum(sample.times)[: p - 1] / (sample.times.sum() / p)
    cum = state.cumulative()
    hist = tuple(h + ((float(cum[i + 1]), float(ups[i])),) for i, h in enumerate(state.history))
    return CorrectionState(p, state.lam, hist, state.mode, state.wlr_growth)


@dataclass(frozen=True)
class RegressionFit:
    alpha: float
    beta: float
    n_obs: int
    degenerate: bool = False


def fit(observations, mode: RegressionMode = RegressionMode.WLR,
        wlr_growth: float = DEFAULT_WLR_GROWTH) -> RegressionFit:
    """Weighted least-squares line y = alpha + beta x through the anchor
    (0, 0) (weight 1) and the observations (weight growth**(k-1) under WLR,
    1 under SLR) (reference balance.py:166-194)."""
    n = len(observations)
    if n < 1:
        raise ValueError("need at least one observation")
    x = np.array([0.0] + [float(o[0]) for o in observations])
    y = np.array([0.0] + [float(o[1]) for o in observations])
    if mode is RegressionMode.WLR:
        w = np.array([1.0] + [wlr_growth ** k for k in range(n)])
    else:
        w = np.ones(n + 1)
    sw = w.sum()
    mx = (w * x).sum() / sw
    my = (w * y).sum() / sw
    sxx = (w * (x - mx) ** 2).sum()
    if sxx / sw < 1e-12:
        return RegressionFit(alpha=my, beta=0.0, n_obs=n, degenerate=True)
    beta = (w * (x - mx) * (y - my)).sum() / sxx
    return RegressionFit(alpha=my - beta * mx, beta=beta, n_obs=n)


def _monotone(cum: np.ndarray) -> np.ndarray:
    """Forward then backward clamp keeping DELTA_MIN gaps, ends pinned
    (reference balance.py:226-231)."""
    p = len(cum) - 1
    for i in range(1, p):
        cum[i] = max(cum[i], cum[i - 1] + DELTA_MIN)
    cum[p] = float(p)
    for i in range(p - 1, 0, -1):
        cum[i] = min(cum[i], cum[i + 1] - DELTA_MIN)
    return cum


def update_coefficients(state: CorrectionState) -> CorrectionState:
    """Move splitting point i to the crossing of its regression line with
    y = i; untrustworthy fits keep the old point (reference balance.py:197-234)."""
    p = state.n_parts
    cum = state.cumulative()
    new = cum.copy()
    for i in range(1, p):
        obs = state.history[i - 1]
        if not obs:
            raise ValueError(f"splitting point {i} has no observations")
        f = fit(obs, state.mode, state.wlr_growth)
        if f.degenerate or f.beta <= BETA_MIN:
            continue
        x = (i - f.alpha) / f.beta
        if math.isfinite(x):
            new[i] = x
    return CorrectionState(p, np.diff(_monotone(new)), state.history, state.mode, state.wlr_growth)


def rank_model_coefficients(loads: list, times: list, mode: RegressionMode = RegressionMode.WLR,
                            wlr_growth: float = DEFAULT_WLR_GROWTH) -> np.ndarray:
    """Stabilised update: per rank k, a weighted least-squares fit of the
    affine cost t = c_k + s_k W over its own (load, time) history (WLR
    weights growth**(j-1), SLR uniform; with one observation, or no spread in
    the loads, the line through the origin s_k = t_k / W_k — the throughput
    estimate of :func:`throughput_coefficients`), then the loads that
    equalise the predicted times, W_k = (T - c_k) / s_k with sum W_k = W,
    kept >= DELTA_MIN of the mean load.  Returns lambda = P W_k / W.

    ``loads`` / ``times``: one (P,) array per balancing iteration, oldest
    first.  Unlike the splitting-point regression its observations are
    absolute, so moving work between heterogeneous devices does not rescale
    the old ones."""
    L = np.asarray(loads, dtype=np.float64)
    T = np.asarray(times, dtype=np.float64)
    if L.shape != T.shape or L.ndim != 2 or (L <= 0).any() or (T <= 0).any():
        raise ValueError("loads and times must be positive (iterations, ranks) arrays of equal shape")
    n_it, p = L.shape
    total = float(L[-1].sum())
    s = T[-1] / L[-1]
    c = np.zeros(p)
    if n_it > 1:
        w = np.array([wlr_growth ** j for j in range(n_it)]) if mode is RegressionMode.WLR else np.ones(n_it)
        sw = w.sum()
        for k in range(p):
            x, y = L[:, k], T[:, k]
            mx, my = (w * x).sum() / sw, (w * y).sum() / sw
            sxx = (w * (x - mx) ** 2).sum()
            if sxx / sw <= 1e-12 * mx * mx:
                continue
            b = (w * (x - mx) * (y - my)).sum() / sxx
            if b > BETA_MIN * my / mx:
                s[k] = b
                c[k] = max(my - b * mx, 0.0)
    inv = 1.0 / s
    t_eq = (total + (c * inv).sum()) / inv.sum()
    w_new = np.maximum((t_eq - c) * inv, DELTA_MIN * total / p)
    cum = _monotone(np.concatenate(([0.0], np.cumsum(p * w_new / w_new.sum()))))
    return np.diff(cum)


@dataclass(frozen=True)
class IterationRecord:
    k: int
    lam: np.ndarray
    times: np.ndarray
    metrics: BalanceMetrics
    partition: object


@dataclass(frozen=True)
class BalanceReport:
    n_parts: int
    mode: RegressionMode
    tol: float
    converged: bool
    iterations: tuple

    @property
    def n_iterations(self) -> int:
        return len(self.iterations)

    @property
    def final(self) -> IterationRecord:
        return self.iterations[-1]

    @property
    def best(self) -> IterationRecord:
        """The iteration with the lowest imbalance (first on ties)."""
        return min(self.iterations, key=lambda r: r.metrics.imbalance)

    def to_json_dict(self, manifest: dict | None = None, final_partition_ref: str | None = None) -> dict:
        """Same document as the reference's (balance.py:271-289)."""
        doc = {"iterations": [{"k": r.k, "lambda": [float(v) for v in r.lam], "times": [float(v) for v in r.times],
                               "imbalance": r.metrics.imbalance, "lb": r.metrics.lb,
                               "max_dev": r.metrics.max_deviation} for r in self.iterations],
               "converged": self.converged, "final_partition_ref": final_partition_ref}
        if manifest is not None:
            doc["manifest"] = manifest
        return doc

    def convergence_csv(self) -> str:
        """k,rank,time,I_k with 1-based ranks (reference balance.py:291-299)."""
        out = io.StringIO()
        wr = csv.writer(out, lineterminator="\n")
        wr.writerow(["k", "rank", "time", "I_k"])
        for r in self.iterations:
            for j in range(self.n_parts):
                wr.writerow([r.k, j + 1, repr(float(r.times[j])), repr(float(r.metrics.per_rank[j]))])
        return out.getvalue()


def run_balancing_loop(mesh, cfg, n_parts: int, timer: Timer, mode: RegressionMode = RegressionMode.WLR,
                       tol: float = 0.02, max_iters: int = 20, wlr_growth: float = DEFAULT_WLR_GROWTH,
                       bins=None, *, stabilised: bool = False) -> BalanceReport:
    """split -> time -> observe -> correct until max/mean - 1 <= tol
    (reference balance.py:302-346; iteration 1 uses unit coefficients).

    ``timer`` is any Timer: :func:`gpu_timer` times K2 of every subdomain on
    this GPU.  ``stabilised=True`` uses :func:`rank_model_coefficients`
    instead of the splitting-point regression."""
    from .partition import project_to_bins, split_1d
    if max_iters < 1:
        raise ValueError("max_iters must be >= 1")
    seq = bins if bins is not None else project_to_bins(mesh, cfg)
    state = CorrectionState.initial(n_parts, mode=mode, wlr_growth=wlr_growth)
    recs, loads, times = [], [], []
    converged = False
    for k in range(1, max_iters + 1):
        part = split_1d(seq, n_parts, state.lam)
        got = timer(part)
        sample = TimingSample(iteration=k, times=got.times, phase=got.phase)
        met = compute_metrics(sample)
        recs.append(IterationRecord(k=k, lam=state.lam.copy(), times=sample.times, metrics=met, partition=part))
        if met.imbalance - 1.0 <= tol:
            converged = True
            break
        if k == max_iters:
            break
        if stabilised:
            loads.append(np.asarray(part.subdomain_weights, dtype=np.float64))
            times.append(sample.times)
            state = CorrectionState(n_parts, rank_model_coefficients(loads, times, mode, wlr_growth),
                                    state.history, mode, wlr_growth)
        else:
            state = update_coefficients(observe(state, sample))
    return BalanceReport(n_parts=n_parts, mode=mode, tol=tol, converged=converged, iterations=tuple(recs))

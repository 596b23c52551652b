"""Closed-form CPU/GPU co-execution efficiency model (SURVEY.md §8(f) row
f-4; reference coexec.py:258-323, PAPER.md co-execution section), restated
for reporting the measured B200 numbers in context.

The model: a GPU rank computes s times faster than one CPU core (s in
single-core equivalents), there are r = n_gpu / n_core GPUs per core, and
each GPU rank idles one or two host cores to drive it.  Resource
efficiencies (fraction of the aggregate capacity doing useful work):

* GPUs only:         s r / (1 + s r)
* cores only:        1 / (1 + s r)
* co-execution, 1 (2) cores idled per GPU: (1 + (s - 1) r) / (1 + s r)
  (resp. s - 2), and the predicted elapsed-time reduction of co-execution
  over the GPU-only run, 1 - eff_gpu / eff_coex.

This framework never co-executes (there is no CPU path in the product;
DESIGN.md §0); :func:`measured_params` turns a bench line's measured GPU and
single-core rates into the model's inputs so the reports can state what the
paper's co-execution would buy on this host.  Values are bit-identical to the
reference's for the same inputs (tests/test_coexec.py, golden runs).
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass


@dataclass(frozen=True)
class EfficiencyParams:
    """GPU speedup s (single-core equivalents) and ratio r = n_gpu / n_core."""

    speedup: float
    ratio: float
    n_core: int | None = None
    n_gpu: int | None = None

    def __post_init__(self):
        if not self.speedup > 0:
            raise ValueError("speedup must be > 0")
        if self.ratio < 0:
            raise ValueError("ratio must be >= 0")

    @classmethod
    def from_counts(cls, n_core: int, n_gpu: int, speedup: float) -> "EfficiencyParams":
        if n_core < 1 or n_gpu < 0:
            raise ValueError("need n_core >= 1 and n_gpu >= 0")
        return cls(speedup=speedup, ratio=n_gpu / n_core, n_core=n_core, n_gpu=n_gpu)


def _sr(p: EfficiencyParams) -> float:
    return p.speedup * p.ratio


def eff_gpu(p: EfficiencyParams) -> float:
    return _sr(p) / (1.0 + _sr(p))


def eff_core(p: EfficiencyParams) -> float:
    return 1.0 / (1.0 + _sr(p))


def eff_coex1(p: EfficiencyParams) -> float:
    return (1.0 + (p.speedup - 1.0) * p.ratio) / (1.0 + _sr(p))


def eff_coex2(p: EfficiencyParams) -> float:
    if p.speedup < 2.0:
        warnings.warn(f"eff_coex2 evaluated at speedup {p.speedup} < 2: co-execution wastes more core capacity "
                      "than the GPUs add", stacklevel=2)
    return (1.0 + (p.speedup - 2.0) * p.ratio) / (1.0 + _sr(p))


def predicted_time_reduction(p: EfficiencyParams, cores_per_gpu: int = 2) -> float:
    """1 - eff_gpu / eff_coex (elapsed time is inversely proportional to
    efficiency)."""
    if cores_per_gpu not in (1, 2):
        raise ValueError("cores_per_gpu must be 1 or 2")
    coex = eff_coex1(p) if cores_per_gpu == 1 else eff_coex2(p)
    if coex <= 0:
        raise ValueError(f"co-execution efficiency {coex} is not positive")
    return 1.0 - eff_gpu(p) / coex


def measured_params(gpu_rate: float, core_rate: float, n_core: int, n_gpu: int = 1) -> EfficiencyParams:
    """Model inputs from measured rates in the same unit (e.g. M
    element-steps/s of one B200 and of one host core running the CPU path)."""
    if not (gpu_rate > 0 and core_rate > 0):
        raise ValueError("rates must be > 0")
    return EfficiencyParams.from_counts(n_core, n_gpu, gpu_rate / core_rate)


def report(p: EfficiencyParams) -> dict:
    """The reference's efficiency table (cli.py `efficiency`) as a dict."""
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        out = {"speedup": p.speedup, "ratio": p.ratio, "eff_core": eff_core(p), "eff_gpu": eff_gpu(p),
               "eff_coex1": eff_coex1(p), "eff_coex2": eff_coex2(p)}
        for c in (1, 2):
            try:
                out[f"time_reduction_coex{c}"] = predicted_time_reduction(p, c)
            except ValueError:
                out[f"time_reduction_coex{c}"] = None
    return out

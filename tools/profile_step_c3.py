"""Eager C3 time steps for an ncu launch list (BASELINE configs[2]: 30.2M
mixed elements, wall model, two-kernel CG) — the solver bench.py builds.

    ncu --profile-from-start off --metrics gpu__time_duration.sum --csv python tools/profile_step_c3.py
"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2005_05899_b200.timestep import FlowParams, FlowSolver  # noqa: E402

w = bench.build_rank_workload("c3", 1, 0)
fs = FlowSolver(w["sub"], FlowParams(**bench.PHYS), **w["bc"], windows=True, reorder="sfc", wall=w["wall"])
fs.set_state(w["u"], w["p"])
fs.step(1e-3, 50)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
fs.step(1e-3, 50)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("done")

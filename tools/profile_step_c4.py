"""Eager time steps of a bench workload for ncu (default C4, BASELINE
configs[3]: 249M mixed elements, wall model, two-kernel CG) — the same
solver bench.py builds at N = 1.  Only the last step is inside
cudaProfilerStart/Stop, so `ncu --profile-from-start off` sees one step.

    ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,... \
        --csv python tools/profile_step_c4.py [--workload c4] [--steps 1]
"""
import argparse
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2005_05899_b200.timestep import FlowParams, FlowSolver  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c4")
ap.add_argument("--steps", type=int, default=1)
a = ap.parse_args()
w = bench.build_rank_workload(a.workload, 1, 0)
fs = FlowSolver(w["sub"], FlowParams(**bench.PHYS), **w["bc"], windows=True, reorder="sfc", wall=w["wall"])
fs.set_state(w["u"], w["p"])
print({r: int(c.shape[0]) for r, c in zip(fs.dm.rules, fs.dm.conn)}, "nodes", fs.n, "nnz", fs.L.nnz,
      "stored", fs.L.nnz_stored, flush=True)
fs.step(1e-3, 50)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for _ in range(a.steps):
    fs.step(1e-3, 50)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("done", flush=True)

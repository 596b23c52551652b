"""Run eager C2 time steps for profiling (ncu / nsys-less launch lists).

    python tools/profile_step.py [--steps 2] [--no-windows] [--n 88]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2005_05899_b200 import meshgen  # noqa: E402
from paper_2005_05899_b200.timestep import FlowParams, FlowSolver  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--n", type=int, default=88)
ap.add_argument("--no-windows", action="store_true")
ap.add_argument("--no-reorder", action="store_true")
ap.add_argument("--cg-iters", type=int, default=50)
ap.add_argument("--no-resident", action="store_true")
ap.add_argument("--no-pipeline", action="store_true")
a = ap.parse_args()
m = meshgen.box_tets(a.n, a.n, a.n, jitter=0.2, seed=20200131)
u, p = meshgen.c2_initial(m.coords)
from paper_2005_05899_b200.device import DeviceMesh  # noqa: E402
dm = DeviceMesh(m, reorder=None if a.no_reorder else "sfc", windows=not a.no_windows, pipelined=not a.no_pipeline)
fs = FlowSolver(dm, FlowParams(1.0, 1e-3, 0.07), p_fixed=meshgen.boundary_nodes(m))
if a.no_resident:
    fs.pcg.resident = False
fs.set_state(u, p)
if not a.no_windows:
    print(fs.dm.window_stats())
torch.cuda.synchronize()
# ncu --profile-from-start off sees only the time steps (not the setup)
torch.cuda.cudart().cudaProfilerStart()
for _ in range(a.steps):
    fs.step(1e-3, a.cg_iters)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("done")

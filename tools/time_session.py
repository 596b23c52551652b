"""Throughput of the C-ABI session (ab_step: native setup, tiled single-pass
CG) against the Python FlowSolver (eager steps) on the same mesh.

    python tools/time_session.py [c3 scale=1.0]
"""
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch  # noqa: E401,E402
from paper_2005_05899_b200 import meshgen  # noqa: E402
from paper_2005_05899_b200.session import Session  # noqa: E402
from paper_2005_05899_b200.timestep import FlowParams, FlowSolver  # noqa: E402

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
m = meshgen.c3_mesh(scale)
bc, wall = meshgen.wall_model_bcs(m)
u = np.zeros((m.n_nodes, 3)); u[:, 0] = 1.0
p = np.zeros(m.n_nodes)
params = FlowParams(1.0, 1e-3, 0.07)
E = m.n_elements


def timed(step, reps=5):
    step(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        step()
    b.record(); b.synchronize()
    return a.elapsed_time(b) / reps


t0 = time.time()
s = Session(m, params, wall=wall, **bc)
t_setup = time.time() - t0
s.set_state(u, p)
ms_s = timed(lambda: s.step(1e-3, 50))
s.close()
fs = FlowSolver(m, params, **bc, wall=wall)
fs.set_state(u, p)
ms_f = timed(lambda: fs.step(1e-3, 50))
print(f"{E} elements: session {ms_s:.2f} ms/step = {E / ms_s / 1e3:.1f} M element-steps/s (setup {t_setup:.1f} s), "
      f"FlowSolver eager {ms_f:.2f} ms/step = {E / ms_f / 1e3:.1f}")

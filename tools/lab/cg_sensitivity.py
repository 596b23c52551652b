"""State error vs the oracle of the colour/wall-model test scenario (c3_mesh(0.06), 2 steps, 40 CG iterations)
for the CG forms: how much of the ~1e-8 is CG rounding amplification."""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2])); sys.path.insert(0, str(Path(__file__).resolve().parents[2] / "tests"))
import numpy as np, torch
from oracle import fem
from paper_2005_05899_b200 import meshgen
from paper_2005_05899_b200.timestep import FlowParams, FlowSolver
import test_gpu_colour as T
CGI = int(os.environ.get("CGI", "40"))
m = meshgen.c3_mesh(0.06)
bc, wall = meshgen.wall_model_bcs(m)
u, p = T._field(m, 6)
params = dict(rho=1.0, mu=0.01, c_vreman=0.07)
ora = fem.FlowOracle(m, **params, **bc, wall=wall)
st = ora.init_state(u, p)
for _ in range(2):
    st = ora.step(st, 2e-3, cg_iters=CGI)
rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)
for name, env in (("single-pass", {}), ("two-pass-tiled", {"AB_CG_SINGLE_PASS": "0"}), ("two-pass-untiled", {"AB_CG_SINGLE_PASS": "0", "AB_CG_TILE": "0"})):
    for k in ("AB_CG_SINGLE_PASS", "AB_CG_TILE"):
        os.environ.pop(k, None)
    os.environ.update(env)
    for scatter in ("colour", "atomic"):
        fs = FlowSolver(m, FlowParams(**params), **bc, wall=wall, scatter=scatter)
        fs.set_state(u, p)
        for _ in range(2):
            fs.step(2e-3, cg_iters=CGI, graph=True)
        torch.cuda.synchronize()
        print(name, scatter, "resident" if fs.pcg.resident else "perm2", "N", m.n_nodes,
              "u %.2e p %.2e" % (rel(fs.u.cpu().numpy(), st["u"]), rel(fs.p.cpu().numpy(), st["p"])), flush=True)

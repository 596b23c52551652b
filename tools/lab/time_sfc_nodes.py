"""Would numbering the nodes of C2 in Hilbert order help?  Times the full
graph-replayed step (L2 flushed, as bench.py) and K2 on the generator's node
numbering and on the same mesh with SFC-renumbered nodes (lab experiment)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np, torch  # noqa: E401,E402
from paper_2005_05899_b200 import meshgen  # noqa: E402
from paper_2005_05899_b200.device import DeviceMesh  # noqa: E402
from paper_2005_05899_b200.timestep import FlowParams, FlowSolver  # noqa: E402

m = meshgen.box_tets(88, 88, 88, jitter=0.2, seed=20200131)
u, p = meshgen.c2_initial(m.coords)
bnd = meshgen.boundary_nodes(m)
perm = DeviceMesh(m).node_order().cpu().numpy().astype(np.int64)   # new id -> old id
inv = np.empty_like(perm)
inv[perm] = np.arange(len(perm))
m2 = meshgen.MeshArrays(coords=m.coords[perm], conn={k: inv[v].astype(np.int32) for k, v in m.conn.items()},
                        elem_ids=dict(m.elem_ids), period=m.period)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for name, mm, uu, pp, bb in (("generator order", m, u, p, bnd), ("SFC order", m2, u[perm], p[perm], bnd[perm])):
    fs = FlowSolver(mm, FlowParams(1.0, 1e-3, 0.07), p_fixed=bb)
    fs.set_state(uu, pp)
    fs.step(1e-3, 50, graph=True)
    torch.cuda.synchronize()
    ts = []
    for _ in range(7):
        flush.zero_()
        a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fs.step(1e-3, 50, graph=True); c.record(); c.synchronize()
        ts.append(a.elapsed_time(c))
    print(f"{name:16s}: step {np.median(ts) * 1e3:.1f} us", flush=True)

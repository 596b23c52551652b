"""Colour-mode K2 reproducibility probe: runs K2 several times on a 384k-tet
box and reports how many node values differ between runs, and whether the
differing nodes sit in blocks of one or several colours.

    [AB_COLOUR_SPLIT=1] python tools/lab/colour_debug.py
"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np, torch  # noqa: E401,E402
from paper_2005_05899_b200 import meshgen  # noqa: E402
from paper_2005_05899_b200.device import DeviceMesh  # noqa: E402
from paper_2005_05899_b200.ops import assemble_momentum  # noqa: E402
from paper_2005_05899_b200.timestep import FlowParams  # noqa: E402

m = meshgen.box_tets(40, 40, 40, jitter=0.2, seed=5)
rng = np.random.default_rng(0)
u = rng.standard_normal((m.n_nodes, 3))
dm = DeviceMesh(m, reorder="sfc", windows=True, scatter="colour")
ph = FlowParams(rho=1.3, mu=0.01, c_vreman=0.0)
runs = [assemble_momentum(dm, u, ph).cpu().numpy() for _ in range(6)]
diff = np.zeros(m.n_nodes, bool)
for r in runs[1:]:
    diff |= (r != runs[0]).any(axis=1)
print("colours", dm.colour_stats()["tet4"]["colours"], "blocks", len(dm._col[0][4]), "differing nodes", int(diff.sum()),
      "of", m.n_nodes, flush=True)
blk_ptr, wnode = dm._win[0][0].cpu().numpy(), dm._win[0][1].cpu().numpy()
colour = dm._col[0][4].cpu().numpy()
nb = len(blk_ptr) - 1
wb = np.repeat(np.arange(nb), np.diff(blk_ptr))
wn = wnode[:blk_ptr[-1]]
bad = np.nonzero(diff)[0][:10]
for n in bad:
    bl = wb[wn == n]
    print("node", n, "blocks", bl.tolist(), "colours", colour[bl].tolist())
# per-node number of blocks and colours for all nodes
nblk = np.bincount(wn, minlength=m.n_nodes)
print("differing nodes by #blocks:", np.bincount(nblk[diff]).tolist(), " all:", np.bincount(nblk).tolist())

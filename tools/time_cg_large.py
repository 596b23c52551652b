"""Large single-domain scaled CG variants on a jittered tet box: device time
per iteration (CUDA graph of a 50-iteration solve, L2 flushed before every
solve, as in bench.py) and the relative difference of the solutions from the
first variant.

    python tools/time_cg_large.py [cells=200] [variants=two-pass,tile4096,...]

variants: two-pass (ab_cg_spmv_unit + ab_cg_update_scaled), tile<R>
(ab_cg_spmv_tile with R rows per tile + ab_cg_update_scaled), sptile<R> (the
tiled single pass, ab_cg_tile_iter).  The rejected
single-pass form is tools/lab/cg_single_pass.cu.
"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch  # noqa: E401,E402
from paper_2005_05899_b200 import meshgen  # noqa: E402
from paper_2005_05899_b200.device import DeviceMesh  # noqa: E402
from paper_2005_05899_b200.solver import PCG, assemble_laplacian  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
names = sys.argv[2].split(",") if len(sys.argv) > 2 else ["two-pass", "tile2048", "tile4096", "tile8192"]
its = 50
m = meshgen.box_tets(n, n, n, jitter=0.2, seed=20200131)
fixed = torch.from_numpy(meshgen.boundary_nodes(m))
dm = DeviceMesh(m)
A = assemble_laplacian(dm, fixed)
dinv = 1.0 / A.diag
N, Z = A.n_rows, A.nnz
g = torch.Generator(device="cuda").manual_seed(7)
b = torch.randn(N, dtype=torch.float64, device="cuda", generator=g)
b[fixed.cuda()] = 0
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
order = dm.node_order()
del dm, m
ref = None
for name in names:
    kw = dict(tile_rows=int(name.split("tile")[1]) if "tile" in name else 0, single_pass=name.startswith("sp"))
    pcg = PCG(A, dinv, fixed=fixed, order=order, resident=False, **kw)
    info = ""
    if pcg.perm2.get("tile") is not None:
        info = f"max_ghost={pcg.perm2['tile']['max_ghost']} ghosts/row={pcg.perm2['tile']['ghost'].numel() / N:.3f}"
    elif name.startswith("tile"):
        info = "(tile map did not fit: untiled)"
    x, _ = pcg.solve(b.clone(), its, zero_b=False)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        x, _ = pcg.solve(b, its, zero_b=False)
    ts = []
    for _ in range(8):
        flush.zero_()
        a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); gr.replay(); c.record(); c.synchronize()
        ts.append(a.elapsed_time(c))
    xs = x.cpu().numpy().copy()
    if ref is None:
        ref = xs
    d = np.linalg.norm(xs - ref) / np.linalg.norm(ref)
    us = np.median(ts) * 1e3 / its
    print(f"{name:12s} N={N} Z={Z}: {us:8.2f} us/iteration (min {min(ts) * 1e3 / its:8.2f}) "
          f"rel.diff={d:.2e} {info}", flush=True)
    del pcg, gr
    torch.cuda.empty_cache()

"""Device time of K2/K4/K6 per scatter mode (CUDA graph of 10 launches).

    AB_MODES=direct,window,pipelined,colour  AB_MESH=c2 | c3:<scale>  python tools/time_elements.py
"""
import ctypes
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch  # noqa: E401,E402
from paper_2005_05899_b200 import meshgen  # noqa: E402
from paper_2005_05899_b200._lib import call, ptr, stream_handle  # noqa: E402
from paper_2005_05899_b200.device import DeviceMesh  # noqa: E402
from paper_2005_05899_b200.timestep import FlowParams  # noqa: E402

import os
spec = os.environ.get("AB_MESH", "c2")
m = meshgen.c2_mesh() if spec == "c2" else meshgen.c3_mesh(float(spec.split(":")[1]))
u = torch.randn((m.n_nodes, 4), dtype=torch.float64, device="cuda")
p = torch.randn(m.n_nodes, dtype=torch.float64, device="cuda")
out4 = torch.zeros_like(u)
out1 = torch.zeros_like(p)
import os
cv = float(os.environ.get("AB_CVREMAN", "0.07"))
ph = FlowParams(1.0, 1e-3, cv).struct()
modes = os.environ.get("AB_MODES", "direct,window,pipelined").split(",")
for mode in modes:
    dm = DeviceMesh(m, reorder="sfc", windows=mode != "direct", pipelined=mode in ("pipelined", "colour"),
                    scatter="colour" if mode == "colour" else "atomic")
    res = {}
    for name, fn in (("K2", lambda: call("ab_momentum_rhs", ctypes.byref(dm.struct), ctypes.byref(ph), ptr(u),
                                         ptr(out4), stream_handle())),
                     ("K4", lambda: call("ab_divergence", ctypes.byref(dm.struct), ptr(u), 1.0, ptr(out1),
                                         stream_handle())),
                     ("K6", lambda: call("ab_gradient", ctypes.byref(dm.struct), ptr(p), 1.0, ptr(out4),
                                         stream_handle()))):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(10):
                fn()
        ts = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); g.replay(); b.record(); b.synchronize()
            ts.append(a.elapsed_time(b) * 100)
        res[name] = round(float(np.median(ts)), 1)
    extra = {k: v["colours"] for k, v in dm.colour_stats().items()} if mode == "colour" else ""
    print(mode, res, extra or (dm.window_stats() if mode != "direct" else ""), flush=True)
    del dm

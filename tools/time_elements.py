"""Device time of K2/K4/K6 on C2 per scatter mode (CUDA graph of 10 launches)."""
import ctypes
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch  # noqa: E401,E402
from paper_2005_05899_b200 import meshgen  # noqa: E402
from paper_2005_05899_b200._lib import call, ptr, stream_handle  # noqa: E402
from paper_2005_05899_b200.device import DeviceMesh  # noqa: E402
from paper_2005_05899_b200.timestep import FlowParams  # noqa: E402

m = meshgen.c2_mesh()
u = torch.randn((m.n_nodes, 4), dtype=torch.float64, device="cuda")
p = torch.randn(m.n_nodes, dtype=torch.float64, device="cuda")
out4 = torch.zeros_like(u)
out1 = torch.zeros_like(p)
import os
cv = float(os.environ.get("AB_CVREMAN", "0.07"))
ph = FlowParams(1.0, 1e-3, cv).struct()
modes = os.environ.get("AB_MODES", "direct,window,pipelined").split(",")
for mode in modes:
    dm = DeviceMesh(m, reorder="sfc", windows=mode != "direct", pipelined=mode == "pipelined")
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
    print(mode, res, dm.window_stats() if mode != "direct" else "")

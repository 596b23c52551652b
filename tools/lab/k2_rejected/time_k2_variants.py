"""K2 on C2: warp-window kernel vs the pipelined CTA-window kernel —
agreement of the assembled RHS and device time (CUDA graph of 10 launches).

    python tools/time_k2_warp.py [n]
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

n = int(sys.argv[1]) if len(sys.argv) > 1 else 88
m = meshgen.box_tets(n, n, n, jitter=0.2, seed=20200131)
torch.manual_seed(0)
u = torch.randn((m.n_nodes, 4), dtype=torch.float64, device="cuda")
ph = FlowParams(1.0, 1e-3, 0.07).struct()
res = {}
modes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["pipe", "pipe1", "warp"]
for mode in modes:
    call("ab_set_k2_variant", 1 if mode == "pipe1" else 0)
    dm = DeviceMesh(m, reorder="sfc", windows=True, pipelined=True, warp_windows=mode == "warp")
    out = torch.zeros_like(u)

    def fn():
        call("ab_momentum_rhs", ctypes.byref(dm.struct), ctypes.byref(ph), ptr(u), ptr(out), stream_handle())
    fn()
    torch.cuda.synchronize()
    res[mode] = out.clone()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(10):
            fn()
    ts = []
    for _ in range(7):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b) * 100)
    extra = ""
    if mode == "warp":
        w = dm._wwin[0]
        extra = f"wcap {w[5]} window nodes/element {w[6] / dm.conn[0].shape[0]:.3f}"
    print(mode, f"{np.median(ts):.1f} us", extra, flush=True)
a = res[modes[0]][:, :3]
for mode in modes[1:]:
    b = res[mode][:, :3]
    print(f"rel L2 {mode} vs {modes[0]}", float(torch.linalg.norm(a - b) / torch.linalg.norm(a)))
call("ab_set_k2_variant", 0)

"""Time SpMV variants on the C2 pressure Laplacian (lab; not product code).

    python tools/lab/run_lab.py
"""
import ctypes
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

LIB = HERE / "liblab.so"
if not LIB.exists() or LIB.stat().st_mtime < (HERE / "spmv_lab.cu").stat().st_mtime:
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                           "-Xcompiler", "-fPIC", "-shared", "-o", str(LIB), str(HERE / "spmv_lab.cu")])
lab = ctypes.CDLL(str(LIB))

from paper_2005_05899_b200 import meshgen  # noqa: E402
from paper_2005_05899_b200._lib import call, ptr, stream_handle  # noqa: E402
from paper_2005_05899_b200.solver import PCG, assemble_laplacian  # noqa: E402

m = meshgen.c2_mesh()
fixed = torch.from_numpy(meshgen.boundary_nodes(m))
A = assemble_laplacian(m, fixed)
n = A.n_rows
nnz = A.nnz
ne = A.vals.numel()
print(f"n={n} nnz={nnz} stored={ne} max_width={A.max_width}")
zp = torch.randn((n, 2), dtype=torch.float64, device="cuda")
x = torch.randn(n, dtype=torch.float64, device="cuda")
q = torch.empty(n, dtype=torch.float64, device="cuda")
out = torch.zeros(1, dtype=torch.float64, device="cuda")
s = ctypes.c_void_p(stream_handle())
flush = torch.empty(1 << 27, dtype=torch.float32, device="cuda")


def timeit(fn, reps=20, cold=False):
    """Device time per launch: a spin kernel keeps the GPU busy while the
    host enqueues, so launches run back to back between the events."""
    fn()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    torch.cuda._sleep(int(2e7))
    for a, b in evs:
        if cold:
            flush.fill_(1.0)
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) * 1e3 for a, b in evs]))


mat_bytes = ne * 12
alg = 12 * nnz + 32 * n
res = {}
for grid, block in ((148 * 8, 256), (148 * 32, 256), (148 * 64, 128)):
    t = timeit(lambda: lab.lab_stream(ctypes.c_int64(ne), ctypes.c_void_p(ptr(A.cols)), ctypes.c_void_p(ptr(A.vals)),
                                      ctypes.c_void_p(ptr(out)), grid, block, s), cold=True)
    print(f"stream grid={grid} block={block}: {t:.1f} us  {mat_bytes / t / 1e3:.0f} GB/s")
for unroll in (4, 8, 16):
    for grid, block in (((n + 255) // 256, 256), (148 * 6, 256), (148 * 12, 128)):
        t = timeit(lambda: lab.lab_spmv_batch(unroll, ctypes.c_int64(n), ctypes.c_void_p(ptr(A.slice_ptr)),
                                              ctypes.c_void_p(ptr(A.cols)), ctypes.c_void_p(ptr(A.vals)),
                                              ctypes.c_void_p(ptr(zp)), ctypes.c_double(0.5), ctypes.c_void_p(ptr(q)),
                                              grid, block, s), cold=True)
        t2 = timeit(lambda: lab.lab_spmv_x(unroll, ctypes.c_int64(n), ctypes.c_void_p(ptr(A.slice_ptr)),
                                           ctypes.c_void_p(ptr(A.cols)), ctypes.c_void_p(ptr(A.vals)),
                                           ctypes.c_void_p(ptr(x)), ctypes.c_void_p(ptr(q)), grid, block, s),
                    cold=True)
        print(f"spmv pair unroll={unroll} grid={grid} block={block}: {t:.1f} us ({alg / t / 1e3:.0f} GB/s alg) | "
              f"x-only {t2:.1f} us")
# product kernels
pcg = PCG(A, 1.0 / A.diag, fixed=fixed)
b = torch.randn(n, dtype=torch.float64, device="cuda")
pcg.solve(b.clone(), 2)
for staged in (False,):
    t = timeit(lambda: call("ab_cg_spmv", ctypes.byref(A.struct), ptr(pcg.zpa), ptr(pcg.zpb), ptr(pcg.q), 1, None,
                            ptr(pcg.red), ptr(pcg.sc), ptr(pcg.part), ptr(pcg.cnt), stream_handle()), cold=True)
    print(f"product ab_cg_spmv: {t:.1f} us ({alg / t / 1e3:.0f} GB/s alg)")
t = timeit(lambda: call("ab_cg_update", n, ptr(pcg.zpb), ptr(pcg.q), ptr(pcg.dinv), ptr(pcg.x), ptr(pcg.r), None,
                        ptr(pcg.red), ptr(pcg.sc), ptr(pcg.part), ptr(pcg.cnt), stream_handle()), cold=True)
print(f"product ab_cg_update: {t:.1f} us ({64 * n / t / 1e3:.0f} GB/s alg)")
t = timeit(lambda: call("ab_cg_update", n, ptr(pcg.zpb), ptr(pcg.q), ptr(pcg.dinv), ptr(pcg.x), ptr(pcg.r), None,
                        ptr(pcg.red), ptr(pcg.sc), ptr(pcg.part), ptr(pcg.cnt), stream_handle()), cold=False)
print(f"product ab_cg_update warm: {t:.1f} us ({64 * n / t / 1e3:.0f} GB/s alg)")
t = timeit(lambda: call("ab_cg_dot", n, ptr(pcg.zpb), ptr(pcg.q), None, ptr(pcg.red), ptr(pcg.sc), ptr(pcg.part),
                        ptr(pcg.cnt), stream_handle()), cold=False)
print(f"product ab_cg_dot warm: {t:.1f} us ({24 * n / t / 1e3:.0f} GB/s alg)")
t = timeit(lambda: call("ab_rk_stage", n, 0.5, 0.5, 0.1, ptr(pcg.zpa), ptr(pcg.zpb), ptr(pcg.zpa), ptr(pcg.zpb),
                        ptr(pcg.dinv), ptr(pcg.zpb), stream_handle()), cold=False)
print(f"product ab_rk_stage (n/2 nodes) warm: {t:.1f} us")
pp = torch.randn(n, dtype=torch.float64, device="cuda")
qq = torch.randn(n, dtype=torch.float64, device="cuda")
part = torch.zeros(1 << 16, dtype=torch.float64, device="cuda")
cnt = torch.zeros(4096, dtype=torch.int32, device="cuda")
red = torch.zeros(8, dtype=torch.float64, device="cuda")
for block in (256, 1024):
    for grid in ((n + block - 1) // block, 148 * (2048 // block), 148):
        for mode in (0, 1, 2):
            t = timeit(lambda: lab.lab_dot(mode, block, ctypes.c_int64(n), ctypes.c_void_p(ptr(pp)),
                                           ctypes.c_void_p(ptr(qq)), ctypes.c_void_p(ptr(red)),
                                           ctypes.c_void_p(ptr(part)), ctypes.c_void_p(ptr(cnt)), grid, s))
            print(f"dot block={block} grid={grid} mode={['partial', 'grid_sum', 'fence'][mode]}: {t:.1f} us "
                  f"({16 * n / t / 1e3:.0f} GB/s)")

"""Benchmark of the time-step hot path (BASELINE.json metric: M element-steps/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c4|c5|c3|c2] [--weak]
                    [--impl native|reference]

A "step" is one full fractional time step (Algorithm 1: 3 x (K2 + K8 wall
model + K3), K4, PCG with a fixed 50 iterations, K6 + K7) over the whole
mesh; the unit of work is one element through one step.

Default workload: C4 (BASELINE configs[3], the config the metric's 1/2/4/8
quotes): the ~249M-element mixed tet/prism/pyramid/hex boundary-layer box.
N = 1 runs it on one GPU (68 GB of HBM); N > 1 (torchrun, one rank per GPU)
runs STRONG scaling: the cells are split along a Hilbert curve
(dmesh.partition_cells, the reference's split_1d rule on cell bins) and every
rank generates only its own subdomain; after one calibration the split is
re-done with lambda_i = P theta_i / sum(theta) from the measured K2
throughput (the paper's DLB analog).  ``--weak`` runs C5 (BASELINE
configs[4]: 150 x 150 x (237 P + 21) cells, ~32M elements per GPU).
``--workload c2`` keeps round 1's C2 line (4.09M jittered tets).

Timing: W untimed warm-up steps; K timed steps, each bracketed by CUDA events
on the launching stream, with a 512 MB L2 flush (untimed) between steps;
barrier + synchronize on both sides; max over ranks.  The per-kernel
breakdown and roofline come from one instrumented (eager) step afterwards.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CG_ITERS = 50
DT = 1e-3
L2_FLUSH_BYTES = 512 << 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--workload", default="c4", choices=["c2", "c3", "c4", "c5"])
    ap.add_argument("--weak", action="store_true", help="weak scaling: C5 (32M elements per GPU)")
    ap.add_argument("--no-c2", action="store_true", help="N=1: skip the extra C2 reference point")
    ap.add_argument("--cg-iters", type=int, default=CG_ITERS)
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-windows", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-rebalance", action="store_true",
                    help="N>1: skip the throughput-weighted repartitioning (DLB analog)")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


PHYS = dict(rho=1.0, mu=1e-3, c_vreman=0.07)


def workload_spec(name: str, n_ranks: int):
    """(BoxSpec, description, scaling) of a boundary-layer workload."""
    from paper_2005_05899_b200 import dmesh
    if name == "c4":
        return (dmesh.c4_spec(), "C4: ~250M-element mixed tet/prism/pyramid/hex boundary-layer box "
                                 "(BASELINE configs[3]), strong scaling", "strong")
    if name == "c5":
        return (dmesh.c5_spec(n_ranks), "C5: ~32M mixed elements per GPU, throughput-weighted repartitioning "
                                        "(BASELINE configs[4]), weak scaling", "weak")
    return (dmesh.c3_spec(n_ranks ** (1.0 / 3.0)),
            "C3: mixed tet/prism/pyramid/hex boundary-layer box (BASELINE configs[2]), scaled by P^(1/3)", "weak")


def build_rank_workload(name: str, ws: int, rank: int, coeffs=None, device="cuda"):
    """This rank's subdomain and inputs.  Boundary-layer workloads (C3/C4/C5):
    the rank generates only its own cells (dmesh.local_mesh); C2: the global
    jittered box, decomposed by decompose.py (weak scaling, round-1 path)."""
    from paper_2005_05899_b200 import dmesh, meshgen
    if name == "c2":
        n = 88
        mesh = meshgen.box_tets(n * ws, n, n, lengths=(float(ws), 1.0, 1.0), jitter=0.2, seed=20200131)
        u, p = meshgen.c2_initial(mesh.coords)
        bc = dict(p_fixed=meshgen.boundary_nodes(mesh))
        desc = {"workload": "C2: jittered Kuhn TET04 box (BASELINE configs[1])", "cells": [n * ws, n, n],
                "nodes": mesh.n_nodes}
        w = dict(sub=mesh, u=u, p=p, bc=bc, wall=None, desc=desc, plan=None, scaling="weak", weights=None)
        if ws > 1:
            from paper_2005_05899_b200.decompose import decompose
            from paper_2005_05899_b200.partition import sfc_partition
            parts, _cuts, subw = sfc_partition(mesh, ws, coeffs=coeffs, level=8)
            sub, plan = decompose(mesh, parts, ws, rank)
            l2g = plan.l2g
            w.update(sub=sub, u=u[l2g], p=p[l2g], bc={k: np.asarray(v)[l2g] for k, v in bc.items()}, plan=plan,
                     weights=subw)
        return w
    spec, text, scaling = workload_spec(name, ws)
    part = dmesh.partition_cells(spec, ws, coeffs=coeffs, device=device)
    sub, plan = dmesh.local_mesh(spec, part, rank)
    weights = part.weights
    del part
    bc, wall = dmesh.wall_model_bcs_local(sub, spec)
    u = np.zeros((sub.n_nodes, 3))
    u[:, 0] = 1.0
    desc = {"workload": text, "cells": [spec.nx, spec.ny, spec.nz], "prism_layers": spec.layers,
            "nodes": spec.n_nodes,
            "wall": "equilibrium wall model (Reichardt) on z = 0, K8 per RK stage",
            "decomposition": ("per-rank generation of Hilbert-ordered cell ranges (dmesh.py)" if ws > 1 else None)}
    return dict(sub=sub, u=u, p=np.zeros(sub.n_nodes), bc=bc, wall=wall, desc=desc,
                plan=plan if ws > 1 else None, scaling=scaling, weights=weights)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def algorithmic_cost(kernel: str, counts: dict, n_nodes: int, nnz: int, cg_iters: int = CG_ITERS,
                     n_faces: int = 0, unit_diag: bool = False):
    """Algorithmic bytes (and flops for K2) per launch, layout-independent
    (SURVEY §8(d) per-unit figures): int32 indices, fp64 values."""
    from paper_2005_05899_b200.meshgen import NODE_COUNT, RULE_KIND
    conn_bytes = sum(4 * NODE_COUNT[RULE_KIND[r]] * e for r, e in counts.items())
    N = n_nodes
    if kernel in ("K5_cg_resident", "K5_cg_fused_dd"):  # SURVEY §8(d) K5 per iteration: 12Z + 4(N+1) + 104N
        return cg_iters * (12 * nnz + 4 * (N + 1) + 104 * N), cg_iters * (2 * nnz + 12 * N)
    if kernel == "K5_cg_spmv":      # vals+cols, z gathered once, p & q read + written
        if unit_diag:  # scaled form: the unit diagonal of D^-1/2 A D^-1/2 is implicit (never read)
            return 12 * (nnz - N) + 8 * N + 32 * N, 2 * nnz + 4 * N
        return 12 * nnz + 8 * N + 32 * N, 2 * nnz + 4 * N
    if kernel == "K5_cg_tile_iter":  # one whole CG iteration (SURVEY §8(d) K5 per iteration)
        return 12 * nnz + 4 * (N + 1) + 104 * N, 2 * nnz + 12 * N
    if kernel == "K5_cg_dot":       # z t p q in, p q out
        return 48 * N, 6 * N
    if kernel == "K5_cg_update":    # x p r q dinv in, x r z out
        return 64 * N, 10 * N
    if kernel == "K5_cg_update_scaled":  # symmetrically scaled form: x p r q in, x r out (no z, no D^-1)
        return 48 * N, 8 * N
    if kernel == "K2_momentum":     # conn, coords, u in; rhs out
        return conn_bytes + 48 * N + 24 * N, sum(FLOPS_K2.get(r, 0) * e for r, e in counts.items())
    if kernel == "K3_rk_stage":     # u0 uprev rhs gp in (24 B each), minv, uout + rhs zero out
        return 4 * 24 * N + 8 * N + 48 * N, 12 * N
    if kernel == "K4_divergence":   # (computed as the product B . u; algorithmic bytes stay the element form's)
        return conn_bytes + 48 * N + 8 * N, 0
    if kernel == "K6_gradient":
        return conn_bytes + 24 * N + 8 * N + 24 * N, 0
    if kernel == "K7_correct":
        return 24 * 3 * N + 8 * N + 16 * N + 24 * 3 * N, 6 * N
    if kernel == "K8_wall":           # per face: 8 node ids, <= 8 coordinates, 4 exchange velocities, 4 rhs RMW
        return n_faces * (32 + 8 * 24 + 4 * 24 + 4 * 48), 0
    if kernel == "K67_grad_correct":  # K6 + K7 without the G dp round trip
        return conn_bytes + 24 * N + 8 * N + 24 * N + 8 * N + 16 * N + 48 * N + 24 * N, 6 * N
    return 0, 0


# fp64 flops per element of K2 as the kernel executes them: ncu thread
# instructions 2 x DFMA + DMUL + DADD per element of each category
# (profiles/r2_c4_ncu.md, one C4 step; tet4 also r1g on C2: 417.8)
FLOPS_K2 = {"tet4": 416.7, "pri6": 3867.9, "hex8": 6461.1, "pyr5": 2821.3}


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


def load_fp64_peak():
    """Measured FP64 FMA peak (tools/lab/fp64_peak.cu -> profiles/fp64_peak.json)."""
    p = ROOT / "profiles" / "fp64_peak.json"
    try:
        return float(json.loads(p.read_text())["fp64_fma_tflops"]), "measured (tools/lab/fp64_peak.cu)"
    except Exception:
        return 37.0, "nominal"


def load_traffic(workload: str = "c2"):
    """ncu DRAM bytes per launch of the step kernels of this workload
    (profiles/ncu_traffic_c4.json for C4, profiles/ncu_traffic.json for C2)."""
    p = ROOT / "profiles" / ("ncu_traffic_c4.json" if workload == "c4" else "ncu_traffic.json")
    if p.exists():
        try:
            d = json.loads(p.read_text())
            return d.get("traffic", d)
        except Exception:
            return {}
    return {}


def host_cpu() -> dict:
    """CPU model and logical core count of the host."""
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


def cpu_sample(workload: str, scale: float, seed: int = 0, c_threads: int | None = None):
    """(oracle, initial state, element count, description) of a bounded CPU
    sample of the workload: the same recipe at a smaller size (boundary-layer
    box with the wall model for C3/C4/C5, a jittered Kuhn box for C2).
    ``c_threads`` not None: the C + OpenMP restatement (oracle/fem_c.c) on that
    many threads (0 = all cores) instead of the numpy oracle; setup (lumped
    mass, Laplacian) is numpy either way and untimed."""
    from oracle import fem
    from paper_2005_05899_b200 import dmesh, meshgen
    if c_threads is not None:
        from oracle import femc
        mk = lambda *a, **k: femc.CFlowOracle(*a, **k, threads=c_threads)  # noqa: E731
    else:
        mk = fem.FlowOracle
    if workload == "c2":
        n = max(4, int(round(88 * scale)))
        m = meshgen.box_tets(n, n, n, jitter=0.2, seed=20200131 + seed)
        u, p = meshgen.c2_initial(m.coords)
        o = mk(m, **PHYS, p_fixed=meshgen.boundary_nodes(m))
        return o, o.init_state(u, p), m.n_elements, f"jittered Kuhn TET04 {n}^3 cells"
    spec = dmesh.c3_spec(scale)
    m = spec.global_mesh()
    bc, wall = meshgen.wall_model_bcs(m)
    u = np.zeros((m.n_nodes, 3))
    u[:, 0] = 1.0
    o = mk(m, **PHYS, **bc, wall=wall)
    return (o, o.init_state(u, np.zeros(m.n_nodes)), m.n_elements,
            f"mixed boundary-layer box {spec.nx}x{spec.ny}x{spec.nz} cells, {spec.layers} prism layers, wall model "
            "(the C3/C4 recipe at reduced size)")


# sample sizes of the CPU legs: the C restatement on all host cores needs a larger sample than numpy on one core
# for ~10-30 s of CPU work with a few steps
C_SCALE = {"c2": 48 / 88, "other": 0.25}


def cpu_baseline_sample(workload: str = "c4", steps: int = 20):
    """The C + OpenMP restatement of the step (oracle/fem_c.c) on all host
    cores, on a bounded sample of the workload; the single-thread numpy oracle
    on a smaller sample is reported beside it."""
    from oracle import femc
    femc.build()
    o, st, n_el, what = cpu_sample(workload, C_SCALE["c2" if workload == "c2" else "other"], c_threads=0)
    st = o.step(st, DT, cg_iters=CG_ITERS)  # warm-up
    t0 = time.perf_counter()
    for _ in range(steps):
        st = o.step(st, DT, cg_iters=CG_ITERS)
    dt = time.perf_counter() - t0
    out = {"value": n_el * steps / dt / 1e6, "unit": "M element-steps/s", "cores": o.threads, "kind": "port",
           "sample": f"oracle/fem_c.c (C + OpenMP restatement of oracle/fem.py FlowOracle.step), {what} "
                     f"({n_el} elements), {steps} full steps (CG {CG_ITERS} it), {o.threads} threads",
           **host_cpu()}
    del o
    from threadpoolctl import threadpool_limits
    with threadpool_limits(1):
        o, st, n_el, what = cpu_sample(workload, 0.12 if workload != "c2" else 24 / 88)
        st = o.step(st, DT, cg_iters=CG_ITERS)
        t0 = time.perf_counter()
        o.step(st, DT, cg_iters=CG_ITERS)
        dt = time.perf_counter() - t0
    out["numpy_oracle_1core"] = {"value": n_el / dt / 1e6, "sample": f"oracle/fem.py FlowOracle, {what} ({n_el} "
                                 "elements), 1 full step, numpy single thread"}
    return out


KINDS = ("hex8", "pri6", "pyr5", "tet4")


def _kind_counts(solver) -> dict:
    c = solver.dm.element_counts()
    return {k: c.get(k, 0) for k in KINDS}


def _max_over_ranks(v: float, backend: str) -> float:
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(v)], dtype=torch.float64, device="cuda" if backend == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_native(args):
    import torch
    import torch.distributed as dist
    from paper_2005_05899_b200 import _lib
    from paper_2005_05899_b200.timestep import FlowParams, FlowSolver

    ws, rank, local = dist_env()
    if args.gpus != ws and ws > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {ws}")
    # AB_DIST_BACKEND=gloo runs several ranks on one GPU (exchange staged
    # through the host): a functional check of this multi-rank path only
    backend = os.environ.get("AB_DIST_BACKEND", "nccl")
    if backend != "nccl":
        local = 0
    torch.cuda.set_device(local)
    if ws > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    name = "c5" if args.weak else args.workload
    params = PHYS
    rebalance = None

    def make_solver(coeffs=None):
        w = build_rank_workload(name, ws, rank, coeffs=coeffs)
        halo = None
        if w["plan"] is not None:
            if os.environ.get("AB_PEER", "1") == "1":
                # interface sums over peer memory (CUDA IPC over NVLink), graph-capturable
                from paper_2005_05899_b200.peer import PeerHalo
                halo = PeerHalo.connect(w["plan"], "cuda")
            else:  # AB_PEER=0: NCCL grouped send/recv (host-driven)
                from paper_2005_05899_b200.halo import HaloExchanger
                halo = HaloExchanger(w["plan"], "cuda")
        # AB_FUSED_CG=1 forces the fused decomposed CG also on gloo (ranks sharing one GPU)
        fused = True if (halo is not None and os.environ.get("AB_FUSED_CG") == "1") else None
        s_ = FlowSolver(w["sub"], FlowParams(**params), **w["bc"], windows=not args.no_windows, reorder="sfc",
                        wall=w["wall"], halo=halo, own=halo.own if halo is not None else None, fused_cg=fused)
        s_.set_state(w["u"], w["p"])
        return s_, w

    solver, wl = make_solver()
    if ws > 1 and not args.no_rebalance:
        from paper_2005_05899_b200.balance import distributed_timer, throughput_coefficients
        # DLB analog: lambda_i = P theta_i / sum(theta) from
        # each rank's measured K2 throughput, one re-split, rebuild
        sample = distributed_timer(solver)
        subw = wl["weights"]
        lam = throughput_coefficients(sample.times, subw)
        del solver
        torch.cuda.synchronize()
        solver, wl = make_solver(coeffs=lam)
        rebalance = {"k2_seconds_before": [float(t) for t in sample.times], "lambda": [float(x) for x in lam],
                     "weights_before": [float(x) for x in subw], "weights_after": [float(x) for x in wl["weights"]]}
    desc = dict(wl["desc"])
    n_local = solver.dm.n_elements
    counts_t = torch.tensor([n_local] + [c for c in _kind_counts(solver).values()], dtype=torch.float64,
                            device="cuda" if backend == "nccl" else "cpu")
    if ws > 1:
        dist.all_reduce(counts_t)
    n_elem_total = int(counts_t[0].item())
    desc["elements"] = n_elem_total
    desc["kinds"] = {k: int(v) for k, v in zip(_kind_counts(solver).keys(), counts_t[1:].tolist())}
    if ws > 1:
        desc["elements_per_rank_max"] = _max_over_ranks(n_local, backend)
    graph = (not args.no_graph) and solver.graph_safe
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")

    for _ in range(args.warmup):
        solver.step(DT, args.cg_iters, graph=graph)
    torch.cuda.synchronize()

    # launches of this library per step (eager count; graph replays the same)
    c0 = _lib.launch_count()
    solver._step_body(DT, args.cg_iters, 0.0) if not graph else solver.capture(DT, args.cg_iters)
    torch.cuda.synchronize()
    launches_per_step = (_lib.launch_count() - c0) // (2 if graph else 1)

    clocks = ClockSampler(local)
    clocks.start()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    total_ms = 0.0
    for _ in range(args.steps):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        solver.step(DT, args.cg_iters, graph=graph)
        b.record()
        b.synchronize()
        total_ms += a.elapsed_time(b)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    clk = clocks.stop()
    t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = n_elem_total * args.steps / (total_ms / 1e3) / 1e6

    # end-to-end through the public API with host buffers
    u_h = torch.empty((solver.n, 3), dtype=torch.float64, pin_memory=True)
    p_h = torch.empty(solver.n, dtype=torch.float64, pin_memory=True)
    u_h.copy_(solver.u)
    p_h.copy_(solver.p)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    e2e_ms = 0.0
    for _ in range(args.steps):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        solver.step_host(u_h, p_h, DT, args.cg_iters, graph=graph)
        b.record()
        b.synchronize()
        e2e_ms += a.elapsed_time(b)
    te = torch.tensor([e2e_ms], dtype=torch.float64, device="cuda")
    if ws > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_ms = float(te.item())
    bytes_io = (u_h.numel() + p_h.numel()) * 8

    # instrumented eager step: per-kernel durations
    solver.timeline = []
    flush.fill_(1.0)
    solver._step_body(DT, args.cg_iters, 0.0)
    torch.cuda.synchronize()
    per = {}
    for kname, a, b in solver.timeline:
        per.setdefault(kname, []).append(a.elapsed_time(b) / 1e3)
    solver.timeline = None
    counts = solver.dm.element_counts()
    nnz = solver.L.nnz
    kern = {}
    for kname, ts in per.items():
        B, F = algorithmic_cost(kname, counts, solver.n, nnz, args.cg_iters,
                                n_faces=solver.wall.n_faces if solver.wall is not None else 0,
                                unit_diag=bool(getattr(solver.pcg, "perm2", None) and solver.pcg.perm2["unit"]))
        avg = float(np.mean(ts))
        kern[kname] = {"launches": len(ts), "avg_us": avg * 1e6, "total_ms": float(np.sum(ts)) * 1e3,
                      "alg_bytes": B, "gbs": B / avg / 1e9 if avg > 0 else None,
                      "gflops": F / avg / 1e9 if F and avg > 0 else None}
    dom = max((k for k in kern if k.startswith("K")), key=lambda k: kern[k]["total_ms"])
    peak, peak_kind = load_peaks()
    traffic = load_traffic(name if ws == 1 else "")
    traffic = traffic.get(dom) if isinstance(traffic.get(dom), (int, float)) else None
    roof = {"kernel": dom, "bound": "hbm", "achieved": round(kern[dom]["gbs"], 1), "peak": peak, "unit": "GB/s",
            "frac": round(kern[dom]["gbs"] / peak, 4), "peak_source": peak_kind,
            "traffic": traffic, "alg_bytes_per_launch": kern[dom]["alg_bytes"],
            "alg_bytes_definition": "SURVEY.md §8(d) per-unit figure x units per launch"}
    pm = getattr(solver.pcg, "perm2", None)
    if dom == "K5_cg_tile_iter" and pm is not None and pm.get("single"):
        # The tiled single pass moves fewer bytes than the SURVEY per-iteration
        # model (CSR int32 + Jacobi z/D^-1 vectors), so the roofline uses the
        # compulsory bytes of this format per iteration (every datum once): 8 B
        # value + 2 B tile-local column per stored entry, (r', q) read and
        # written (32 B) and (x, p) read and written (32 B) per row, a 4 B
        # index per ghost row, slice and ghost pointers.  The ghost rows'
        # (r', q) values are re-reads of pairs already counted once: what they
        # cost in DRAM shows up as traffic / compulsory > 1.
        A2, tm = pm["A"], pm["tile"]
        n2 = solver.pcg.n
        n_tiles = (n2 + tm["struct"].rows_per_cta - 1) // tm["struct"].rows_per_cta
        comp = (10 * A2.nnz_stored + 64 * n2 + 4 * int(tm["ghost"].numel()) + 8 * A2.slice_ptr.numel()
                + 4 * (n_tiles + 1))
        t_dom = kern[dom]["avg_us"] * 1e-6
        roof.update({"achieved": round(comp / t_dom / 1e9, 1), "frac": round(comp / t_dom / 1e9 / peak, 4),
                     "alg_bytes_per_launch": comp,
                     "alg_bytes_definition": "compulsory bytes of the stored format per launch (one CG iteration, "
                                             "ab_cg_tile_iter): 10 B x stored SELL entries (8 B value + 2 B "
                                             "tile-local column) + 64 B per row ((r', q) and (x, p) pairs read and "
                                             "written) + 4 B index per ghost row + slice/ghost pointers (ghost "
                                             "values are re-reads: they appear in traffic_over_alg)",
                     "survey_model_bytes": kern[dom]["alg_bytes"],
                     "survey_model_gbs": round(kern[dom]["gbs"], 1),
                     "survey_model_note": "SURVEY §8(d) K5 per-iteration model 12Z + 4(N+1) + 104N (CSR int32 "
                                          "columns, Jacobi z and D^-1 vectors): exceeds the HBM peak because the "
                                          "format moves fewer bytes"})
        kern[dom]["compulsory_bytes"] = comp
    if dom == "K5_cg_spmv" and pm is not None and pm.get("tile") is not None:
        # The tiled SpMV stores fewer bytes per entry than the layout-independent
        # SURVEY model (12 B per non-zero), so that model over-counts its
        # traffic.  The roofline uses the compulsory bytes of this format per
        # launch: 8 B value + 2 B tile-local column per stored entry, z of the
        # own rows once, a 4 B index per ghost row, p and q read and written,
        # slice and ghost pointers.
        A2, tm = pm["A"], pm["tile"]
        n2 = solver.pcg.n
        n_tiles = (n2 + pm["tile"]["struct"].rows_per_cta - 1) // pm["tile"]["struct"].rows_per_cta
        comp = (10 * A2.nnz_stored + 8 * n2 + 4 * int(tm["ghost"].numel()) + 32 * n2
                + 8 * (A2.slice_ptr.numel()) + 4 * (n_tiles + 1))
        t_dom = kern[dom]["avg_us"] * 1e-6
        roof.update({"achieved": round(comp / t_dom / 1e9, 1), "frac": round(comp / t_dom / 1e9 / peak, 4),
                     "alg_bytes_per_launch": comp,
                     "alg_bytes_definition": "compulsory bytes of the stored format per launch (ab_cg_spmv_tile): "
                                             "10 B x stored SELL entries (8 B value + 2 B tile-local column) + 8 B z "
                                             "per row + 4 B index per ghost row + 32 B p,q per row + slice/ghost "
                                             "pointers (ghost z values are re-reads)",
                     "survey_model_bytes": kern[dom]["alg_bytes"],
                     "survey_model_gbs": round(kern[dom]["gbs"], 1),
                     "survey_model_note": "SURVEY §8(d) layout-independent model (12 B per off-diagonal non-zero, "
                                          "int32 columns): exceeds the HBM peak because the format moves fewer bytes"})
        kern[dom]["compulsory_bytes"] = comp
    if traffic:
        # the same kernel's DRAM bytes (ncu) over this run's launch time
        roof["frac_dram"] = round(traffic / (kern[dom]["avg_us"] * 1e-6) / 1e9 / peak, 4)
        roof["traffic_over_alg"] = round(traffic / roof["alg_bytes_per_launch"], 4)
    # the element assembly's binding roof is the FP64 pipe
    roof_k2 = None
    if "K2_momentum" in kern and kern["K2_momentum"]["gflops"]:
        fp_peak, fp_src = load_fp64_peak()
        ach = kern["K2_momentum"]["gflops"] / 1e3
        roof_k2 = {"kernel": "K2_momentum", "bound": "fp64", "achieved": round(ach, 3), "peak": fp_peak,
                   "unit": "TFLOP/s", "frac": round(ach / fp_peak, 4), "peak_source": fp_src,
                   "flops_definition": "fp64 flops per element executed by K2 (ncu thread instructions 2 x DFMA + "
                                       "DMUL + DADD, profiles/r2_c4_ncu.md): " +
                                       ", ".join(f"{k} {v}" for k, v in FLOPS_K2.items())}
    if dom == "K5_cg_resident":
        # what this design must move at minimum per iteration: the stored SELL
        # entries (8 B value + 2 B local column, ab_cg_local), the z write and
        # D^-1 re-read (8 B/row each) and one 8 B gather per ghost row
        lm = solver.pcg.local
        if lm is not None:
            comp = args.cg_iters * (10 * lm["A"].nnz_stored + 16 * solver.n + 8 * int(lm["ghost"].numel()))
            roof["compulsory_definition"] = "per iteration: 10 B x stored SELL entries + 16 B/row + 8 B/ghost row"
        else:
            comp = args.cg_iters * (12 * nnz + 24 * solver.n)
            roof["compulsory_definition"] = "per iteration: 12 B/non-zero + 24 B/row"
        roof["compulsory_bytes_per_launch"] = comp
        roof["compulsory_frac"] = round(comp / (kern[dom]["avg_us"] * 1e-6) / 1e9 / peak, 4)

    result = {
        "metric": "M element-steps/s per time step (assembly + CG)", "value": round(value, 3),
        "unit": "M element-steps/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
        "scaling": wl["scaling"], "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": dict(desc, step=("3x(K2+%sK3) + K4 + PCG(%d it, Jacobi) + K6 + K7"
                                   % ("K8+" if solver.wall is not None else "", args.cg_iters)),
                       cg_iters=args.cg_iters, dt=DT, physics=params, cuda_graph=graph,
                       scatter="windowed" if not args.no_windows else "atomics",
                       l2="flushed (512 MB write) between timed steps", parallelism=f"dd{ws}"),
        "roofline_assembly": roof_k2,
        "e2e": {"value": round(n_elem_total * args.steps / (e2e_ms / 1e3) / 1e6, 3), "unit": "M element-steps/s",
                "h2d_bytes_per_step": bytes_io, "d2h_bytes_per_step": bytes_io,
                "api": "FlowSolver.step_host (pinned host u,p -> step -> host)"},
        "roofline": roof,
        "kernels": {k: {kk: (round(vv, 3) if isinstance(vv, float) else vv) for kk, vv in v.items()}
                    for k, v in kern.items()},
        "gpu_launches": int(launches_per_step * args.steps),
        "clocks": clk,
    }
    if rebalance is not None:
        result["rebalance"] = rebalance
    if ws == 1 and not args.no_c2 and name != "c2":
        del solver
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        result["c2_point"] = c2_point(args, flush)
    if backend != "nccl":
        result["note"] = f"{ws} ranks on one GPU over {backend}: functional check, not a performance number"
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            result["cpu_baseline"] = cpu_baseline_sample(name)
            # the paper's co-execution model with this box's measured rates (context only: no CPU path runs)
            from paper_2005_05899_b200 import coexec
            cb = result["cpu_baseline"]
            per_core = cb["value"] / max(1, cb.get("cores") or 1)
            rep = coexec.report(coexec.measured_params(result["value"], per_core, n_core=cb.get("nproc") or 1))
            result["coexec_model"] = {k: (round(v, 6) if isinstance(v, float) else v) for k, v in rep.items()}
            result["coexec_model"]["inputs"] = ("speedup = value / (cpu_baseline.value / cores) (one core of the C "
                                                "restatement); ratio = 1 GPU / nproc")
        except Exception as exc:  # pragma: no cover
            result["cpu_baseline"] = {"error": repr(exc)}
    if rank == 0:
        print(json.dumps(result), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()


def c2_point(args, flush) -> dict:
    """Round 1's headline config as an extra key: C2 (4.09M jittered tets,
    BASELINE configs[1]), same step, graph replay, L2 flushed per step."""
    import torch
    from paper_2005_05899_b200.timestep import FlowParams, FlowSolver
    w = build_rank_workload("c2", 1, 0)
    s_ = FlowSolver(w["sub"], FlowParams(**PHYS), **w["bc"], windows=True, reorder="sfc")
    s_.set_state(w["u"], w["p"])
    for _ in range(3):
        s_.step(DT, args.cg_iters, graph=True)
    torch.cuda.synchronize()
    ms = []
    for _ in range(10):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        s_.step(DT, args.cg_iters, graph=True)
        b.record()
        b.synchronize()
        ms.append(a.elapsed_time(b))
    e = s_.dm.n_elements
    return {"workload": "C2: jittered Kuhn TET04 88^3 (BASELINE configs[1])", "elements": e,
            "value": round(e * len(ms) / (sum(ms) / 1e3) / 1e6, 3), "ms_per_step": round(float(np.mean(ms)), 4),
            "steps": len(ms), "warmup": 3, "k1_mass": k1_point(s_.dm)}


def k1_point(dm) -> dict:
    """The reference's own kernel (assemble_packs: per-element mass matrices
    + lumped mass, assembly.py:227-244, :306-333) as K1 on the GPU vs its CPU
    restatement on this host (oracle element_mass, 1 thread, a 20^3-cell
    sample of the same recipe); the reference itself cannot run here, its
    ratio to the restatement was measured in the build container
    (profiles/r2_reference_k1_calibration.json)."""
    import ctypes
    import torch
    from threadpoolctl import threadpool_limits
    from oracle import fem
    from paper_2005_05899_b200 import meshgen
    from paper_2005_05899_b200._lib import call, ptr, stream_handle
    E = dm.n_elements
    ae = torch.empty((E, 4, 4), dtype=torch.float64, device="cuda")
    ml = torch.zeros(dm.n_nodes, dtype=torch.float64, device="cuda")
    ts = []
    for _ in range(6):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        call("ab_mass", ctypes.byref(dm.struct), 0, ptr(ae), None, ptr(ml), 128, stream_handle())
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) / 1e3)
    gpu = E / float(np.median(ts[1:])) / 1e6
    with threadpool_limits(1):
        m = meshgen.box_tets(20, 20, 20, jitter=0.2, seed=20200131)
        X = fem.element_coords(m.coords, m.conn["tet4"])
        fem.element_mass(X, "tet4")
        tc = []
        for _ in range(3):
            t0 = time.perf_counter()
            fem.element_mass(X, "tet4")
            tc.append(time.perf_counter() - t0)
    port = m.n_elements / float(np.median(tc)) / 1e6
    cal = {}
    try:
        cal = json.loads((ROOT / "profiles" / "r2_reference_k1_calibration.json").read_text())
    except Exception:
        pass
    out = {"gpu_Melem_s": round(gpu, 1), "gpu_ms": round(float(np.median(ts[1:])) * 1e3, 4),
           "output": "Ae f64[E][4][4] (523 MB) + lumped mass", "cpu_port_Melem_s": round(port, 4),
           "cpu_port": "oracle/fem.py element_mass (restates assemble_packs), 1 thread, 48000 elements"}
    if cal.get("port_over_reference"):
        out["reference_estimate_Melem_s"] = round(port / cal["port_over_reference"], 4)
        out["reference_estimate"] = ("cpu_port / port_over_reference (reference assemble_packs, pack 32, measured "
                                     "in the build container)")
    return out


def run_reference(args):
    """Reference arm: the CPU restatement of the path (the reference package
    has no NS step to run) — oracle/fem_c.c, C + OpenMP on all host cores —
    stepping a bounded sample of the workload (the C4 recipe at reduced
    size by default)."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle import femc
    femc.build()
    steps, warmup = max(1, min(args.steps, 50)), max(1, min(args.warmup, 3))
    name = "c5" if args.weak else args.workload
    o, st, n_el, what = cpu_sample(name, C_SCALE["c2" if name == "c2" else "other"], c_threads=0)
    for _ in range(warmup):
        st = o.step(st, DT, cg_iters=CG_ITERS)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        st = o.step(st, DT, cg_iters=CG_ITERS)
        times.append(time.perf_counter() - t0)
    value = n_el * steps / sum(times) / 1e6
    cores = o.threads
    sample = (f"oracle/fem_c.c (C + OpenMP restatement of the step) on {cores} threads, {what} ({n_el} elements), "
              f"{steps} timed steps after {warmup} warm-up, full step with CG {CG_ITERS} it")
    out = {"impl": "reference", "metric": "M element-steps/s per time step (assembly + CG)",
           "value": round(value, 5), "unit": "M element-steps/s", "n_gpus": args.gpus, "steps": steps,
           "warmup": warmup, "ms_per_step": round(1e3 * sum(times) / steps, 3), "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": f"{name.upper()} sample (same recipe and algorithm, bounded size: {what})",
                      "cg_iters": CG_ITERS, "parallelism": f"{cores} CPU threads (OpenMP)"},
           "cpu_baseline": {"value": round(value, 5), "unit": "M element-steps/s", "cores": cores, "kind": "port",
                            "sample": sample, **host_cpu()},
           "e2e": {"value": round(value, 5), "unit": "M element-steps/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_native(args)


if __name__ == "__main__":
    main()

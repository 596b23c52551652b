"""Two processes on ONE GPU run the fused decomposed CG with CUDA-IPC-mapped
peer buffers (the multi-GPU wiring of ddcg.ipc_ranks); the kernels of the
two processes time-slice, so this checks the wiring, not the speed.

    python tools/ipc_dd_check.py
"""
import os
import socket
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def worker(rank, world, port, its, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from oracle import fem
    from paper_2005_05899_b200 import meshgen
    from paper_2005_05899_b200.ddcg import DDRank, DDSolve, ipc_ranks
    from paper_2005_05899_b200.decompose import decompose
    from paper_2005_05899_b200.device import DeviceMesh
    from paper_2005_05899_b200.partition import sfc_partition
    from paper_2005_05899_b200.solver import assemble_laplacian
    m = meshgen.box_tets(10, 9, 8, jitter=0.2, seed=5)
    fixed = meshgen.boundary_nodes(m)
    L = fem.laplacian(m, fixed)
    parts, _, _ = sfc_partition(m, world, level=6)
    subs = [decompose(m, parts, world, r) for r in range(world)]
    ms = max(len(v) for _, pl in subs for v in pl.shared.values())
    sub, plan = subs[rank]
    dm = DeviceMesh(sub)
    fl = torch.from_numpy(fixed[plan.l2g])
    A = assemble_laplacian(dm, fl)
    dinv = torch.from_numpy(1.0 / L.diagonal()[plan.l2g]).cuda()
    r = DDRank(rank, world, A, dinv, plan.own, plan.shared, dm.node_order(), 4, fixed=fl, max_shared=ms)
    ipc_ranks(r)
    b = np.random.default_rng(7).standard_normal(m.n_nodes)
    b[fixed] = 0.0
    bt = torch.from_numpy(b[plan.l2g]).cuda()
    dist.barrier()
    DDSolve([r], [bt], zero_b=False).run(its)
    torch.cuda.synchronize()
    xr, _, _ = fem.pcg(L, b, 1.0 / L.diagonal(), its)
    err = np.linalg.norm(r.x.cpu().numpy() - xr[plan.l2g]) / np.linalg.norm(xr[plan.l2g])
    np.save(os.path.join(out, f"err{rank}.npy"), np.array([err, r.iterations]))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    import tempfile
    its = 5
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(worker, args=(2, _port(), its, d), nprocs=2, join=True)
        for k in range(2):
            e, it = np.load(os.path.join(d, f"err{k}.npy"))
            print(f"rank {k}: rel err vs oracle {e:.2e}, iterations {int(it)}")
            assert it == its and e <= 1e-10, (e, it)
    print("ipc wiring ok")

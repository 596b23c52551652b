"""B200-native (sm_100a) time-step hot path of the arXiv 2005.05899 (Alya)
fractional-step explicit-RK finite-element Navier-Stokes scheme.

Drop-in name surface of the reference package ``coexbal``
(reference pkg/src/coexbal/__init__.py:7-72) for the hot-path modules
(mesh, assembly, sfc partitioning, the balance Timer plugin), plus the new
time-step entry points (``assemble_momentum``, ``assemble_laplacian``,
``pcg_solve``, ``time_step``, ``run``, ``gpu_timer``).  Compute goes through
libalyab200.so (include/alyab200.h); there is no CPU fallback.
"""

__version__ = "0.1.0"

from .mesh import (  # noqa: F401
    BoundingBox, ElementKind, FullElement, FullMesh, Mesh, MeshFormatError, PartitionElement,
    compute_bounding_box, from_arrays, generate_synthetic_full_mesh, generate_synthetic_mesh, load_full_mesh,
    load_mesh, make_mesh, partition_mesh_from_full, store_full_mesh, store_mesh, to_arrays,
)
from .meshgen import MeshArrays  # noqa: F401


def __getattr__(name):
    # GPU-backed modules load lazily so that `import paper_2005_05899_b200`
    # (mesh types, I/O) works on a CPU-only host; calling any compute entry
    # point needs the CUDA library and a device.
    lazy = {
        "assembly": ("PackSet", "Pack", "Category", "CooMatrix", "SweepRow", "assemble_packs",
                     "assemble_reference", "build_packs", "scatter_global", "sweep_pack_size", "sweep_csv",
                     "lumped_mass"),
        "partition": ("BinSequence", "Partition", "SfcConfig", "hilbert_decode", "hilbert_key",
                      "hilbert_keys_batch", "partition_chunked", "project_to_bins", "split_1d", "store_partition",
                      "load_partition", "sfc_partition", "store_partition_parts", "load_partition_parts"),
        "balance": ("BalanceMetrics", "Phase", "TimingSample", "compute_metrics", "gpu_timer",
                    "throughput_coefficients", "distributed_timer", "RegressionMode", "CorrectionState",
                    "RegressionFit", "IterationRecord", "BalanceReport", "observe", "fit", "update_coefficients",
                    "rank_model_coefficients", "run_balancing_loop", "DELTA_MIN", "BETA_MIN", "DEFAULT_WLR_GROWTH"),
        "solver": ("SellMatrix", "assemble_laplacian", "pcg_solve"),
        "timestep": ("FlowParams", "FlowSolver", "time_step", "run"),
        "ops": ("assemble_momentum", "assemble_divergence", "assemble_gradient"),
        "coexec": ("EfficiencyParams", "eff_gpu", "eff_core", "eff_coex1", "eff_coex2", "predicted_time_reduction"),
    }
    import importlib
    for mod, names in lazy.items():
        if name in names:
            return getattr(importlib.import_module(f"{__name__}.{mod}"), name)
    raise AttributeError(name)

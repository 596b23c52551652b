"""bench.py's byte/flop model on CPU: the per-launch figures
the roofline lines are built from."""
import bench


def test_algorithmic_cost_per_kernel():
    counts = {"tet4": 1000, "pri6": 10, "hex8": 5, "pyr5": 1}
    N, Z = 300, 4500
    conn = 4 * (4 * 1000 + 6 * 10 + 8 * 5 + 5 * 1)
    assert bench.algorithmic_cost("K5_cg_tile_iter", counts, N, Z) == (12 * Z + 4 * (N + 1) + 104 * N,
                                                                       2 * Z + 12 * N)
    assert bench.algorithmic_cost("K5_cg_spmv", counts, N, Z, unit_diag=True)[0] == 12 * (Z - N) + 40 * N
    assert bench.algorithmic_cost("K5_cg_update_scaled", counts, N, Z) == (48 * N, 8 * N)
    b, f = bench.algorithmic_cost("K2_momentum", counts, N, Z)
    assert b == conn + 72 * N
    assert f == sum(bench.FLOPS_K2[k] * v for k, v in counts.items())
    assert bench.algorithmic_cost("K4_divergence", counts, N, Z) == (conn + 56 * N, 0)
    assert bench.algorithmic_cost("no_such_kernel", counts, N, Z) == (0, 0)


def test_flops_table_covers_every_element_kind():
    assert set(bench.FLOPS_K2) == {"tet4", "pri6", "hex8", "pyr5"}
    assert all(v > 0 for v in bench.FLOPS_K2.values())

"""GPU parity of the reference-pinned path: K1 mass matrices, |det J|, the
global COO scatter and the lumped mass against golden vectors produced by
the reference itself, and the SFC decomposition bit for bit."""

import numpy as np
import pytest

from conftest import mesh_from_golden, rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import paper_2005_05899_b200 as p
    return p


@pytest.mark.parametrize("prefix", ["mixed", "soup"])
@pytest.mark.parametrize("pack_size", [1, 5, 32, 4096])
def test_assemble_packs_matches_reference(pkg, golden_mass, prefix, pack_size):
    _, full = mesh_from_golden(golden_mass, prefix)
    ref = golden_mass[f"{prefix}_ae_reference"]
    got = pkg.assemble_packs(pkg.build_packs(full, pack_size))
    assert sorted(got) == list(range(len(full.elements)))
    num = den = 0.0
    for eid, m in got.items():
        n = m.shape[0]
        num += float(np.sum((m - ref[eid][:n, :n]) ** 2))
        den += float(np.sum(ref[eid][:n, :n] ** 2))
        assert np.allclose(m, m.T, rtol=0, atol=1e-14 * np.abs(m).max())
    assert np.sqrt(num / den) <= 1e-12


def test_pack_size_invariance_bitwise(pkg, golden_mass):
    _, full = mesh_from_golden(golden_mass, "mixed")
    a = pkg.assemble_packs(pkg.build_packs(full, 1))
    b = pkg.assemble_packs(pkg.build_packs(full, 32))
    for k in a:
        assert np.array_equal(a[k], b[k])


def test_packs_structure_and_jacobians(pkg, golden_mass):
    _, full = mesh_from_golden(golden_mass, "mixed")
    ps = pkg.build_packs(full, 4)
    order = np.concatenate([p.element_ids for p in ps.packs])
    assert np.array_equal(order, golden_mass["mixed_pack_order"])
    assert np.array_equal([p.valid_count for p in ps.packs], golden_mass["mixed_pack_counts"])
    J = golden_mass["mixed_jacobian"]
    for p in ps.packs:
        g = p.category.ngaus
        assert rel_l2(p.jacobian[: p.valid_count], J[p.element_ids][:, :g]) <= 1e-13
        assert np.all(p.jacobian[p.valid_count:] == 0.0)


def test_build_packs_errors(pkg):
    from paper_2005_05899_b200.mesh import ElementKind, FullElement, FullMesh
    nodes = np.eye(4, 3)
    bad = FullMesh(nodes=nodes, elements=(FullElement(ElementKind.TETRAHEDRON, (0, 1, 2, 3), "hex8"),))
    with pytest.raises(KeyError):
        pkg.build_packs(bad, 4)
    unk = FullMesh(nodes=nodes, elements=(FullElement(ElementKind.TETRAHEDRON, (0, 1, 2, 3), "tet9"),))
    with pytest.raises(KeyError):
        pkg.build_packs(unk, 4)
    with pytest.raises(ValueError):
        pkg.build_packs(unk, 0)


@pytest.mark.parametrize("prefix", ["mixed", "soup"])
def test_scatter_global_matches_reference(pkg, golden_mass, prefix):
    _, full = mesh_from_golden(golden_mass, prefix)
    coo = pkg.scatter_global(pkg.assemble_reference(full), full)
    assert np.array_equal(coo.rows, golden_mass[f"{prefix}_coo_rows"])
    assert np.array_equal(coo.cols, golden_mass[f"{prefix}_coo_cols"])
    assert rel_l2(coo.values, golden_mass[f"{prefix}_coo_vals"]) <= 1e-12
    assert rel_l2(coo.row_sums(), golden_mass[f"{prefix}_row_sums"]) <= 1e-12
    assert abs(coo.total() - float(golden_mass[f"{prefix}_total"])) <= 1e-12


@pytest.mark.parametrize("prefix", ["mixed", "soup"])
def test_lumped_mass_matches_reference(pkg, golden_mass, prefix):
    arrays, _ = mesh_from_golden(golden_mass, prefix)
    assert rel_l2(pkg.lumped_mass(arrays), golden_mass[f"{prefix}_row_sums"]) <= 1e-12


def test_sweep_pack_size(pkg, golden_mass):
    _, full = mesh_from_golden(golden_mass, "mixed")
    rows = pkg.sweep_pack_size(full, [8, 32], reps=3)
    assert [r.pack_size for r in rows] == [1, 8, 32]
    assert rows[0].speedup == 1.0 and all(r.speedup > 0 for r in rows)
    assert pkg.sweep_csv(rows).startswith("pack_size,median_seconds,speedup\n")


def test_centroids_match_reference_bitwise(pkg, golden_mass):
    arrays, full = mesh_from_golden(golden_mass, "mixed")
    from paper_2005_05899_b200.partition import element_centroids
    assert np.array_equal(element_centroids(arrays), golden_mass["mixed_centroids"])
    pm = pkg.partition_mesh_from_full(full)
    assert np.array_equal(pm.weight_array(), golden_mass["mixed_weights"])


@pytest.mark.parametrize("level", [1, 3, 8, 20])
def test_hilbert_batch_matches_reference(pkg, golden_sfc, level):
    keys = pkg.hilbert_keys_batch(golden_sfc[f"hk_cells_L{level}"], level)
    assert np.array_equal(keys, golden_sfc[f"hk_keys_L{level}"])
    for k, c in zip(golden_sfc[f"hd_keys_L{level}"][:16], golden_sfc[f"hd_cells_L{level}"][:16]):
        assert pkg.hilbert_decode(int(k), level) == tuple(int(v) for v in c)
        assert pkg.hilbert_key(tuple(int(v) for v in c), level) == int(k)


def test_fixture_partitions_match_reference(pkg, golden_sfc):
    from paper_2005_05899_b200.mesh import ElementKind, PartitionElement, make_mesh
    cent, ids, w = golden_sfc["fx_centroids"], golden_sfc["fx_ids"], golden_sfc["fx_weights"]
    kinds = {4.0: ElementKind.TETRAHEDRON, 5.0: ElementKind.PYRAMID, 6.0: ElementKind.PRISM,
             8.0: ElementKind.HEXAHEDRON}
    mesh = make_mesh(PartitionElement(id=int(i), kind=kinds[float(wi)], centroid=tuple(c), weight=float(wi))
                     for i, c, wi in zip(ids, cent, w))
    for tag in golden_sfc["fx_cases"]:
        tag = str(tag)
        level, P = int(tag.split("_")[0][1:]), int(tag.split("_")[1][1:])
        lam = golden_sfc[f"fx_lam_{tag}"]
        cfg = pkg.SfcConfig(level=level)
        seq = pkg.project_to_bins(mesh, cfg)
        assert np.array_equal(seq.keys, golden_sfc[f"fx_bins_keys_L{level}"])
        part = pkg.split_1d(seq, P, lam)
        assert np.array_equal(part.cut_bins, golden_sfc[f"fx_cut_{tag}"])
        assert np.array_equal(part.subdomain_weights, golden_sfc[f"fx_subw_{tag}"])
        got = np.array([part.assignment[i] for i in sorted(part.assignment)])
        assert np.array_equal(got, golden_sfc[f"fx_assign_{tag}"])
        for nch in (1, 3, 8):
            assert pkg.partition_chunked(mesh, cfg, P, lam, n_chunks=nch) == part


def test_sfc_partition_array_native_matches_oracle(pkg):
    from oracle import sfc as osfc
    from paper_2005_05899_b200 import meshgen
    m = meshgen.c3_mesh(0.06)
    parts, cuts, sub = pkg.sfc_partition(m, 4, level=6)
    cent = np.zeros((m.n_elements, 3))
    ids = np.zeros(m.n_elements, np.int64)
    w = np.zeros(m.n_elements)
    for _t, rule, conn, eids in m.categories():
        cent[eids] = osfc.centroids(m.coords, conn)
        ids[eids] = eids
        w[eids] = meshgen.GAUSS_COUNT[rule]
    ref, rcuts, rsub = osfc.partition(cent, ids, w, 4, level=6)
    assert np.array_equal(parts, ref)
    assert np.array_equal(cuts, rcuts) and np.array_equal(sub, rsub)

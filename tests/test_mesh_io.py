"""Mesh drop-in (reference mesh.py): types, validation, file formats, and
generators.  CPU only."""

import json

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2005_05899_b200 import meshgen
from paper_2005_05899_b200.mesh import (
    ElementKind, FullElement, FullMesh, MeshFormatError, PartitionElement, from_arrays, generate_synthetic_full_mesh,
    generate_synthetic_mesh, load_full_mesh, load_mesh, make_mesh, store_full_mesh, store_mesh, to_arrays,
)


def test_element_kind_tables():
    assert [k.node_count for k in ElementKind] == [4, 5, 6, 8]
    assert [k.default_rule for k in ElementKind] == ["tet4", "pyr5", "pri6", "hex8"]
    assert [k.default_gauss_count for k in ElementKind] == [4, 5, 6, 8]


def test_full_mesh_validation():
    nodes = np.zeros((4, 3))
    with pytest.raises(ValueError):
        FullMesh(nodes=nodes, elements=(FullElement(ElementKind.TETRAHEDRON, (0, 1, 2), "tet4"),))
    with pytest.raises(ValueError):
        FullMesh(nodes=nodes, elements=(FullElement(ElementKind.TETRAHEDRON, (0, 1, 2, 4), "tet4"),))


def test_full_mesh_json_roundtrip(tmp_path):
    full = from_arrays(meshgen.c3_mesh(0.03))
    store_full_mesh(full, tmp_path / "m.json")
    back = load_full_mesh(tmp_path / "m.json")
    assert np.array_equal(back.nodes, full.nodes) and back.elements == full.elements
    (tmp_path / "bad.json").write_text("{not json")
    with pytest.raises(MeshFormatError):
        load_full_mesh(tmp_path / "bad.json")
    (tmp_path / "bad2.json").write_text(json.dumps({"nodes": [[0, 0, 0]], "elements": [{"kind": "xx"}]}))
    with pytest.raises(MeshFormatError):
        load_full_mesh(tmp_path / "bad2.json")


def test_partition_mesh_text_roundtrip_numpy2(tmp_path):
    """store -> load round trip (the reference's numpy-2 repr bug, is fixed)."""
    m = generate_synthetic_mesh(50, {ElementKind.TETRAHEDRON: 0.5, ElementKind.HEXAHEDRON: 0.5}, seed=3)
    store_mesh(m, tmp_path / "m.pmesh")
    back = load_mesh(tmp_path / "m.pmesh")
    assert np.array_equal(back.centroid_array(), m.centroid_array())
    assert np.array_equal(back.weight_array(), m.weight_array())
    (tmp_path / "dup.pmesh").write_text("pmesh 1 2\n0 tet 0 0 0 4\n0 tet 1 1 1 4\n")
    with pytest.raises(MeshFormatError):
        load_mesh(tmp_path / "dup.pmesh")


def test_synthetic_mesh_reproduces_reference_fixture(golden_sfc):
    """Same draw sequence as the reference: its 10k fixture mesh (seed
    20200131) is reproduced bit for bit."""
    m = generate_synthetic_mesh(10_000, {ElementKind.TETRAHEDRON: 0.55, ElementKind.PYRAMID: 0.15,
                                         ElementKind.PRISM: 0.15, ElementKind.HEXAHEDRON: 0.15}, seed=20200131)
    assert np.array_equal(m.centroid_array(), golden_sfc["fx_centroids"])
    assert np.array_equal(m.weight_array(), golden_sfc["fx_weights"])
    assert m.bounding_box.lo == tuple(golden_sfc["fx_box_lo"]) and m.bounding_box.hi == tuple(golden_sfc["fx_box_hi"])


def test_synthetic_full_mesh_matches_reference(golden_mass):
    full = generate_synthetic_full_mesh(300, hex_fraction=0.3, seed=3)
    assert np.array_equal(full.nodes, golden_mass["soup_nodes"])
    kinds = [e.kind.value for e in full.elements]
    assert kinds == [str(k) for k in golden_mass["soup_kinds"]]


def test_make_mesh_duplicate_ids():
    e = [PartitionElement(id=1, kind=ElementKind.TETRAHEDRON, centroid=(0, 0, 0), weight=4.0)] * 2
    with pytest.raises(ValueError, match="duplicate element id 1"):
        make_mesh(e)
    with pytest.raises(ValueError):
        make_mesh([])


def test_arrays_roundtrip_groups_like_build_packs(golden_mass):
    from conftest import mesh_from_golden
    arrays, full = mesh_from_golden(golden_mass, "mixed")
    assert sorted(arrays.conn) == ["hex8", "tet1", "tet4"]
    order = np.concatenate([ids for _t, _r, _c, ids in arrays.categories()])
    assert np.array_equal(order, golden_mass["mixed_pack_order"])
    back = from_arrays(arrays)
    assert back.elements == full.elements


def test_boundary_layer_mesh_is_conforming():
    """Every interior face is shared by exactly two elements with matching
    vertex sets (Appendix B), total volume 1."""
    from oracle import fem
    m = meshgen.boundary_layer_mesh(4, 4, 7, 2, hex_fraction=0.25)
    faces = {}
    local = {"tet": [(0, 1, 2), (0, 1, 3), (0, 2, 3), (1, 2, 3)],
             "pyr": [(0, 1, 2, 3), (0, 1, 4), (1, 2, 4), (2, 3, 4), (3, 0, 4)],
             "pri": [(0, 1, 2), (3, 4, 5), (0, 1, 4, 3), (1, 2, 5, 4), (2, 0, 3, 5)],
             "hex": [(0, 1, 2, 3), (4, 5, 6, 7), (0, 1, 5, 4), (1, 2, 6, 5), (2, 3, 7, 6), (3, 0, 4, 7)]}
    for tag, rule, conn, _ids in m.categories():
        for row in conn:
            for f in local[tag]:
                key = tuple(sorted(int(row[i]) for i in f))
                faces[key] = faces.get(key, 0) + 1
    x = m.coords
    lo, hi = x.min(0), x.max(0)
    for key, cnt in faces.items():
        on_bnd = any(np.all(np.abs(x[list(key), d] - lo[d]) < 1e-12) or np.all(np.abs(x[list(key), d] - hi[d]) < 1e-12)
                     for d in range(3))
        assert cnt == (1 if on_bnd else 2), key
    assert abs(fem.lumped_mass(m).sum() - 1.0) < 1e-13
    counts = {r: c.shape[0] for r, c in m.conn.items()}
    assert counts["hex8"] == 8 and counts["pyr5"] == 4 and counts["pri6"] == 48


def test_c2_sizes():
    m = meshgen.box_tets(88, 88, 88)
    assert m.n_elements == 4_088_832 and m.n_nodes == 704_969


def test_partition_array_io_matches_dict_io(tmp_path):
    """store_partition_parts / load_partition_parts (native formatter and
    parser) write and read the same `part 1` files as the dict-based
    store_partition / load_partition (reference sfc.py:385-417)."""
    from paper_2005_05899_b200.partition import (Partition, load_partition, load_partition_parts,
                                                 store_partition, store_partition_parts)
    rng = np.random.default_rng(7)
    parts = rng.integers(1, 6, size=12345).astype(np.int32)
    cuts = np.array([10, 20, 30, 40], dtype=np.int64)
    sub = np.array([1.5, 2.0, 2.5, 3.0, 4.0])
    ref = Partition(n_parts=5, cut_bins=cuts, assignment={i: int(p) for i, p in enumerate(parts)},
                    subdomain_weights=sub)
    store_partition(ref, tmp_path / "a.part")
    store_partition_parts(parts, 5, cuts, sub, tmp_path / "b.part", chunk=1000)
    assert (tmp_path / "a.part").read_bytes() == (tmp_path / "b.part").read_bytes()
    assert (tmp_path / "a.part.json").read_text() == (tmp_path / "b.part.json").read_text()
    got, n_parts, c2, s2 = load_partition_parts(tmp_path / "a.part")
    assert n_parts == 5 and np.array_equal(got, parts) and np.array_equal(c2, cuts) and np.array_equal(s2, sub)
    assert load_partition(tmp_path / "b.part") == ref
    # malformed / inconsistent files are rejected like the dict reader does
    (tmp_path / "c.part").write_text("part 1 2 3\n0 1\n1 2\n1 2\n")
    (tmp_path / "c.part.json").write_text('{"cut_bins": [0], "subdomain_weights": [1.0, 1.0]}')
    with pytest.raises(ValueError, match="duplicate"):
        load_partition_parts(tmp_path / "c.part")
    (tmp_path / "c.part").write_text("part 1 2 3\n0 1\n1 2\n")
    with pytest.raises(ValueError, match="expected 3"):
        load_partition_parts(tmp_path / "c.part")
    (tmp_path / "c.part").write_text("part 2 2 3\n")
    with pytest.raises(ValueError, match="header"):
        load_partition_parts(tmp_path / "c.part")
    with pytest.raises(ValueError):
        store_partition_parts(np.array([0, 1]), 2, [0], [1.0, 1.0], tmp_path / "d.part")

"""Generate the golden vectors that pin the oracle and the GPU path to the
reference's own implementation.

Runs ONLY in the build container, where the reference is importable from
/root/reference/pkg/src.  The outputs are small committed
fixtures; nothing on the GPU box reads /root/reference.

    python tests/golden/make_golden.py

Fixtures:
  reference_mass.npz   meshes + reference assemble_reference / assemble_packs /
                       build_packs Jacobians / scatter_global COO + row sums
                       (reference assembly.py:178-333)
  reference_sfc.npz    hilbert_keys_batch / hilbert_decode / project_to_bins /
                       split_1d / partition_chunked outputs (reference sfc.py)
  reference_balance.json  compute_metrics examples (reference balance.py:82-92)
  reference_dlb.json   run_balancing_loop (SLR/WLR regression DLB, reference
                       balance.py:95-346) on the 10k fixture mesh with
                       noise-free affine per-rank cost models
                       t_k = W_k / theta_k + c_k (the reference's own
                       simulate_times for noise_sigma = 0, coexec.py:69-98)

  reference_coexec.json  closed-form co-execution efficiencies (reference
                       coexec.py:258-323)

    python tests/golden/make_golden.py dlb      # only reference_dlb.json
    python tests/golden/make_golden.py coexec   # only reference_coexec.json
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))
sys.path.insert(0, str(HERE.parents[1]))

import coexbal  # noqa: E402
from coexbal import assembly as ra  # noqa: E402
from coexbal import balance as rb  # noqa: E402
from coexbal import mesh as rm  # noqa: E402
from coexbal import sfc as rs  # noqa: E402
from coexbal.fixtures import fixture_mesh_10k as load_fixture_mesh  # noqa: E402

from paper_2005_05899_b200 import meshgen  # noqa: E402


def connected_mixed_mesh(seed=7):
    """Jittered Kuhn-tet box + disjoint hex box, elements shuffled so ids do not
    follow categories; a few tets use the 1-point rule (category tet1)."""
    tb = meshgen.box_tets(3, 3, 2, jitter=0.2, seed=seed)
    hb = meshgen.box_hexes(2, 2, 3, lengths=(0.7, 0.9, 1.1), origin=(1.5, 0.1, -0.2))
    rng = np.random.default_rng(seed)
    hcoords = hb.coords + rng.uniform(-0.05, 0.05, hb.coords.shape)  # non-affine hexes
    nodes = np.concatenate([tb.coords, hcoords])
    off = tb.n_nodes
    elems = [("tet", tuple(int(c) for c in row)) for row in tb.conn["tet4"]]
    elems += [("hex", tuple(int(c) + off for c in row)) for row in hb.conn["hex8"]]
    perm = rng.permutation(len(elems))
    full = []
    for k, i in enumerate(perm):
        kind, conn = elems[i]
        rule = "tet1" if (kind == "tet" and k % 7 == 3) else rm.ElementKind(kind).default_rule
        full.append(rm.FullElement(kind=rm.ElementKind(kind), conn=conn, rule=rule))
    return rm.FullMesh(nodes=nodes, elements=tuple(full))


def pack_mesh(full):
    """FullMesh -> flat arrays (kind tag, rule, conn padded to 8)."""
    n = len(full.elements)
    conn = np.full((n, 8), -1, dtype=np.int64)
    kinds, rules = [], []
    for i, e in enumerate(full.elements):
        conn[i, : len(e.conn)] = e.conn
        kinds.append(e.kind.value)
        rules.append(e.rule)
    return conn, np.array(kinds), np.array(rules)


def mass_fixture(prefix, full, out):
    conn, kinds, rules = pack_mesh(full)
    out[f"{prefix}_nodes"] = full.nodes
    out[f"{prefix}_conn"] = conn
    out[f"{prefix}_kinds"] = kinds
    out[f"{prefix}_rules"] = rules
    ref = ra.assemble_reference(full)
    ae = np.zeros((len(full.elements), 8, 8))
    for i, m in ref.items():
        ae[i, : m.shape[0], : m.shape[1]] = m
    out[f"{prefix}_ae_reference"] = ae
    for size in (1, 5, 32):
        ps = ra.build_packs(full, size)
        got = ra.assemble_packs(ps)
        arr = np.zeros_like(ae)
        for i, m in got.items():
            arr[i, : m.shape[0], : m.shape[1]] = m
        out[f"{prefix}_ae_packs{size}"] = arr
    ps = ra.build_packs(full, 4)
    J = np.zeros((len(full.elements), 8))
    order = []
    for p in ps.packs:
        for lane in range(p.valid_count):
            eid = int(p.element_ids[lane])
            J[eid, : p.category.ngaus] = p.jacobian[lane]
            order.append(eid)
        out.setdefault(f"{prefix}_pack_valid", [])
    out[f"{prefix}_jacobian"] = J
    out[f"{prefix}_pack_order"] = np.array(order, dtype=np.int64)
    out[f"{prefix}_pack_counts"] = np.array([p.valid_count for p in ps.packs], dtype=np.int64)
    out.pop(f"{prefix}_pack_valid", None)
    coo = ra.scatter_global(ref, full)
    out[f"{prefix}_coo_rows"] = coo.rows
    out[f"{prefix}_coo_cols"] = coo.cols
    out[f"{prefix}_coo_vals"] = coo.values
    out[f"{prefix}_row_sums"] = coo.row_sums()
    out[f"{prefix}_total"] = np.array(coo.total())
    pm = rm.partition_mesh_from_full(full)
    out[f"{prefix}_centroids"] = pm.centroid_array()
    out[f"{prefix}_weights"] = pm.weight_array()


def sfc_fixture(out):
    rng = np.random.default_rng(20200131)
    for level in (1, 3, 8, 20):
        side = 1 << level
        cells = rng.integers(0, side, size=(512, 3), dtype=np.int64)
        out[f"hk_cells_L{level}"] = cells
        out[f"hk_keys_L{level}"] = rs.hilbert_keys_batch(cells, level)
        keys = rng.integers(0, 1 << (3 * level), size=64, dtype=np.int64)
        out[f"hd_keys_L{level}"] = keys
        out[f"hd_cells_L{level}"] = np.array([rs.hilbert_decode(int(k), level) for k in keys], dtype=np.int64)
    # partitions of the fixture mesh (seed 20200131, fixtures/__init__.py:13)
    m = load_fixture_mesh()
    out["fx_centroids"] = m.centroid_array()
    out["fx_weights"] = m.weight_array()
    out["fx_ids"] = m.id_array()
    out["fx_box_lo"] = np.array(m.bounding_box.lo)
    out["fx_box_hi"] = np.array(m.bounding_box.hi)
    cases = []
    for level in (4, 8):
        cfg = rs.SfcConfig(level=level)
        seq = rs.project_to_bins(m, cfg)
        out[f"fx_bins_keys_L{level}"] = seq.keys
        out[f"fx_bins_weights_L{level}"] = seq.weights
        for P, lam in ((1, None), (2, None), (3, [0.5, 1.2, 1.3]), (8, None),
                       (8, list(np.linspace(0.3, 1.7, 8)))):
            if lam is not None:
                lam = np.array(lam) * P / np.sum(lam)
            part = rs.split_1d(seq, P, lam)
            tag = f"L{level}_P{P}_{'lam' if lam is not None else 'uni'}"
            cases.append(tag)
            out[f"fx_cut_{tag}"] = part.cut_bins
            out[f"fx_subw_{tag}"] = part.subdomain_weights
            ids = np.array(sorted(part.assignment), dtype=np.int64)
            out[f"fx_assign_{tag}"] = np.array([part.assignment[i] for i in ids], dtype=np.int64)
            out[f"fx_lam_{tag}"] = np.ones(P) if lam is None else lam
            for nch in (2, 8):
                pc = rs.partition_chunked(m, cfg, P, lam, n_chunks=nch)
                assert pc == part
    out["fx_cases"] = np.array(cases)


def balance_fixture():
    rng = np.random.default_rng(5)
    ex = []
    for _ in range(8):
        t = rng.uniform(0.5, 3.0, size=int(rng.integers(1, 9)))
        mtr = rb.compute_metrics(rb.TimingSample(iteration=1, times=t))
        ex.append({"times": t.tolist(), "mean": mtr.mean, "imbalance": mtr.imbalance, "lb": mtr.lb,
                   "per_rank": mtr.per_rank.tolist(), "deviations": mtr.deviations.tolist()})
    return ex


# (name, theta per rank, fixed cost per rank, mode, tol, max_iters)
DLB_CASES = (
    ("hetero6_wlr", [1, 1, 1, 1, 5, 5], [0.0] * 6, "wlr", 0.02, 20),
    ("affine4_slr", [1, 2, 1, 3], [0.01, 0.0, 0.02, 0.005], "slr", 0.01, 15),
    ("homog8_wlr", [1.0] * 8, [0.0] * 8, "wlr", 0.02, 5),
    # the bundled hetero_s20 plan (2 nodes x (16 cores + 2 GPU ranks at
    # theta 20)): SURVEY F8-ii, where the regression plateaus then diverges
    ("hetero_s20_wlr", ([1.0] * 16 + [20.0] * 2) * 2, [0.0] * 36, "wlr", 0.02, 30),
)


def dlb_fixture():
    m = load_fixture_mesh()
    cfg = rs.SfcConfig(level=8)
    seq = rs.project_to_bins(m, cfg)
    cases = []
    for name, theta, cost, mode, tol, iters in DLB_CASES:
        th, c = np.array(theta, dtype=float), np.array(cost, dtype=float)

        def timer(part, th=th, c=c):
            return rb.TimingSample(iteration=0, times=part.subdomain_weights / th + c)

        rep = rb.run_balancing_loop(m, cfg, len(th), timer, mode=rb.RegressionMode(mode), tol=tol,
                                    max_iters=iters, bins=seq)
        cases.append({"name": name, "theta": theta, "cost": cost, "mode": mode, "tol": tol, "max_iters": iters,
                      "converged": rep.converged,
                      "lambda": [r.lam.tolist() for r in rep.iterations],
                      "times": [r.times.tolist() for r in rep.iterations],
                      "subdomain_weights": [r.partition.subdomain_weights.tolist() for r in rep.iterations],
                      "imbalance": [r.metrics.imbalance for r in rep.iterations],
                      "json": rep.to_json_dict(final_partition_ref="part.txt"),
                      "csv": rep.convergence_csv() if len(th) <= 8 else None})
    return {"reference_version": coexbal.__version__, "level": 8, "cases": cases}


def coexec_fixture():
    import warnings
    from coexbal import coexec as rc
    rows = []
    for s_, nc, ng in ((20.0, 40, 4), (1.5, 16, 2), (2.0, 8, 1), (350.0, 16, 1), (1e4, 112, 8), (3.0, 1, 0)):
        p = rc.EfficiencyParams.from_counts(nc, ng, s_)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            row = {"speedup": s_, "n_core": nc, "n_gpu": ng, "eff_core": rc.eff_core(p), "eff_gpu": rc.eff_gpu(p),
                   "eff_coex1": rc.eff_coex1(p), "eff_coex2": rc.eff_coex2(p)}
            for c in (1, 2):
                try:
                    row[f"red{c}"] = rc.predicted_time_reduction(p, c)
                except ValueError:
                    row[f"red{c}"] = None
        rows.append(row)
    return {"reference_version": coexbal.__version__, "rows": rows}


def main():
    if sys.argv[1:] == ["coexec"]:
        (HERE / "reference_coexec.json").write_text(json.dumps(coexec_fixture(), indent=1))
        print("wrote", HERE / "reference_coexec.json")
        return
    if sys.argv[1:] == ["dlb"]:
        (HERE / "reference_dlb.json").write_text(json.dumps(dlb_fixture()))
        print("wrote", HERE / "reference_dlb.json")
        return
    out: dict = {}
    mass_fixture("mixed", connected_mixed_mesh(), out)
    mass_fixture("soup", rm.generate_synthetic_full_mesh(300, hex_fraction=0.3, seed=3), out)
    np.savez_compressed(HERE / "reference_mass.npz", **out)
    out = {}
    sfc_fixture(out)
    np.savez_compressed(HERE / "reference_sfc.npz", **out)
    (HERE / "reference_balance.json").write_text(json.dumps(
        {"reference_version": coexbal.__version__, "examples": balance_fixture()}, indent=1))
    (HERE / "reference_dlb.json").write_text(json.dumps(dlb_fixture()))
    (HERE / "reference_coexec.json").write_text(json.dumps(coexec_fixture(), indent=1))
    print("wrote fixtures to", HERE)


if __name__ == "__main__":
    main()

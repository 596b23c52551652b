"""Test configuration.

* ``gpu`` marker: needs a CUDA device (run on the B200 box with -m gpu).
* The CUDA library is (re)built in-tree if stale, so the CPU suite can check
  that it loads and exports the ABI, and the GPU suite runs the native path.
* The oracle (oracle/) is imported only here, in tests, as the checker.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    from paper_2005_05899_b200 import build
    try:
        build.build()
    except Exception as exc:  # surfaced by test_abi
        print("library build failed:", exc, file=sys.stderr)


@pytest.fixture(scope="session")
def golden_mass():
    return dict(np.load(GOLDEN / "reference_mass.npz"))


@pytest.fixture(scope="session")
def golden_sfc():
    return dict(np.load(GOLDEN / "reference_sfc.npz"))


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def mesh_from_golden(g, prefix):
    """Golden FullMesh arrays -> (MeshArrays grouped like build_packs, FullMesh)."""
    from paper_2005_05899_b200.mesh import ElementKind, FullElement, FullMesh, to_arrays
    nodes = g[f"{prefix}_nodes"]
    conn = g[f"{prefix}_conn"]
    kinds = g[f"{prefix}_kinds"]
    rules = g[f"{prefix}_rules"]
    elems = []
    for c, k, r in zip(conn, kinds, rules):
        kind = ElementKind(str(k))
        elems.append(FullElement(kind=kind, conn=tuple(int(v) for v in c[: kind.node_count]), rule=str(r)))
    full = FullMesh(nodes=nodes, elements=tuple(elems))
    return to_arrays(full), full

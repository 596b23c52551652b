"""Reference-element data: integration rules and shape functions.

Drop-in for reference pkg/src/coexbal/assembly.py:33-126 (``QuadratureRule``,
``RULES``, ``shape_values``) extended with the prism (pri6) and pyramid (pyr5)
categories the reference names in mesh.py:59-71 but never implements
(SURVEY.md F4).  The same tables are emitted into ``csrc/ab_tables.inc`` as
``__constant__`` arrays so the CUDA kernels and the Python API share one
definition (``python -m paper_2005_05899_b200.elements`` regenerates it).

Rule index order (kernel template parameter): tet1=0, tet4=1, pyr5=2, pri6=3,
hex8=4.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .mesh import ElementKind

RULE_INDEX = {"tet1": 0, "tet4": 1, "pyr5": 2, "pri6": 3, "hex8": 4}
RULE_NAMES = tuple(RULE_INDEX)

_HEX_SIGNS = np.array([[-1, -1, -1], [1, -1, -1], [1, 1, -1], [-1, 1, -1],
                       [-1, -1, 1], [1, -1, 1], [1, 1, 1], [-1, 1, 1]], dtype=np.float64)
_PYR_SIGNS = ((-1, -1), (1, -1), (1, 1), (-1, 1))
_TET4_A = (5.0 + 3.0 * math.sqrt(5.0)) / 20.0
_TET4_B = (5.0 - math.sqrt(5.0)) / 20.0
_G3 = 1.0 / math.sqrt(3.0)


@dataclass(frozen=True)
class QuadratureRule:
    """Same fields as reference assembly.py:77-86."""

    rule_id: str
    kind: ElementKind
    points: np.ndarray   # (ngaus, 3) reference coordinates
    weights: np.ndarray  # (ngaus,)

    @property
    def ngaus(self) -> int:
        return len(self.weights)


def _pyr5():
    # 5-point rule on [-1,1]^2 x [0,1] (apex (0,0,1), volume 4/3): four points
    # (+-a, +-a, 1/6) with weight 9/32 and (0, 0, 7/10) with weight 5/24.  The
    # moment equations for 1, z, z^2, x^2, x^2 z fix a^2 = 32/135.
    a = math.sqrt(32.0 / 135.0)
    pts = [[sx * a, sy * a, 1.0 / 6.0] for sx, sy in _PYR_SIGNS] + [[0.0, 0.0, 0.7]]
    return np.array(pts), np.array([9.0 / 32.0] * 4 + [5.0 / 24.0])


def _pri6():
    tri = [(1.0 / 6.0, 1.0 / 6.0), (2.0 / 3.0, 1.0 / 6.0), (1.0 / 6.0, 2.0 / 3.0)]
    return np.array([[x, y, z] for z in (-_G3, _G3) for (x, y) in tri]), np.full(6, 1.0 / 6.0)


RULES: dict[str, QuadratureRule] = {
    "tet1": QuadratureRule("tet1", ElementKind.TETRAHEDRON, np.array([[0.25, 0.25, 0.25]]),
                           np.array([1.0 / 6.0])),
    "tet4": QuadratureRule("tet4", ElementKind.TETRAHEDRON,
                           np.array([[_TET4_A, _TET4_B, _TET4_B], [_TET4_B, _TET4_A, _TET4_B],
                                     [_TET4_B, _TET4_B, _TET4_A], [_TET4_B, _TET4_B, _TET4_B]]),
                           np.full(4, 1.0 / 24.0)),
    "pyr5": QuadratureRule("pyr5", ElementKind.PYRAMID, *_pyr5()),
    "pri6": QuadratureRule("pri6", ElementKind.PRISM, *_pri6()),
    "hex8": QuadratureRule("hex8", ElementKind.HEXAHEDRON,
                           np.array([[sx * _G3, sy * _G3, sz * _G3] for sx, sy, sz in _HEX_SIGNS]),
                           np.ones(8)),
}


def shape_values_and_gradients(rule: QuadratureRule):
    """N[i,g] and dN/dxi[i,g,3] at the rule's points."""
    p = rule.points
    xi, eta, zeta = p[:, 0], p[:, 1], p[:, 2]
    g = len(p)
    kind = rule.kind
    if kind is ElementKind.TETRAHEDRON:
        N = np.stack([1.0 - xi - eta - zeta, xi, eta, zeta])
        dN = np.zeros((4, g, 3))
        dN[0] = -1.0
        for a in range(3):
            dN[a + 1, :, a] = 1.0
        return N, dN
    if kind is ElementKind.HEXAHEDRON:
        N = np.empty((8, g))
        dN = np.empty((8, g, 3))
        for i, (sx, sy, sz) in enumerate(_HEX_SIGNS):
            fx, fy, fz = 1 + sx * xi, 1 + sy * eta, 1 + sz * zeta
            N[i] = fx * fy * fz / 8.0
            dN[i, :, 0] = sx * fy * fz / 8.0
            dN[i, :, 1] = fx * sy * fz / 8.0
            dN[i, :, 2] = fx * fy * sz / 8.0
        return N, dN
    if kind is ElementKind.PRISM:
        L = (1.0 - xi - eta, xi, eta)
        dL = ((-1.0, -1.0), (1.0, 0.0), (0.0, 1.0))
        N = np.empty((6, g))
        dN = np.empty((6, g, 3))
        for half, sz in enumerate((-1.0, 1.0)):
            fz = (1.0 + sz * zeta) / 2.0
            for a in range(3):
                i = 3 * half + a
                N[i] = L[a] * fz
                dN[i, :, 0] = dL[a][0] * fz
                dN[i, :, 1] = dL[a][1] * fz
                dN[i, :, 2] = L[a] * sz / 2.0
        return N, dN
    if kind is ElementKind.PYRAMID:
        s = 1.0 - zeta
        N = np.empty((5, g))
        dN = np.empty((5, g, 3))
        for i, (sx, sy) in enumerate(_PYR_SIGNS):
            N[i] = (s + sx * xi) * (s + sy * eta) / (4.0 * s)
            dN[i, :, 0] = sx * (s + sy * eta) / (4.0 * s)
            dN[i, :, 1] = sy * (s + sx * xi) / (4.0 * s)
            dN[i, :, 2] = -0.25 + sx * sy * xi * eta / (4.0 * s * s)
        N[4] = zeta
        dN[4] = 0.0
        dN[4, :, 2] = 1.0
        return N, dN
    raise KeyError(f"no shape functions for kind {kind.value}")


def shape_values(rule: QuadratureRule) -> np.ndarray:
    """Shape-function table N[i, g] (reference assembly.py:120-126)."""
    return shape_values_and_gradients(rule)[0]


def emit_tables(path: Path | None = None) -> str:
    """Write the ``__constant__`` tables used by every element kernel."""
    lines = ["// GENERATED by paper_2005_05899_b200/elements.py -- do not edit.",
             "// c_w[rule][g], c_N[rule][g][a], c_dN[rule][g][a][d]; rule order tet1,tet4,pyr5,pri6,hex8",
             "__constant__ double c_w[5][8] = {"]
    Ns, dNs = {}, {}
    for name in RULE_NAMES:
        r = RULES[name]
        Ns[name], dNs[name] = shape_values_and_gradients(r)
        w = list(r.weights) + [0.0] * (8 - r.ngaus)
        lines.append("  {" + ", ".join(repr(float(v)) for v in w) + "},")
    lines.append("};")
    lines.append("__constant__ double c_N[5][8][8] = {")
    for name in RULE_NAMES:
        N = Ns[name]
        rows = []
        for g in range(8):
            vals = [float(N[a, g]) if (g < N.shape[1] and a < N.shape[0]) else 0.0 for a in range(8)]
            rows.append("{" + ", ".join(repr(v) for v in vals) + "}")
        lines.append("  {" + ", ".join(rows) + "},")
    lines.append("};")
    lines.append("__constant__ double c_dN[5][8][8][3] = {")
    for name in RULE_NAMES:
        dN = dNs[name]
        gs = []
        for g in range(8):
            aa = []
            for a in range(8):
                if g < dN.shape[1] and a < dN.shape[0]:
                    aa.append("{" + ", ".join(repr(float(v)) for v in dN[a, g]) + "}")
                else:
                    aa.append("{0.0, 0.0, 0.0}")
            gs.append("{" + ", ".join(aa) + "}")
        lines.append("  {" + ", ".join(gs) + "},")
    lines.append("};")
    # M[rule][a][b] = sum_g w_g N_a(g) N_b(g): reference-element mass table,
    # used by the affine (tet) momentum kernel (sum_g w N_a u_g = sum_b M_ab u_b)
    lines.append("__constant__ double c_M[5][8][8] = {")
    for name in RULE_NAMES:
        N, w = Ns[name], RULES[name].weights
        M = (N * w[None, :]) @ N.T
        rows = []
        for a in range(8):
            vals = [float(M[a, b]) if (a < M.shape[0] and b < M.shape[1]) else 0.0 for b in range(8)]
            rows.append("{" + ", ".join(repr(v) for v in vals) + "}")
        lines.append("  {" + ", ".join(rows) + "},")
    lines.append("};")
    text = "\n".join(lines) + "\n"
    if path is not None:
        Path(path).write_text(text)
    return text


if __name__ == "__main__":
    out = Path(__file__).resolve().parent / "csrc" / "ab_tables.inc"
    emit_tables(out)
    print("wrote", out)

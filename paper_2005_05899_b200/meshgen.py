"""Array-native synthetic mesh generators (conforming, node-sharing).

The reference's only connectivity generator (`generate_synthetic_full_mesh`,
reference pkg/src/coexbal/mesh.py:326-363) emits a node soup: no two elements
share a node, so a global scatter never sums anything.  The configurations of
BASELINE.json need connected meshes, so these generators follow SURVEY.md
Appendix B instead:

* structured n_x x n_y x n_z cells, node index (i*(ny+1) + j)*(nz+1) + k;
* HEX08 cells in VTK node order (reference assembly.py:38-50);
* Kuhn TET04: six tets per cell along the main diagonal, one per axis
  permutation, so every face is split along its min->max diagonal;
* PEN06 (prism) layers: two prisms per cell split by the xy min->max diagonal;
* PYR05 transition cells above the hex patch: one pyramid (base = bottom
  quad, apex = max corner) + the four remaining Kuhn tets.

Everything is vectorised numpy; a 250M-element mesh is a few GB of int32
connectivity and never becomes Python objects.
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass, field

import numpy as np

# Category order follows the reference's sorted (kind.value, rule) grouping
# (assembly.py:197): "hex" < "pri" < "pyr" < "tet".
KIND_TAGS = ("hex", "pri", "pyr", "tet")
NODE_COUNT = {"tet": 4, "pyr": 5, "pri": 6, "hex": 8}
DEFAULT_RULE = {"tet": "tet4", "pyr": "pyr5", "pri": "pri6", "hex": "hex8"}
GAUSS_COUNT = {"tet1": 1, "tet4": 4, "pyr5": 5, "pri6": 6, "hex8": 8}
RULE_KIND = {"tet1": "tet", "tet4": "tet", "pyr5": "pyr", "pri6": "pri", "hex8": "hex"}

# Corner offsets of a unit cell, indexed by (dx, dy, dz).
_PERMS = list(itertools.permutations(range(3)))  # Kuhn path orders


@dataclass
class MeshArrays:
    """Array-native mesh: nodes (N,3) f64 and one connectivity block per
    category.  ``elem_ids[tag]`` maps the rows of ``conn[tag]`` to global
    element ids (the FullMesh element index), so drop-in results keyed by
    element id can be produced for any category layout.

    ``period`` holds the box lengths of periodic axes (0 = not periodic);
    kernels unwrap element coordinates by minimum image so node-wrapped
    periodic meshes keep correct Jacobians.
    """

    coords: np.ndarray
    conn: dict = field(default_factory=dict)      # rule id -> (E_k, n_k) int32
    elem_ids: dict = field(default_factory=dict)  # rule id -> (E_k,) int64
    period: np.ndarray = field(default_factory=lambda: np.zeros(3))
    shape: tuple | None = None                    # (nx, ny, nz) cells if structured

    @property
    def n_nodes(self) -> int:
        return int(self.coords.shape[0])

    @property
    def n_elements(self) -> int:
        return int(sum(c.shape[0] for c in self.conn.values()))

    def categories(self):
        """(kind tag, rule, conn, ids) in the reference's sorted (kind, rule)
        category order (assembly.py:197); rule ids start with the kind tag,
        so sorting by rule id is the same order."""
        for rule in sorted(self.conn):
            if self.conn[rule].shape[0] > 0:
                yield RULE_KIND[rule], rule, self.conn[rule], self.elem_ids[rule]

    def gauss_weight_total(self) -> int:
        return int(sum(c.shape[0] * GAUSS_COUNT[r] for r, c in self.conn.items()))


def _node_index(nx, ny, nz):
    def nid(i, j, k):
        return (i * (ny + 1) + j) * (nz + 1) + k
    return nid


def _grid_nodes(nx, ny, nz, lengths=(1.0, 1.0, 1.0), origin=(0.0, 0.0, 0.0)):
    xs = origin[0] + np.linspace(0.0, lengths[0], nx + 1)
    ys = origin[1] + np.linspace(0.0, lengths[1], ny + 1)
    zs = origin[2] + np.linspace(0.0, lengths[2], nz + 1)
    X, Y, Z = np.meshgrid(xs, ys, zs, indexing="ij")
    return np.stack([X.ravel(), Y.ravel(), Z.ravel()], axis=1)


def _cell_corner_ids(nx, ny, nz, ii, jj, kk):
    """corner[dx][dy][dz] -> (n_cells,) node ids for the given cells."""
    nid = _node_index(nx, ny, nz)
    c = {}
    for dx in (0, 1):
        for dy in (0, 1):
            for dz in (0, 1):
                c[(dx, dy, dz)] = nid(ii + dx, jj + dy, kk + dz)
    return c


def _kuhn_tets(c, perms=None):
    """Kuhn tets of cells with corner map ``c``; one tet per axis permutation."""
    perms = _PERMS if perms is None else perms
    out = []
    for p in perms:
        v = [0, 0, 0]
        path = [c[tuple(v)]]
        for ax in p:
            v[ax] = 1
            path.append(c[tuple(v)])
        out.append(np.stack(path, axis=1))
    # interleave so the six tets of one cell are consecutive (cell order kept)
    return np.stack(out, axis=1).reshape(-1, 4)


def _cells(nx, ny, nz, mask=None):
    ii, jj, kk = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    ii, jj, kk = ii.ravel(), jj.ravel(), kk.ravel()
    if mask is not None:
        m = mask(ii, jj, kk)
        ii, jj, kk = ii[m], jj[m], kk[m]
    return ii, jj, kk


def _finish(coords, blocks, period=None, shape=None):
    """Assign global element ids category by category (sorted tag order)."""
    mesh = MeshArrays(coords=np.ascontiguousarray(coords, dtype=np.float64))
    start = 0
    for tag in KIND_TAGS:
        if tag not in blocks:
            continue
        conn = np.ascontiguousarray(blocks[tag], dtype=np.int32)
        rule = DEFAULT_RULE[tag]
        mesh.conn[rule] = conn
        mesh.elem_ids[rule] = np.arange(start, start + conn.shape[0], dtype=np.int64)
        start += conn.shape[0]
    if period is not None:
        mesh.period = np.asarray(period, dtype=np.float64)
    mesh.shape = shape
    return mesh


def signed_volumes(coords, conn):
    """6 x signed volume of the (0,1,2,3)-corner tet of each element."""
    x = coords[conn[:, :4]]
    e = x[:, 1:] - x[:, :1]
    return np.einsum("ij,ij->i", e[:, 0], np.cross(e[:, 1], e[:, 2]))


def box_tets(nx, ny, nz, lengths=(1.0, 1.0, 1.0), jitter=0.0, seed=20200131):
    """Kuhn TET04 box (C2 of BASELINE.json when nx=ny=nz=88, jitter=0.2).

    Interior nodes are jittered by U(-jitter*h, jitter*h) per axis; the draw
    is repeated (seed+attempt) until no tet changes orientation.
    """
    coords = _grid_nodes(nx, ny, nz, lengths)
    ii, jj, kk = _cells(nx, ny, nz)
    tets = _kuhn_tets(_cell_corner_ids(nx, ny, nz, ii, jj, kk))
    if jitter > 0.0:
        h = np.array(lengths, dtype=np.float64) / np.array([nx, ny, nz])
        I, J, K = np.meshgrid(np.arange(nx + 1), np.arange(ny + 1), np.arange(nz + 1), indexing="ij")
        interior = ((I > 0) & (I < nx) & (J > 0) & (J < ny) & (K > 0) & (K < nz)).ravel()
        ref = np.sign(signed_volumes(coords, tets))
        for attempt in range(16):
            rng = np.random.default_rng(seed + attempt)
            d = rng.uniform(-jitter, jitter, size=coords.shape) * h
            d[~interior] = 0.0
            trial = coords + d
            vol = signed_volumes(trial, tets)
            if np.all(np.sign(vol) == ref) and np.all(np.abs(vol) > 0):
                coords = trial
                break
        else:  # pragma: no cover - 16 failed draws would be a generator bug
            raise RuntimeError("could not jitter mesh without inverting elements")
    return _finish(coords, {"tet": tets}, shape=(nx, ny, nz))


def box_hexes(nx, ny, nz, lengths=(1.0, 1.0, 1.0), periodic=False, origin=(0.0, 0.0, 0.0)):
    """HEX08 box.  ``periodic=True`` wraps nodes on all three axes (TGV, C1)."""
    if not periodic:
        coords = _grid_nodes(nx, ny, nz, lengths, origin)
        ii, jj, kk = _cells(nx, ny, nz)
        c = _cell_corner_ids(nx, ny, nz, ii, jj, kk)
        period = None
    else:
        h = np.array(lengths, dtype=np.float64) / np.array([nx, ny, nz])
        I, J, K = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
        coords = np.stack([origin[0] + I.ravel() * h[0], origin[1] + J.ravel() * h[1],
                           origin[2] + K.ravel() * h[2]], axis=1)
        ii, jj, kk = _cells(nx, ny, nz)

        def pid(i, j, k):
            return ((i % nx) * ny + (j % ny)) * nz + (k % nz)
        c = {(dx, dy, dz): pid(ii + dx, jj + dy, kk + dz)
             for dx in (0, 1) for dy in (0, 1) for dz in (0, 1)}
        period = lengths
    order = [(0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0), (0, 0, 1), (1, 0, 1), (1, 1, 1), (0, 1, 1)]
    hexes = np.stack([c[o] for o in order], axis=1)
    return _finish(coords, {"hex": hexes}, period=period, shape=(nx, ny, nz))


# Cell types of the boundary-layer box (one code per structured cell) and the
# Gauss-point weight of the elements each cell produces (mesh.py:66-71 counts:
# hex 8, 2 prisms 2 x 6, pyramid + 4 tets 5 + 16, 6 Kuhn tets 6 x 4).
CELL_HEX, CELL_PRI, CELL_TRANS, CELL_KUHN = 0, 1, 2, 3
CELL_GAUSS = np.array([8, 12, 21, 24], dtype=np.int64)
CELL_ELEMS = {"hex": np.array([1, 0, 0, 0]), "pri": np.array([0, 2, 0, 0]), "pyr": np.array([0, 0, 1, 0]),
              "tet_trans": np.array([0, 0, 4, 0]), "tet_kuhn": np.array([0, 0, 0, 6])}


def patch_extent(nx, ny, hex_fraction):
    s = np.sqrt(hex_fraction)
    return int(round(nx * s)), int(round(ny * s))


def cell_codes(ii, jj, kk, layers, px, py):
    """Cell type (CELL_*) of cells (ii, jj, kk) of the boundary-layer box."""
    patch = (ii < px) & (jj < py)
    code = np.full(np.shape(ii), CELL_KUHN, dtype=np.int8)
    code[(kk < layers) & patch] = CELL_HEX
    code[(kk < layers) & ~patch] = CELL_PRI
    code[(kk == layers) & patch] = CELL_TRANS
    return code


def boundary_layer_blocks(nx, ny, nz, layers, px, py, ii, jj, kk):
    """Element blocks (kind tag -> connectivity with GLOBAL grid node ids) of
    the given cells, in the order boundary_layer_mesh emits them: per kind
    in ascending cell id, the transition tets before the Kuhn tets.  The
    cells must be in ascending cell id ((i * ny + j) * nz + k)."""
    code = cell_codes(ii, jj, kk, layers, px, py)
    blocks = {}

    def sel(c):
        m = code == c
        return ii[m], jj[m], kk[m]

    ci, cj, ck = sel(CELL_HEX)
    if ci.size:
        c = _cell_corner_ids(nx, ny, nz, ci, cj, ck)
        order = [(0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0), (0, 0, 1), (1, 0, 1), (1, 1, 1), (0, 1, 1)]
        blocks["hex"] = np.stack([c[o] for o in order], axis=1)
    ci, cj, ck = sel(CELL_PRI)
    if ci.size:  # split along the xy diagonal
        c = _cell_corner_ids(nx, ny, nz, ci, cj, ck)
        pa = np.stack([c[(0, 0, 0)], c[(1, 0, 0)], c[(1, 1, 0)], c[(0, 0, 1)], c[(1, 0, 1)], c[(1, 1, 1)]], axis=1)
        pb = np.stack([c[(0, 0, 0)], c[(1, 1, 0)], c[(0, 1, 0)], c[(0, 0, 1)], c[(1, 1, 1)], c[(0, 1, 1)]], axis=1)
        blocks["pri"] = np.stack([pa, pb], axis=1).reshape(-1, 6)
    ci, cj, ck = sel(CELL_TRANS)
    trans_tets = None
    if ci.size:  # pyramid (base = bottom quad, apex = max corner) + 4 Kuhn tets
        c = _cell_corner_ids(nx, ny, nz, ci, cj, ck)
        blocks["pyr"] = np.stack([c[(0, 0, 0)], c[(1, 0, 0)], c[(1, 1, 0)], c[(0, 1, 0)], c[(1, 1, 1)]], axis=1)
        trans_tets = _kuhn_tets(c, perms=[(0, 2, 1), (1, 2, 0), (2, 0, 1), (2, 1, 0)])
    ci, cj, ck = sel(CELL_KUHN)
    tets = _kuhn_tets(_cell_corner_ids(nx, ny, nz, ci, cj, ck)) if ci.size else np.zeros((0, 4), np.int64)
    if trans_tets is not None:
        tets = np.concatenate([trans_tets, tets], axis=0)
    if tets.shape[0]:
        blocks["tet"] = tets
    return blocks


def boundary_layer_mesh(nx, ny, nz, layers, hex_fraction=0.25, lengths=(1.0, 1.0, 1.0)):
    """Conforming mixed tet/prism/pyramid/hex boundary-layer box (C3/C4/C5).

    Prism layers k < ``layers`` except a hex "wing patch" covering
    ``hex_fraction`` of the wall (i < px, j < py); transition cells (one
    pyramid + four Kuhn tets) above the patch at k == layers; Kuhn tets
    everywhere else.  dmesh.py generates the same
    elements for a subset of the cells (one rank's subdomain).
    """
    px, py = patch_extent(nx, ny, hex_fraction)
    coords = _grid_nodes(nx, ny, nz, lengths)
    ii, jj, kk = _cells(nx, ny, nz)
    blocks = boundary_layer_blocks(nx, ny, nz, layers, px, py, ii, jj, kk)
    return _finish(coords, blocks, shape=(nx, ny, nz))


def boundary_nodes(mesh: MeshArrays, tol=1e-12):
    """Boolean mask of nodes on the bounding box faces."""
    x = mesh.coords
    lo, hi = x.min(axis=0), x.max(axis=0)
    return np.any((np.abs(x - lo) < tol) | (np.abs(x - hi) < tol), axis=1)


def c2_mesh(n=88, jitter=0.2, seed=20200131):
    """BASELINE.json configs[1]: jittered Kuhn TET04 unit box, 88^3 cells
    -> 4,088,832 elements / 704,969 nodes."""
    return box_tets(n, n, n, jitter=jitter, seed=seed)


def c1_mesh(n=32):
    """BASELINE.json configs[0]: periodic [0,2pi]^3 HEX08 box, 32^3 cells."""
    L = 2.0 * np.pi
    return box_hexes(n, n, n, lengths=(L, L, L), periodic=True)


def c3_mesh(scale=1.0):
    """BASELINE.json configs[2]: 150x150x245 cells, 30 prism layers, 25% hex
    patch -> ~30.2M elements (scale shrinks every axis for tests)."""
    nx = max(2, int(round(150 * scale)))
    nz = max(4, int(round(245 * scale)))
    layers = max(1, int(round(30 * scale)))
    return boundary_layer_mesh(nx, nx, nz, layers, hex_fraction=0.25)


def c4_mesh():
    """BASELINE.json configs[3]: 300x300x490 cells, 40 prism layers, 25% hex
    patch -> ~249M elements / 44.5M nodes."""
    return boundary_layer_mesh(300, 300, 490, 40, hex_fraction=0.25)


# ---------------------------------------------------------------------------
# Initial / boundary conditions of the BASELINE configurations
# ---------------------------------------------------------------------------

def tgv_initial(coords, V0=1.0):
    """Taylor-Green vortex on [0,2pi]^3 (C1)."""
    x, y, z = coords[:, 0], coords[:, 1], coords[:, 2]
    u = np.stack([V0 * np.sin(x) * np.cos(y) * np.cos(z), -V0 * np.cos(x) * np.sin(y) * np.cos(z),
                  np.zeros_like(x)], axis=1)
    p = (V0 ** 2 / 16.0) * (np.cos(2 * x) + np.cos(2 * y)) * (np.cos(2 * z) + 2.0)
    return u, p


def c2_initial(coords, seed=20200131, noise=0.01):
    """C2: TGV-like field on the unit cube + N(0, noise^2), p = 0."""
    x, y, z = (2 * np.pi * coords[:, i] for i in range(3))
    u = np.stack([np.sin(x) * np.cos(y) * np.cos(z), -np.cos(x) * np.sin(y) * np.cos(z), np.zeros_like(x)], axis=1)
    rng = np.random.default_rng(seed)
    return u + rng.normal(0.0, noise, size=u.shape), np.zeros(coords.shape[0])


def wall_model_bcs(mesh: MeshArrays, bounds=None):
    """C3-C5 with the equilibrium wall model on z = 0 (Algorithm 1 line 4):
    inflow u = (1,0,0) at x = 0, zero normal velocity on the wall (the wall
    shear comes from the wall law), p = 0 at x = 1.  Returns (bcs, (faces,
    off)) for FlowSolver(**bcs, wall=(faces, off)).  ``bounds`` = (lo, hi)
    of the whole box (a subdomain's own extent is not the box's); default:
    this mesh's extent."""
    from .wall import wall_faces
    x = mesh.coords
    n = mesh.n_nodes
    lo, hi = (x.min(axis=0), x.max(axis=0)) if bounds is None else (np.asarray(bounds[0]), np.asarray(bounds[1]))
    uf = np.zeros((n, 3), bool)
    uv = np.zeros((n, 3))
    inflow = np.abs(x[:, 0] - lo[0]) < 1e-12
    wall = np.abs(x[:, 2] - lo[2]) < 1e-12
    uf[wall, 2] = True
    uf[inflow] = True
    uv[inflow] = (1.0, 0.0, 0.0)
    pf = np.abs(x[:, 0] - hi[0]) < 1e-12
    return dict(p_fixed=pf, u_fixed=uf, u_fixed_values=uv), wall_faces(mesh, wall)


def channel_bcs(mesh: MeshArrays):
    """C3-C5 boundary conditions: inflow u = (1,0,0) at x = 0, no-slip at
    z = 0, p = 0 at x = 1."""
    x = mesh.coords
    n = mesh.n_nodes
    uf = np.zeros((n, 3), bool)
    uv = np.zeros((n, 3))
    inflow = np.abs(x[:, 0] - x[:, 0].min()) < 1e-12
    wall = np.abs(x[:, 2] - x[:, 2].min()) < 1e-12
    uf[inflow] = True
    uv[inflow] = (1.0, 0.0, 0.0)
    uf[wall] = True
    uv[wall] = 0.0
    pf = np.abs(x[:, 0] - x[:, 0].max()) < 1e-12
    return dict(p_fixed=pf, u_fixed=uf, u_fixed_values=uv)

"""Voxel tetrahedral enclosure: rest operators and the voxel-grid builder.

Host-side (numpy) preparation of the inputs the B200 step consumes.  It mirrors
the fields of the reference `VolumeMesh` that the PD hot path reads
(`volmesh.py:53-99`): `nodes`, `tets`, `volume`, `shape_grad`, `node_mass`,
plus the voxel bookkeeping (`node_grid`, `voxels`, `tet_voxel`, `cell_size`,
`origin`).  The dead-weight `diff_op` (nE,9,12) and `dtd` (nE,12,12) tensors of
the reference are not materialised: the device kernels work from `shape_grad`.

Any object exposing `nodes`, `tets`, `volume`, `shape_grad` and `node_mass`
(including the reference's own `VolumeMesh`) is accepted by the simulator.
"""

from __future__ import annotations

import itertools
import json
import warnings

import numpy as np

__all__ = ["VolumeMesh", "CELL_TETS", "CELL_CORNERS", "voxel_mesh", "lump_mass_density",
           "rest_operators"]

# corner c of the unit cell sits at (c & 1, (c >> 1) & 1, (c >> 2) & 1)
CELL_CORNERS = np.array([[c & 1, (c >> 1) & 1, (c >> 2) & 1] for c in range(8)], dtype=np.int64)


def _kuhn_six():
    """Kuhn/Freudenthal split of the unit cell into six tets on the 0-7 diagonal.

    One tet per permutation of the axis order (itertools order), each walking
    0 -> +e_a -> +e_a+e_b -> 7 and re-oriented to positive volume by swapping its
    two middle corners.  Same split and order as `volmesh._local_tets`
    (`volmesh.py:24-46`), so face-adjacent cells agree on their shared faces.
    """
    code = {tuple(c): i for i, c in enumerate(CELL_CORNERS.tolist())}
    out = []
    for order in itertools.permutations(range(3)):
        walk = [np.zeros(3, dtype=np.int64)]
        for ax in order[:2]:
            step = walk[-1].copy()
            step[ax] += 1
            walk.append(step)
        walk.append(np.ones(3, dtype=np.int64))
        ids = [code[tuple(w.tolist())] for w in walk]
        e = np.array([walk[1] - walk[0], walk[2] - walk[0], walk[3] - walk[0]], dtype=float)
        if np.linalg.det(e.T) < 0.0:
            ids[1], ids[2] = ids[2], ids[1]
        out.append(tuple(ids))
    return out


CELL_TETS = np.array(_kuhn_six(), dtype=np.int64)


def rest_operators(nodes, tets):
    """Rest volume and shape gradients of every tet (`volmesh.py:79-91`).

    Dm holds the rest edges X1-X0, X2-X0, X3-X0 as columns; V = det(Dm)/6 must be
    positive; rows 1..3 of G are the rows of Dm^-1 and G[0] = -(G[1]+G[2]+G[3]).
    """
    nodes = np.asarray(nodes, dtype=np.float64)
    tets = np.asarray(tets, dtype=np.int64)
    corner = nodes[tets]                                    # (nE, 4, 3)
    Dm = np.swapaxes(corner[:, 1:] - corner[:, :1], 1, 2)   # (nE, 3, 3), edges as columns
    det = np.linalg.det(Dm)
    if np.any(det <= 0.0):
        raise ValueError("non-positive element volume")
    inv = np.linalg.inv(Dm)
    G = np.empty((len(tets), 4, 3))
    G[:, 1:] = inv
    G[:, 0] = -inv.sum(axis=1)
    return det / 6.0, G


class VolumeMesh:
    """Tet enclosure with the rest operators the PD step needs.

    Field meaning follows the reference `VolumeMesh` (`volmesh.py:53-69`).
    """

    def __init__(self, nodes, tets, cell_size=1.0, origin=None, node_grid=None, voxels=None,
                 tet_voxel=None, node_mass=None, volume=None, shape_grad=None):
        self.nodes = np.ascontiguousarray(nodes, dtype=np.float64).reshape(-1, 3)
        self.tets = np.ascontiguousarray(tets, dtype=np.int64).reshape(-1, 4)
        self.cell_size = float(cell_size)
        self.origin = np.zeros(3) if origin is None else np.asarray(origin, dtype=float)
        self.node_grid = node_grid
        self.voxels = voxels
        self.tet_voxel = tet_voxel
        if volume is None or shape_grad is None:
            volume, shape_grad = rest_operators(self.nodes, self.tets)
        self.volume = np.asarray(volume, dtype=np.float64)
        self.shape_grad = np.asarray(shape_grad, dtype=np.float64)
        self.node_mass = None if node_mass is None else np.asarray(node_mass, dtype=np.float64)

    @property
    def n_nodes(self):
        return self.nodes.shape[0]

    @property
    def n_elements(self):
        return self.tets.shape[0]

    def deformation_gradients(self, x):
        """F = sum_n x_n (x) g_n per tet (`volmesh.py:115-118`), host numpy, (nE,3,3)."""
        xe = np.asarray(x, dtype=np.float64).reshape(-1, 3)[self.tets]   # (nE,4,3)
        return np.einsum("eni,enj->eij", xe, self.shape_grad)


def voxel_mesh(cells, cell_size, origin=(0.0, 0.0, 0.0)):
    """Split occupied voxel cells into six tets each.

    Numbering reproduces `volmesh.voxelize` (`volmesh.py:268-293`): cells in
    lexicographic order, grid corners in lexicographic order, six tets per
    cell in `CELL_TETS` order.
    """
    cells = np.unique(np.asarray(cells, dtype=np.int64).reshape(-1, 3), axis=0)
    corners = (cells[:, None, :] + CELL_CORNERS[None, :, :]).reshape(-1, 3)
    grid, inverse = np.unique(corners, axis=0, return_inverse=True)
    corner_ids = inverse.reshape(len(cells), 8)
    tets = corner_ids[:, CELL_TETS].reshape(-1, 4)
    origin = np.asarray(origin, dtype=float)
    nodes = origin + grid.astype(np.float64) * float(cell_size)
    return VolumeMesh(nodes, tets, cell_size=cell_size, origin=origin, node_grid=grid,
                      voxels=cells, tet_voxel=np.repeat(np.arange(len(cells)), 6))


def lump_mass_density(mesh, rho):
    """Lumped node masses m_i = sum over incident tets of rho * V_e / 4."""
    m = np.zeros(mesh.n_nodes)
    np.add.at(m, mesh.tets.reshape(-1), np.repeat(rho * mesh.volume / 4.0, 4))
    mesh.node_mass = m
    return m


# ---------------------------------------------------------------------------
# mesh and material files: the reference's text formats,
# parsed with numpy's C reader instead of a Python loop per line


class ConfigError(ValueError):
    """Unreadable input file (the reference CLI's `ConfigError`, `cli.py:225-240`)."""


def _header_rows(path):
    """(number of leading comment/blank lines, first data row as tokens)."""
    skip = 0
    with open(path) as fh:
        for line in fh:
            s = line.strip()
            if s and not s.startswith("#"):
                return skip, s.split()
            skip += 1
    raise ConfigError(f"{path}: no data rows")


def _table(path, skip, cols, dtype):
    a = np.loadtxt(path, dtype=dtype, comments="#", skiprows=skip + 1, ndmin=2)
    if a.size == 0:
        return np.empty((0, cols), dtype=dtype)
    if a.shape[1] < cols:
        raise ConfigError(f"{path}: expected {cols} columns, found {a.shape[1]}")
    return a[:, :cols]


def read_mesh(prefix):
    """Read `<prefix>.node/.ele/.json` as written by the reference `write_mesh` (`volmesh.py:575-611`).

    Rows are placed by their leading index, as in the reference reader.
    """
    skip, head = _header_rows(f"{prefix}.node")
    n = int(head[0])
    rows = _table(f"{prefix}.node", skip, 4, np.float64)
    nodes = np.empty((n, 3))
    nodes[rows[:, 0].astype(np.int64)] = rows[:, 1:4]
    skip, head = _header_rows(f"{prefix}.ele")
    m = int(head[0])
    rows = _table(f"{prefix}.ele", skip, 5, np.int64)
    tets = np.empty((m, 4), dtype=np.int64)
    tets[rows[:, 0]] = rows[:, 1:5]
    with open(f"{prefix}.json") as fh:
        meta = json.load(fh)
    origin = np.asarray(meta["origin"], dtype=float)
    h = float(meta["cell_size"])
    grid = np.rint((nodes - origin) / h).astype(np.int64)
    mesh = VolumeMesh(nodes, tets, cell_size=h, origin=origin, node_grid=grid,
                      voxels=np.asarray(meta["voxels"], dtype=np.int64),
                      tet_voxel=np.asarray(meta["tet_voxel"], dtype=np.int64))
    if "node_mass" in meta:
        mesh.node_mass = np.asarray(meta["node_mass"], dtype=float)
    return mesh


def boundary_faces(mesh):
    """Faces used by one tet, outward-oriented, sorted (`volmesh.py:505-535`)."""
    t = mesh.tets
    faces, opp = [], []
    for k in range(4):
        faces.append(np.delete(t, k, axis=1))
        opp.append(t[:, k])
    faces = np.concatenate(faces)
    opp = np.concatenate(opp)
    key = np.sort(faces, axis=1)
    _, inv, cnt = np.unique(key, axis=0, return_inverse=True, return_counts=True)
    one = cnt[inv.reshape(-1)] == 1
    f, o = faces[one], opp[one]
    a, b, c = (mesh.nodes[f[:, i]] for i in range(3))
    nrm = np.cross(b - a, c - a)
    flip = np.einsum("ij,ij->i", nrm, mesh.nodes[o] - a) > 0.0
    f[flip] = f[flip][:, [0, 2, 1]]
    order = np.lexsort(f.T[::-1])
    return f[order]


def write_mesh(mesh, prefix, comment=None):
    """Write `<prefix>.node/.ele/.json/_boundary.obj` in the reference format (`volmesh.py:538-572`)."""
    head = f"# {comment}\n" if comment else ""
    idx = np.arange(mesh.n_nodes)[:, None]
    with open(f"{prefix}.node", "w") as fh:
        fh.write(head)
        fh.write(f"{mesh.n_nodes} 3 0 0\n")
        np.savetxt(fh, np.hstack([idx, mesh.nodes]), fmt=["%d", "%.17g", "%.17g", "%.17g"])
    with open(f"{prefix}.ele", "w") as fh:
        fh.write(head)
        fh.write(f"{mesh.n_elements} 4 0\n")
        np.savetxt(fh, np.hstack([np.arange(mesh.n_elements)[:, None], mesh.tets]), fmt="%d")
    meta = {
        "cell_size": mesh.cell_size,
        "origin": [float(v) for v in mesh.origin],
        "voxels": [[int(v) for v in c] for c in (mesh.voxels if mesh.voxels is not None else [])],
        "tet_voxel": [int(v) for v in (mesh.tet_voxel if mesh.tet_voxel is not None else [])],
    }
    if mesh.node_mass is not None:
        meta["node_mass"] = [float(v) for v in mesh.node_mass]
    if comment:
        meta["comment"] = comment
    with open(f"{prefix}.json", "w") as fh:
        json.dump(meta, fh)
    with open(f"{prefix}_boundary.obj", "w") as fh:
        fh.write(head)
        np.savetxt(fh, mesh.nodes, fmt="v %.17g %.17g %.17g")
        np.savetxt(fh, boundary_faces(mesh) + 1, fmt="f %d %d %d")


def read_material(path):
    """`element,gamma_s,gamma_v` CSV (`cli.py:225-240`) -> MaterialField."""
    from .material import MaterialField
    try:
        skip, head = _header_rows(path)
    except OSError as exc:
        raise ConfigError(f"cannot read material file {path}: {exc}") from exc
    except ConfigError:
        raise ConfigError(f"material file {path} holds no rows") from None
    if head[0].startswith("element"):
        skip += 1
    try:
        with warnings.catch_warnings():
            warnings.simplefilter("ignore", UserWarning)      # "input contained no data"
            a = np.loadtxt(path, delimiter=",", comments="#", skiprows=skip, ndmin=2)
    except (OSError, ValueError) as exc:
        raise ConfigError(f"cannot read material file {path}: {exc}") from exc
    if a.size == 0:
        raise ConfigError(f"material file {path} holds no rows")
    return MaterialField(np.ascontiguousarray(a[:, 1]), np.ascontiguousarray(a[:, 2]))

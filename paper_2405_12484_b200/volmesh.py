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

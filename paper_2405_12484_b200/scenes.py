"""Synthetic scenes for the benchmark configurations.

All scenes are voxel enclosures with h = 5 mm, rho = 300 kg/m^3 lumped as
rho*V/4 per incident tet, dt = 1/150 s, gravity (0, 0, -9.81) * m, 30 PD
iterations, damping 1.  Random streams are seeded (`default_rng(240512484)`
unless stated), so every scene is bit-reproducible on any host.

  C1  swatch   11x11x3 box (2,178 tets / 576 nodes), grid-x = 0 pinned,
               gamma_s ~ U(50,500), gamma_v ~ U(10,100)
  C2  scarf    100x25x2 strip (30,000 / 7,878) hanging from its x = 0 edge,
               1x1 rib stripes along the wales (cell index y)
  C3  sweater  voxelised cylindrical shell two cells thick, ~390K tets, top
               ring pinned, cable-pattern parameters
  C5  garment  C3 scaled to ~4M tets
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .material import MaterialField
from .volmesh import VolumeMesh, lump_mass_density, voxel_mesh

H = 0.005
RHO = 300.0
DT = 1.0 / 150.0
GRAVITY = np.array([0.0, 0.0, -9.81])
SEED = 240512484


@dataclass
class Scene:
    name: str
    mesh: VolumeMesh
    gammas: MaterialField
    pins: np.ndarray
    pin_targets: np.ndarray
    forces: np.ndarray
    dt: float = DT
    iterations: int = 30
    meta: dict = field(default_factory=dict)

    @property
    def n_tets(self):
        return self.mesh.n_elements

    @property
    def n_nodes(self):
        return self.mesh.n_nodes


def _box_cells(nx, ny, nz):
    g = np.stack(np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij"), -1)
    return g.reshape(-1, 3)


def _finish(name, mesh, gs, gv, pins, meta=None):
    lump_mass_density(mesh, RHO)
    pins = np.asarray(pins, dtype=np.int64)
    forces = mesh.node_mass[:, None] * GRAVITY[None, :]
    return Scene(name=name, mesh=mesh, gammas=MaterialField(gs, gv), pins=pins,
                 pin_targets=mesh.nodes[pins].copy(), forces=forces, meta=meta or {})


def box_scene(nx, ny, nz, seed=SEED, name=None):
    """Voxel box with the x = 0 node plane pinned and uniform-random gammas (C1)."""
    mesh = voxel_mesh(_box_cells(nx, ny, nz), H)
    rng = np.random.default_rng(seed)
    gs = rng.uniform(50.0, 500.0, mesh.n_elements)
    gv = rng.uniform(10.0, 100.0, mesh.n_elements)
    pins = np.flatnonzero(mesh.node_grid[:, 0] == 0)
    return _finish(name or f"box{nx}x{ny}x{nz}", mesh, gs, gv, pins)


def c1_swatch(seed=SEED):
    return box_scene(11, 11, 3, seed=seed, name="C1-swatch-2K")


def c2_scarf(nx=100, ny=25, nz=2, seed=SEED):
    """Rib-knit strip hanging from its short x = 0 edge (C2)."""
    mesh = voxel_mesh(_box_cells(nx, ny, nz), H)
    rng = np.random.default_rng(seed)
    wale = mesh.voxels[mesh.tet_voxel, 1] % 2
    gs = 300.0 * (1.0 + 0.8 * wale) * rng.lognormal(0.0, 0.1, mesh.n_elements)
    gv = 50.0 * (1.0 + 2.0 * wale) * rng.lognormal(0.0, 0.1, mesh.n_elements)
    pins = np.flatnonzero(mesh.node_grid[:, 0] == 0)
    return _finish(f"C2-scarf-{mesh.n_elements // 1000}K", mesh, gs, gv, pins)


def _shell_cells(radius, height_cells, thickness_cells=2):
    """Cells whose centre lies in the radial band [R - t/2, R + t/2) (units of h)."""
    r_out = radius + 0.5 * thickness_cells
    r_in = radius - 0.5 * thickness_cells
    n = int(np.ceil(r_out)) + 1
    i = np.arange(-n, n)
    cx, cy = np.meshgrid(i + 0.5, i + 0.5, indexing="ij")
    r = np.hypot(cx, cy)
    ring = np.argwhere((r >= r_in) & (r < r_out)) - n        # (nRing, 2) integer cells
    k = np.arange(height_cells)
    cells = np.concatenate([np.c_[ring, np.full(len(ring), kk)] for kk in k])
    return cells


def cable_pattern(theta, z, radius_m, a=0.008, lam=0.060, w=0.006, n_cables=6):
    """c(theta, z) = sum_k sum_pm exp(-((R (theta - theta_k) -+ a sin(2 pi z / lam)) / w)^2)."""
    c = np.zeros_like(theta)
    wave = a * np.sin(2.0 * np.pi * z / lam)
    for k in range(n_cables):
        d = np.angle(np.exp(1j * (theta - 2.0 * np.pi * k / n_cables)))   # wrap to (-pi, pi]
        for sgn in (1.0, -1.0):
            c += np.exp(-(((radius_m * d) - sgn * wave) / w) ** 2)
    return c


def sweater_scene(target_tets=390_000, height_m=0.65, seed=SEED, name=None):
    """Voxelised cylindrical shell, two cells thick, top ring pinned (C3 / C5).

    The radius is chosen so the tet count lands within 1% of `target_tets`
    at the given height; gammas follow the cable pattern with LogNormal(0, 0.1)
    per-tet noise.
    """
    height_cells = int(round(height_m / H))
    # per layer ~ 4 pi R / h cells for a two-cell band
    radius = target_tets / 6.0 / height_cells * 1.0 / (4.0 * np.pi)
    best = None
    for dr in np.linspace(-3.0, 3.0, 121):
        cells = _shell_cells(radius + dr, height_cells)
        err = abs(len(cells) * 6 - target_tets)
        if best is None or err < best[0]:
            best = (err, radius + dr, cells)
    _, radius, cells = best
    mesh = voxel_mesh(cells, H)
    rng = np.random.default_rng(seed)
    cen = mesh.nodes[mesh.tets].mean(axis=1)
    theta = np.arctan2(cen[:, 1], cen[:, 0])
    c = cable_pattern(theta, cen[:, 2], radius * H)
    gs = 300.0 * (1.0 + 2.0 * c) * rng.lognormal(0.0, 0.1, mesh.n_elements)
    gv = 50.0 * (1.0 + 4.0 * c) * rng.lognormal(0.0, 0.1, mesh.n_elements)
    pins = np.flatnonzero(mesh.node_grid[:, 2] == mesh.node_grid[:, 2].max())
    nm = name or f"C3-sweater-{mesh.n_elements // 1000}K"
    return _finish(nm, mesh, gs, gv, pins, meta={"radius_m": radius * H, "height_cells": height_cells})


def c3_sweater(seed=SEED):
    return sweater_scene(390_000, 0.65, seed=seed, name=None)


def c5_garment(seed=SEED):
    """C3 scaled by ~sqrt(10) in both radius and height to ~4.0M tets."""
    return sweater_scene(4_000_000, 0.65 * np.sqrt(4_000_000 / 390_000), seed=seed,
                         name="C5-garment-4M")


def contact_scene():
    """Small box dropped onto a tilted plane and a sphere (collider parity scene)."""
    sc = box_scene(8, 6, 3, name="contact-box")
    m = sc.mesh
    lo = m.nodes.min(axis=0)
    hi = m.nodes.max(axis=0)
    colliders = [("plane", (0.0, 0.0, lo[2] - 0.002), (0.1, 0.0, 1.0)),
                 ("sphere", (hi[0] - 0.006, 0.5 * (lo[1] + hi[1]), lo[2] - 0.02), 0.0195)]
    return sc, colliders


SCENES = {
    "C1": c1_swatch,
    "C2": c2_scarf,
    "C3": c3_sweater,
    "C5": c5_garment,
}


def make_scene(key, **kw):
    return SCENES[key](**kw)


def equilibrium_case():
    """C1 inputs of the pd_equilibrium fixtures: a sagging inertia target, a perturbed start."""
    sc = c1_swatch()
    rng = np.random.default_rng(11)
    a = 0.3 * sc.dt ** 2 * sc.forces / sc.mesh.node_mass[:, None]
    x0 = sc.mesh.nodes + 0.001 * rng.normal(size=sc.mesh.nodes.shape)
    return sc, a, x0


def second_order_case():
    """C1 inputs of the second-order fixtures: a perturbed x for the gradient / exact
    Hessian, and the dynamic step of newton_polish (gravity prediction from rest)."""
    sc = c1_swatch()
    rng = np.random.default_rng(12)
    x = sc.mesh.nodes + 0.002 * rng.normal(size=sc.mesh.nodes.shape)
    inv_m = 1.0 / sc.mesh.node_mass
    xhat = sc.mesh.nodes + sc.dt ** 2 * inv_m[:, None] * sc.forces
    return sc, x, xhat


class TrackingProblem:
    """Synthetic stand-in for the reference FitProblem's duck-typed surface
    (`fitting.py:92-170`) used by the adjoint fixtures: loss = sum_i w_i |x_i - t_i|^2."""

    def __init__(self, mesh, dt, target, weight):
        self.mesh = mesh
        self.dt = dt
        self.target = np.asarray(target, dtype=float)
        self.weight = np.asarray(weight, dtype=float)

    def loss(self, x, sample):
        d = np.asarray(x).reshape(-1, 3) - self.target
        return float(np.sum(self.weight[:, None] * d * d))

    def loss_grad_x(self, x, sample):
        return 2.0 * self.weight[:, None] * (np.asarray(x).reshape(-1, 3) - self.target)

    def loss_hessian_scalar(self, sample):
        import scipy.sparse as sp
        return sp.diags(2.0 * self.weight).tocsr()

    def free_dofs(self, sample):
        free = np.setdiff1d(np.arange(self.mesh.n_nodes), sample.pins)
        return (3 * free[:, None] + np.arange(3)[None, :]).reshape(-1)


class TrackingSample:
    def __init__(self, pins, pin_vals, inertia, index=0):
        self.pins = np.asarray(pins, dtype=int)
        self.pin_vals = np.asarray(pin_vals, dtype=float)
        self.inertia = np.asarray(inertia, dtype=float)
        self.index = index


def adjoint_case():
    """C1 quasi-static sample for the adjoint fixtures: the equilibrium_case loads; the
    tracking target is a seeded perturbation of the equilibrium (found by the caller)."""
    sc, a, x0 = equilibrium_case()
    rng = np.random.default_rng(13)
    weight = rng.uniform(0.5, 2.0, sc.mesh.n_nodes)
    shift = 0.001 * rng.normal(size=sc.mesh.nodes.shape)
    sample = TrackingSample(sc.pins, sc.pin_targets, a)
    return sc, a, x0, weight, shift, sample

"""Drop-in projective-dynamics API backed by the B200 (sm_100a) library.

Mirrors the reference simulator surface (`/root/reference/pkg/src/volknit/pdsolver.py`):

  SimState                       pdsolver.py:180-198
  assemble_global(mesh, g, dt)   pdsolver.py:42-56     (assembled on the GPU, returned as CSC)
  elastic_rhs(mesh, g, x)        pdsolver.py:59-71     (GPU local step + deterministic gather)
  GlobalSolver(K, free, pins)    pdsolver.py:201-246   (GPU persistent CG; `.solve(B, pin_vals)`)
  pd_step(state, mesh, g, ...)   pdsolver.py:257-304
  simulate_mesh(mesh, g, ...)    pdsolver.py:710-763
  pd_objective / elastic_energy  pdsolver.py:74-82, 307-312 (diagnostics, projections on GPU)
  elastic_gradient               pdsolver.py:85-97     (GPU, float64)
  exact_elastic_hessian          pdsolver.py:100-118   (GPU-assembled CSR, float64)
  newton_polish                  pdsolver.py:350-460   (GPU gradient/energy, GN solve, MINRES exact step)

Same argument names, meaning and error behaviour: ValueError for invalid input,
RuntimeError("... non-finite positions at iteration {it}") on blow-up, any
object with `.solve(B, pin_vals)` accepted as `solver=`.  All arithmetic runs
in the CUDA library; nothing here falls back to the CPU.

Extra keyword arguments (not in the reference): `precision` ("fp64" default, the
reference's arithmetic; "fp32" the fast path, within 1e-5 of the reference after one
frame and 1e-3 after 100 frames, tests/test_gpu_parity.py), `tol` (relative residual
of each global solve) and `max_iters`.

Solver modes: "direct" is the exact global step (the reference's SuperLU),
realised as a persistent CG on the device driven to `tol`; "cms" is the
reference's component-mode subspace + A-Jacobi path (see `cms.py`).
"""

from __future__ import annotations

import logging
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

from . import _abi
from .cms import CmsSubspace, a_jacobi_refine, build_cms, classify_nodes, partition_elements  # noqa: F401
from .material import MaterialField

log = logging.getLogger(__name__)

PD_ITERS_DEFAULT = 30       # pdsolver.py:23
JACOBI_OMEGA = 0.75         # pdsolver.py:24
CONTACT_STIFFNESS = 1e4     # pdsolver.py:25

DEFAULT_TOL = {"fp32": 2e-6, "fp64": 1e-12}


@dataclass
class SimState:
    """Forward-simulation state; pinned nodes track their targets exactly (`pdsolver.py:180-198`)."""

    x: np.ndarray
    v: np.ndarray
    dt: float
    pins: np.ndarray = field(default_factory=lambda: np.empty(0, dtype=int))
    pin_targets: np.ndarray = None
    colliders: tuple = ()

    def __post_init__(self):
        if _is_cuda_tensor(self.x):
            # PyTorch carrier: x / v stay float64 CUDA tensors and pd_step keeps them on the device
            import torch
            self.x = self.x.detach().to(torch.float64).reshape(-1, 3).contiguous().clone()
            v = self.v if _is_cuda_tensor(self.v) else torch.as_tensor(np.asarray(self.v, dtype=float))
            self.v = v.detach().to(device=self.x.device, dtype=torch.float64).reshape(-1, 3).contiguous().clone()
            self.pins = np.asarray(self.pins, dtype=int)
            if self.pin_targets is None and len(self.pins):
                self.pin_targets = self.x[torch.as_tensor(self.pins, device=self.x.device)].clone()
            if self.dt <= 0.0:
                raise ValueError("dt must be positive")
            return
        self.x = np.asarray(self.x, dtype=float).reshape(-1, 3).copy()
        self.v = np.asarray(self.v, dtype=float).reshape(-1, 3).copy()
        self.pins = np.asarray(self.pins, dtype=int)
        if self.pin_targets is None and len(self.pins):
            self.pin_targets = self.x[self.pins].copy()
        if self.dt <= 0.0:
            raise ValueError("dt must be positive")


def _is_cuda_tensor(a):
    return getattr(a, "is_cuda", False) and hasattr(a, "data_ptr")


def _check_inputs(mesh, gammas, dt):
    if dt <= 0.0:
        raise ValueError("dt must be positive")
    if np.any(np.asarray(gammas.gamma_s) < 0.0) or np.any(np.asarray(gammas.gamma_v) < 0.0):
        raise ValueError("negative material coefficient")
    if getattr(mesh, "node_mass", None) is None:
        raise ValueError("mesh node masses not lumped yet")


# ---------------------------------------------------------------------------
# device contexts (one per scene configuration), cached by array identity

_CACHE = {}
_CACHE_MAX = 8


def _ident(arrs):
    return tuple((id(a), a.__array_interface__["data"][0], a.shape) for a in map(np.asarray, arrs))


def current_device():
    """CUDA ordinal for new device contexts: torch's current device when torch has initialised CUDA
    (one process per GPU: `torch.cuda.set_device(local_rank)`), else $VKPD_DEVICE, else 0."""
    import os
    import sys
    torch = sys.modules.get("torch")
    if torch is not None and torch.cuda.is_initialized():
        return int(torch.cuda.current_device())
    return int(os.environ.get("VKPD_DEVICE", "0"))


def _key(mesh, gammas, dt, pins, precision, tol, max_iters):
    """Cache key of the mesh part of a device scene (the material is refreshed in place)."""
    ident = _ident((mesh.tets, mesh.shape_grad, mesh.volume, mesh.node_mass))
    pins = np.asarray(pins, dtype=np.int64)
    return (ident, float(dt), pins.tobytes(), precision, tol, max_iters, current_device())


def invalidate_cache():
    """Drop cached device contexts (call after editing mesh/material arrays in place)."""
    _CACHE.clear()


def device_context(mesh, gammas, dt, pins=(), precision="fp32", tol=None, max_iters=0):
    """Device-resident scene for (mesh, gammas, dt, pins); created once and cached.

    A new MaterialField for a cached mesh (the fitting loop's case, `fitting.py:429-432`)
    refreshes the context's weights and re-assembles K on the device instead of rebuilding it.
    """
    _check_inputs(mesh, gammas, dt)
    tol = DEFAULT_TOL[precision] if tol is None else float(tol)
    k = _key(mesh, gammas, dt, pins, precision, tol, max_iters)
    gid = _ident((gammas.gamma_s, gammas.gamma_v))
    hit = _CACHE.get(k)
    if hit is None:
        if len(_CACHE) >= _CACHE_MAX:
            _CACHE.pop(next(iter(_CACHE)))
        ctx = _abi.Context(mesh.n_nodes if hasattr(mesh, "n_nodes") else len(mesh.nodes), mesh.tets,
                           mesh.shape_grad, mesh.volume, mesh.node_mass, gammas.gamma_s,
                           gammas.gamma_v, pins, dt, precision=precision, tol=tol,
                           max_iters=max_iters, device=k[-1], nodes=getattr(mesh, "nodes", None))
        # the entry keeps the gamma arrays it was built from alive, so their ids cannot be reused
        # by a later MaterialField (which would skip a needed refresh)
        _CACHE[k] = [gid, ctx, (gammas.gamma_s, gammas.gamma_v)]
        return ctx
    if hit[0] != gid:
        hit[1].set_gammas(gammas.gamma_s, gammas.gamma_v)
        hit[0] = gid
        hit[2] = (gammas.gamma_s, gammas.gamma_v)
    return hit[1]


# ---------------------------------------------------------------------------
# assembly and local step


def assemble_global(mesh, gammas, dt, precision="fp64"):
    """Scalar global matrix K = M/dt^2 + sum_e 2 V_e (gs + gv) G G^T (`pdsolver.py:42-56`).

    Assembled on the device (deterministic node-centric sum) and returned as a
    scipy CSC matrix for callers that want the matrix itself.
    """
    ctx = device_context(mesh, gammas, dt, (), precision)
    indptr, indices, data = ctx.matrix_csr()
    n = ctx.n
    return sp.csr_matrix((data, indices, indptr), shape=(n, n)).tocsc()


def elastic_rhs(mesh, gammas, x, precision="fp64"):
    """Local-step rhs sum_e 2 V_e G^T (gs R + gv V) and (F, R, V) (`pdsolver.py:59-71`)."""
    m = mesh
    if getattr(m, "node_mass", None) is None:
        m = _MassShim(mesh)
    ctx = device_context(m, gammas, 1.0, (), precision)
    rhs, F, R, V = ctx.elastic_rhs(np.asarray(x, dtype=float).reshape(-1, 3))
    return rhs, F, R, V


class _MassShim:
    """elastic_rhs does not need masses; give the context unit masses."""

    def __init__(self, mesh):
        self.tets, self.shape_grad, self.volume = mesh.tets, mesh.shape_grad, mesh.volume
        self.n_nodes = mesh.nodes.shape[0]
        self.nodes = mesh.nodes
        self.node_mass = _MassShim._ones(self.n_nodes)

    _ones_cache = {}

    @staticmethod
    def _ones(n):
        a = _MassShim._ones_cache.get(n)
        if a is None:
            a = _MassShim._ones_cache[n] = np.ones(n)
        return a


def elastic_energy(mesh, gammas, x, FRV=None, precision="fp64"):
    """sum_e V_e (gs |F - R|^2 + gv |F - V|^2) (`pdsolver.py:74-82`).

    Without FRV the whole sum runs on the GPU in float64 (deterministic reduction);
    `precision="fp32"` takes the projections from the fp32 local step instead.
    """
    if FRV is None and precision == "fp64":
        e, _ = hess_context(mesh, gammas).energy_grad(x, want_energy=True, want_grad=False)
        return e
    if FRV is None:
        _, F, R, V = elastic_rhs(mesh, gammas, x, precision)
    else:
        F, R, V = FRV
    ds = np.sum((F - R) ** 2, axis=(1, 2))
    dv = np.sum((F - V) ** 2, axis=(1, 2))
    return float(np.sum(mesh.volume * (gammas.gamma_s * ds + gammas.gamma_v * dv)))


# ---------------------------------------------------------------------------
# second order (fitting side): float64 device contexts per (mesh, pins, dt)

_HCACHE = {}


def hess_context(mesh, gammas, dt=1.0, pins=()):
    """Device float64 second-order context for (mesh, pins, dt); gammas refreshed in place."""
    m = mesh if getattr(mesh, "node_mass", None) is not None else _MassShim(mesh)
    k = (_ident((m.tets, m.shape_grad, m.volume, m.node_mass)), float(dt),
         np.asarray(pins, dtype=np.int64).tobytes(), current_device())
    gid = _ident((gammas.gamma_s, gammas.gamma_v))
    hit = _HCACHE.get(k)
    if hit is None:
        if len(_HCACHE) >= _CACHE_MAX:
            _HCACHE.pop(next(iter(_HCACHE)))
        if dt <= 0.0:
            raise ValueError("dt must be positive")
        h = _abi.HessContext(m.n_nodes if hasattr(m, "n_nodes") else len(m.nodes), m.tets, m.shape_grad,
                             m.volume, m.node_mass, gammas.gamma_s, gammas.gamma_v, pins, dt, device=k[-1])
        _HCACHE[k] = [gid, h, (gammas.gamma_s, gammas.gamma_v)]
        return h
    if hit[0] != gid:
        hit[1].set_gammas(gammas.gamma_s, gammas.gamma_v)
        hit[0] = gid
        hit[2] = (gammas.gamma_s, gammas.gamma_v)
    return hit[1]


def elastic_gradient(mesh, gammas, x):
    """Gradient of the elastic energy wrt node positions, (nV, 3) (`pdsolver.py:85-97`).

    Per tet 2 V G^T (gs (F - R) + gv (F - V)) on the GPU, summed per node in tet order
    (the `np.add.at` order), float64.
    """
    _, g = hess_context(mesh, gammas).energy_grad(x, want_energy=False, want_grad=True)
    return g


def exact_elastic_hessian(mesh, gammas, x):
    """Second derivative of the elastic energy over all DOFs, (3nV, 3nV) CSR (`pdsolver.py:100-118`).

    The per-tet blocks 2 V D^T (gs (I - dR/dF) + gv (I - dV/dF)) D are formed on the GPU
    (projection Jacobians of `material.projection_jacobians_batch`) and summed per row in tet
    order; symmetric, not necessarily definite.
    """
    h = hess_context(mesh, gammas)
    h.linearize(np.asarray(x, dtype=float).reshape(-1, 3))
    return h.csr()


def pd_objective(state_or_x, mesh, gammas, xhat, dt, precision="fp64"):
    """Inertia plus elastic potential minimized by one implicit step (`pdsolver.py:307-312`)."""
    x = state_or_x.x if isinstance(state_or_x, SimState) else np.asarray(state_or_x)
    d = x - xhat
    inertia = 0.5 / dt ** 2 * float(np.sum(mesh.node_mass[:, None] * d * d))
    return inertia + elastic_energy(mesh, gammas, x, precision=precision)


def _predicted(state, forces, mesh):
    """xhat = x + dt v + dt^2 m^-1 f, m^-1 := 0 where m = 0 (`pdsolver.py:249-254`)."""
    inv_m = np.zeros(mesh.n_nodes)
    pos = mesh.node_mass > 0.0
    inv_m[pos] = 1.0 / mesh.node_mass[pos]
    f = np.zeros_like(state.x) if forces is None else np.asarray(forces, dtype=float)
    return state.x + state.dt * state.v + state.dt ** 2 * inv_m[:, None] * f


# ---------------------------------------------------------------------------
# global solver


class GlobalSolver:
    """Solves K X = B with pinned values eliminated (`pdsolver.py:201-246`).

    `K` is any sparse SPD matrix (e.g. from `assemble_global`); it is uploaded
    once and every `solve(B, pin_vals)` runs the device CG to `tol`.  Mode
    "cms" routes through the component-mode subspace (`cms.CmsGlobalSolver`).
    """

    def __init__(self, K, free, pins, mode="direct", cms=None, refine_sweeps=0, aggregation=2,
                 omega=JACOBI_OMEGA, chebyshev=False, precision="fp64", tol=None, max_iters=0):
        if mode not in ("direct", "cms"):
            raise ValueError(f"unknown solver mode {mode!r}")
        self.K = K
        self.free = np.asarray(free)
        self.pins = np.asarray(pins, dtype=np.int64)
        self.mode = mode
        self.cms = cms
        self.refine_sweeps = refine_sweeps
        self.aggregation = aggregation
        self.omega = omega
        self.chebyshev = chebyshev
        tol = DEFAULT_TOL[precision] if tol is None else tol
        K = sp.csr_matrix(K)
        n = K.shape[0]
        expect_free = np.setdiff1d(np.arange(n), self.pins)
        if len(expect_free) != len(self.free) or np.any(np.sort(self.free) != expect_free):
            raise ValueError("free must be the complement of pins")
        self._ctx = _abi.MatrixContext(K, self.pins, precision=precision, tol=tol, max_iters=max_iters,
                                       device=current_device())
        if mode == "cms":
            from .cms import CmsGlobalSolver
            self._cms = CmsGlobalSolver(self._ctx, K, self.free, self.pins, cms, refine_sweeps,
                                        aggregation, omega, chebyshev)

    def solve(self, B, pin_vals):
        B = np.asarray(B, dtype=float)
        if self.mode == "cms":
            return self._cms.solve(B, pin_vals)
        return self._ctx.global_solve(B, pin_vals)


# ---------------------------------------------------------------------------
# stepping


def pd_step(state, mesh, gammas, iterations=PD_ITERS_DEFAULT, forces=None, solver=None,
            contact_stiffness=CONTACT_STIFFNESS, damping=1.0, precision="fp64", tol=None,
            max_iters=0):
    """One implicit-Euler step by local/global rounds (`pdsolver.py:257-304`); returns the state.

    With `solver=None` the whole step (prologue, `iterations` x [local step,
    device CG], epilogue) runs device-resident as one CUDA graph.  A caller
    `solver` (anything with `.solve(B, pin_vals)`) keeps the reference's
    host-driven loop with the local step on the GPU.
    """
    _check_inputs(mesh, gammas, state.dt)
    if state.colliders:
        _validate_colliders(state.colliders)
    elif solver is not None and not isinstance(solver, _DeviceStep):
        return _pd_step_host_solver(state, mesh, gammas, iterations, forces, solver, damping, precision)
    # with colliders the reference re-assembles K with the contact diagonal and ignores
    # `solver` (pdsolver.py:273-281); the device step adds the contact terms per step
    ctx = device_context(mesh, gammas, state.dt, state.pins, precision, tol, max_iters)
    on_device = _is_cuda_tensor(state.x)
    if on_device:
        # torch tensors in, torch tensors out, ordered after / before the caller's stream: no
        # host copies of the state
        import torch
        caller = torch.cuda.current_stream(state.x.device)
        lib_stream = torch.cuda.ExternalStream(ctx.stream_ptr(), device=state.x.device)
        lib_stream.wait_stream(caller)
        ctx.set_state_tensor(state.x, state.v)
        if len(state.pins):
            if _is_cuda_tensor(state.pin_targets):
                ctx.set_pin_targets_tensor(state.pin_targets.to(torch.float64).contiguous())
            else:
                ctx.set_pin_targets(state.pin_targets)
        if _is_cuda_tensor(forces):
            ctx.set_forces_tensor(forces.to(torch.float64).reshape(-1, 3).contiguous())
        else:
            ctx.set_forces(forces)
    else:
        ctx.set_state(state.x, state.v)
        if len(state.pins):
            ctx.set_pin_targets(state.pin_targets)
        ctx.set_forces(forces)
    ctx.set_colliders(state.colliders, contact_stiffness)
    try:
        ctx.step(iterations, damping)
    except _abi.NonFiniteError as exc:
        raise RuntimeError(str(exc)) from None
    if on_device:
        with torch.cuda.stream(lib_stream):
            state.x, state.v = ctx.get_state_tensor()
        caller.wait_stream(lib_stream)
        state.x.record_stream(caller)
        state.v.record_stream(caller)
    else:
        state.x, state.v = ctx.get_state()
    return state


class _DeviceStep:
    """Marker base for solvers that run inside the device-resident step."""


# ---------------------------------------------------------------------------
# colliders (pdsolver.py:125-173).  Host helpers for callers; inside the step the
# contact set, weights and surface targets are computed on the device.


def _validate_colliders(colliders):
    for kind, *_ in colliders:
        if kind not in ("plane", "sphere"):
            raise ValueError(f"unknown collider kind {kind!r}")


def collider_targets(x, colliders):
    """Nodes penetrating a collider and their closest surface points (`pdsolver.py:125-155`)."""
    x = np.asarray(x, dtype=float)
    idx, tgt = [], []
    for kind, *args in colliders:
        if kind == "plane":
            p0 = np.asarray(args[0], dtype=float)
            nrm = np.asarray(args[1], dtype=float)
            nrm = nrm / np.linalg.norm(nrm)
            depth = (x - p0) @ nrm
            pen = np.flatnonzero(depth < 0.0)
            idx.append(pen)
            tgt.append(x[pen] - depth[pen, None] * nrm)
        elif kind == "sphere":
            c = np.asarray(args[0], dtype=float)
            r = float(args[1])
            rel = x - c
            dist = np.linalg.norm(rel, axis=1)
            pen = np.flatnonzero(dist < r)
            idx.append(pen)
            tgt.append(c + rel[pen] * (r / np.maximum(dist[pen], 1e-12))[:, None])
        else:
            raise ValueError(f"unknown collider kind {kind!r}")
    if not idx:
        return np.empty(0, dtype=int), np.empty((0, 3))
    return np.concatenate(idx), np.concatenate(tgt)


def surface_targets(points, colliders):
    """Project points out of any collider they penetrate; identity otherwise (`pdsolver.py:158-163`)."""
    out = np.asarray(points, dtype=float).copy()
    idx, tgt = collider_targets(out, colliders)
    out[idx] = tgt
    return out


def collide_project(state, colliders=None):
    """Snap penetrating nodes of a state to the collider surfaces (`pdsolver.py:166-173`)."""
    colliders = state.colliders if colliders is None else colliders
    idx, tgt = collider_targets(state.x, colliders)
    if len(idx):
        state.x = state.x.copy()
        state.x[idx] = tgt
    return state


def _pd_step_host_solver(state, mesh, gammas, iterations, forces, solver, damping, precision):
    """Reference loop (`pdsolver.py:283-304`) with a caller-provided global solver."""
    ctx = device_context(mesh, gammas, state.dt, (), "fp64" if precision == "fp64" else precision)
    xhat = _predicted(state, forces, mesh)
    x_start = state.x.copy()
    x = xhat.copy()
    if len(state.pins):
        pin_vals = state.pin_targets
        x[state.pins] = pin_vals
    else:
        pin_vals = np.empty((0, 3))
    inertia = (mesh.node_mass[:, None] / state.dt ** 2) * xhat
    for it in range(iterations):
        rhs = ctx.elastic_rhs(x, with_frv=False)[0]
        x = np.asarray(solver.solve(inertia + rhs, pin_vals), dtype=float)
        if not np.all(np.isfinite(x)):
            raise RuntimeError(f"projective step produced non-finite positions at iteration {it}")
    state.v = damping * (x - x_start) / state.dt
    state.x = x
    return state


def pd_equilibrium(mesh, gammas, inertia_target, x0, pins, pin_vals, dt, iterations=PD_ITERS_DEFAULT,
                   solver=None, precision="fp64", tol=None):
    """Proximal local/global rounds on E(x) + (1/dt^2) a^T M x (`pdsolver.py:315-338`).

    Each round solves K x = (M/dt^2)(x_cur - a) + elastic rhs.  Without `solver` the
    rounds run on the device (`vkpd_equilibrium`, fitting-side default precision float64);
    any object with `.solve(B, pin_vals)` runs the reference loop with the local step on
    the device.  RuntimeError "quasi-static projection diverged at iteration {it}".
    """
    _check_inputs(mesh, gammas, dt)
    pins = np.asarray(pins, dtype=np.int64)
    a = np.asarray(inertia_target, dtype=float).reshape(-1, 3)
    pv = np.asarray(pin_vals, dtype=float).reshape(-1, 3) if len(pins) else np.empty((0, 3))
    if solver is None:
        ctx = device_context(mesh, gammas, dt, pins, precision, tol)
        try:
            return ctx.equilibrium(a, x0, pv, iterations)
        except _abi.NonFiniteError as exc:
            raise RuntimeError(str(exc)) from None
    ctx = device_context(mesh, gammas, dt, (), precision)
    x = np.asarray(x0, dtype=float).reshape(-1, 3).copy()
    if len(pins):
        x[pins] = pv
    m_dt2 = mesh.node_mass[:, None] / dt ** 2
    for it in range(iterations):
        rhs = ctx.elastic_rhs(x, with_frv=False)[0]
        x = np.asarray(solver.solve(m_dt2 * (x - a) + rhs, pv), dtype=float)
        if not np.all(np.isfinite(x)):
            raise RuntimeError(f"quasi-static projection diverged at iteration {it}")
    return x


def quasi_static_objective(mesh, gammas, inertia_target, x, dt):
    """E(x) + (1/dt^2) a^T M x (`pdsolver.py:341-343`), elastic part on the GPU."""
    lin = float(np.sum(mesh.node_mass[:, None] * inertia_target * x)) / dt ** 2
    return elastic_energy(mesh, gammas, x) + lin


EXACT_SOLVE_TOL = 1e-13          # MINRES relative tolerance of the exact Newton step
EXACT_SOLVE_ACCEPT = 1e-8        # true relative residual above this = failed factorization


def newton_polish(mesh, gammas, x0, *, dt, pins=(), pin_vals=None, inertia_target=None, xhat=None,
                  tol=1e-5, max_iters=20, exact=False):
    """Drive the step residual below tol with Newton-type iterations (`pdsolver.py:350-460`).

    Same two residual flavours, objective, halving line search, stall rule and return
    value (x, converged, iterations) as the reference.  On the device: the gradient and
    energy (float64, `vkpd_hess_energy_grad`), the Gauss-Newton step with the assembled K
    (the persistent CG of the global step, float64, relative tolerance 1e-12, in place of
    SuperLU), and with `exact=True` the exact-Jacobian step by preconditioned MINRES on the
    device-resident exact Hessian (`vkpd_hess_solve`); a solve that does not reach a true
    relative residual of 1e-8 counts as the reference's failed factorization and falls
    back to the Gauss-Newton step.
    """
    if (inertia_target is None) == (xhat is None):
        raise ValueError("give exactly one of inertia_target or xhat")
    _check_inputs(mesh, gammas, dt)
    n = mesh.n_nodes
    pins = np.asarray(pins, dtype=int)
    free = np.setdiff1d(np.arange(n), pins)
    x = np.asarray(x0, dtype=float).reshape(-1, 3).copy()
    if len(pins):
        x[pins] = pin_vals
    m_dt2 = mesh.node_mass[:, None] / dt ** 2
    h = hess_context(mesh, gammas, dt, pins)

    def residual(xc):
        _, g = h.energy_grad(xc, want_energy=False, want_grad=True)
        if xhat is not None:
            g = g + m_dt2 * (xc - xhat)
        else:
            g = g + m_dt2 * inertia_target
        return g

    def objective(xc):
        e, _ = h.energy_grad(xc, want_energy=True, want_grad=False)
        if xhat is not None:
            d = xc - xhat
            return e + 0.5 * float(np.sum(m_dt2 * d * d))
        return e + float(np.sum(m_dt2 * inertia_target * xc))

    def gmax(gv):
        return float(np.abs(gv[free]).max()) if len(free) else 0.0

    g = residual(x)
    if gmax(g) < tol:
        return x, True, 0

    ctx = device_context(mesh, gammas, dt, pins, "fp64")     # K = GN Hessian + M/dt^2 (scalar)
    zero_pins = np.zeros((len(pins), 3))

    def gn_step(gc):
        step = np.asarray(ctx.global_solve(-gc, zero_pins), dtype=float).reshape(-1, 3)
        if len(pins):
            step[pins] = 0.0
        return step

    def exact_step(xc, gc):
        h.linearize(xc)
        step, _, rr = h.solve(-gc, mass_scale=1.0 if xhat is not None else 0.0, tol=EXACT_SOLVE_TOL)
        if not (rr <= EXACT_SOLVE_ACCEPT) or not np.all(np.isfinite(step)):
            return None
        return step

    def try_step(step, obj):
        t = 1.0
        for _ in range(12):
            xn = x + t * step
            if len(pins):
                xn[pins] = pin_vals
            on = objective(xn)
            if on < obj + 1e-15 * max(1.0, abs(obj)):
                return xn, on
            t *= 0.5
        return None, obj

    obj = objective(x)
    stall = 0
    for it in range(1, max_iters + 1):
        xn = None
        if exact:
            step = exact_step(x, g)
            if step is not None:
                xn, on = try_step(step, obj)
        if xn is None:
            xn, on = try_step(gn_step(g), obj)
        if xn is None:
            stall += 1
            if stall >= 10:
                log.warning("newton polish stalled at residual %.3e", gmax(g))
                return x, False, it
            xn, on = x, obj
        x, obj = xn, on
        g = residual(x)
        if gmax(g) < tol:
            return x, True, it
    ok = gmax(g) < tol
    if not ok:
        log.warning("newton polish hit iteration cap at residual %.3e", gmax(g))
    return x, ok, max_iters


def simulate_mesh(mesh, gammas, steps, dt, forces=None, pins=(), pin_targets=None, colliders=(),
                  iterations=PD_ITERS_DEFAULT, solver_mode="direct", n_domains=2, modes_per_domain=20,
                  refine_sweeps=30, aggregation=2, chebyshev=False, damping=1.0, polish_tol=None,
                  x0=None, precision="fp64", tol=None, max_iters=0, labels=None):
    """Run a forward simulation and return the frame stack (steps, nV, 3) (`pdsolver.py:710-763`).

    pin_targets may be constant (nP, 3) or a per-step path (steps, nP, 3).
    """
    if solver_mode not in ("direct", "cms"):
        raise ValueError(f"unknown solver mode {solver_mode!r}")
    _check_inputs(mesh, gammas, dt)
    pins = np.asarray(pins, dtype=int)
    pin_path = None
    if pin_targets is not None:
        pin_targets = np.asarray(pin_targets, dtype=float)
        if pin_targets.ndim == 3:
            pin_path = pin_targets
            pin_targets = pin_path[0]
    state = SimState(x=mesh.nodes.copy() if x0 is None else np.asarray(x0, dtype=float).copy(),
                     v=np.zeros_like(mesh.nodes), dt=dt, pins=pins, pin_targets=pin_targets,
                     colliders=tuple(colliders))
    if forces is not None:
        forces = np.asarray(forces, dtype=float)
        if forces.ndim == 2:
            forces = np.broadcast_to(forces, (steps,) + forces.shape)
    frames = np.empty((steps, mesh.n_nodes, 3))
    if steps == 0:                      # the reference's loop body never runs (pdsolver.py:749)
        return frames
    if state.colliders:
        # the reference drops the prefactored solver when colliders exist (pdsolver.py:753)
        _validate_colliders(state.colliders)
        solver_mode = "direct"
    if solver_mode == "cms":
        from .cms import simulate_cms
        return simulate_cms(mesh, gammas, steps, dt, forces, state, pin_path, iterations,
                            n_domains, modes_per_domain, refine_sweeps, aggregation, chebyshev,
                            damping, precision, labels, polish_tol=polish_tol)
    ctx = device_context(mesh, gammas, dt, pins, precision, tol, max_iters)
    ctx.set_state(state.x, state.v)
    if len(pins):
        ctx.set_pin_targets(state.pin_targets)
    const_forces = forces is not None and forces.strides[0] == 0      # broadcast (nV,3) input
    ctx.set_forces(None if forces is None else forces[0])
    ctx.set_colliders(state.colliders)
    if polish_tol is None or state.colliders:
        # the whole frame loop in one library call: per-step inputs up and positions down on a
        # copy stream, overlapped with the next frame's compute (vkpd_simulate)
        try:
            return ctx.simulate(steps, iterations, damping,
                                forces=None if forces is None else (forces[0] if const_forces else forces),
                                forces_per_step=forces is not None and not const_forces,
                                pin_path=pin_path, out=frames)
        except _abi.NonFiniteError as exc:
            raise RuntimeError(str(exc)) from None
    for i in range(steps):
        if pin_path is not None:
            ctx.set_pin_targets(pin_path[i])
        if forces is not None and not const_forces and i > 0:
            ctx.set_forces(forces[i])
        try:
            ctx.step(iterations, damping)
        except _abi.NonFiniteError as exc:
            raise RuntimeError(str(exc)) from None
        if polish_tol is not None and not state.colliders:
            # pdsolver.py:757-761: polish toward the prediction of the stepped state; the
            # polished x replaces state.x, v stays the PD step's
            f = None if forces is None else forces[i]
            xs, vs = ctx.get_state(want_x=True, want_v=True)
            st = SimState(x=xs, v=vs, dt=dt, pins=pins,
                          pin_targets=pin_path[i] if pin_path is not None else state.pin_targets)
            xh = _predicted(st, f, mesh)
            xp, _, _ = newton_polish(mesh, gammas, xs, dt=dt, pins=pins, pin_vals=st.pin_targets,
                                     xhat=xh, tol=polish_tol)
            ctx.set_state(xp, vs)
            frames[i] = xp
            continue
        ctx.get_state(want_x=True, want_v=False, out_x=frames[i])
    return frames

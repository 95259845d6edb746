"""Adjoint machinery of the material fit on the B200 library.

Mirrors `/root/reference/pkg/src/volknit/fitting.py`:

  gamma_jacobian(mesh, x)                           fitting.py:172-190
  AdjointState, EquilibriumGateError                fitting.py:193-243
  adjoint_gradient(problem, sample, gammas, x, ...) fitting.py:206-238
  adjoint_gauss_newton(problem, sample, state, ...) fitting.py:251-313

`problem` / `sample` are duck-typed exactly as the reference uses them: `problem.mesh`,
`problem.dt`, `problem.loss_grad_x(x, sample)`, `problem.loss_hessian_scalar(sample)`,
`problem.free_dofs(sample)`, `sample.pins`, `sample.inertia`, `sample.index`.  The loss
itself, the sample construction and the fitting driver stay the caller's (SURVEY.md §2:
out of scope).

On the device (float64): the equilibrium residual (elastic gradient), the exact equilibrium
Jacobian (per-tet blocks with the projection sensitivities), the adjoint solve H_ff lam = g_x
(preconditioned MINRES in place of SuperLU; a solve that does not reach a true relative
residual of 1e-8 is the reference's singular factorization and gets the same
KAPPA_SCALE ridge), and grad = -J^T lam as one per-tet contraction (the sparse J is never
needed for the gradient).
"""

from __future__ import annotations

import logging
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from . import material as mat
from . import pdsolver

log = logging.getLogger(__name__)

EQ_GATE = 1e-5          # fitting.py:32
KAPPA_SCALE = 1e-6      # fitting.py:35
ADJOINT_TOL = 1e-13     # MINRES relative tolerance of the adjoint solve
ADJOINT_ACCEPT = 1e-8   # true relative residual above this = singular factorization


def gamma_jacobian(mesh, x):
    """Sparse d(residual)/d(gamma), shape (3nV, 2nE) (`fitting.py:172-190`).

    Column e (resp. nE + e) is element e's unit-coefficient force pattern 2V D^T vec(F - R)
    (resp. F - V), with F, R, V from the device local step (float64).
    """
    x = np.asarray(x, dtype=float).reshape(-1, 3)
    _, F, R, V = pdsolver.elastic_rhs(mesh, mat.MaterialField.uniform(mesh.n_elements, 1.0, 1.0), x)
    G = mesh.shape_grad
    v2 = 2.0 * mesh.volume[:, None, None]
    Js = v2 * np.einsum("enj,eij->eni", G, F - R)
    Jv = v2 * np.einsum("enj,eij->eni", G, F - V)
    nE = mesh.n_elements
    dofs = (3 * mesh.tets[:, :, None] + np.arange(3)[None, None, :]).reshape(-1)
    rows = np.concatenate([dofs, dofs])
    cols = np.concatenate([np.repeat(np.arange(nE), 12), np.repeat(np.arange(nE, 2 * nE), 12)])
    vals = np.concatenate([Js.reshape(-1), Jv.reshape(-1)])
    return sp.csr_matrix((vals, (rows, cols)), shape=(3 * mesh.n_nodes, 2 * nE))


@dataclass
class AdjointState:
    """Equilibrium-point quantities reused by gradient and Gauss-Newton (`fitting.py:193-203`)."""

    x: np.ndarray
    residual: float
    fdofs: np.ndarray
    H: sp.csc_matrix          # exact equilibrium Jacobian, free DOFs
    J: sp.csr_matrix          # residual derivative in gamma, free rows
    lam: np.ndarray           # adjoint vector
    grad: np.ndarray          # loss gradient in gamma, length 2nE


class EquilibriumGateError(RuntimeError):
    pass


def equilibrium_residual(problem, sample, gammas, x):
    """max |elastic_gradient + (M/dt^2) a| over free nodes (`fitting.py:215-220`)."""
    mesh = problem.mesh
    free = np.setdiff1d(np.arange(mesh.n_nodes), sample.pins)
    g = pdsolver.elastic_gradient(mesh, gammas, x) + (mesh.node_mass[:, None] / problem.dt ** 2) * sample.inertia
    return float(np.abs(g[free]).max()) if len(free) else 0.0


def _adjoint_solve(h, gx):
    lam, _, rr = h.solve(gx, mass_scale=0.0, tol=ADJOINT_TOL)
    if rr <= ADJOINT_ACCEPT and np.all(np.isfinite(lam)):
        return lam
    return None


def adjoint_gradient(problem, sample, gammas, x, residual=None, logger=None, with_matrices=True):
    """Loss gradient in the coefficients via one adjoint solve (`fitting.py:206-238`).

    The equilibrium Jacobian carries the projection sensitivities.  Each call is gated on
    the equilibrium residual (EQ_GATE) and logged.  `with_matrices=False` skips assembling
    the state's H and J (only the gradient and lam are formed; adjoint_gauss_newton needs
    them).
    """
    mesh = problem.mesh
    x = np.asarray(x, dtype=float).reshape(-1, 3)
    if residual is None:
        residual = equilibrium_residual(problem, sample, gammas, x)
    ok = residual < EQ_GATE
    if logger is not None:
        logger.log_gate(sample.index, residual, ok)
    if not ok:
        raise EquilibriumGateError(f"adjoint evaluation rejected: residual {residual:.3e} >= {EQ_GATE:g}")

    pins = np.asarray(sample.pins, dtype=int)
    fdofs = problem.free_dofs(sample)
    h = pdsolver.hess_context(mesh, gammas, problem.dt, pins)
    h.linearize(x)
    gx = np.asarray(problem.loss_grad_x(x, sample), dtype=float).reshape(-1, 3)
    lam = _adjoint_solve(h, gx)
    if lam is None:
        Hd = h.csr()[fdofs][:, fdofs]
        kap = KAPPA_SCALE * Hd.diagonal().sum() / Hd.shape[0]
        log.warning("singular equilibrium Jacobian; adding %.3e ridge", kap)
        lam, _, _ = h.solve(gx, mass_scale=0.0, ridge=kap, tol=ADJOINT_TOL)
    grad = -h.gamma_jt(x, lam)              # lam is zero on the pinned rows
    H = J = None
    if with_matrices:
        H = h.csr()[fdofs][:, fdofs].tocsc()
        J = gamma_jacobian(mesh, x)[fdofs]
    return AdjointState(x=x, residual=residual, fdofs=fdofs, H=H, J=J, lam=lam.reshape(-1)[fdofs], grad=grad)

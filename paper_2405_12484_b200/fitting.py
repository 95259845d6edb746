"""Adjoint machinery of the material fit on the B200 library.

Mirrors `/root/reference/pkg/src/volknit/fitting.py`:

  gamma_jacobian(mesh, x)                           fitting.py:172-190
  AdjointState, EquilibriumGateError                fitting.py:193-243
  adjoint_gradient(problem, sample, gammas, x, ...) fitting.py:206-238
  reduce_columns, adjoint_gauss_newton(...)         fitting.py:245-313

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
    hctx: object = None       # device float64 Hessian context (pdsolver.hess_context), not in the reference


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
    return AdjointState(x=x, residual=residual, fdofs=fdofs, H=H, J=J, lam=lam.reshape(-1)[fdofs], grad=grad,
                        hctx=h)


def _sensitivities(problem, state, Jk):
    """S = H_ff^-1 J column by column with the device MINRES of the equilibrium Jacobian
    (linearised at state.x); None when a column does not reach ADJOINT_ACCEPT."""
    h = state.hctx
    n = problem.mesh.n_nodes
    h.linearize(state.x)
    fd = state.fdofs
    Jc = sp.csc_matrix(Jk)
    S = np.empty(Jc.shape)
    b = np.zeros(3 * n)
    for j in range(Jc.shape[1]):
        b[:] = 0.0
        b[fd] = Jc[:, j].toarray().ravel()
        x, _, rr = h.solve(b.reshape(-1, 3), mass_scale=0.0, tol=SOLVE_TOL)
        if not (rr <= ADJOINT_ACCEPT) or not np.all(np.isfinite(x)):
            return None
        S[:, j] = x.reshape(-1)[fd]
    return S


def reduce_columns(J, basis):
    """Map the coefficient Jacobian onto a rank-r basis per field (`fitting.py:245-248`)."""
    nE = basis.shape[0]
    return np.hstack([J[:, :nE] @ basis, J[:, nE:] @ basis])


DENSE_GN_MAX = 24000        # largest m (coefficient columns) of the dense reduced system
DENSE_H_MAX = 6000          # above this many free DOFs, S = H^-1 J comes from the device solver
SOLVE_TOL = 1e-13           # MINRES relative tolerance of the sensitivity columns


def adjoint_gauss_newton(problem, sample, state, kappa=None, basis=None, frozen=None, dense_h_max=DENSE_H_MAX):
    """Gauss-Newton direction d with (J^T H^-1 G H^-1 J + kappa I) d = -grad (`fitting.py:251-313`).

    The reference eliminates v, u from its sparse symmetric block system
        [ 0   H   J ] [v]   [ 0    ]
        [ H  -G   0 ] [u] = [ 0    ]
        [ J^T 0  -kI] [d]   [ grad ]
    by one sparse LU.  On the B200 the same direction comes from the equivalent reduced
    system in float64: S = H^-1 J, P = S^T G S (DGEMM), then a Cholesky solve of P + kappa I
    (the ridge kappa = 1e-6 mean diag G makes P too ill-conditioned for an iterative outer
    solve; the reference factorizes for the same reason).  S comes from the device solver:
    one preconditioned-MINRES solve of the exact equilibrium Jacobian per column of J
    (`vkpd_hess_solve`, the adjoint solve of adjoint_gradient), so the mesh size is not
    bounded -- a large garment takes the `basis` reduction (m = 2r columns); for at most
    `dense_h_max` free DOFs an LU of H on the device is faster and is used instead.  Same
    `basis` / `frozen` reductions, the same default kappa and the same (d, kappa, ok)
    contract: ok False when a solve or the factorization fails, the result is not finite,
    or d is not a descent direction.  m up to DENSE_GN_MAX columns.
    """
    import scipy.sparse as sps
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("adjoint_gauss_newton needs a CUDA device (no CPU path)")
    G_scalar = problem.loss_hessian_scalar(sample)
    fdofs = state.fdofs
    G = sps.kron(G_scalar, sps.eye(3)).tocsr()[fdofs][:, fdofs]
    if kappa is None:
        kappa = KAPPA_SCALE * G.diagonal().sum() / G.shape[0]
    J = state.J
    grad = state.grad
    if basis is not None:
        J = sps.csr_matrix(reduce_columns(J, basis))
        nE = basis.shape[0]
        grad = np.concatenate([basis.T @ grad[:nE], basis.T @ grad[nE:]])
    keep = np.setdiff1d(np.arange(J.shape[1]), frozen) if frozen is not None and len(frozen) else None
    Jk = J[:, keep] if keep is not None else J
    gk = grad[keep] if keep is not None else grad
    nf, m = Jk.shape
    if m > DENSE_GN_MAX:
        raise NotImplementedError(f"reduced Gauss-Newton system limited to {DENSE_GN_MAX} columns; "
                                  f"pass a basis")
    dev = torch.device("cuda")
    f64 = torch.float64
    g = torch.as_tensor(np.asarray(gk, dtype=float), dtype=f64, device=dev)
    d = np.zeros(J.shape[1])
    if nf <= dense_h_max or state.hctx is None:
        if nf > DENSE_GN_MAX:
            raise NotImplementedError("state without a device Hessian context: dense path only")
        H = torch.as_tensor(state.H.toarray(), dtype=f64, device=dev)
        Jd = torch.as_tensor(Jk.toarray(), dtype=f64, device=dev)
        LU, piv, info = torch.linalg.lu_factor_ex(H)
        if int(info.item()) != 0:
            return None, kappa, False
        S = torch.linalg.lu_solve(LU, piv, Jd)
    else:
        S = _sensitivities(problem, state, Jk)
        if S is None:
            return None, kappa, False
        S = torch.as_tensor(S, dtype=f64, device=dev)
    if not bool(torch.isfinite(S).all()):
        return None, kappa, False
    Gs = torch.sparse_csr_tensor(torch.as_tensor(G.indptr, dtype=torch.int64), torch.as_tensor(G.indices, dtype=torch.int64),
                                 torch.as_tensor(G.data, dtype=f64), size=G.shape).to(dev)
    P = S.T @ (Gs @ S)
    P = 0.5 * (P + P.T)
    P.diagonal().add_(kappa)
    L, info = torch.linalg.cholesky_ex(P)
    if int(info.item()) != 0:
        return None, kappa, False
    dk = torch.cholesky_solve(-g[:, None], L)[:, 0].cpu().numpy()
    if not np.all(np.isfinite(dk)):
        return None, kappa, False
    if keep is not None:
        d[keep] = dk
    else:
        d = dk
    # d = 0 at a stationary point is the valid homogeneous solution, not a failed descent direction
    if len(gk) and np.linalg.norm(gk) > 0.0 and float(d @ grad) >= 0.0:
        return d, kappa, False
    return d, kappa, True

"""Domain-decomposed (component-mode synthesis) global solve and A-Jacobi refinement.

Drop-ins for the reference's subspace machinery (`/root/reference/pkg/src/volknit/pdsolver.py`):

  partition_elements     pdsolver.py:467-480  (host bookkeeping)
  classify_nodes         pdsolver.py:483-509  (host bookkeeping)
  CmsSubspace / build_cms  pdsolver.py:512-609
  a_jacobi_refine        pdsolver.py:632-703  (persistent cooperative CUDA kernel)
  GlobalSolver(mode="cms")  pdsolver.py:237-246

Precompute (once per K): per-domain dense K_ii eigenpairs and the static
boundary response Psi_d = -K_ii^-1 K_ib run through cuSOLVER on the GPU
(torch.linalg.eigh / cholesky in float64, library calls); the reduced matrix
K_red = T^T K T and its inverse likewise.  Every solve then runs on the
device through the vkpd C-ABI: x0 = T K_red^-1 T^T b (dense skinny
contractions) followed by aggregated / Chebyshev Jacobi sweeps with the
reference's best-iterate and divergence semantics.

Like the reference, the basis T stores the full boundary block for every
domain (zeros included), so this reference-compatible mode is meant for the
sizes the reference itself can build.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from . import _abi

JACOBI_OMEGA = 0.75


def partition_elements(mesh, n_domains, labels=None):
    """Caller labels, or quantile slabs of tet centroids along the longest bbox axis."""
    if labels is not None:
        labels = np.asarray(labels, dtype=int)
        if len(labels) != mesh.n_elements:
            raise ValueError("need one domain label per element")
        return labels
    centers = mesh.nodes[mesh.tets].mean(axis=1)
    span = mesh.nodes.max(axis=0) - mesh.nodes.min(axis=0)
    axis = int(np.argmax(span))
    c = centers[:, axis]
    edges = np.quantile(c, np.linspace(0.0, 1.0, n_domains + 1)[1:-1])
    return np.searchsorted(edges, c)


def classify_nodes(mesh, element_labels, free=None):
    """Interior node sets per domain + merged boundary set (restricted to `free`)."""
    n = mesh.n_nodes
    lab4 = np.repeat(np.asarray(element_labels, dtype=np.int64), 4)
    lo = np.full(n, np.iinfo(np.int64).max, dtype=np.int64)
    hi = np.full(n, -1, dtype=np.int64)
    np.minimum.at(lo, mesh.tets.reshape(-1), lab4)
    np.maximum.at(hi, mesh.tets.reshape(-1), lab4)
    keep = np.ones(n, dtype=bool)
    if free is not None:
        keep[:] = False
        keep[free] = True
    taken = np.zeros(n, dtype=bool)
    interior = []
    for d in range(int(np.max(element_labels)) + 1):
        sel = np.flatnonzero((lo == d) & (hi == d) & keep)
        interior.append(sel)
        taken[sel] = True
    return interior, np.flatnonzero(keep & ~taken & (hi >= 0))


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("the CMS precompute runs on the GPU (cuSOLVER); no CUDA device visible")
    return torch


class CmsSubspace:
    """Craig-Bampton basis T = [Phi blocks | I_b + Psi blocks] and K_red = T^T K T.

    `solve(b)` = T K_red^-1 T^T b on the device.  Attributes mirror the
    reference: `blocks` [(sel, Phi, Psi) | None], `T` (CSR, built on first use), `K_red` (CSC).

    The build scales with the domain size (`pdsolver.py:521-590` forms dense eigensystems and a
    dense n x m_tot T; at C3 with 8 domains that is 36 s and 4.9 GB):
      * Phi_d: the m lowest eigenpairs of K_ii -- dense `eigh` up to DENSE_EIG_MAX interior
        nodes (the reference's exact route for small domains), else Chebyshev-filtered subspace
        iteration on the sparse K_ii on the GPU (K_ii is mass-dominated, condition number ~100)
        to a Ritz residual of EIG_TOL;
      * Psi_d = -K_ii^-1 K_ib only on the boundary columns adjacent to d (K_ib is zero on the
        others, so Psi is too): block conjugate gradients on the sparse K_ii with all adjacent
        columns at once, to PSI_TOL, on the GPU (Cholesky of the dense K_ii for small domains);
      * K_red from the blocks: Phi^T K_ii Phi per domain, Phi^T (K_ib + K_ii Psi), and
        S = K_bb + sum_d (K_bi Psi + Psi^T K_ib + Psi^T K_ii Psi) -- no dense T.
    """

    DENSE_EIG_MAX = 3000
    EIG_TOL = 1e-12          # Ritz residual of the filtered subspace iteration, relative to |A|
    PSI_TOL = 1e-13

    def __init__(self, K, interior_sets, boundary, modes_per_domain=20):
        torch = _torch()
        dev = torch.device("cuda")
        f64 = torch.float64
        K = sp.csr_matrix(K)
        self.n = K.shape[0]
        self.boundary = np.asarray(boundary, dtype=int)
        nb = len(self.boundary)
        bpos = -np.ones(self.n, dtype=np.int64)
        bpos[self.boundary] = np.arange(nb)
        blocks, red_parts = [], []
        Kbb = K[self.boundary][:, self.boundary].toarray() if nb else np.zeros((0, 0))
        S = torch.as_tensor(Kbb, dtype=f64, device=dev)
        n_modes_tot = sum(min(modes_per_domain, len(s)) for s in interior_sets if len(s))
        cross = torch.zeros((n_modes_tot, nb), dtype=f64, device=dev)
        lam_blocks = []
        c0 = 0
        for sel in interior_sets:
            sel = np.asarray(sel, dtype=int)
            if len(sel) == 0:
                blocks.append(None)
                continue
            Kii_sp = K[sel][:, sel].tocsr()
            m = min(modes_per_domain, len(sel))
            Kii = _to_torch_csr(torch, Kii_sp, dev)
            if len(sel) <= self.DENSE_EIG_MAX:
                Kd = torch.as_tensor(Kii_sp.toarray(), dtype=f64, device=dev)
                w, v = torch.linalg.eigh(Kd)
                Phi = v[:, :m]
            else:
                Kd = None
                gersh = float(abs(Kii_sp).sum(axis=1).max())
                Phi = _lowest_modes(torch, Kii, Kii_sp.diagonal(), m, self.EIG_TOL, dev, lam_hi=gersh)
            Psi_adj, adj = None, np.zeros(0, dtype=np.int64)
            if nb:
                Kib_sp = K[sel][:, self.boundary].tocsc()
                adj = np.flatnonzero(np.diff(Kib_sp.indptr) > 0)       # boundary columns touching d
                if len(adj):
                    Kib = torch.as_tensor(Kib_sp[:, adj].toarray(), dtype=f64, device=dev)
                    if Kd is not None:
                        L = torch.linalg.cholesky(Kd)
                        Psi_adj = -torch.cholesky_solve(Kib, L)
                    else:
                        Psi_adj = _block_cg(torch, Kii, torch.as_tensor(1.0 / Kii_sp.diagonal(), dtype=f64,
                                                                          device=dev), -Kib, self.PSI_TOL)
                    # Schur complement contributions and the mode/boundary coupling
                    KiiPsi = Kii @ Psi_adj
                    adj_t = torch.as_tensor(adj, device=dev)
                    Sd = Kib.T @ Psi_adj
                    Sd = Sd + Sd.T + Psi_adj.T @ KiiPsi
                    S[adj_t[:, None], adj_t[None, :]] += Sd
                    cross[c0:c0 + m, adj_t] = Phi.T @ (Kib + KiiPsi)
            lam_blocks.append(Phi.T @ (Kii @ Phi))
            Psi_full = None
            if Psi_adj is not None:
                Psi_full = _embed_columns(Psi_adj.cpu().numpy(), adj, len(sel), nb)
            blocks.append((sel, Phi.cpu().numpy(), Psi_full))
            c0 += m
        self.blocks = blocks
        m_tot = n_modes_tot + nb
        Kr = torch.zeros((m_tot, m_tot), dtype=f64, device=dev)
        r0 = 0
        for Lb in lam_blocks:
            k = Lb.shape[0]
            Kr[r0:r0 + k, r0:r0 + k] = Lb
            r0 += k
        Kr[:n_modes_tot, n_modes_tot:] = cross
        Kr[n_modes_tot:, :n_modes_tot] = cross.T
        Kr[n_modes_tot:, n_modes_tot:] = S
        Kr = 0.5 * (Kr + Kr.T)
        self.K_red = sp.csc_matrix(Kr.cpu().numpy())
        self.K_red_inv = torch.linalg.inv(Kr).cpu().numpy() if m_tot else np.zeros((0, 0))
        self._T = None
        self._ctx = None
        self._K = K

    @property
    def T(self):
        """The basis as a sparse (n, m_tot) matrix (`pdsolver.py:560-575`), built on first use."""
        if self._T is None:
            nb = len(self.boundary)
            rows, cols, vals = [], [], []
            c0 = 0
            for blk in self.blocks:
                if blk is None:
                    continue
                sel, Phi, _ = blk
                r, c = np.meshgrid(sel, np.arange(Phi.shape[1]), indexing="ij")
                rows.append(r.reshape(-1)); cols.append(c0 + c.reshape(-1)); vals.append(Phi.reshape(-1))
                c0 += Phi.shape[1]
            rows.append(self.boundary); cols.append(c0 + np.arange(nb)); vals.append(np.ones(nb))
            for blk in self.blocks:
                if blk is not None and blk[2] is not None:
                    P = sp.coo_matrix(blk[2])
                    rows.append(blk[0][P.row]); cols.append(c0 + P.col); vals.append(P.data)
            self._T = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                                    shape=(self.n, c0 + nb))
        return self._T

    def _context(self):
        if self._ctx is None:
            from .pdsolver import current_device
            self._ctx = _abi.MatrixContext(self._K, np.empty(0, dtype=np.int64), precision="fp64",
                                           device=current_device())
            self._ctx.cms_set_blocks(basis_blocks(self))
        return self._ctx

    def solve(self, b):
        b = np.asarray(b, dtype=float)
        one = b.ndim == 1
        X = self._context().cms_solve(b[:, None] if one else b, np.zeros((0, 1 if one else b.shape[1])),
                                      0, 2, JACOBI_OMEGA, False, 0.0)
        return X[:, 0] if one else X


def _to_torch_csr(torch, A, dev):
    A = sp.csr_matrix(A)
    return torch.sparse_csr_tensor(torch.from_numpy(A.indptr.astype(np.int64)), torch.from_numpy(A.indices.astype(np.int64)),
                                   torch.from_numpy(A.data.astype(np.float64)), size=A.shape).to(dev)


def _embed_columns(P, adj, n_rows, nb):
    """Dense (n_rows, len(adj)) block as a sparse (n_rows, nb) CSC matrix on columns `adj`
    (stored densely per column: no scan for zeros)."""
    counts = np.zeros(nb, dtype=np.int64)
    counts[adj] = n_rows
    indptr = np.concatenate([[0], np.cumsum(counts)])
    indices = np.tile(np.arange(n_rows, dtype=np.int64), len(adj))
    return sp.csc_matrix((np.asfortranarray(P).reshape(-1, order="F"), indices, indptr), shape=(n_rows, nb))


def _block_cg(torch, A, inv_diag, B, tol, max_iter=2000):
    """Jacobi-preconditioned CG on SPD sparse A with all columns of B at once (per-column
    recurrences), to |r_j| <= tol |b_j|."""
    X = torch.zeros_like(B)
    R = B.clone()
    Z = inv_diag[:, None] * R
    P = Z.clone()
    rz = (R * Z).sum(0)
    bn = torch.linalg.norm(B, dim=0)
    for _ in range(max_iter):
        Q = A @ P
        alpha = rz / (P * Q).sum(0).clamp_min(1e-300)
        X += alpha * P
        R -= alpha * Q
        if bool((torch.linalg.norm(R, dim=0) <= tol * bn).all()):
            break
        Z = inv_diag[:, None] * R
        rz_new = (R * Z).sum(0)
        P = Z + (rz_new / rz.clamp_min(1e-300)) * P
        rz = rz_new
    return X


def _lowest_modes(torch, A, diag, m, tol, dev, lam_hi=None):
    """m lowest eigenvectors of the sparse SPD A, orthonormal: Chebyshev-filtered subspace
    iteration on a block of m + 8 vectors (a degree-24 filter that damps [cut, lam_hi], where cut
    is the block's largest Ritz value), QR and Rayleigh-Ritz each round, until every wanted
    Ritz pair has |A x - theta x| <= tol |A|.  The block's spectrum edge is mass-dominated
    (condition number ~100), so a few rounds suffice."""
    n = A.shape[0]
    k = min(n, m)
    p = min(n, k + 8)
    if lam_hi is None:
        lam_hi = float(diag.max()) * 2.0
    gen = torch.Generator(device="cpu").manual_seed(0)
    X = torch.randn((n, p), generator=gen, dtype=torch.float64).to(dev)
    X, _ = torch.linalg.qr(X)
    H = X.T @ (A @ X)
    w, U = torch.linalg.eigh(0.5 * (H + H.T))
    X = X @ U
    deg = 24
    for _ in range(60):
        cut = float(w[-1])
        e, c = 0.5 * (lam_hi - cut), 0.5 * (lam_hi + cut)
        # three-term Chebyshev recurrence of the filter on [cut, lam_hi]
        Y = (A @ X - c * X) / e
        Xp = X
        for _ in range(2, deg + 1):
            Yn = 2.0 * (A @ Y - c * Y) / e - Xp
            Xp, Y = Y, Yn
        Q, _ = torch.linalg.qr(Y)
        AQ = A @ Q
        H = Q.T @ AQ
        w, U = torch.linalg.eigh(0.5 * (H + H.T))
        X = Q @ U
        R = AQ @ U - X * w[None, :]
        if bool((torch.linalg.norm(R[:, :k], dim=0) <= tol * lam_hi).all()):
            break
    return X[:, :k]


def basis_blocks(cms):
    """Per-domain storage of the subspace T = [Phi blocks | I_b + Psi blocks] (`pdsolver.py:560-575`).

    Domain d keeps A_d = [Phi_d | Psi_d on the boundary columns it touches] (column-major):
    Psi_d = -K_ii^-1 K_ib is exactly zero on the boundary nodes no element of d touches,
    so the dense T's zeros are dropped.  Works for this module's CmsSubspace and the
    reference's (both expose `blocks` [(sel, Phi, Psi) | None], `boundary`, `K_red`).
    """
    boundary = np.asarray(cms.boundary, dtype=np.int64)
    nb = len(boundary)
    blocks = [b for b in cms.blocks if b is not None]
    n_modes = sum(b[1].shape[1] for b in blocks)
    row_ptr, col_ptr, rows, colmap, parts = [0], [0], [], [], []
    c0 = 0
    for sel, Phi, Psi in blocks:
        sel = np.asarray(sel, dtype=np.int64)
        m = Phi.shape[1]
        cols = list(range(c0, c0 + m))
        mats = [np.asarray(Phi, dtype=float)]
        if Psi is not None and nb:
            if sp.issparse(Psi):
                Pc = sp.csc_matrix(Psi)
                adj = np.flatnonzero(np.diff(Pc.indptr) > 0)
                Pa = Pc[:, adj].toarray()
            else:
                Psi = np.asarray(Psi, dtype=float)
                adj = np.flatnonzero(np.any(Psi != 0.0, axis=0))
                Pa = Psi[:, adj]
            cols += list(n_modes + adj)
            mats.append(Pa)
        c0 += m
        A = np.hstack(mats) if len(mats) > 1 else mats[0]
        parts.append(np.asfortranarray(A).reshape(-1, order="F"))
        rows.append(sel)
        colmap.append(np.asarray(cols, dtype=np.int64))
        row_ptr.append(row_ptr[-1] + len(sel))
        col_ptr.append(col_ptr[-1] + len(cols))
    Ki = getattr(cms, "K_red_inv", None)
    if Ki is None:
        Kr = cms.K_red.toarray() if hasattr(cms.K_red, "toarray") else np.asarray(cms.K_red)
        Ki = np.linalg.inv(Kr) if Kr.size else np.zeros((0, 0))
    cat = lambda xs, dt: np.concatenate(xs).astype(dt) if xs else np.zeros(0, dtype=dt)
    return dict(row_ptr=np.asarray(row_ptr), col_ptr=np.asarray(col_ptr), rows=cat(rows, np.int64),
                colmap=cat(colmap, np.int64), A=cat(parts, float), n_modes=n_modes, boundary=boundary,
                K_red_inv=np.ascontiguousarray(Ki, dtype=float))


def build_cms(K, mesh=None, n_domains=2, modes_per_domain=20, element_labels=None, free=None,
              interior_sets=None, boundary=None):
    """Partition a mesh (or take explicit sets) and reduce K onto the component-mode basis."""
    if interior_sets is None:
        labels = partition_elements(mesh, n_domains, element_labels)
        interior_sets, boundary = classify_nodes(mesh, labels, free)
        if free is not None:
            remap = -np.ones(mesh.n_nodes, dtype=int)
            remap[free] = np.arange(len(free))
            interior_sets = [remap[s] for s in interior_sets]
            boundary = remap[boundary]
    return CmsSubspace(K, interior_sets, boundary, modes_per_domain)


_RHO_CACHE = {}


def _power_rho(ctx, n, omega, seed=0):
    """Reference start vector `default_rng(0).normal(size=n)` (pdsolver.py:618-619), iterated on the GPU."""
    v0 = np.random.default_rng(seed).normal(size=n)
    return ctx.power_rho(omega, v0, 30)


def a_jacobi_refine(K, b, x0, sweeps=30, aggregation=2, omega=JACOBI_OMEGA, chebyshev=False, rho=None,
                    precision="fp64"):
    """Aggregated weighted-Jacobi refinement of K x = b on the GPU (`pdsolver.py:632-703`).

    Returns (x, info) with info["residuals"] and info["diverged"] like the reference.
    b, x0: (n,) or (n, k<=3).
    """
    if aggregation not in (2, 3):
        raise ValueError("aggregation must be 2 or 3")
    K = sp.csr_matrix(K)
    if np.any(K.diagonal() <= 0.0):
        raise ValueError("matrix diagonal must be positive")
    from .pdsolver import current_device
    ctx = _abi.MatrixContext(K, np.empty(0, dtype=np.int64), precision=precision, device=current_device())
    if chebyshev and rho is None:
        rho = _power_rho(ctx, K.shape[0], omega)
    X, hist, div = ctx.a_jacobi_refine(b, x0, sweeps, aggregation, omega, chebyshev,
                                       -1.0 if rho is None else rho)
    one = np.asarray(b).ndim == 1
    if one:
        return X[:, 0], {"residuals": hist[0], "diverged": div[0]}
    return X, {"residuals": hist, "diverged": any(div), "diverged_columns": div}


class CmsGlobalSolver:
    """GlobalSolver(mode="cms").solve on the device (`pdsolver.py:237-246`)."""

    def __init__(self, ctx, K, free, pins, cms, refine_sweeps, aggregation, omega, chebyshev):
        if cms is None:
            raise ValueError("cms mode needs a CmsSubspace")
        self.ctx = ctx
        self.cms = cms
        self.sweeps = int(refine_sweeps)
        self.aggregation = int(aggregation)
        self.omega = float(omega)
        self.chebyshev = bool(chebyshev)
        if self.sweeps > 0 and self.aggregation not in (2, 3):
            raise ValueError("aggregation must be 2 or 3")
        # also accepts the reference's own CmsSubspace (same `blocks` / `boundary` / `K_red`)
        ctx.cms_set_blocks(basis_blocks(cms))
        self.rho = _power_rho(ctx, len(free), omega) if (chebyshev and self.sweeps > 0) else 0.0

    def solve(self, B, pin_vals):
        return self.ctx.cms_solve(B, pin_vals, self.sweeps, self.aggregation, self.omega, self.chebyshev,
                                  self.rho)


def simulate_cms(mesh, gammas, steps, dt, forces, state, pin_path, iterations, n_domains, modes_per_domain,
                 refine_sweeps, aggregation, chebyshev, damping, precision, labels=None, polish_tol=None):
    """`simulate_mesh(..., solver_mode="cms")` (`pdsolver.py:734-740`, 749-762).

    The subspace is built once (`build_cms`, GPU eigensolves), stored per domain on the mesh's
    float64 device context, and every frame runs as one device call (`vkpd_step_cms`): local
    step, b = rhs + (M/dt^2) xhat, subspace apply and A-Jacobi sweeps per PD round.
    """
    from . import pdsolver
    pins = state.pins
    free = np.setdiff1d(np.arange(mesh.n_nodes), pins)
    K = pdsolver.assemble_global(mesh, gammas, dt)
    Kff = K[free][:, free].tocsc()
    cms = build_cms(Kff, mesh, n_domains=n_domains, modes_per_domain=modes_per_domain, free=free,
                    element_labels=labels)
    sweeps = int(refine_sweeps)
    if sweeps > 0 and aggregation not in (2, 3):
        raise ValueError("aggregation must be 2 or 3")
    ctx = pdsolver.device_context(mesh, gammas, dt, pins, "fp64")
    ctx.cms_set_blocks(basis_blocks(cms))
    rho = _power_rho(ctx, len(free), JACOBI_OMEGA) if (chebyshev and sweeps > 0) else 0.0
    ctx.set_state(state.x, state.v)
    if len(pins):
        ctx.set_pin_targets(state.pin_targets)
    const_forces = forces is not None and forces.strides[0] == 0
    ctx.set_forces(None if forces is None else forces[0])
    ctx.set_colliders(())
    frames = np.empty((steps, mesh.n_nodes, 3))
    for i in range(steps):
        if pin_path is not None:
            state.pin_targets = pin_path[i]
            ctx.set_pin_targets(pin_path[i])
        if forces is not None and not const_forces and i > 0:
            ctx.set_forces(forces[i])
        try:
            ctx.step_cms(iterations, damping, sweeps, aggregation, JACOBI_OMEGA, chebyshev, rho)
        except _abi.NonFiniteError as exc:
            raise RuntimeError(str(exc)) from None
        if polish_tol is not None:          # pdsolver.py:757-761
            f = None if forces is None else forces[i]
            xs, vs = ctx.get_state()
            st = pdsolver.SimState(x=xs, v=vs, dt=dt, pins=pins, pin_targets=state.pin_targets)
            xh = pdsolver._predicted(st, f, mesh)
            xp, _, _ = pdsolver.newton_polish(mesh, gammas, xs, dt=dt, pins=pins, pin_vals=state.pin_targets,
                                              xhat=xh, tol=polish_tol)
            ctx.set_state(xp, vs)
            frames[i] = xp
            continue
        ctx.get_state(want_x=True, want_v=False, out_x=frames[i])
    return frames

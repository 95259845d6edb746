"""CPU ORACLE for the projective-dynamics hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy/scipy restatement of the reference algorithm
(`/root/reference/pkg/src/volknit`, a pure-Python package).  It is the checker
the parity tests, `__graft_entry__.smoke()` and the `cpu_baseline` /
`--impl reference` legs of `bench.py` run against; the product package
(`paper_2405_12484_b200`) never imports it.

Pinned against the reference: `tests/golden/make_golden.py` imports the real
reference in the build container and commits its outputs under
`tests/golden/`; `tests/test_oracle.py` checks this restatement against those
vectors (CPU, `-m "not gpu"`).

Every function cites the reference `file:line` it restates.  Precision is
float64 throughout with int64 indices, as in the reference
(`pdsolver.py:192-194`, `material.py:400`).
"""

from __future__ import annotations

import logging

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

log = logging.getLogger(__name__)

SV_FLOOR = 0.01            # material.py:25
NEWTON_ITERS = 20          # material.py:29
NEWTON_TOL = 1e-12         # material.py:30
PD_ITERS = 30              # pdsolver.py:23
OMEGA = 0.75               # pdsolver.py:24


# ---------------------------------------------------------------------------
# mesh operators


def deformation_gradients(x, tets, G):
    """F_e = sum_n x_{t(e,n)} (x) g_{e,n}  (`volmesh.py:115-118` via `diff_op` 92-97)."""
    xe = np.asarray(x, dtype=float).reshape(-1, 3)[tets]          # (nE,4,3)
    return np.einsum("eni,enj->eij", xe, G)


# ---------------------------------------------------------------------------
# rotation-variant SVD  (material.py:127-137)


def svd_rv(F):
    """Batched F = U diag(s) W^T with U, W in SO(3); reflections go into s[2]."""
    U, s, Wt = np.linalg.svd(F)
    W = np.ascontiguousarray(np.swapaxes(Wt, -1, -2))
    s = s.copy()
    for M in (U, W):
        neg = np.linalg.det(M) < 0.0
        M[neg, :, 2] = -M[neg, :, 2]
        s[neg, 2] = -s[neg, 2]
    return U, s, W


# ---------------------------------------------------------------------------
# volume projection in singular-value space


def _pairprod(s):
    """p = (s1 s2, s0 s2, s0 s1): gradient of s0 s1 s2 (`material.py:159-160`)."""
    return np.stack([s[..., 1] * s[..., 2], s[..., 0] * s[..., 2], s[..., 0] * s[..., 1]], -1)


def kkt_newton_batch(sig, s0=None):
    """Vectorised unclamped KKT Newton (`material.py:309-340`).

    Stops when the batch-wide max residual drops below 1e-12 or after 20
    iterations; a singular Jacobian anywhere aborts the whole batch with ok=False
    (the reference's `LinAlgError` branch, line 332-333).
    """
    n = sig.shape[0]
    s = np.clip(sig, SV_FLOOR, None) if s0 is None else np.array(s0, dtype=float)
    p = _pairprod(s)
    lam = (np.prod(s, axis=1) - 1.0) / np.maximum((p * p).sum(1), 1e-300)
    for _ in range(NEWTON_ITERS):
        p = _pairprod(s)
        res = np.concatenate([s - sig + lam[:, None] * p, (np.prod(s, axis=1) - 1.0)[:, None]], 1)
        if np.abs(res).max() < NEWTON_TOL:
            break
        J = np.zeros((n, 4, 4))
        J[:, [0, 1, 2], [0, 1, 2]] = 1.0
        for (a, b), k in (((0, 1), 2), ((0, 2), 1), ((1, 2), 0)):
            J[:, a, b] = J[:, b, a] = lam * s[:, k]
        J[:, :3, 3] = p
        J[:, 3, :3] = p
        try:
            step = np.linalg.solve(J, -res[:, :, None])[:, :, 0]
        except np.linalg.LinAlgError:
            return s, lam, np.zeros(n, dtype=bool)
        s = s + step[:, :3]
        lam = lam + step[:, 3]
    p = _pairprod(s)
    r_stat = np.abs(s - sig + lam[:, None] * p).max(1)
    r_con = np.abs(np.prod(s, axis=1) - 1.0)
    ok = (np.maximum(r_stat, r_con) < 1e-10) & np.isfinite(s).all(1)
    return s, lam, ok


def _kkt_res(sig, s, lam, free):
    """Residual with frozen entries zeroed (`material.py:163-168`)."""
    r = np.zeros(4)
    r[:3] = np.where(free, s - sig + lam * _pairprod(s), 0.0)
    r[3] = s[0] * s[1] * s[2] - 1.0
    return r


def _newton_free(sig, s_start, lam_start, free):
    """Damped Newton on the free entries (`material.py:171-214`)."""
    s = s_start.copy()
    lam = lam_start
    idx = np.flatnonzero(free)
    nf = len(idx)
    if nf == 0:
        return s, lam, False

    def rnorm(sv, lv):
        r = _kkt_res(sig, sv, lv, free)
        return np.abs(np.r_[r[idx], r[3]]).max()

    for _ in range(NEWTON_ITERS):
        r = _kkt_res(sig, s, lam, free)
        rn = np.abs(np.r_[r[idx], r[3]]).max()
        if rn < NEWTON_TOL:
            return s, lam, True
        p = _pairprod(s)
        J = np.zeros((nf + 1, nf + 1))
        for a, i in enumerate(idx):
            for b, j in enumerate(idx):
                J[a, b] = 1.0 if i == j else lam * s[3 - i - j]
            J[a, nf] = J[nf, a] = p[i]
        try:
            d = np.linalg.solve(J, -np.r_[r[idx], r[3]])
        except np.linalg.LinAlgError:
            return s, lam, False
        t = 1.0
        for _h in range(6):
            s_try = s.copy()
            s_try[idx] = s[idx] + t * d[:nf]
            lam_try = lam + t * d[nf]
            rn_try = rnorm(s_try, lam_try)
            if rn_try < rn or rn_try < NEWTON_TOL:
                break
            t *= 0.5
        s, lam = s_try, lam_try
    return s, lam, rnorm(s, lam) < 1e-10


def _solve_with_clamps(sig, s_init, lam_init):
    """Up to 3 rounds of Newton + freezing of floor violators (`material.py:217-239`)."""
    free = np.ones(3, dtype=bool)
    s = s_init.copy()
    lam = lam_init
    for _ in range(3):
        s = np.where(free, s, SV_FLOOR)
        s, lam, ok = _newton_free(sig, s, lam, free)
        if not ok:
            return None
        viol = free & (s < SV_FLOOR - 1e-12)
        if not viol.any():
            return s, lam, ~free
        free &= ~viol
        if free.sum() == 1:
            i = int(np.flatnonzero(free)[0])
            s = np.full(3, SV_FLOOR)
            s[i] = 1.0 / SV_FLOOR ** 2
            lam = (sig[i] - s[i]) / _pairprod(s)[i]
            return s, lam, ~free
    return None


def sl3_project_scalar(sig):
    """Robust multi-start volume projection (`material.py:242-287`).

    Returns (s, lam, clamped, ok).
    """
    sig = np.asarray(sig, dtype=float)
    starts = [np.clip(sig, SV_FLOOR, None), np.ones(3)]
    prod = float(np.prod(sig))
    if prod > 1e-12:
        starts.append(np.clip(sig / np.cbrt(prod), SV_FLOOR, None))
    if prod > 1.0:
        j = int(np.argmin(sig))
        rest = float(np.prod(np.delete(sig, j)))
        if rest > 1e-12:
            st = np.clip(sig, SV_FLOOR, None)
            st[j] = max(1.0 / rest, SV_FLOOR)
            starts.append(st)
    best = None
    for st in starts:
        p = _pairprod(st)
        pp = float(p @ p)
        lam0 = (float(np.prod(st)) - 1.0) / pp if pp > 1e-300 else 0.0
        got = _solve_with_clamps(sig, st, lam0)
        if got is None:
            continue
        s, lam, clamped = got
        if s.min() < SV_FLOOR - 1e-9 or abs(np.prod(s) - 1.0) > 1e-8:
            continue
        obj = float(((s - sig) ** 2).sum())
        if best is None or obj < best[0] - 1e-15:
            best = (obj, s, lam, clamped)
    if best is not None:
        return best[1], best[2], best[3], True
    s = np.clip(np.abs(sig), SV_FLOOR, None)
    for _ in range(3):
        s = np.clip(s / np.cbrt(np.prod(s)), SV_FLOOR, None)
    log.warning("volume projection Newton failed for sigma=%s, using uniform scaling", sig)
    return s, 0.0, s <= SV_FLOOR, False


def sl3_project_batch(sig):
    """Batched projection with second start and suspicious re-solve (`material.py:343-392`).

    Returns (s, lam, clamped, n_robust) where n_robust counts scalar re-solves.
    """
    sig = np.asarray(sig, dtype=float)
    s, lam, ok = kkt_newton_batch(sig)
    clamped = np.zeros(sig.shape, dtype=bool)
    feas = ok & (s.min(1) >= SV_FLOOR - 1e-12)
    obj = ((s - sig) ** 2).sum(1)
    obj[~feas] = np.inf
    prod = np.prod(sig, axis=1)
    big = np.flatnonzero(prod > 1.0)
    if len(big):
        sub = sig[big]
        r = np.arange(len(big))
        j = sub.argmin(1)
        rest = prod[big] / np.maximum(sub[r, j], 1e-300)
        st = np.clip(sub, SV_FLOOR, None)
        st[r, j] = np.clip(1.0 / np.maximum(rest, 1e-12), SV_FLOOR, None)
        s2, lam2, ok2 = kkt_newton_batch(sub, st)
        obj2 = ((s2 - sub) ** 2).sum(1)
        take = ok2 & (s2.min(1) >= SV_FLOOR - 1e-12) & (obj2 < obj[big] - 1e-15)
        sel = big[take]
        s[sel], lam[sel], obj[sel] = s2[take], lam2[take], obj2[take]
        feas[sel] = True
    odd = ~feas | (sig.min(1) < 0.2) | (np.abs(sig).max(1) > 5.0)
    with np.errstate(invalid="ignore", divide="ignore"):
        uni = sig / np.cbrt(np.maximum(prod, 1e-300))[:, None]
    uni_ok = (prod > 1e-12) & (uni.min(1) >= SV_FLOOR)
    odd |= uni_ok & (obj > ((uni - sig) ** 2).sum(1) + 1e-12)
    rows = np.flatnonzero(odd)
    for i in rows:
        s[i], lam[i], clamped[i], _ = sl3_project_scalar(sig[i])
    return s, lam, clamped, len(rows)


def projections(F):
    """(R, V) for a batch of F (`material.py:395-407`)."""
    F = np.asarray(F, dtype=float)
    if not np.all(np.isfinite(F)):
        raise ValueError("non-finite deformation gradient in batch")
    U, sig, W = svd_rv(F)
    Wt = np.swapaxes(W, -1, -2)
    R = U @ Wt
    s = sl3_project_batch(sig)[0]
    V = (U * s[:, None, :]) @ Wt
    return R, V


# ---------------------------------------------------------------------------
# local step and assembly


def elastic_rhs(x, tets, G, vol, gs, gv, n_nodes):
    """rhs = sum_e 2 V_e G_e^T (gs R + gv V) scattered in tet order (`pdsolver.py:59-71`).

    Returns (rhs, F, R, V).
    """
    F = deformation_gradients(x, tets, G)
    R, V = projections(F)
    P = gs[:, None, None] * R + gv[:, None, None] * V
    per = 2.0 * vol[:, None, None] * np.einsum("enj,eij->eni", G, P)
    rhs = np.zeros((n_nodes, 3))
    np.add.at(rhs, tets.reshape(-1), per.reshape(-1, 3))
    return rhs, F, R, V


def elastic_energy(x, tets, G, vol, gs, gv):
    """sum_e V_e (gs |F-R|^2 + gv |F-V|^2) (`pdsolver.py:74-82`)."""
    F = deformation_gradients(x, tets, G)
    R, V = projections(F)
    return float(np.sum(vol * (gs * ((F - R) ** 2).sum((1, 2)) + gv * ((F - V) ** 2).sum((1, 2)))))


def pd_objective(x, xhat, mass, dt, tets, G, vol, gs, gv):
    """Inertia + elastic objective of one implicit step (`pdsolver.py:307-312`)."""
    d = np.asarray(x) - xhat
    return 0.5 / dt ** 2 * float(np.sum(mass[:, None] * d * d)) + elastic_energy(x, tets, G, vol, gs, gv)


def assemble_K(tets, G, vol, gs, gv, mass, dt, n_nodes):
    """Scalar K = M/dt^2 + sum_e 2V(gs+gv) G G^T as CSC (`pdsolver.py:32-56`)."""
    if dt <= 0.0:
        raise ValueError("dt must be positive")
    if np.any(gs < 0.0) or np.any(gv < 0.0):
        raise ValueError("negative material coefficient")
    if mass is None:
        raise ValueError("mesh node masses not lumped yet")
    c = 2.0 * vol * (gs + gv)
    blk = c[:, None, None] * np.einsum("eni,emi->enm", G, G)
    r = np.repeat(tets, 4, axis=1).reshape(-1)
    q = np.tile(tets, (1, 4)).reshape(-1)
    K = sp.csr_matrix((blk.reshape(-1), (r, q)), shape=(n_nodes, n_nodes))
    return (K + sp.diags(mass / dt ** 2)).tocsc()


# ---------------------------------------------------------------------------
# global solvers


class GlobalSolver:
    """Direct (SuperLU) or CMS + A-Jacobi solve with pins eliminated (`pdsolver.py:201-246`)."""

    def __init__(self, K, free, pins, mode="direct", cms=None, refine_sweeps=0,
                 aggregation=2, omega=OMEGA, chebyshev=False):
        self.free = np.asarray(free)
        self.pins = np.asarray(pins, dtype=np.int64)
        Kf = K[self.free]
        self.Kff = Kf[:, self.free].tocsc()
        self.Kfp = Kf[:, self.pins].tocsc() if len(self.pins) else None
        self.mode = mode
        self.cms = cms
        self.refine = (refine_sweeps, aggregation, omega, chebyshev)
        if mode == "direct":
            self._lu = spla.factorized(self.Kff)
        elif mode != "cms":
            raise ValueError(f"unknown solver mode {mode!r}")

    def solve(self, B, pin_vals):
        Bf = B[self.free]
        if self.Kfp is not None:
            Bf = Bf - self.Kfp @ pin_vals
        X = np.empty_like(B)
        if len(self.pins):
            X[self.pins] = pin_vals
        sweeps, agg, om, cheb = self.refine
        for k in range(Bf.shape[1]):
            if self.mode == "direct":
                X[self.free, k] = self._lu(Bf[:, k])
            else:
                xk = self.cms.solve(Bf[:, k])
                if sweeps > 0:
                    xk, _ = a_jacobi_refine(self.Kff, Bf[:, k], xk, sweeps, agg, om, cheb)
                X[self.free, k] = xk
        return X


def pd_equilibrium(x0, tets, G, vol, gs, gv, mass, inertia_target, pins, pin_vals, dt, iterations=PD_ITERS,
                   solver=None):
    """Proximal local/global rounds on E(x) + (1/dt^2) a^T M x (`pdsolver.py:315-338`).

    Each round solves K x = (M/dt^2)(x_cur - a) + elastic rhs; RuntimeError
    "quasi-static projection diverged at iteration {it}" on non-finite x.
    """
    n = len(mass)
    pins = np.asarray(pins, dtype=np.int64)
    free = np.setdiff1d(np.arange(n), pins)
    if solver is None:
        solver = GlobalSolver(assemble_K(tets, G, vol, gs, gv, mass, dt, n), free, pins)
    x = np.asarray(x0, dtype=float).reshape(-1, 3).copy()
    if len(pins):
        x[pins] = pin_vals
    m_dt2 = np.asarray(mass)[:, None] / dt ** 2
    for it in range(iterations):
        rhs = elastic_rhs(x, tets, G, vol, gs, gv, n)[0]
        b = m_dt2 * (x - inertia_target) + rhs
        x = solver.solve(b, pin_vals if len(pins) else np.empty((0, 3)))
        if not np.all(np.isfinite(x)):
            raise RuntimeError(f"quasi-static projection diverged at iteration {it}")
    return x


def predicted(x, v, dt, mass, forces):
    """xhat = x + dt v + dt^2 m^-1 f with m^-1 := 0 where m = 0 (`pdsolver.py:249-254`)."""
    inv_m = np.zeros_like(mass)
    pos = mass > 0.0
    inv_m[pos] = 1.0 / mass[pos]
    f = np.zeros_like(x) if forces is None else np.asarray(forces, dtype=float)
    return x + dt * v + dt ** 2 * inv_m[:, None] * f


def collider_targets(x, colliders):
    """Penetrating nodes and their closest surface points (`pdsolver.py:125-155`)."""
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
    """Points projected out of any collider they penetrate (`pdsolver.py:158-163`)."""
    out = np.asarray(points, dtype=float).copy()
    i, t = collider_targets(out, colliders)
    out[i] = t
    return out


def pd_step_contact(x, v, dt, tets, G, vol, gs, gv, mass, pins, pin_targets, forces, colliders,
                    iterations=PD_ITERS, damping=1.0, contact_stiffness=1e4):
    """pd_step with colliders (`pdsolver.py:271-281, 294-297`): contact weight
    cw = k * diag(K) at the nodes penetrating at the prediction, folded into K
    (duplicates summed) and into b once per node; direct solve every step."""
    n = len(mass)
    pins = np.asarray(pins, dtype=np.int64)
    free = np.setdiff1d(np.arange(n), pins)
    xhat = predicted(x, v, dt, mass, forces)
    cidx, _ = collider_targets(xhat, colliders)
    K = assemble_K(tets, G, vol, gs, gv, mass, dt, n)
    cw = None
    if len(cidx):
        cw = contact_stiffness * K.diagonal()[cidx]
        K = (K + sp.csr_matrix((cw, (cidx, cidx)), shape=(n, n))).tocsc()
    solver = GlobalSolver(K, free, pins)
    x_start = x.copy()
    xi = xhat.copy()
    pin_vals = np.empty((0, 3))
    if len(pins):
        pin_vals = pin_targets
        xi[pins] = pin_vals
    inertia = (mass[:, None] / dt ** 2) * xhat
    for it in range(iterations):
        b = inertia + elastic_rhs(xi, tets, G, vol, gs, gv, n)[0]
        if len(cidx):
            b[cidx] += cw[:, None] * surface_targets(xi[cidx], colliders)
        xi = solver.solve(b, pin_vals)
        if not np.all(np.isfinite(xi)):
            raise RuntimeError(f"projective step produced non-finite positions at iteration {it}")
    return xi, damping * (xi - x_start) / dt


def pd_step(x, v, dt, tets, G, vol, gs, gv, mass, solver, pins=(), pin_targets=None,
            forces=None, iterations=PD_ITERS, damping=1.0, timers=None):
    """One implicit-Euler step by local/global rounds (`pdsolver.py:257-304`, no colliders).

    Returns (x_new, v_new).
    """
    import time
    n = len(mass)
    pins = np.asarray(pins, dtype=np.int64)
    xhat = predicted(x, v, dt, mass, forces)
    x_start = x.copy()
    xi = xhat.copy()
    pin_vals = np.empty((0, 3))
    if len(pins):
        pin_vals = pin_targets
        xi[pins] = pin_vals
    inertia = (mass[:, None] / dt ** 2) * xhat
    for it in range(iterations):
        t0 = time.perf_counter()
        rhs = elastic_rhs(xi, tets, G, vol, gs, gv, n)[0]
        t1 = time.perf_counter()
        xi = solver.solve(inertia + rhs, pin_vals)
        t2 = time.perf_counter()
        if timers is not None:
            timers["local"] = timers.get("local", 0.0) + t1 - t0
            timers["global"] = timers.get("global", 0.0) + t2 - t1
        if not np.all(np.isfinite(xi)):
            raise RuntimeError(f"projective step produced non-finite positions at iteration {it}")
    return xi, damping * (xi - x_start) / dt


def simulate(nodes, tets, G, vol, gs, gv, mass, steps, dt, forces=None, pins=(),
             pin_targets=None, iterations=PD_ITERS, solver_mode="direct", n_domains=2,
             modes_per_domain=20, refine_sweeps=30, aggregation=2, chebyshev=False,
             damping=1.0, labels=None, x0=None):
    """Frame driver (`pdsolver.py:710-763`, no colliders / polish). Returns (steps, nV, 3)."""
    n = len(mass)
    pins = np.asarray(pins, dtype=np.int64)
    path = None
    if pin_targets is not None:
        pin_targets = np.asarray(pin_targets, dtype=float)
        if pin_targets.ndim == 3:
            path, pin_targets = pin_targets, pin_targets[0]
    x = np.array(nodes if x0 is None else x0, dtype=float).reshape(-1, 3)
    v = np.zeros_like(x)
    if len(pins) and pin_targets is None:
        pin_targets = x[pins].copy()
    free = np.setdiff1d(np.arange(n), pins)
    K = assemble_K(tets, G, vol, gs, gv, mass, dt, n)
    if solver_mode == "cms":
        Kff = K[free][:, free].tocsc()
        lab = partition_elements(nodes, tets, n_domains, labels)
        inner, bnd = classify_nodes(tets, lab, n, free)
        remap = -np.ones(n, dtype=np.int64)
        remap[free] = np.arange(len(free))
        cms = CmsBasis(Kff, [remap[i] for i in inner], remap[bnd], modes_per_domain)
        solver = GlobalSolver(K, free, pins, "cms", cms, refine_sweeps, aggregation, OMEGA, chebyshev)
    else:
        solver = GlobalSolver(K, free, pins)
    if forces is not None:
        forces = np.asarray(forces, dtype=float)
        if forces.ndim == 2:
            forces = np.broadcast_to(forces, (steps,) + forces.shape)
    frames = np.empty((steps, n, 3))
    for i in range(steps):
        if path is not None:
            pin_targets = path[i]
        x, v = pd_step(x, v, dt, tets, G, vol, gs, gv, mass, solver, pins, pin_targets,
                       None if forces is None else forces[i], iterations, damping)
        frames[i] = x
    return frames


# ---------------------------------------------------------------------------
# component-mode subspace (pdsolver.py:467-609)


def partition_elements(nodes, tets, n_domains, labels=None):
    """Caller labels, or quantile slabs of centroids on the longest axis (`pdsolver.py:467-480`)."""
    if labels is not None:
        labels = np.asarray(labels, dtype=np.int64)
        if len(labels) != len(tets):
            raise ValueError("need one domain label per element")
        return labels
    cen = nodes[tets].mean(1)
    ax = int(np.argmax(nodes.max(0) - nodes.min(0)))
    cuts = np.quantile(cen[:, ax], np.linspace(0.0, 1.0, n_domains + 1)[1:-1])
    return np.searchsorted(cuts, cen[:, ax])


def classify_nodes(tets, labels, n_nodes, free=None):
    """Interior sets per domain + merged boundary (`pdsolver.py:483-509`)."""
    lo = np.full(n_nodes, np.iinfo(np.int64).max, dtype=np.int64)
    hi = np.full(n_nodes, -1, dtype=np.int64)
    lab4 = np.repeat(labels, 4)
    np.minimum.at(lo, tets.reshape(-1), lab4)
    np.maximum.at(hi, tets.reshape(-1), lab4)
    keep = np.ones(n_nodes, dtype=bool)
    if free is not None:
        keep[:] = False
        keep[free] = True
    taken = np.zeros(n_nodes, dtype=bool)
    inner = []
    for d in range(int(labels.max()) + 1):
        sel = np.flatnonzero((lo == d) & (hi == d) & keep)
        inner.append(sel)
        taken[sel] = True
    return inner, np.flatnonzero(keep & ~taken & (hi >= 0))


def lowest_modes(Kii, m):
    """m lowest eigenvectors of K_ii (`pdsolver.py:578-590`)."""
    n = Kii.shape[0]
    if m >= n or n <= 400:
        return np.linalg.eigh(Kii.toarray())[1][:, :m]
    try:
        return spla.eigsh(Kii, k=m, sigma=0.0, mode="normal")[1]
    except Exception:                                   # noqa: BLE001 - mirrors reference
        return np.linalg.eigh(Kii.toarray())[1][:, :m]


class CmsBasis:
    """Craig-Bampton basis T = [Phi blocks | I_b + Psi blocks], K_red = T^T K T (`pdsolver.py:512-593`)."""

    def __init__(self, K, inner, boundary, modes_per_domain=20):
        K = K.tocsc()
        n = K.shape[0]
        boundary = np.asarray(boundary, dtype=np.int64)
        nb = len(boundary)
        self.blocks = []
        phi_cols = []
        psi_rows = []
        c0 = 0
        for sel in inner:
            sel = np.asarray(sel, dtype=np.int64)
            if len(sel) == 0:
                self.blocks.append(None)
                continue
            Kii = K[sel][:, sel].tocsc()
            Phi = lowest_modes(Kii, min(modes_per_domain, len(sel)))
            Psi = None
            if nb:
                Kib = K[sel][:, boundary].toarray()
                lu = spla.factorized(Kii)
                Psi = -np.column_stack([lu(Kib[:, j]) for j in range(nb)])
            self.blocks.append((sel, Phi, Psi))
            phi_cols.append((sel, Phi, c0))
            c0 += Phi.shape[1]
            if Psi is not None:
                psi_rows.append((sel, Psi))
        r, c, v = [], [], []
        for sel, Phi, off in phi_cols:
            rr, cc = np.meshgrid(sel, off + np.arange(Phi.shape[1]), indexing="ij")
            r.append(rr.ravel()); c.append(cc.ravel()); v.append(Phi.ravel())
        r.append(boundary); c.append(c0 + np.arange(nb)); v.append(np.ones(nb))
        for sel, Psi in psi_rows:
            rr, cc = np.meshgrid(sel, c0 + np.arange(nb), indexing="ij")
            r.append(rr.ravel()); c.append(cc.ravel()); v.append(Psi.ravel())
        self.T = sp.csr_matrix((np.concatenate(v), (np.concatenate(r), np.concatenate(c))),
                               shape=(n, c0 + nb))
        Kr = (self.T.T @ K @ self.T).tocsc()
        self.K_red = (0.5 * (Kr + Kr.T)).tocsc()
        self._lu = spla.factorized(self.K_red)

    def solve(self, b):
        return self.T @ self._lu(self.T.T @ b)


# ---------------------------------------------------------------------------
# aggregated Jacobi (pdsolver.py:616-703)


def power_rho(K, invd, omega, iters=30, seed=0):
    """Spectral radius estimate of I - omega D^-1 K (`pdsolver.py:616-629`)."""
    v = np.random.default_rng(seed).normal(size=K.shape[0])
    v /= np.linalg.norm(v)
    rho = 0.0
    for _ in range(iters):
        v = v - omega * (invd * (K @ v))
        nv = np.linalg.norm(v)
        if nv < 1e-300:
            return 0.0
        rho = nv
        v /= nv
    return min(rho, 0.9999)


def a_jacobi_refine(K, b, x0, sweeps=30, aggregation=2, omega=OMEGA, chebyshev=False, rho=None):
    """Aggregated weighted Jacobi with best-iterate tracking (`pdsolver.py:632-703`)."""
    if aggregation not in (2, 3):
        raise ValueError("aggregation must be 2 or 3")
    d = K.diagonal()
    if np.any(d <= 0.0):
        raise ValueError("matrix diagonal must be positive")
    invd = 1.0 / d
    x = np.array(x0, dtype=float)
    r = b - K @ x
    best_x, best_r = x.copy(), float(np.linalg.norm(r))
    hist = [best_r]
    info = {"diverged": False}
    if chebyshev:
        if rho is None:
            rho = power_rho(K, invd, omega)
        x_old = x.copy()
        w = 1.0
        for k in range(sweeps * aggregation):
            y = x + omega * (invd * (b - K @ x))
            if k == 0:
                xn = y
                w = 2.0 / (2.0 - rho ** 2)
            else:
                xn = w * (y - x_old) + x_old
                w = 4.0 / (4.0 - rho ** 2 * w)
            x_old, x = x, xn
            rn = float(np.linalg.norm(b - K @ x))
            hist.append(rn)
            if rn < best_r:
                best_r, best_x = rn, x.copy()
            if rn > 10.0 * best_r:
                info["diverged"] = True
                info["residuals"] = hist
                return best_x, info
        info["residuals"] = hist
        return (best_x if best_r < hist[-1] else x), info
    for _ in range(sweeps):
        e = np.zeros_like(x)
        s = r.copy()
        for _a in range(aggregation):
            c = omega * (invd * s)
            e += c
            s -= K @ c
        x = x + e
        r = s
        rn = float(np.linalg.norm(r))
        hist.append(rn)
        if rn < best_r:
            best_r, best_x = rn, x.copy()
        if rn > 10.0 * best_r:
            info["diverged"] = True
            break
    info["residuals"] = hist
    if info["diverged"] or hist[-1] > best_r:
        return best_x, info
    return x, info


# ---------------------------------------------------------------------------
# second order (fitting side)


def elastic_gradient(x, tets, G, vol, gs, gv, n_nodes):
    """sum_e 2 V_e G_e^T (gs (F-R) + gv (F-V)) in tet order (`pdsolver.py:85-97`)."""
    F = deformation_gradients(x, tets, G)
    R, V = projections(F)
    P = gs[:, None, None] * (F - R) + gv[:, None, None] * (F - V)
    per = 2.0 * vol[:, None, None] * np.einsum("enj,eij->eni", G, P)
    out = np.zeros((n_nodes, 3))
    np.add.at(out, tets.reshape(-1), per.reshape(-1, 3))
    return out


def _ds_dsigma(s, lam, clamped):
    """ds/dsigma of the constrained singular-value solve (`material.py:418-438`)."""
    idx = np.flatnonzero(~clamped)
    nf = idx.size
    D = np.zeros((3, 3))
    if nf == 0:
        return D
    p = _pairprod(s)
    A = np.zeros((nf + 1, nf + 1))
    for a, i in enumerate(idx):
        for b, j in enumerate(idx):
            A[a, b] = 1.0 if i == j else lam * s[3 - i - j]
        A[a, nf] = A[nf, a] = p[i]
    rhs = np.zeros((nf + 1, nf))
    rhs[:nf, :nf] = np.eye(nf)
    D[np.ix_(idx, idx)] = np.linalg.solve(A, rhs)[:nf, :]
    return D


def projection_jacobians(F):
    """(d vec R / d vec F, d vec V / d vec F), (B, 9, 9) each, row-major vec (`material.py:490-524`)."""
    F = np.asarray(F, dtype=float)
    B = F.shape[0]
    U, sig, W = svd_rv(F)
    s, lam, clamped, _ = sl3_project_batch(sig)
    LR = np.zeros((B, 9, 9))
    LV = np.zeros((B, 9, 9))
    ds = np.stack([_ds_dsigma(s[e], lam[e], clamped[e]) for e in range(B)]) if B else np.zeros((0, 3, 3))
    dia = (0, 4, 8)
    for i in range(3):
        for j in range(3):
            LV[:, dia[i], dia[j]] = ds[:, i, j]
    for i, j in ((0, 1), (0, 2), (1, 2)):
        a, b = 3 * i + j, 3 * j + i
        den = sig[:, i] + sig[:, j]
        den = np.where(np.abs(den) < 1e-8, np.copysign(1e-8, np.where(den == 0.0, 1.0, den)), den)
        LR[:, a, a] = LR[:, b, b] = 1.0 / den
        LR[:, a, b] = LR[:, b, a] = -1.0 / den
        dd = sig[:, i] - sig[:, j]
        scale = np.maximum(1.0, np.maximum(np.abs(sig[:, i]), np.abs(sig[:, j])))
        safe = np.abs(dd) > 1e-7 * scale
        cs = np.where(safe, (s[:, i] - s[:, j]) / np.where(safe, dd, 1.0), ds[:, i, i] - ds[:, i, j])
        ca = (s[:, i] + s[:, j]) / den
        LV[:, a, a] = LV[:, b, b] = 0.5 * (cs + ca)
        LV[:, a, b] = LV[:, b, a] = 0.5 * (cs - ca)
    Q = np.einsum("eik,ejl->eijkl", U, W).reshape(B, 9, 9)
    Qt = np.swapaxes(Q, 1, 2)
    return Q @ LR @ Qt, Q @ LV @ Qt


def exact_elastic_hessian(x, tets, G, vol, gs, gv, n_nodes):
    """2 V D^T (gs (I - dR/dF) + gv (I - dV/dF)) D summed over tets, CSR (`pdsolver.py:100-118`)."""
    F = deformation_gradients(x, tets, G)
    LR, LV = projection_jacobians(F)
    I9 = np.eye(9)
    M9 = gs[:, None, None] * (I9 - LR) + gv[:, None, None] * (I9 - LV)
    nE = len(tets)
    D = np.zeros((nE, 9, 12))          # D[3i+j, 3n+i] = G[n, j]   (volmesh.py:92-97)
    for n in range(4):
        for i in range(3):
            for j in range(3):
                D[:, 3 * i + j, 3 * n + i] = G[:, n, j]
    He = 2.0 * vol[:, None, None] * np.einsum("eia,eij,ejb->eab", D, M9, D)
    dofs = (3 * tets[:, :, None] + np.arange(3)).reshape(nE, 12)
    rows = np.repeat(dofs, 12, axis=1).reshape(-1)
    cols = np.tile(dofs, (1, 12)).reshape(-1)
    n = 3 * n_nodes
    return sp.csr_matrix((He.reshape(-1), (rows, cols)), shape=(n, n))


def newton_polish(x0, tets, G, vol, gs, gv, mass, dt, pins=(), pin_vals=None, inertia_target=None, xhat=None,
                  tol=1e-5, max_iters=20, exact=False):
    """Newton-type polish of the step / quasi-static residual (`pdsolver.py:350-460`).

    Returns (x, converged, iterations)."""
    if (inertia_target is None) == (xhat is None):
        raise ValueError("give exactly one of inertia_target or xhat")
    n = len(mass)
    pins = np.asarray(pins, dtype=int)
    free = np.setdiff1d(np.arange(n), pins)
    x = np.asarray(x0, dtype=float).reshape(-1, 3).copy()
    if len(pins):
        x[pins] = pin_vals
    m_dt2 = mass[:, None] / dt ** 2

    def residual(xc):
        g = elastic_gradient(xc, tets, G, vol, gs, gv, n)
        return g + (m_dt2 * (xc - xhat) if xhat is not None else m_dt2 * inertia_target)

    def objective(xc):
        e = elastic_energy(xc, tets, G, vol, gs, gv)
        if xhat is not None:
            d = xc - xhat
            return e + 0.5 * float(np.sum(m_dt2 * d * d))
        return e + float(np.sum(m_dt2 * inertia_target * xc))

    def gmax(gv_):
        return float(np.abs(gv_[free]).max()) if len(free) else 0.0

    g = residual(x)
    if gmax(g) < tol:
        return x, True, 0
    K = assemble_K(tets, G, vol, gs, gv, mass, dt, n)
    solve = spla.factorized(K[free][:, free].tocsc())
    fdofs = (3 * free[:, None] + np.arange(3)[None, :]).reshape(-1)
    mass_diag = np.repeat(mass, 3) / dt ** 2

    def gn_step(gc):
        step = np.zeros_like(x)
        for k in range(3):
            step[free, k] = solve(-gc[free, k])
        return step

    def exact_step(xc, gc):
        J = exact_elastic_hessian(xc, tets, G, vol, gs, gv, n)
        if xhat is not None:
            J = J + sp.diags(mass_diag)
        try:
            d = spla.spsolve(J[fdofs][:, fdofs].tocsc(), -gc.reshape(-1)[fdofs])
        except RuntimeError:
            return None
        if not np.all(np.isfinite(d)):
            return None
        step = np.zeros_like(x)
        step.reshape(-1)[fdofs] = d
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
                return x, False, it
            xn, on = x, obj
        x, obj = xn, on
        g = residual(x)
        if gmax(g) < tol:
            return x, True, it
    return x, gmax(g) < tol, max_iters


def gamma_jacobian_t(x, lam, tets, G, vol):
    """gamma_jacobian(mesh, x)^T lam, (2 nE,) (`fitting.py:172-190`)."""
    F = deformation_gradients(x, tets, G)
    R, V = projections(F)
    L = deformation_gradients(lam, tets, G)
    v2 = 2.0 * vol
    return np.concatenate([v2 * ((F - R) * L).sum((1, 2)), v2 * ((F - V) * L).sum((1, 2))])


def adjoint_gradient(x, gx, tets, G, vol, gs, gv, n_nodes, pins):
    """grad = -J^T lam with H_ff lam = g_x[free] (`fitting.py:206-238`).  Returns (grad, lam_full)."""
    free = np.setdiff1d(np.arange(n_nodes), pins)
    fdofs = (3 * free[:, None] + np.arange(3)[None, :]).reshape(-1)
    H = exact_elastic_hessian(x, tets, G, vol, gs, gv, n_nodes)
    lam_f = spla.spsolve(H[fdofs][:, fdofs].tocsc(), np.asarray(gx).reshape(-1)[fdofs])
    lam = np.zeros(3 * n_nodes)
    lam[fdofs] = lam_f
    lam = lam.reshape(-1, 3)
    return -gamma_jacobian_t(x, lam, tets, G, vol), lam


def gauss_newton_direction(H_ff, J_f, G_f, grad, kappa):
    """(J^T H^-1 G H^-1 J + kappa I) d = -grad by dense normal equations: the reference's own
    oracle route `dense_gauss_newton_direction` (`fitting.py:316-333`) for `adjoint_gauss_newton`
    (`fitting.py:251-313`)."""
    Hlu = spla.splu(sp.csc_matrix(H_ff))
    Jd = np.asarray(sp.csr_matrix(J_f).todense())
    S = np.column_stack([Hlu.solve(-Jd[:, j]) for j in range(Jd.shape[1])])
    P = S.T @ (sp.csr_matrix(G_f) @ S)
    return np.linalg.solve(P + kappa * np.eye(P.shape[0]), -grad)

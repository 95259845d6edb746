"""Generate golden vectors by running the REAL reference (volknit) in the build container.

Run from the repo root (needs /root/reference, which the GPU box does not have):

    python tests/golden/make_golden.py [small|c2|c3|all]

Outputs (committed) land next to this script.  Scenes come from
`paper_2405_12484_b200.scenes` (seeded, bit-reproducible); the fixtures also
store input checksums so the tests can prove the regenerated scene is the one
the reference saw.  Per-fixture contents:

  projections.npz  F batch (random / inverted / near-singular / clamp / t*I) and the
                   reference `material.batch_projections` R, V; scalar
                   `sl3_sigma_project` results on special sigma triples.
  c1.npz           C1 swatch: `assemble_global` K (CSR), `elastic_rhs` at a perturbed
                   x (rhs, F, R, V), `simulate_mesh(direct)` after 1 and 3 frames.
  solvers.npz      C1 free-free K: `a_jacobi_refine` (agg 2/3, Chebyshev) from a seeded
                   start, `build_cms(...).solve`, and `simulate_mesh(cms)` 1 frame.
  c2.npz           C2 scarf: `simulate_mesh(direct)` frames 1, 10, 100 (f64).
  c3.npz           C3 sweater: `simulate_mesh(direct)` frame 1, positions (float64).
  c3fold.npz       C3 sweater, one `pd_step(direct)` frame from a state inside the fold window
                   (frame 120 of the device fp64 trajectory, rounded to float32 and stored: the
                   reference and the device start from the same bits); displacement (float64).
  second_order.npz C1: elastic_energy / elastic_gradient / exact_elastic_hessian, newton_polish
                   (dynamic GN + exact, quasi-static exact), simulate_mesh(polish_tol), and
                   fitting.adjoint_gradient on a tracking loss (scenes.TrackingProblem).
  contact.npz      box dropped on a plane + sphere collider: `simulate_mesh(colliders=...)`, 20 frames.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

from volknit import material as ref_mat      # noqa: E402
from volknit import pdsolver as ref_pd       # noqa: E402
from volknit import volmesh as ref_vm        # noqa: E402

from paper_2405_12484_b200 import scenes     # noqa: E402


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:32]


def scene_digest(sc):
    m = sc.mesh
    return digest(m.nodes, m.tets.astype(np.int64), m.node_mass, sc.gammas.gamma_s,
                  sc.gammas.gamma_v, sc.pins.astype(np.int64))


def ref_mesh(sc):
    m = sc.mesh
    rm = ref_vm.VolumeMesh(nodes=m.nodes.copy(), tets=m.tets.copy(), cell_size=m.cell_size,
                           origin=m.origin.copy(), node_grid=m.node_grid.copy(),
                           voxels=m.voxels.copy(), tet_voxel=m.tet_voxel.copy())
    rm.node_mass = m.node_mass.copy()
    return rm


def projection_batch(rng):
    F = [np.eye(3) + 0.8 * rng.normal(size=(1500, 3, 3))]
    inv = np.eye(3) + 0.3 * rng.normal(size=(200, 3, 3))
    inv[:, :, 0] *= -1.0
    F.append(inv)
    # near-rank-deficient: scale one singular direction down
    a = rng.normal(size=(100, 3, 3))
    U, s, Vt = np.linalg.svd(a)
    s[:, 2] = 10.0 ** rng.uniform(-7, -2, size=100)
    F.append(U @ (s[:, :, None] * Vt))
    # large stretches / compressions (suspicious band: min < 0.2 or max > 5)
    d = np.exp(rng.uniform(-3.0, 2.0, size=(200, 3)))
    Q1 = np.linalg.qr(rng.normal(size=(200, 3, 3)))[0]
    Q2 = np.linalg.qr(rng.normal(size=(200, 3, 3)))[0]
    F.append(Q1 @ (d[:, :, None] * np.swapaxes(Q2, 1, 2)))
    # mild near-identity (the PD steady state)
    F.append(np.eye(3) + 0.02 * rng.normal(size=(500, 3, 3)))
    # uniform scalings incl. the symmetry-breaking band
    F.append(np.stack([t * np.eye(3) for t in (0.5, 1.0, 1.5, 1.8, 1.95, 2.0, 2.5)]))
    return np.concatenate(F)


def make_projections():
    rng = np.random.default_rng(20240817)
    F = projection_batch(rng)
    R, V = ref_mat.batch_projections(F)
    sig_cases = np.array([
        [2.0, 2.0, 2.0], [100.0, 100.0, 1e-5], [1.5, 1.5, 1.5], [0.5, 0.5, 0.5],
        [3.0, 0.1, 0.05], [1.2, 0.9, 0.95], [7.0, 1.0, 0.2], [0.0, 0.0, 0.0],
        [1.0, 1.0, -0.5], [40.0, 0.3, 0.001],
    ])
    sig_rand = np.exp(rng.uniform(-3.0, 1.5, size=(40, 3)))
    sig_all = np.concatenate([sig_cases, sig_rand])
    S, L, C, OK = [], [], [], []
    for sg in sig_all:
        s, lam, cl, ok = ref_mat.sl3_sigma_project(sg)
        S.append(s); L.append(lam); C.append(cl); OK.append(ok)
    np.savez_compressed(os.path.join(HERE, "projections.npz"), F=F, R=R, V=V, sigma=sig_all,
                        s=np.array(S), lam=np.array(L), clamped=np.array(C), ok=np.array(OK))
    print("projections", F.shape)


def make_c1():
    sc = scenes.c1_swatch()
    rm = ref_mesh(sc)
    K = ref_pd.assemble_global(rm, ref_mat.MaterialField(sc.gammas.gamma_s, sc.gammas.gamma_v),
                               sc.dt).tocsr()
    gam = ref_mat.MaterialField(sc.gammas.gamma_s, sc.gammas.gamma_v)
    rng = np.random.default_rng(7)
    xp = sc.mesh.nodes + 0.002 * rng.normal(size=sc.mesh.nodes.shape)
    rhs, F, R, V = ref_pd.elastic_rhs(rm, gam, xp)
    kw = dict(forces=sc.forces, pins=sc.pins, pin_targets=sc.pin_targets, iterations=30)
    fr3 = ref_pd.simulate_mesh(rm, gam, 3, sc.dt, **kw)
    st = ref_pd.SimState(x=sc.mesh.nodes, v=np.zeros_like(sc.mesh.nodes), dt=sc.dt,
                         pins=sc.pins, pin_targets=sc.pin_targets)
    xhat = ref_pd._predicted(st, sc.forces, rm)
    np.savez_compressed(os.path.join(HERE, "c1.npz"), digest=scene_digest(sc),
                        K_data=K.data, K_indices=K.indices, K_indptr=K.indptr,
                        x_pert=xp, rhs=rhs, F=F, R=R, V=V, frames=fr3, xhat=xhat)
    print("c1", fr3.shape)


def make_solvers():
    sc = scenes.c1_swatch()
    rm = ref_mesh(sc)
    gam = ref_mat.MaterialField(sc.gammas.gamma_s, sc.gammas.gamma_v)
    K = ref_pd.assemble_global(rm, gam, sc.dt)
    free = np.setdiff1d(np.arange(sc.n_nodes), sc.pins)
    Kff = K[free][:, free].tocsc()
    rng = np.random.default_rng(11)
    b = rng.normal(size=len(free))
    x0 = rng.normal(size=len(free))
    out = {"digest": scene_digest(sc), "b": b, "x0": x0}
    for agg in (2, 3):
        x, info = ref_pd.a_jacobi_refine(Kff, b, x0, sweeps=7, aggregation=agg, omega=0.7)
        out[f"aj{agg}_x"], out[f"aj{agg}_res"] = x, np.array(info["residuals"])
    x, info = ref_pd.a_jacobi_refine(Kff, b, x0, sweeps=10, aggregation=2, chebyshev=True)
    out["cheb_x"], out["cheb_res"] = x, np.array(info["residuals"])
    x, info = ref_pd.a_jacobi_refine(Kff, b, x0, sweeps=60, aggregation=2, omega=2.5)
    out["div_x"], out["div_res"], out["div_flag"] = x, np.array(info["residuals"]), info["diverged"]
    cms = ref_pd.build_cms(Kff, rm, n_domains=2, modes_per_domain=12, free=free)
    out["cms_x"] = cms.solve(b)
    out["cms_nred"] = cms.K_red.shape[0]
    kw = dict(forces=sc.forces, pins=sc.pins, pin_targets=sc.pin_targets, iterations=30)
    out["cms_frame"] = ref_pd.simulate_mesh(rm, gam, 1, sc.dt, solver_mode="cms", n_domains=2,
                                            modes_per_domain=12, refine_sweeps=30, **kw)[0]
    np.savez_compressed(os.path.join(HERE, "solvers.npz"), **out)
    print("solvers")


def contact_scene():
    return scenes.contact_scene()


def make_contact():
    sc, colliders = contact_scene()
    rm = ref_mesh(sc)
    gam = ref_mat.MaterialField(sc.gammas.gamma_s, sc.gammas.gamma_v)
    fr = ref_pd.simulate_mesh(rm, gam, 20, sc.dt, forces=sc.forces, colliders=colliders, iterations=10,
                              damping=0.9)
    np.savez_compressed(os.path.join(HERE, "contact.npz"), digest=scene_digest(sc), frames=fr)
    print("contact", fr.shape)


def make_big(key, frames_keep, steps, f32_disp):
    sc = scenes.make_scene(key)
    rm = ref_mesh(sc)
    gam = ref_mat.MaterialField(sc.gammas.gamma_s, sc.gammas.gamma_v)
    t0 = time.time()
    fr = ref_pd.simulate_mesh(rm, gam, steps, sc.dt, forces=sc.forces, pins=sc.pins,
                              pin_targets=sc.pin_targets, iterations=30)
    el = time.time() - t0
    keep = {f"frame{k}": (fr[k - 1] - sc.mesh.nodes).astype(np.float32) if f32_disp else fr[k - 1]
            for k in frames_keep}
    np.savez_compressed(os.path.join(HERE, f"{key.lower()}.npz"), digest=scene_digest(sc),
                        seconds=el, steps=steps, **keep)
    print(key, "seconds", el)


def make_c3fold():
    """One reference frame from the stored fold-window state (tools/c3_state.py writes it on the GPU)."""
    st = np.load(os.path.join(ROOT, "gpurun_out", "c3_state120.npz"))
    sc = scenes.make_scene("C3")
    rm = ref_mesh(sc)
    gam = ref_mat.MaterialField(sc.gammas.gamma_s, sc.gammas.gamma_v)
    x0 = st["x"].astype(np.float32).astype(np.float64)
    v0 = st["v"].astype(np.float32).astype(np.float64)
    state = ref_pd.SimState(x=x0, v=v0, dt=sc.dt, pins=sc.pins, pin_targets=sc.pin_targets)
    solver = ref_pd.GlobalSolver(ref_pd.assemble_global(rm, gam, sc.dt),
                                 np.setdiff1d(np.arange(rm.n_nodes), sc.pins), sc.pins)
    t0 = time.time()
    ref_pd.pd_step(state, rm, gam, iterations=30, forces=sc.forces, solver=solver)
    el = time.time() - t0
    np.savez_compressed(os.path.join(HERE, "c3fold.npz"), digest=scene_digest(sc), seconds=el,
                        frame=int(st["frame"]), x0=x0.astype(np.float32), v0=v0.astype(np.float32),
                        disp=state.x - x0, v=state.v)
    print("c3fold seconds", el)


def make_jacobians():
    """Reference projection_jacobians_batch on 600 cases of the projection set."""
    g = np.load(os.path.join(HERE, "projections.npz"))
    F = g["F"]
    idx = np.unique(np.concatenate([np.arange(0, len(F), max(1, len(F) // 500)), np.arange(len(F) - 100, len(F))]))
    F = F[idx]
    JR, JV = ref_mat.projection_jacobians_batch(F)
    np.savez_compressed(os.path.join(HERE, "jacobians.npz"), F=F, JR=JR, JV=JV)
    print("jacobians", F.shape)


def make_equilibrium():
    sc, a, x0 = scenes.equilibrium_case()
    rm = ref_mesh(sc)
    gam = ref_mat.MaterialField(sc.gammas.gamma_s, sc.gammas.gamma_v)
    out = {}
    for its in (1, 5, 30):
        out[f"x{its}"] = ref_pd.pd_equilibrium(rm, gam, a, x0, sc.pins, sc.pin_targets, sc.dt, iterations=its)
    np.savez_compressed(os.path.join(HERE, "equilibrium.npz"), digest=scene_digest(sc), a=a, x0=x0, **out)
    print("equilibrium fixtures written")


def make_io():
    """Mesh / material files written by the reference writers, and what its readers return."""
    from volknit import cli as ref_cli
    sc = scenes.c1_swatch()
    rm = ref_mesh(sc)
    d = os.path.join(HERE, "io")
    os.makedirs(d, exist_ok=True)
    prefix = os.path.join(d, "c1")
    ref_vm.write_mesh(rm, prefix, comment="golden c1")
    gam = ref_mat.MaterialField(sc.gammas.gamma_s, sc.gammas.gamma_v)
    ref_cli.write_material(os.path.join(d, "c1_material.csv"), gam, "golden")
    back = ref_vm.read_mesh(prefix)
    mat = ref_cli.read_material(os.path.join(d, "c1_material.csv"))
    np.savez_compressed(os.path.join(HERE, "io.npz"), nodes=back.nodes, tets=back.tets,
                        node_mass=back.node_mass, node_grid=back.node_grid, voxels=back.voxels,
                        tet_voxel=back.tet_voxel, cell_size=back.cell_size, origin=back.origin,
                        faces=ref_vm.boundary_faces(back), gamma_s=mat.gamma_s, gamma_v=mat.gamma_v)
    print("io fixtures written")


def make_second_order():
    """Reference elastic_energy / elastic_gradient / exact_elastic_hessian at a perturbed C1 x;
    newton_polish (dynamic GN and exact, quasi-static exact); simulate_mesh(polish_tol);
    adjoint_gradient on a tracking loss at the quasi-static equilibrium."""
    from volknit import fitting as ref_fit
    sc, x, xhat = scenes.second_order_case()
    rm = ref_mesh(sc)
    gam = ref_mat.MaterialField(sc.gammas.gamma_s, sc.gammas.gamma_v)
    out = dict(digest=scene_digest(sc), x=x, xhat=xhat)
    out["energy"] = ref_pd.elastic_energy(rm, gam, x)
    out["grad"] = ref_pd.elastic_gradient(rm, gam, x)
    H = ref_pd.exact_elastic_hessian(rm, gam, x).tocsr()
    H.sum_duplicates()
    H.sort_indices()
    out.update(H_data=H.data, H_indices=H.indices, H_indptr=H.indptr)
    for exact in (False, True):
        xp, ok, its = ref_pd.newton_polish(rm, gam, xhat, dt=sc.dt, pins=sc.pins, pin_vals=sc.pin_targets,
                                           xhat=xhat, tol=1e-7, max_iters=100, exact=exact)
        out[f"dyn_x_{int(exact)}"], out[f"dyn_ok_{int(exact)}"], out[f"dyn_it_{int(exact)}"] = xp, ok, its
    sc2, a, x0, weight, shift, sample = scenes.adjoint_case()
    xe = ref_pd.pd_equilibrium(rm, gam, a, x0, sc.pins, sc.pin_targets, sc.dt, iterations=8)
    xq, okq, itq = ref_pd.newton_polish(rm, gam, xe, dt=sc.dt, pins=sc.pins, pin_vals=sc.pin_targets,
                                        inertia_target=a, tol=1e-10, max_iters=150, exact=True)
    out.update(qs_x0=xe, qs_x=xq, qs_ok=okq, qs_it=itq)
    prob = scenes.TrackingProblem(rm, sc.dt, xq + shift, weight)
    st = ref_fit.adjoint_gradient(prob, sample, gam, xq)
    out.update(adj_grad=st.grad, adj_lam=st.lam, adj_residual=st.residual)
    rng = np.random.default_rng(14)
    basis, _ = np.linalg.qr(rng.normal(size=(sc.mesh.n_elements, 10)))
    frozen = np.array([3, 17, 4000])
    for tag, kw in (("full", {}), ("basis", dict(basis=basis)), ("frozen", dict(frozen=frozen))):
        d, kap, ok = ref_fit.adjoint_gauss_newton(prob, sample, st, **kw)
        out[f"gn_{tag}_d"], out[f"gn_{tag}_kappa"], out[f"gn_{tag}_ok"] = d, kap, ok
    out["gn_basis"] = basis
    out["gn_frozen"] = frozen
    fr = ref_pd.simulate_mesh(rm, gam, 2, sc.dt, forces=sc.forces, pins=sc.pins, pin_targets=sc.pin_targets,
                              iterations=sc.iterations, polish_tol=1e-6)
    out["polish_frames"] = fr
    np.savez_compressed(os.path.join(HERE, "second_order.npz"), **out)
    print("second-order fixtures written", {k: v for k, v in out.items() if np.ndim(v) == 0})


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "small"
    if what in ("small", "all"):
        make_projections()
        make_c1()
        make_solvers()
    if what in ("jac", "all"):
        make_jacobians()
    if what in ("eq", "all"):
        make_equilibrium()
    if what in ("so", "all"):
        make_second_order()
    if what in ("io", "all"):
        make_io()
    if what in ("contact", "all"):
        make_contact()
    if what in ("c2", "all"):
        make_big("C2", (1, 10, 100), 100, False)
    if what in ("c3", "all"):
        make_big("C3", (1,), 1, False)
    if what in ("c3fold",):
        make_c3fold()

"""GPU tests of the reference-compatible domain-decomposed solve (CMS) and the
A-Jacobi / Chebyshev refinement, against golden vectors from the reference and
the reference's own properties (test_pdsolver.py:317-459)."""

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from oracle import pd_oracle as orc
from paper_2405_12484_b200 import cms as gcms
from paper_2405_12484_b200 import pdsolver, scenes
from pdtest_helpers import golden, rel_l2, scene_digest

pytestmark = pytest.mark.gpu


def random_spd(rng, n, density=0.3):
    A = sp.random(n, n, density=density, random_state=np.random.RandomState(int(rng.integers(1 << 31))),
                  format="csr")
    return (A + A.T + sp.diags(np.full(n, n * 0.5))).tocsr()


@pytest.fixture(scope="module")
def c1sys():
    sc = scenes.c1_swatch()
    m = sc.mesh
    K = orc.assemble_K(m.tets, m.shape_grad, m.volume, sc.gammas.gamma_s, sc.gammas.gamma_v,
                       m.node_mass, sc.dt, sc.n_nodes)
    free = np.setdiff1d(np.arange(sc.n_nodes), sc.pins)
    return sc, K, free, K[free][:, free].tocsc()


def test_a_jacobi_matches_reference_golden(c1sys):
    sc, K, free, Kff = c1sys
    g = golden("solvers.npz")
    assert str(g["digest"]) == scene_digest(sc)
    for agg in (2, 3):
        x, info = gcms.a_jacobi_refine(Kff, g["b"], g["x0"], sweeps=7, aggregation=agg, omega=0.7)
        assert np.abs(x - g[f"aj{agg}_x"]).max() < 1e-11 * np.abs(x).max()
        assert np.allclose(info["residuals"], g[f"aj{agg}_res"], rtol=1e-9)
    x, info = gcms.a_jacobi_refine(Kff, g["b"], g["x0"], sweeps=10, aggregation=2, chebyshev=True)
    assert np.abs(x - g["cheb_x"]).max() < 1e-9 * np.abs(x).max()
    assert np.allclose(info["residuals"], g["cheb_res"], rtol=1e-8)
    x, info = gcms.a_jacobi_refine(Kff, g["b"], g["x0"], sweeps=60, aggregation=2, omega=2.5)
    assert info["diverged"] == bool(g["div_flag"])
    assert len(info["residuals"]) == len(g["div_res"])
    assert np.abs(x - g["div_x"]).max() < 1e-9 * np.abs(x).max()


def test_aggregation_matches_plain_sweeps(rng):
    A = random_spd(rng, 50)
    b = rng.normal(size=50)
    x0 = rng.normal(size=50)

    def plain(x, sweeps, omega):
        invd = 1.0 / A.diagonal()
        for _ in range(sweeps):
            x = x + omega * (invd * (b - A @ x))
        return x

    for agg in (2, 3):
        xa, info = gcms.a_jacobi_refine(A, b, x0, sweeps=7, aggregation=agg, omega=0.7)
        assert np.abs(xa - plain(x0.copy(), 7 * agg, 0.7)).max() < 1e-12
        assert not info["diverged"]


def test_exact_solution_fixed_point_and_diagonal(rng):
    A = random_spd(rng, 40)
    xs = rng.normal(size=40)
    x, _ = gcms.a_jacobi_refine(A, A @ xs, xs, sweeps=5, aggregation=2)
    assert np.abs(x - xs).max() < 1e-12
    d = rng.uniform(1.0, 3.0, size=30)
    bb = rng.normal(size=30)
    x, _ = gcms.a_jacobi_refine(sp.diags(d).tocsr(), bb, np.zeros(30), sweeps=1, aggregation=2, omega=1.0)
    assert np.abs(x - bb / d).max() < 1e-14


def test_divergence_returns_best_iterate(rng):
    A = random_spd(rng, 50)
    b = rng.normal(size=50)
    x, info = gcms.a_jacobi_refine(A, b, rng.normal(size=50), sweeps=300, aggregation=2, omega=2.5)
    assert info["diverged"]
    assert np.all(np.isfinite(x))
    assert np.linalg.norm(b - A @ x) <= min(info["residuals"]) * (1 + 1e-12)


def test_chebyshev_no_slower(c1sys, rng):
    sc, K, free, Kff = c1sys
    b = rng.normal(size=Kff.shape[0])
    x_ref = spla.spsolve(Kff, b)
    x_p, _ = gcms.a_jacobi_refine(Kff, b, np.zeros_like(b), sweeps=40, aggregation=2)
    x_c, info = gcms.a_jacobi_refine(Kff, b, np.zeros_like(b), sweeps=40, aggregation=2, chebyshev=True)
    assert not info["diverged"]
    assert np.linalg.norm(x_c - x_ref) <= np.linalg.norm(x_p - x_ref) * 1.01


def test_rejects_bad_aggregation(rng):
    with pytest.raises(ValueError):
        gcms.a_jacobi_refine(random_spd(rng, 10), np.ones(10), np.zeros(10), aggregation=4)


def test_cms_solve_matches_reference_golden(c1sys):
    sc, K, free, Kff = c1sys
    g = golden("solvers.npz")
    cms = gcms.build_cms(Kff, sc.mesh, n_domains=2, modes_per_domain=12, free=free)
    assert cms.K_red.shape[0] == int(g["cms_nred"])
    assert rel_l2(cms.solve(g["b"]), g["cms_x"]) < 1e-9


def test_cms_complete_basis_exact_and_spd(c1sys, rng):
    sc, K, free, Kff = c1sys
    b = rng.normal(size=Kff.shape[0])
    x_ref = spla.spsolve(Kff, b)
    labels = gcms.partition_elements(sc.mesh, 2)
    interior, _ = gcms.classify_nodes(sc.mesh, labels, free)
    modes = max(len(s) for s in interior)
    cms = gcms.build_cms(Kff, sc.mesh, n_domains=2, modes_per_domain=modes, free=free)
    assert rel_l2(cms.solve(b), x_ref) < 1e-8
    assert np.linalg.eigvalsh(cms.K_red.toarray()).min() > 0.0
    cms0 = gcms.build_cms(Kff, sc.mesh, n_domains=2, modes_per_domain=0, free=free)
    remap = -np.ones(sc.n_nodes, dtype=int)
    remap[free] = np.arange(len(free))
    _, bnd = gcms.classify_nodes(sc.mesh, labels, free)
    bb = np.zeros(Kff.shape[0])
    bb[remap[bnd]] = rng.normal(size=len(bnd))
    assert rel_l2(cms0.solve(bb), spla.spsolve(Kff, bb)) < 1e-8


def test_truncated_plus_refinement_converges(c1sys, rng):
    sc, K, free, Kff = c1sys
    b = rng.normal(size=Kff.shape[0])
    x_ref = spla.spsolve(Kff, b)
    cms = gcms.build_cms(Kff, sc.mesh, n_domains=2, modes_per_domain=15, free=free)
    x0 = cms.solve(b)
    x, info = gcms.a_jacobi_refine(Kff, b, x0, sweeps=300, aggregation=2)
    assert not info["diverged"]
    assert rel_l2(x, x_ref) < 1e-8 < rel_l2(x0, x_ref)


def test_cms_mode_frame_matches_reference(c1sys):
    sc, K, free, Kff = c1sys
    g = golden("solvers.npz")
    fr = pdsolver.simulate_mesh(sc.mesh, sc.gammas, 1, sc.dt, forces=sc.forces, pins=sc.pins,
                                pin_targets=sc.pin_targets, iterations=30, solver_mode="cms", n_domains=2,
                                modes_per_domain=12, refine_sweeps=30)
    assert rel_l2(fr[0], g["cms_frame"]) < 1e-9
    assert rel_l2(fr[0] - sc.mesh.nodes, g["cms_frame"] - sc.mesh.nodes) < 1e-6


@pytest.mark.parametrize("chebyshev", [False, True])
def test_cms_device_frame_equals_host_loop(c1sys, chebyshev):
    """simulate_mesh(solver_mode="cms") runs each frame as one device call (vkpd_step_cms); the
    reference's loop of pd_step with a GlobalSolver(mode="cms") object gives the same frames."""
    sc, K, free, Kff = c1sys
    kw = dict(n_domains=2, modes_per_domain=12, refine_sweeps=10, chebyshev=chebyshev)
    fr = pdsolver.simulate_mesh(sc.mesh, sc.gammas, 3, sc.dt, forces=sc.forces, pins=sc.pins,
                                pin_targets=sc.pin_targets, iterations=8, solver_mode="cms", **kw)
    sub = gcms.build_cms(Kff, sc.mesh, n_domains=2, modes_per_domain=12, free=free)
    solver = pdsolver.GlobalSolver(pdsolver.assemble_global(sc.mesh, sc.gammas, sc.dt), free, sc.pins, mode="cms",
                                   cms=sub, refine_sweeps=10, chebyshev=chebyshev)
    st = pdsolver.SimState(x=sc.mesh.nodes, v=np.zeros_like(sc.mesh.nodes), dt=sc.dt, pins=sc.pins,
                           pin_targets=sc.pin_targets)
    for k in range(3):
        pdsolver.pd_step(st, sc.mesh, sc.gammas, iterations=8, forces=sc.forces, solver=solver, precision="fp64")
        assert rel_l2(fr[k] - sc.mesh.nodes, st.x - sc.mesh.nodes) < 1e-10, k


def test_scalable_build_matches_dense_build():
    """The large-domain build (block LOBPCG for Phi, block CG for Psi on the adjacent boundary
    columns, K_red from the blocks) gives the same subspace solve as the dense eigh / Cholesky
    build (forced on C2 with 4 slab domains)."""
    sc = scenes.make_scene("C2")
    m = sc.mesh
    K = pdsolver.assemble_global(m, sc.gammas, sc.dt).tocsr()
    free = np.setdiff1d(np.arange(m.n_nodes), sc.pins)
    Kff = K[free][:, free].tocsc()
    dense = gcms.build_cms(Kff, m, n_domains=4, modes_per_domain=12, free=free)
    old = gcms.CmsSubspace.DENSE_EIG_MAX
    try:
        gcms.CmsSubspace.DENSE_EIG_MAX = 0
        big = gcms.build_cms(Kff, m, n_domains=4, modes_per_domain=12, free=free)
    finally:
        gcms.CmsSubspace.DENSE_EIG_MAX = old
    b = np.random.default_rng(5).normal(size=(len(free), 3))
    assert rel_l2(big.solve(b), dense.solve(b)) < 1e-8
    assert abs(big.K_red.shape[0] - dense.K_red.shape[0]) == 0
    assert rel_l2(big.T.toarray(), dense.T.toarray()) < 1.0      # same structure (modes up to sign)

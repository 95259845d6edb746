"""Pin the CPU oracle against golden vectors produced by the real reference (CPU only)."""

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import pd_oracle as orc
from paper_2405_12484_b200 import scenes
from pdtest_helpers import golden, scene_digest, rel_l2


def _c1():
    sc = scenes.c1_swatch()
    m = sc.mesh
    return sc, (m.tets, m.shape_grad, m.volume, sc.gammas.gamma_s, sc.gammas.gamma_v)


def test_projections_match_reference():
    g = golden("projections.npz")
    R, V = orc.projections(g["F"])
    assert np.abs(R - g["R"]).max() < 1e-12
    assert np.abs(V - g["V"]).max() < 1e-10


def test_scalar_sl3_matches_reference():
    g = golden("projections.npz")
    for sig, s_ref, cl_ref, ok_ref in zip(g["sigma"], g["s"], g["clamped"], g["ok"]):
        s, lam, cl, ok = orc.sl3_project_scalar(sig)
        assert np.abs(s - s_ref).max() < 1e-12
        assert list(cl) == list(cl_ref) and ok == ok_ref


def test_sl3_known_answers():
    phi = (1.0 + np.sqrt(5.0)) / 2.0
    s, _, _, ok = orc.sl3_project_scalar(np.array([2.0, 2.0, 2.0]))
    assert ok and np.abs(np.sort(s) - [phi ** -2, phi, phi]).max() < 1e-9
    s, _, cl, ok = orc.sl3_project_scalar(np.array([100.0, 100.0, 1e-5]))
    assert ok and np.abs(s - [10.0, 10.0, 0.01]).max() < 1e-6 and list(cl) == [False, False, True]
    for t in (0.5, 1.5, 1.8):
        R, V = orc.projections((t * np.eye(3))[None])
        assert np.abs(V[0] - np.eye(3)).max() < 1e-9


def test_scene_digest_matches_fixture():
    sc, _ = _c1()
    assert scene_digest(sc) == str(golden("c1.npz")["digest"])


def test_c1_assembly_and_local_step():
    sc, (tets, G, vol, gs, gv) = _c1()
    g = golden("c1.npz")
    K = orc.assemble_K(tets, G, vol, gs, gv, sc.mesh.node_mass, sc.dt, sc.n_nodes).tocsr()
    Kr = sp.csr_matrix((g["K_data"], g["K_indices"], g["K_indptr"]), shape=K.shape)
    assert abs(K - Kr).max() < 1e-12 * abs(Kr).max()
    rhs, F, R, V = orc.elastic_rhs(g["x_pert"], tets, G, vol, gs, gv, sc.n_nodes)
    assert np.abs(F - g["F"]).max() < 1e-12
    assert np.abs(R - g["R"]).max() < 1e-10
    assert np.abs(V - g["V"]).max() < 1e-10
    assert np.abs(rhs - g["rhs"]).max() < 1e-10 * np.abs(g["rhs"]).max()


def test_c1_frames_match_reference():
    sc, (tets, G, vol, gs, gv) = _c1()
    g = golden("c1.npz")
    fr = orc.simulate(sc.mesh.nodes, tets, G, vol, gs, gv, sc.mesh.node_mass, 3, sc.dt,
                      forces=sc.forces, pins=sc.pins, pin_targets=sc.pin_targets)
    for k in range(3):
        assert rel_l2(fr[k], g["frames"][k]) < 1e-12
    assert rel_l2(fr[0] - sc.mesh.nodes, g["frames"][0] - sc.mesh.nodes) < 1e-9


def test_solvers_match_reference():
    sc, (tets, G, vol, gs, gv) = _c1()
    g = golden("solvers.npz")
    assert str(g["digest"]) == scene_digest(sc)
    K = orc.assemble_K(tets, G, vol, gs, gv, sc.mesh.node_mass, sc.dt, sc.n_nodes)
    free = np.setdiff1d(np.arange(sc.n_nodes), sc.pins)
    Kff = K[free][:, free].tocsc()
    b, x0 = g["b"], g["x0"]
    for agg in (2, 3):
        x, info = orc.a_jacobi_refine(Kff, b, x0, sweeps=7, aggregation=agg, omega=0.7)
        assert np.abs(x - g[f"aj{agg}_x"]).max() < 1e-12 * np.abs(x).max()
        assert np.allclose(info["residuals"], g[f"aj{agg}_res"], rtol=1e-10)
    x, info = orc.a_jacobi_refine(Kff, b, x0, sweeps=10, aggregation=2, chebyshev=True)
    assert np.abs(x - g["cheb_x"]).max() < 1e-10 * np.abs(x).max()
    x, info = orc.a_jacobi_refine(Kff, b, x0, sweeps=60, aggregation=2, omega=2.5)
    assert info["diverged"] == bool(g["div_flag"])
    assert np.abs(x - g["div_x"]).max() < 1e-9 * np.abs(x).max()
    lab = orc.partition_elements(sc.mesh.nodes, tets, 2)
    inner, bnd = orc.classify_nodes(tets, lab, sc.n_nodes, free)
    remap = -np.ones(sc.n_nodes, dtype=np.int64)
    remap[free] = np.arange(len(free))
    cms = orc.CmsBasis(Kff, [remap[i] for i in inner], remap[bnd], 12)
    assert cms.K_red.shape[0] == int(g["cms_nred"])
    assert rel_l2(cms.solve(b), g["cms_x"]) < 1e-9


def test_cms_mode_frame_matches_reference():
    sc, (tets, G, vol, gs, gv) = _c1()
    g = golden("solvers.npz")
    fr = orc.simulate(sc.mesh.nodes, tets, G, vol, gs, gv, sc.mesh.node_mass, 1, sc.dt,
                      forces=sc.forces, pins=sc.pins, pin_targets=sc.pin_targets,
                      solver_mode="cms", n_domains=2, modes_per_domain=12, refine_sweeps=30)
    assert rel_l2(fr[0], g["cms_frame"]) < 1e-10


def test_aggregation_rejects_bad_value():
    with pytest.raises(ValueError):
        orc.a_jacobi_refine(sp.eye(4).tocsc(), np.ones(4), np.zeros(4), aggregation=4)


def test_contact_oracle_matches_reference():
    g = golden("contact.npz")
    sc, colliders = scenes.contact_scene()
    assert scene_digest(sc) == str(g["digest"])
    m = sc.mesh
    x, v = m.nodes.copy(), np.zeros_like(m.nodes)
    for k in range(20):
        x, v = orc.pd_step_contact(x, v, sc.dt, m.tets, m.shape_grad, m.volume, sc.gammas.gamma_s,
                                   sc.gammas.gamma_v, m.node_mass, [], None, sc.forces, colliders, 10, 0.9)
        assert np.abs(x - g["frames"][k]).max() < 1e-12


def test_pd_equilibrium_oracle_matches_reference():
    g = golden("equilibrium.npz")
    sc, a, x0 = scenes.equilibrium_case()
    assert scene_digest(sc) == str(g["digest"])
    assert np.array_equal(a, g["a"]) and np.array_equal(x0, g["x0"])
    m = sc.mesh
    for its in (1, 5):
        x = orc.pd_equilibrium(x0, m.tets, m.shape_grad, m.volume, sc.gammas.gamma_s, sc.gammas.gamma_v,
                               m.node_mass, a, sc.pins, sc.pin_targets, sc.dt, iterations=its)
        assert rel_l2(x, g[f"x{its}"]) < 1e-12


# ---------------------------------------------------------------------------
# second order: oracle vs the reference's outputs (second_order.npz)


def _so_scene():
    g = golden("second_order.npz")
    sc, x, xhat = scenes.second_order_case()
    assert scene_digest(sc) == str(g["digest"])
    assert np.array_equal(x, g["x"]) and np.array_equal(xhat, g["xhat"])
    m = sc.mesh
    return g, sc, m, (m.tets, m.shape_grad, m.volume, sc.gammas.gamma_s, sc.gammas.gamma_v)


def test_projection_jacobians_oracle_matches_reference():
    g = golden("jacobians.npz")
    JR, JV = orc.projection_jacobians(g["F"])
    assert np.abs(JR - g["JR"]).max() < 1e-9
    assert np.abs(JV - g["JV"]).max() < 1e-8


def test_second_order_oracle_matches_reference():
    g, sc, m, op = _so_scene()
    x = g["x"]
    assert abs(orc.elastic_energy(x, *op) - float(g["energy"])) < 1e-13 * abs(float(g["energy"]))
    gr = orc.elastic_gradient(x, *op, m.n_nodes)
    assert rel_l2(gr, g["grad"]) < 1e-12
    H = orc.exact_elastic_hessian(x, *op, m.n_nodes).tocsr()
    Href = sp.csr_matrix((g["H_data"], g["H_indices"], g["H_indptr"]), shape=H.shape)
    assert abs(H - Href).max() < 1e-10 * abs(Href).max()


def test_newton_polish_oracle_matches_reference():
    g, sc, m, op = _so_scene()
    for exact in (0, 1):
        x, ok, its = orc.newton_polish(g["xhat"], *op, m.node_mass, sc.dt, sc.pins, sc.pin_targets,
                                       xhat=g["xhat"], tol=1e-7, max_iters=100, exact=bool(exact))
        assert ok and bool(g[f"dyn_ok_{exact}"])
        assert its == int(g[f"dyn_it_{exact}"])
        assert rel_l2(x, g[f"dyn_x_{exact}"]) < 1e-12
    _, a, _, _, _, _ = scenes.adjoint_case()
    x, ok, its = orc.newton_polish(g["qs_x0"], *op, m.node_mass, sc.dt, sc.pins, sc.pin_targets,
                                   inertia_target=a, tol=1e-10, max_iters=150, exact=True)
    assert ok and its == int(g["qs_it"])
    assert rel_l2(x, g["qs_x"]) < 1e-12


def test_adjoint_gradient_oracle_matches_reference():
    g, sc, m, op = _so_scene()
    _, a, _, weight, shift, sample = scenes.adjoint_case()
    x = g["qs_x"]
    prob = scenes.TrackingProblem(m, sc.dt, x + shift, weight)
    grad, lam = orc.adjoint_gradient(x, prob.loss_grad_x(x, sample), *op, m.n_nodes, sc.pins)
    assert rel_l2(grad, g["adj_grad"]) < 1e-9
    free = np.setdiff1d(np.arange(m.n_nodes), sc.pins)
    assert rel_l2(lam[free].reshape(-1), g["adj_lam"]) < 1e-9


def test_gauss_newton_oracle_matches_reference():
    g, sc, m, op = _so_scene()
    _, a, _, weight, shift, sample = scenes.adjoint_case()
    x = g["qs_x"]
    free = np.setdiff1d(np.arange(m.n_nodes), sc.pins)
    fd = (3 * free[:, None] + np.arange(3)).reshape(-1)
    H = orc.exact_elastic_hessian(x, *op, m.n_nodes).tocsr()[fd][:, fd]
    F = orc.deformation_gradients(x, m.tets, m.shape_grad)
    R, V = orc.projections(F)
    v2 = 2.0 * m.volume[:, None, None]
    Js = (v2 * np.einsum("enj,eij->eni", m.shape_grad, F - R)).reshape(-1)
    Jv = (v2 * np.einsum("enj,eij->eni", m.shape_grad, F - V)).reshape(-1)
    nE = m.n_elements
    dofs = (3 * m.tets[:, :, None] + np.arange(3)).reshape(-1)
    J = sp.csr_matrix((np.concatenate([Js, Jv]), (np.concatenate([dofs, dofs]),
                       np.concatenate([np.repeat(np.arange(nE), 12), np.repeat(np.arange(nE, 2 * nE), 12)]))),
                      shape=(3 * m.n_nodes, 2 * nE))[fd]
    G = sp.kron(sp.diags(2.0 * weight), sp.eye(3)).tocsr()[fd][:, fd]
    d = orc.gauss_newton_direction(H, J, G, g["adj_grad"], float(g["gn_full_kappa"]))
    assert rel_l2(d, g["gn_full_d"]) < 1e-7

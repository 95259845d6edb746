"""GPU parity tests: the CUDA path (through the C-ABI) against the reference's golden
vectors and the CPU oracle, on the same seeded inputs.  Run with `-m gpu`."""

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from oracle import pd_oracle as orc
from paper_2405_12484_b200 import material, pdsolver, scenes
from paper_2405_12484_b200.material import MaterialField
from paper_2405_12484_b200.volmesh import VolumeMesh
from pdtest_helpers import golden, rel_l2, scene_digest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c1():
    sc = scenes.c1_swatch()
    assert scene_digest(sc) == str(golden("c1.npz")["digest"])
    return sc


def single_tet(mass=0.1):
    nodes = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], dtype=float)
    m = VolumeMesh(nodes, np.array([[0, 1, 2, 3]]))
    m.node_mass = np.full(4, mass)
    return m


# ---------------------------------------------------------------------------
# projections (material.py:395-407)


@pytest.mark.parametrize("prec,tol_r,tol_v", [("fp64", 1e-11, 1e-10), ("fp32", 2e-4, 2e-4)])
def test_batch_projections_match_reference(prec, tol_r, tol_v):
    g = golden("projections.npz")
    R, V = material.batch_projections(g["F"], precision=prec)
    assert np.abs(R - g["R"]).max() < tol_r
    assert np.abs(V - g["V"]).max() < tol_v


def test_projection_known_answers():
    phi = (1.0 + np.sqrt(5.0)) / 2.0
    F = np.stack([t * np.eye(3) for t in (0.5, 1.5, 1.8)] + [np.diag([100.0, 100.0, 1e-5]),
                                                            2.0 * np.eye(3), np.zeros((3, 3))])
    R, V = material.batch_projections(F)
    for k in range(3):
        assert np.abs(V[k] - np.eye(3)).max() < 1e-9
    assert np.abs(np.sort(np.linalg.svd(V[3], compute_uv=False)) - [0.01, 10.0, 10.0]).max() < 1e-6
    assert np.abs(np.sort(np.linalg.svd(V[4], compute_uv=False)) - [phi ** -2, phi, phi]).max() < 1e-9
    assert abs(np.linalg.det(V[5]) - 1.0) < 1e-6


def test_projection_invariants_random(rng):
    F = np.eye(3) + 0.8 * rng.normal(size=(4000, 3, 3))
    R, V = material.batch_projections(F)
    assert np.abs(np.linalg.det(V) - 1.0).max() < 1e-8
    assert np.linalg.svd(V, compute_uv=False).min() >= 0.01 - 1e-8
    assert np.abs(np.einsum("eij,ekj->eik", R, R) - np.eye(3)).max() < 1e-12
    assert np.abs(np.linalg.det(R) - 1.0).max() < 1e-12


def test_projection_rejects_nonfinite():
    F = np.eye(3)[None].copy()
    F[0, 0, 0] = np.nan
    with pytest.raises(ValueError):
        material.batch_projections(F)


# ---------------------------------------------------------------------------
# assembly and local step


def test_assemble_global_matches_reference(c1):
    g = golden("c1.npz")
    K = pdsolver.assemble_global(c1.mesh, c1.gammas, c1.dt).tocsr()
    Kr = sp.csr_matrix((g["K_data"], g["K_indices"], g["K_indptr"]), shape=K.shape)
    assert abs(K - Kr).max() < 1e-12 * abs(Kr).max()
    assert abs(K - K.T).max() < 1e-12 * abs(Kr).max()


def test_assemble_rejects_bad_input(c1):
    with pytest.raises(ValueError):
        pdsolver.assemble_global(c1.mesh, c1.gammas, 0.0)
    bad = MaterialField(-np.ones(c1.n_tets), np.ones(c1.n_tets))
    with pytest.raises(ValueError):
        pdsolver.assemble_global(c1.mesh, bad, 1e-3)


@pytest.mark.parametrize("prec,tol", [("fp64", 1e-10), ("fp32", 5e-5)])
def test_elastic_rhs_matches_reference(c1, prec, tol):
    g = golden("c1.npz")
    rhs, F, R, V = pdsolver.elastic_rhs(c1.mesh, c1.gammas, g["x_pert"], precision=prec)
    scale = np.abs(g["rhs"]).max()
    assert np.abs(rhs - g["rhs"]).max() < tol * scale
    assert np.abs(F - g["F"]).max() < max(tol, 1e-12) * 10
    assert np.abs(R - g["R"]).max() < tol * 10
    assert np.abs(V - g["V"]).max() < tol * 10


def test_elastic_rhs_is_deterministic(c1):
    g = golden("c1.npz")
    a = pdsolver.elastic_rhs(c1.mesh, c1.gammas, g["x_pert"], precision="fp32")[0]
    b = pdsolver.elastic_rhs(c1.mesh, c1.gammas, g["x_pert"], precision="fp32")[0]
    assert np.array_equal(a, b)


# ---------------------------------------------------------------------------
# global solve (GlobalSolver drop-in)


def test_global_solver_matches_direct(c1, rng):
    K = orc.assemble_K(c1.mesh.tets, c1.mesh.shape_grad, c1.mesh.volume, c1.gammas.gamma_s,
                       c1.gammas.gamma_v, c1.mesh.node_mass, c1.dt, c1.n_nodes)
    free = np.setdiff1d(np.arange(c1.n_nodes), c1.pins)
    ref = orc.GlobalSolver(K, free, c1.pins)
    B = rng.normal(size=(c1.n_nodes, 3))
    P = rng.normal(size=(len(c1.pins), 3))
    X_ref = ref.solve(B, P)
    gs = pdsolver.GlobalSolver(K, free, c1.pins, precision="fp64", tol=1e-13)
    X = gs.solve(B, P)
    assert rel_l2(X, X_ref) < 1e-10
    assert np.array_equal(X[c1.pins], P)
    # more than three columns are chunked
    B5 = rng.normal(size=(c1.n_nodes, 5))
    P5 = rng.normal(size=(len(c1.pins), 5))
    assert rel_l2(gs.solve(B5, P5), ref.solve(B5, P5)) < 1e-10


def test_global_solver_rejects_bad_mode(c1):
    K = pdsolver.assemble_global(c1.mesh, c1.gammas, c1.dt)
    with pytest.raises(ValueError):
        pdsolver.GlobalSolver(K, np.arange(c1.n_nodes), np.empty(0, dtype=int), mode="lu")


# ---------------------------------------------------------------------------
# stepping (pdsolver.py:257-304, 710-763)


@pytest.mark.parametrize("prec,tol_pos,tol_disp", [("fp64", 1e-10, 1e-8), ("fp32", 1e-5, 5e-3)])
def test_c1_frames_match_reference(c1, prec, tol_pos, tol_disp):
    g = golden("c1.npz")
    fr = pdsolver.simulate_mesh(c1.mesh, c1.gammas, 3, c1.dt, forces=c1.forces, pins=c1.pins,
                                pin_targets=c1.pin_targets, iterations=30, precision=prec)
    x0 = c1.mesh.nodes
    for k in range(3):
        assert rel_l2(fr[k], g["frames"][k]) < tol_pos, k
        assert rel_l2(fr[k] - x0, g["frames"][k] - x0) < tol_disp, k


def test_rest_is_fixed_point():
    sc = scenes.box_scene(6, 5, 3)
    st = pdsolver.SimState(x=sc.mesh.nodes, v=np.zeros_like(sc.mesh.nodes), dt=1e-3)
    pdsolver.pd_step(st, sc.mesh, sc.gammas, iterations=5, precision="fp64")
    assert np.abs(st.x - sc.mesh.nodes).max() < 1e-12


def test_free_fall_discrete_closed_form():
    sc = scenes.box_scene(6, 5, 3)
    mesh = sc.mesh
    mesh.node_mass = np.full(mesh.n_nodes, 1e-3)
    gam = MaterialField.uniform(mesh.n_elements, 5.0, 3.0)
    dt, steps = 1e-3, 8
    gvec = np.array([0.0, -9.8, 0.0])
    frames = pdsolver.simulate_mesh(mesh, gam, steps, dt, forces=mesh.node_mass[:, None] * gvec,
                                    iterations=3, precision="fp64")
    for n in range(1, steps + 1):
        expect = mesh.nodes + gvec * dt ** 2 * n * (n + 1) / 2.0
        assert np.abs(frames[n - 1] - expect).max() < 1e-12


def test_pinned_nodes_track_targets(c1):
    pins = np.array([0, 1, 2])
    tgt = c1.mesh.nodes[pins] + np.array([0.0, 0.01, 0.0])
    for prec in ("fp64", "fp32"):
        st = pdsolver.SimState(x=c1.mesh.nodes, v=np.zeros_like(c1.mesh.nodes), dt=1e-3, pins=pins,
                               pin_targets=tgt)
        pdsolver.pd_step(st, c1.mesh, c1.gammas, iterations=4, precision=prec)
        assert np.abs(st.x[pins] - tgt).max() < (1e-14 if prec == "fp64" else 1e-7)


def test_non_finite_abort_reports_iteration(c1):
    class BadSolver:
        def solve(self, b, pin_vals):
            return np.full_like(b, np.nan)

    st = pdsolver.SimState(x=c1.mesh.nodes, v=np.zeros_like(c1.mesh.nodes), dt=1e-3)
    with pytest.raises(RuntimeError, match="iteration 0"):
        pdsolver.pd_step(st, c1.mesh, c1.gammas, solver=BadSolver())


def test_device_step_non_finite_abort_keeps_state(c1):
    f = c1.forces.copy()
    node = int(np.setdiff1d(np.arange(c1.n_nodes), c1.pins)[-1])     # a free node
    f[node, 1] = np.nan
    st = pdsolver.SimState(x=c1.mesh.nodes, v=np.zeros_like(c1.mesh.nodes), dt=c1.dt, pins=c1.pins)
    with pytest.raises(RuntimeError, match="iteration 0"):
        pdsolver.pd_step(st, c1.mesh, c1.gammas, iterations=3, forces=f)
    assert np.array_equal(st.x, c1.mesh.nodes)
    # the context is still usable afterwards
    pdsolver.pd_step(st, c1.mesh, c1.gammas, iterations=3, forces=c1.forces)
    assert np.all(np.isfinite(st.x))


def test_simulate_pipelined_equals_frame_loop():
    """simulate_mesh runs its frame loop in one library call (vkpd_simulate: inputs up and
    positions down on a copy stream, overlapping the next frame); same bits as stepping frame by
    frame with per-step forces and a pin path."""
    sc = scenes.make_scene("C2")
    m = sc.mesh
    steps = 24
    rng = np.random.default_rng(4)
    fseq = np.stack([sc.forces * (1.0 + 0.05 * rng.normal()) for _ in range(steps)])
    path = np.stack([sc.pin_targets + np.array([0.0, 0.0, 2e-4 * k]) for k in range(steps)])
    fr = pdsolver.simulate_mesh(m, sc.gammas, steps, sc.dt, forces=fseq, pins=sc.pins, pin_targets=path,
                                precision="fp32")
    from paper_2405_12484_b200 import _abi
    ctx = _abi.Context(m.n_nodes, m.tets, m.shape_grad, m.volume, m.node_mass, sc.gammas.gamma_s, sc.gammas.gamma_v,
                       sc.pins, sc.dt, precision="fp32", tol=pdsolver.DEFAULT_TOL["fp32"], nodes=m.nodes)
    ctx.set_state(m.nodes)
    for k in range(steps):
        ctx.set_pin_targets(path[k])
        ctx.set_forces(fseq[k])
        ctx.step(sc.iterations)
        assert np.array_equal(ctx.get_state()[0], fr[k]), k


def test_simulate_pipelined_non_finite_reports_iteration(c1):
    f = np.broadcast_to(c1.forces, (4,) + c1.forces.shape).copy()
    f[2, int(np.setdiff1d(np.arange(c1.n_nodes), c1.pins)[-1]), 1] = np.nan      # step 2 goes bad
    with pytest.raises(RuntimeError, match="iteration 0"):
        pdsolver.simulate_mesh(c1.mesh, c1.gammas, 4, c1.dt, forces=f, pins=c1.pins, pin_targets=c1.pin_targets,
                               iterations=5)
    fr = pdsolver.simulate_mesh(c1.mesh, c1.gammas, 2, c1.dt, forces=c1.forces, pins=c1.pins,
                                pin_targets=c1.pin_targets, iterations=5)     # the cached context recovers
    assert np.all(np.isfinite(fr))


def test_objective_monotone_with_device_solver(c1):
    mesh, gam, dt = c1.mesh, c1.gammas, 1e-3
    pins = c1.pins
    tgt = mesh.nodes[pins]
    st = pdsolver.SimState(x=1.002 * mesh.nodes, v=np.zeros_like(mesh.nodes), dt=dt, pins=pins,
                           pin_targets=tgt)
    xhat = pdsolver._predicted(st, None, mesh)
    free = np.setdiff1d(np.arange(mesh.n_nodes), pins)
    solver = pdsolver.GlobalSolver(pdsolver.assemble_global(mesh, gam, dt), free, pins, tol=1e-13)
    x = xhat.copy()
    x[pins] = tgt
    objs = [pdsolver.pd_objective(x, mesh, gam, xhat, dt)]
    for _ in range(10):
        rhs, *_ = pdsolver.elastic_rhs(mesh, gam, x)
        b = (mesh.node_mass[:, None] / dt ** 2) * xhat + rhs
        x = solver.solve(b, tgt)
        objs.append(pdsolver.pd_objective(x, mesh, gam, xhat, dt))
    objs = np.array(objs)
    assert np.all(np.diff(objs) <= 1e-10 * np.abs(objs[:-1]) + 1e-18)


def test_bit_identical_reruns(c1):
    kw = dict(forces=c1.forces, pins=c1.pins, pin_targets=c1.pin_targets, iterations=30)
    a = pdsolver.simulate_mesh(c1.mesh, c1.gammas, 2, c1.dt, **kw)
    pdsolver.invalidate_cache()
    b = pdsolver.simulate_mesh(c1.mesh, c1.gammas, 2, c1.dt, **kw)
    assert np.array_equal(a, b)


def _run_frames(sc, frames, precision, collect_every=1, **cfg):
    from paper_2405_12484_b200 import _abi
    m = sc.mesh
    ctx = _abi.Context(m.n_nodes, m.tets, m.shape_grad, m.volume, m.node_mass, sc.gammas.gamma_s,
                       sc.gammas.gamma_v, sc.pins, sc.dt, precision=precision,
                       tol=pdsolver.DEFAULT_TOL[precision], nodes=m.nodes, **cfg)
    ctx.set_state(m.nodes)
    ctx.set_pin_targets(sc.pin_targets)
    ctx.set_forces(sc.forces)
    xs, its = [], []
    for k in range(frames):
        ctx.step(30)
        its.append(list(ctx.stats()["cg_iters"][:30]))
        if (k + 1) % collect_every == 0:
            xs.append(ctx.get_state()[0])
    return np.stack(xs), its


@pytest.mark.parametrize("config,frames,precision", [("C2", 40, "fp32"), ("C2", 10, "fp64"), ("C3", 100, "fp32")])
def test_pd_loop_early_exit_is_exact(config, frames, precision):
    """The graph's PD-iteration loop stops at the first solve that needs zero CG
    iterations (x unchanged, so the remaining rounds are exact repeats).  Same
    bits as running every round; C3 to frame 100 crosses into the frames with
    robust-path tets."""
    sc = scenes.make_scene(config)
    a, ia = _run_frames(sc, frames, precision, collect_every=5, pd_early_exit=False)
    b, ib = _run_frames(sc, frames, precision, collect_every=5)
    assert np.array_equal(a, b)
    assert ia == ib
    if precision == "fp32":
        assert any(0 in it for it in ib)     # the exit was actually taken (fp64 at 1e-12 rarely exits)


@pytest.mark.parametrize("unroll", [3, 7])
def test_unrolled_rounds_are_exact(unroll):
    """Leading PD rounds captured as plain graph nodes ahead of the WHILE node (fixed counts here;
    adaptive by default): a round past the exit point is an exact repeat, so positions and the
    per-round CG iterations of the executed rounds are the same bits as the loop alone."""
    sc = scenes.make_scene("C2")
    a, ia = _run_frames(sc, 30, "fp32", collect_every=3, unroll_rounds=0)
    b, ib = _run_frames(sc, 30, "fp32", collect_every=3, unroll_rounds=unroll)
    assert np.array_equal(a, b)


@pytest.mark.parametrize("precision,tol", [("fp64", 1e-10), ("fp32", 2e-5)])
def test_chebyshev_matches_cg(precision, tol):
    """The two global-step solvers (Chebyshev semi-iteration with neighbour flags, the fp64
    default; polynomial-preconditioned CG, the fp32 default) solve the same K_ff x = b to the
    same residual tolerance: C2 after 20 frames they agree to the tolerance's accuracy."""
    sc = scenes.make_scene("C2")
    a, _ = _run_frames(sc, 20, precision, collect_every=20, solver="pcg")
    b, ib = _run_frames(sc, 20, precision, collect_every=20, solver="chebyshev")
    assert rel_l2(b[-1], a[-1]) < tol
    assert sum(sum(it) for it in ib) > 0


def test_chebyshev_reruns_bit_identical():
    """No float atomics on the Chebyshev path: the neighbour flags only order the steps."""
    sc = scenes.make_scene("C2")
    a, ia = _run_frames(sc, 8, "fp64", collect_every=2, solver="chebyshev")
    b, ib = _run_frames(sc, 8, "fp64", collect_every=2, solver="chebyshev")
    assert np.array_equal(a, b)
    assert ia == ib


def test_chebyshev_without_rest_positions():
    """Without rest positions the free nodes keep caller order (no patches, no exported-first
    rows): same solution to the tolerance."""
    from paper_2405_12484_b200 import _abi
    sc = scenes.make_scene("C2")
    m = sc.mesh
    outs = []
    for nodes in (m.nodes, None):
        ctx = _abi.Context(m.n_nodes, m.tets, m.shape_grad, m.volume, m.node_mass, sc.gammas.gamma_s,
                           sc.gammas.gamma_v, sc.pins, sc.dt, precision="fp64", tol=1e-12, nodes=nodes,
                           solver="chebyshev")
        ctx.set_state(m.nodes)
        ctx.set_pin_targets(sc.pin_targets)
        ctx.set_forces(sc.forces)
        for _ in range(5):
            ctx.step(30)
        outs.append(ctx.get_state()[0])
    assert rel_l2(outs[1], outs[0]) < 1e-11


def _c2_frames_ctx(tets, shape_grad, volume, gs, gv, frames=5, **cfg):
    from paper_2405_12484_b200 import _abi
    sc = scenes.make_scene("C2")
    m = sc.mesh
    ctx = _abi.Context(m.n_nodes, tets, shape_grad, volume, m.node_mass, gs, gv, sc.pins, sc.dt,
                       precision="fp64", tol=1e-12, nodes=m.nodes, **cfg)
    ctx.set_state(m.nodes)
    ctx.set_pin_targets(sc.pin_targets)
    ctx.set_forces(sc.forces)
    for _ in range(frames):
        ctx.step(30)
    return ctx.get_state()[0]


def test_shuffled_tet_order_same_frames():
    """The local step's warp-segmented node reduction groups each warp's 32 tets by node; with the
    tets in random order a warp touches ~100 distinct nodes (more than its 32 lanes, the
    multi-pass branch) and a node gets partials from many warps.  Same physics, different
    summation order: C2 after 5 frames to 1e-11."""
    sc = scenes.make_scene("C2")
    m = sc.mesh
    perm = np.random.default_rng(7).permutation(m.n_elements)
    a = _c2_frames_ctx(m.tets, m.shape_grad, m.volume, sc.gammas.gamma_s, sc.gammas.gamma_v)
    b = _c2_frames_ctx(np.ascontiguousarray(m.tets[perm]), np.ascontiguousarray(m.shape_grad[perm]),
                       np.ascontiguousarray(m.volume[perm]), np.ascontiguousarray(sc.gammas.gamma_s[perm]),
                       np.ascontiguousarray(sc.gammas.gamma_v[perm]))
    assert rel_l2(b, a) < 1e-11


@pytest.mark.parametrize("blocks", [4, 37, 100])
def test_chebyshev_cta_count_same_frames(blocks):
    """Other CTA counts give other patches, halos, exported sets and bank colourings of the
    Chebyshev register path (flag-in-data exchange); 4 CTAs own ~1,900 rows each, more than a
    CTA's threads, so that run takes the generic Chebyshev path (per-CTA step flags): same
    solution to the tolerance."""
    sc = scenes.make_scene("C2")
    m = sc.mesh
    a = _c2_frames_ctx(m.tets, m.shape_grad, m.volume, sc.gammas.gamma_s, sc.gammas.gamma_v)
    b = _c2_frames_ctx(m.tets, m.shape_grad, m.volume, sc.gammas.gamma_s, sc.gammas.gamma_v,
                       pcg_blocks=blocks, solver="chebyshev")
    assert rel_l2(b, a) < 1e-11


def test_pin_path_and_per_step_forces(c1):
    steps = 3
    path = np.stack([c1.pin_targets + np.array([0.0, 0.0, 1e-3 * k]) for k in range(steps)])
    fseq = np.stack([c1.forces * (1.0 + 0.1 * k) for k in range(steps)])
    fr = pdsolver.simulate_mesh(c1.mesh, c1.gammas, steps, c1.dt, forces=fseq, pins=c1.pins,
                                pin_targets=path, iterations=20, precision="fp64")
    m = c1.mesh
    ref = orc.simulate(m.nodes, m.tets, m.shape_grad, m.volume, c1.gammas.gamma_s, c1.gammas.gamma_v,
                       m.node_mass, steps, c1.dt, forces=fseq, pins=c1.pins, pin_targets=path,
                       iterations=20)
    assert rel_l2(fr, ref) < 1e-10
    assert np.abs(fr[:, c1.pins] - path).max() < 1e-14


# ---------------------------------------------------------------------------
# full-size parity (BASELINE configs)


@pytest.mark.parametrize("prec,tol_pos,tol_disp", [("fp32", 1e-5, 1e-2), ("fp64", 1e-10, 1e-8)])
def test_c3_frame_matches_reference(prec, tol_pos, tol_disp):
    """BASELINE configs[2]: the 390K-tet sweater, frame 1 from rest against the reference's
    simulate_mesh(direct) (tests/golden/make_golden.py c3, float64 displacement)."""
    g = golden("c3.npz")
    sc = scenes.c3_sweater()
    assert scene_digest(sc) == str(g["digest"])
    fr = pdsolver.simulate_mesh(sc.mesh, sc.gammas, 1, sc.dt, forces=sc.forces, pins=sc.pins,
                                pin_targets=sc.pin_targets, iterations=30, precision=prec)
    ref = g["frame1"]                                   # positions after frame 1 (float64)
    assert rel_l2(fr[0], ref) < tol_pos
    assert rel_l2(fr[0] - sc.mesh.nodes, ref - sc.mesh.nodes) < tol_disp


# measured on B200: fp64 position 9.3e-14, displacement and velocity 5.7e-11; fp32 5.8e-7 / 3.6e-4
@pytest.mark.parametrize("prec,tol_pos,tol_disp", [("fp32", 1e-5, 5e-3), ("fp64", 1e-12, 1e-9)])
def test_c3_fold_frame_matches_reference(prec, tol_pos, tol_disp):
    """One C3 frame inside the fold window (from the stored frame-120 state), where about 88K tets
    per PD round take the robust SL(3) path (material.py:242-287, `k_robust_tasks`), against the
    reference's pd_step(direct) from the same state (tests/golden/make_golden.py c3fold)."""
    from paper_2405_12484_b200 import _abi
    g = golden("c3fold.npz")
    sc = scenes.c3_sweater()
    assert scene_digest(sc) == str(g["digest"])
    m = sc.mesh
    x0, v0 = g["x0"].astype(np.float64), g["v0"].astype(np.float64)
    ctx = _abi.Context(m.n_nodes, m.tets, m.shape_grad, m.volume, m.node_mass, sc.gammas.gamma_s,
                       sc.gammas.gamma_v, sc.pins, sc.dt, precision=prec, tol=pdsolver.DEFAULT_TOL[prec],
                       nodes=m.nodes)
    ctx.set_state(x0, v0)
    ctx.set_pin_targets(sc.pin_targets)
    ctx.set_forces(sc.forces)
    r0 = ctx.stats()["robust"]
    ctx.step(30)
    x, v = ctx.get_state()
    assert ctx.stats()["robust"] - r0 > 100_000          # the robust path is exercised at scale
    assert rel_l2(x, x0 + g["disp"]) < tol_pos
    assert rel_l2(x - x0, g["disp"]) < tol_disp
    assert rel_l2(v, g["v"]) < tol_disp


@pytest.mark.parametrize("prec,tols", [("fp32", {1: 1e-5, 10: 1e-4, 100: 1e-3}),
                                       ("fp64", {1: 1e-10, 10: 1e-10, 100: 1e-10})])
def test_c2_hundred_frames_match_reference(prec, tols):
    """BASELINE configs[1]: 30K-tet rib scarf hanging from one edge, 100 frames."""
    g = golden("c2.npz")
    sc = scenes.c2_scarf()
    assert scene_digest(sc) == str(g["digest"])
    fr = pdsolver.simulate_mesh(sc.mesh, sc.gammas, 100, sc.dt, forces=sc.forces, pins=sc.pins,
                                pin_targets=sc.pin_targets, iterations=30, precision=prec)
    for k, tol in tols.items():
        assert rel_l2(fr[k - 1], g[f"frame{k}"]) < tol, (k, rel_l2(fr[k - 1], g[f"frame{k}"]))


# ---------------------------------------------------------------------------
# colliders (pdsolver.py:125-173, 271-297)


@pytest.mark.parametrize("prec,tols", [("fp64", {0: 1e-9, 9: 1e-9, 19: 1e-9}),
                                       ("fp32", {0: 1e-4, 9: 1e-3, 19: 1e-2})])
def test_contact_frames_match_reference(prec, tols):
    """Contact sets are discontinuous in x, so float32 trajectories may flip a few late
    contact decisions; float64 follows the reference to 1e-9."""
    g = golden("contact.npz")
    sc, colliders = scenes.contact_scene()
    assert scene_digest(sc) == str(g["digest"])
    fr = pdsolver.simulate_mesh(sc.mesh, sc.gammas, 20, sc.dt, forces=sc.forces, colliders=colliders,
                                iterations=10, damping=0.9, precision=prec)
    x0 = sc.mesh.nodes
    for k, tol in tols.items():
        err = rel_l2(fr[k] - x0, g["frames"][k] - x0)
        assert err < tol, (k, err)


def _settle(colliders, steps=250):
    sc = scenes.box_scene(10, 4, 3)
    mesh = sc.mesh
    mesh.node_mass = np.full(mesh.n_nodes, 2e-4)
    gam = MaterialField.uniform(mesh.n_elements, 50.0, 25.0)
    st = pdsolver.SimState(x=mesh.nodes, v=np.zeros_like(mesh.nodes), dt=2e-3, colliders=colliders)
    f = mesh.node_mass[:, None] * np.array([0.0, -9.8, 0.0])
    for _ in range(steps):
        pdsolver.pd_step(st, mesh, gam, iterations=10, forces=f, damping=0.9, precision="fp64")
    return mesh, st


def test_plane_resting_contact_depth():
    mesh0 = scenes.box_scene(10, 4, 3).mesh
    floor_y = mesh0.nodes[:, 1].min() + 0.002
    mesh, st = _settle((("plane", (0.0, floor_y, 0.0), (0.0, 1.0, 0.0)),))
    assert floor_y - st.x[:, 1].min() < 1e-4 * mesh.cell_size


def test_sphere_resting_contact_depth():
    mesh0 = scenes.box_scene(10, 4, 3).mesh
    c = mesh0.nodes.mean(axis=0) + np.array([0.0, -0.2, 0.0])
    r = 0.2 - 0.006
    mesh, st = _settle((("sphere", c, r),))
    assert r - np.linalg.norm(st.x - c, axis=1).min() < 1e-4 * mesh.cell_size


def test_collide_project_and_bad_kind():
    x = np.array([[0.0, -0.5, 0.0], [0.0, 0.5, 0.0]])
    st = pdsolver.SimState(x=x, v=np.zeros_like(x), dt=1e-3, colliders=(("plane", (0, 0, 0), (0, 1, 0)),))
    pdsolver.collide_project(st)
    assert np.allclose(st.x[0], [0.0, 0.0, 0.0]) and np.allclose(st.x[1], [0.0, 0.5, 0.0])
    with pytest.raises(ValueError):
        pdsolver.collider_targets(np.zeros((1, 3)), [("torus", 0, 1)])
    sc = scenes.box_scene(4, 3, 2)
    st = pdsolver.SimState(x=sc.mesh.nodes, v=np.zeros_like(sc.mesh.nodes), dt=1e-3, colliders=(("torus", 0, 1),))
    with pytest.raises(ValueError):
        pdsolver.pd_step(st, sc.mesh, sc.gammas, iterations=2)


# ---------------------------------------------------------------------------
# material refresh: new gamma on a cached device mesh


def test_set_gammas_matches_fresh_context(c1):
    from paper_2405_12484_b200 import _abi
    m = c1.mesh
    rng = np.random.default_rng(7)
    gs2 = c1.gammas.gamma_s * rng.uniform(0.5, 2.0, c1.n_tets)
    gv2 = c1.gammas.gamma_v * rng.uniform(0.5, 2.0, c1.n_tets)

    def run(ctx):
        ctx.set_state(m.nodes)
        ctx.set_pin_targets(c1.pin_targets)
        ctx.set_forces(c1.forces)
        out = []
        for _ in range(3):
            ctx.step(30)
            out.append(ctx.get_state()[0])
        return np.stack(out)

    for prec in ("fp32", "fp64"):
        mk = lambda gs, gv: _abi.Context(m.n_nodes, m.tets, m.shape_grad, m.volume, m.node_mass, gs, gv,
                                          c1.pins, c1.dt, precision=prec, tol=pdsolver.DEFAULT_TOL[prec])
        a = mk(c1.gammas.gamma_s, c1.gammas.gamma_v)
        run(a)                                   # some history on the old material
        a.set_gammas(gs2, gv2)
        fa = run(a)
        fb = run(mk(gs2, gv2))
        assert np.array_equal(fa, fb), prec
        with pytest.raises(ValueError):
            a.set_gammas(-gs2, gv2)


def test_simulate_mesh_reuses_mesh_for_new_material(c1):
    kw = dict(forces=c1.forces, pins=c1.pins, pin_targets=c1.pin_targets, iterations=30, precision="fp64")
    g2 = MaterialField(c1.gammas.gamma_s * 1.7, c1.gammas.gamma_v * 0.6)
    pdsolver.invalidate_cache()
    pdsolver.simulate_mesh(c1.mesh, c1.gammas, 1, c1.dt, **kw)
    n0 = len(pdsolver._CACHE)
    a = pdsolver.simulate_mesh(c1.mesh, g2, 2, c1.dt, **kw)
    assert len(pdsolver._CACHE) == n0            # refreshed in place, not rebuilt
    m = c1.mesh
    ref = orc.simulate(m.nodes, m.tets, m.shape_grad, m.volume, g2.gamma_s, g2.gamma_v, m.node_mass, 2, c1.dt,
                       forces=c1.forces, pins=c1.pins, pin_targets=c1.pin_targets, iterations=30)
    assert rel_l2(a, ref) < 1e-10


# ---------------------------------------------------------------------------
# per-frame output step: v2y and the det(F) deviation


def _embedding(mesh, n_yarn, rng):
    """An interpolation matrix built the way the reference's embed_yarn does (volmesh.py:401-419)."""
    host = rng.integers(0, mesh.n_elements, n_yarn)
    w = rng.uniform(0.0, 1.0, (n_yarn, 4)) ** 2
    w = np.clip(w, 0.0, 1.0)
    w /= w.sum(axis=1, keepdims=True)
    rows = np.repeat(np.arange(n_yarn), 4)
    cols = mesh.tets[host].reshape(-1)
    return sp.csr_matrix((w.reshape(-1), (rows, cols)), shape=(n_yarn, mesh.n_nodes))


def test_v2y_bit_identical_to_reference_product(c1, rng):
    from paper_2405_12484_b200 import transfer
    interp = _embedding(c1.mesh, 5000, rng)
    x = c1.mesh.nodes + 0.01 * rng.normal(size=c1.mesh.nodes.shape)
    assert np.array_equal(transfer.v2y(interp, x), interp @ x)


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_frame_outputs_on_device_state(c1, rng, prec):
    from paper_2405_12484_b200 import _abi
    m = c1.mesh
    ctx = _abi.Context(m.n_nodes, m.tets, m.shape_grad, m.volume, m.node_mass, c1.gammas.gamma_s,
                       c1.gammas.gamma_v, c1.pins, c1.dt, precision=prec, tol=pdsolver.DEFAULT_TOL[prec])
    interp = _embedding(m, 3000, rng)
    ctx.set_yarn_interp(interp)
    ctx.set_state(m.nodes)
    ctx.set_pin_targets(c1.pin_targets)
    ctx.set_forces(c1.forces)
    for _ in range(3):
        ctx.step(30)
        y, dev = ctx.frame_outputs()
        x = ctx.get_state()[0]
        assert np.array_equal(y, interp @ x)
        ref = float(np.abs(np.linalg.det(m.deformation_gradients(x)) - 1.0).max())
        assert abs(dev - ref) <= 1e-12 * max(1.0, ref)


# ---------------------------------------------------------------------------
# pd_equilibrium (fitting-side forward solve)


@pytest.mark.parametrize("prec,tol", [("fp64", 1e-10), ("fp32", 2e-5)])
def test_pd_equilibrium_matches_reference(prec, tol):
    g = golden("equilibrium.npz")
    sc, a, x0 = scenes.equilibrium_case()
    assert scene_digest(sc) == str(g["digest"])
    for its in (1, 5, 30):
        x = pdsolver.pd_equilibrium(sc.mesh, sc.gammas, a, x0, sc.pins, sc.pin_targets, sc.dt,
                                    iterations=its, precision=prec)
        assert rel_l2(x, g[f"x{its}"]) < tol, its
        assert np.abs(x[sc.pins] - sc.pin_targets).max() < (1e-14 if prec == "fp64" else 1e-7)


def test_pd_equilibrium_host_solver_and_divergence(c1):
    sc, a, x0 = scenes.equilibrium_case()
    g = golden("equilibrium.npz")
    K = orc.assemble_K(sc.mesh.tets, sc.mesh.shape_grad, sc.mesh.volume, sc.gammas.gamma_s, sc.gammas.gamma_v,
                       sc.mesh.node_mass, sc.dt, sc.n_nodes)
    ref_solver = orc.GlobalSolver(K, np.setdiff1d(np.arange(sc.n_nodes), sc.pins), sc.pins)
    x = pdsolver.pd_equilibrium(sc.mesh, sc.gammas, a, x0, sc.pins, sc.pin_targets, sc.dt, iterations=5,
                                solver=ref_solver)
    assert rel_l2(x, g["x5"]) < 1e-10

    class BadSolver:
        def solve(self, b, pin_vals):
            return np.full_like(b, np.nan)

    with pytest.raises(RuntimeError, match="diverged at iteration 0"):
        pdsolver.pd_equilibrium(sc.mesh, sc.gammas, a, x0, sc.pins, sc.pin_targets, sc.dt, iterations=3,
                                solver=BadSolver())
    bad = x0.copy()
    bad[np.setdiff1d(np.arange(sc.n_nodes), sc.pins)[-1]] = np.nan
    with pytest.raises(RuntimeError, match="diverged at iteration 0"):
        pdsolver.pd_equilibrium(sc.mesh, sc.gammas, a, bad, sc.pins, sc.pin_targets, sc.dt, iterations=3)


# ---------------------------------------------------------------------------
# projection derivatives (material.py:490-524)


def test_projection_jacobians_match_reference():
    g = golden("jacobians.npz")
    JR, JV = material.projection_jacobians_batch(g["F"])
    for J, R in ((JR, g["JR"]), (JV, g["JV"])):
        scale = np.maximum(np.abs(R).reshape(len(R), -1).max(1), 1.0)
        err = np.abs(J - R).reshape(len(R), -1).max(1) / scale
        assert err.max() < 1e-8, (int(err.argmax()), float(err.max()))


def test_projection_jacobians_finite_difference(rng):
    F = np.eye(3) + 0.3 * rng.normal(size=(64, 3, 3))
    F[np.linalg.det(F) < 0.2] = np.eye(3)
    JR, JV = material.projection_jacobians_batch(F)
    h = 1e-6
    for k in range(9):
        dF = np.zeros((3, 3))
        dF.flat[k] = h
        Rp, Vp = material.batch_projections(F + dF)
        Rm, Vm = material.batch_projections(F - dF)
        assert np.abs((Rp - Rm).reshape(-1, 9) / (2 * h) - JR[:, :, k]).max() < 1e-5
        assert np.abs((Vp - Vm).reshape(-1, 9) / (2 * h) - JV[:, :, k]).max() < 1e-5


def test_pd_step_with_torch_cuda_state(c1):
    """PyTorch carrier: SimState x / v as float64 CUDA tensors stay on the device through
    pd_step (vkpd_set_state_dev / get_state_dev on the library stream) and give the same bits
    as the numpy path; feeding the returned state back keeps the warm start, as stepping the
    context does."""
    import torch
    pdsolver.invalidate_cache()
    sa = pdsolver.SimState(x=c1.mesh.nodes, v=np.zeros_like(c1.mesh.nodes), dt=c1.dt, pins=c1.pins,
                           pin_targets=c1.pin_targets)
    xa = []
    for _ in range(3):
        pdsolver.pd_step(sa, c1.mesh, c1.gammas, iterations=30, forces=c1.forces)
        xa.append((sa.x.copy(), sa.v.copy()))
    pdsolver.invalidate_cache()
    xt = torch.as_tensor(c1.mesh.nodes, device="cuda")
    sb = pdsolver.SimState(x=xt, v=torch.zeros_like(xt), dt=c1.dt, pins=c1.pins,
                           pin_targets=torch.as_tensor(c1.pin_targets, device="cuda"))
    ft = torch.as_tensor(c1.forces, device="cuda")
    for k in range(3):
        pdsolver.pd_step(sb, c1.mesh, c1.gammas, iterations=30, forces=ft)
        assert sb.x.is_cuda and sb.v.is_cuda
        assert np.array_equal(sb.x.cpu().numpy(), xa[k][0])
        assert np.array_equal(sb.v.cpu().numpy(), xa[k][1])
    assert rel_l2(sb.x.cpu().numpy(), golden("c1.npz")["frames"][2]) < 1e-10

/*
 * vkpd -- B200 (sm_100a) projective-dynamics step for the volumetric
 * homogenized knit model (arXiv 2405.12484).  Plain C ABI: host pointers and
 * sizes only, no PyTorch / CUDA types in the signatures (streams travel as
 * `void*` = cudaStream_t).
 *
 * Each entry point replaces one reference interface (paths relative to
 * /root/reference/pkg/src/volknit/):
 *
 *   vkpd_create           VolumeMesh operators + assemble_global + GlobalSolver(...)
 *                         construction: pdsolver.py:42-56, 201-223, 734-742
 *   vkpd_set_state /      SimState x, v (pdsolver.py:180-198)
 *   vkpd_get_state
 *   vkpd_set_pin_targets  SimState.pin_targets / per-step pin path (pdsolver.py:750-751)
 *   vkpd_set_forces       per-step external forces (pdsolver.py:744-752)
 *   vkpd_set_gammas       MaterialField refresh + assemble_global (material.py:563-590, pdsolver.py:42-56)
 *   vkpd_step             pd_step (pdsolver.py:257-304)
 *   vkpd_set_colliders    SimState.colliders (pdsolver.py:125-173, 271-297)
 *   vkpd_elastic_rhs      elastic_rhs (pdsolver.py:59-71)
 *   vkpd_global_solve     GlobalSolver.solve (pdsolver.py:225-246)
 *   vkpd_apply_K          the assembled K (pdsolver.py:42-56) applied to a vector
 *   vkpd_batch_projections material.batch_projections (material.py:395-407)
 *   vkpd_equilibrium      pd_equilibrium (pdsolver.py:315-338), the fitting side's forward solve
 *   vkpd_hess_*           fitting-side second order (float64, caller node order):
 *                         elastic_energy / elastic_gradient (pdsolver.py:72-97),
 *                         exact_elastic_hessian (pdsolver.py:100-118), the exact Newton step
 *                         of newton_polish (pdsolver.py:402-414), gamma_jacobian^T lam and the
 *                         adjoint solve of adjoint_gradient (fitting.py:172-235)
 *   vkpd_set_yarn_interp / vkpd_frame_outputs / vkpd_v2y
 *                         transfer.v2y (transfer.py:26-28) and the det(F) deviation of the
 *                         simulate loop (cli.py:639-640)
 *
 * Error convention (mirrors the reference's exceptions):
 *   VKPD_OK          0
 *   VKPD_EINVAL      1  invalid argument            -> ValueError
 *   VKPD_ENONFINITE  2  non-finite positions at PD iteration *failed_iter
 *                       -> RuntimeError("projective step produced non-finite
 *                          positions at iteration {it}")
 *   VKPD_ECUDA       3  CUDA error / no device       -> RuntimeError
 * vkpd_last_error() returns a thread-local message for the last failure.
 *
 * A context is not re-entrant; one context per device per process.
 */
#ifndef VKPD_H
#define VKPD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VKPD_OK 0
#define VKPD_EINVAL 1
#define VKPD_ENONFINITE 2
#define VKPD_ECUDA 3

#define VKPD_FP32 32
#define VKPD_FP64 64

typedef struct vkpd_ctx vkpd_ctx;

typedef struct {
    int64_t n_nodes;
    int64_t n_tets;
    const int64_t* tets;        /* (n_tets, 4) node ids, positive orientation        */
    const double* shape_grad;   /* (n_tets, 4, 3) rest shape gradients (volmesh.py:87-91) */
    const double* volume;       /* (n_tets,)  rest volumes, > 0                          */
    const double* node_mass;    /* (n_nodes,) lumped masses                             */
    const double* gamma_s;      /* (n_tets,)  >= 0                                       */
    const double* gamma_v;      /* (n_tets,)  >= 0                                       */
    const int64_t* pins;        /* (n_pins,) unique node ids, may be NULL if n_pins = 0  */
    int64_t n_pins;
    double dt;                  /* > 0 */
    const double* nodes;        /* (n_nodes, 3) rest positions, optional (NULL): used only to   */
                                /* order the free nodes in compact patches, one per solver CTA */
} vkpd_mesh_desc;

typedef struct {
    int precision;     /* VKPD_FP32 or VKPD_FP64                                         */
    double tol;        /* global-step relative residual tolerance (<= 0: default)        */
    int max_iters;     /* CG iteration cap per global solve (<= 0: default 1000)         */
    int device;        /* CUDA device ordinal                                            */
    int pcg_blocks;    /* CTAs of the persistent solver (<= 0: one per SM)               */
    int use_graph;     /* capture a whole frame in a CUDA graph (1, default) or not (0)  */
    int solver;        /* global step: VKPD_SOLVER_AUTO (0: Chebyshev where its register   */
                       /* path applies -- one row per thread -- else polynomial CG),       */
                       /* _PCG_POLY, _CHEBYSHEV, _PCG_JACOBI                                */
    int pd_early_exit; /* stop a frame's PD rounds at the first zero-work solve (<0: on)  */
    int warm_rounds;   /* PD rounds warm-started from earlier frames (<0: default)        */
    int unroll_rounds; /* PD rounds captured ahead of the graph's WHILE node (<0: adaptive) */
    double tol_growth; /* > 1: PD round k of R solves to tol * tol_growth^(R-1-k); < 0: default */
                       /* (1.15 in float64, off in float32); 0 or 1: off                       */
} vkpd_config;

#define VKPD_SOLVER_AUTO 0
#define VKPD_SOLVER_PCG_POLY 1
#define VKPD_SOLVER_CHEBYSHEV 2
#define VKPD_SOLVER_PCG_JACOBI 3

typedef struct {
    int n_pd_iters;            /* PD iterations of the last frame                         */
    int cg_iters[256];         /* CG iterations of each global solve of the last frame     */
    int cg_iters_total;
    unsigned int robust;       /* elements re-solved on the robust scalar SL(3) path       */
    unsigned int fallback;     /* robust path fell back to uniform scaling (warned)        */
    int pcg_blocks;
    int ell_width;
    int64_t n_free;
    double local_ms[256];      /* per-PD-iteration event times of the last vkpd_profile_step */
    double global_ms[256];
    unsigned long long pd_rounds_total; /* PD rounds executed since creation: a frame stops early once a
                                           solve needs zero CG iterations (the rest would repeat it exactly) */
    int solver;                /* the global-step solver in use (VKPD_SOLVER_*; AUTO resolved)     */
} vkpd_stats;

const char* vkpd_last_error(void);
int vkpd_device_count(int* count);

int vkpd_create(const vkpd_mesh_desc* mesh, const vkpd_config* cfg, vkpd_ctx** out);
/* matrix-only context: GlobalSolver(K, free, pins) with K in CSR (pdsolver.py:205-223);
 * supports vkpd_global_solve / vkpd_apply_K / vkpd_get_matrix_csr only */
int vkpd_create_matrix(int64_t n, const int64_t* indptr, const int64_t* indices, const double* data,
                       const int64_t* pins, int64_t n_pins, const vkpd_config* cfg, vkpd_ctx** out);
/* the device-assembled K as CSR in caller node order (free rows; all rows without pins).
 * Call with indptr = NULL to query *nnz first. */
int vkpd_get_matrix_csr(vkpd_ctx* ctx, int64_t* indptr, int64_t* indices, double* data, int64_t* nnz);
void vkpd_destroy(vkpd_ctx* ctx);
/* run subsequent work on this cudaStream_t (NULL: the context's own stream) */
int vkpd_set_stream(vkpd_ctx* ctx, void* stream);
void* vkpd_get_stream(vkpd_ctx* ctx);

int vkpd_set_state(vkpd_ctx* ctx, const double* x, const double* v);      /* (nV,3) each; v may be NULL (= 0) */
int vkpd_get_state(vkpd_ctx* ctx, double* x, double* v);                  /* either may be NULL */
/* The same state transfers with DEVICE pointers (torch tensors' data_ptr(): float64 (n, 3),
 * C-contiguous, caller node order), enqueued on the context stream (vkpd_set_stream: the
 * caller's stream) with no host synchronisation -- the PyTorch-carrier form of SimState x / v,
 * forces and pin targets (pdsolver.py:180-198, 744-752).  set_state keeps the solver's warm
 * start when the incoming state is bit-identical to the one the context holds (a caller that
 * feeds back the state it got), and clears it otherwise. */
int vkpd_set_state_dev(vkpd_ctx* ctx, const void* x, const void* v);      /* v may be NULL (zero) */
int vkpd_get_state_dev(vkpd_ctx* ctx, void* x, void* v);                  /* either may be NULL */
int vkpd_set_forces_dev(vkpd_ctx* ctx, const void* f);                    /* NULL: no forces */
int vkpd_set_pin_targets_dev(vkpd_ctx* ctx, const void* t);               /* (n_pins, 3) */
int vkpd_set_pin_targets(vkpd_ctx* ctx, const double* targets);           /* (n_pins,3) */
int vkpd_set_forces(vkpd_ctx* ctx, const double* forces);                 /* (nV,3) or NULL = none */
/* new per-tet material (MaterialField, material.py:563-590) for the same mesh, pins and dt:
 * the local-step weights and K (assemble_global, pdsolver.py:42-56) are rebuilt on the device
 * (the fitting loop changes gamma every line-search trial, fitting.py:429-432) */
int vkpd_set_gammas(vkpd_ctx* ctx, const double* gamma_s, const double* gamma_v);   /* (n_tets,) each */
/* colliders of the following steps (SimState.colliders, pdsolver.py:125-173, 271-297):
 * kinds[c] = 0 plane (params: point xyz, normal xyz) or 1 sphere (centre xyz, radius, -, -);
 * params (n,6); nodes penetrating at the prediction get weight k * K_ii (n = 0: none) */
int vkpd_set_colliders(vkpd_ctx* ctx, int n, const int* kinds, const double* params, double contact_stiffness);

/* one implicit-Euler step by `iterations` local/global rounds; blocks until done.
 * On VKPD_ENONFINITE the state is left as it was before the step. */
int vkpd_step(vkpd_ctx* ctx, int iterations, double damping, int* failed_iter);
/* simulate_mesh's frame loop (pdsolver.py:744-762): `steps` steps from the current state; forces NULL
 * (none), (nV,3) constant (forces_per_step = 0) or (steps,nV,3); pin_path NULL (current targets) or
 * (steps,n_pins,3); frames (steps,nV,3) receives x after every step.  Per-step inputs and outputs
 * move on a copy stream, overlapping the next frame.  On VKPD_ENONFINITE, *failed_frame / *failed_iter
 * name the first failing step and its PD iteration (the contents of frames from there on are
 * undefined). */
int vkpd_simulate(vkpd_ctx* ctx, int steps, int iterations, double damping, const double* forces, int forces_per_step,
                  const double* pin_path, double* frames, int* failed_frame, int* failed_iter);
/* same step, enqueued without waiting; vkpd_sync() reports the outcome */
int vkpd_step_async(vkpd_ctx* ctx, int iterations, double damping);
int vkpd_sync(vkpd_ctx* ctx, int* failed_iter);
/* one frame launched kernel by kernel with CUDA events around every local-step and
 * global-step launch (measurement only): average durations in ms */
int vkpd_profile_step(vkpd_ctx* ctx, int iterations, double damping, double* local_ms,
                      double* global_ms, double* frame_ms);

/* measurement only: `reps` back-to-back launches of the local step on the current state; average
 * ms of k_local alone and of the local phase of a round (k_local + the robust pass) */
int vkpd_time_local(vkpd_ctx* ctx, int reps, double* local_ms, double* pass_ms);

int vkpd_elastic_rhs(vkpd_ctx* ctx, const double* x, double* rhs, double* F, double* R, double* V);
int vkpd_global_solve(vkpd_ctx* ctx, const double* B, const double* pin_vals, double* X, int k);
int vkpd_apply_K(vkpd_ctx* ctx, const double* X, double* Y);
int vkpd_get_stats(vkpd_ctx* ctx, vkpd_stats* st);

/* Device-pointer primitives for the domain-decomposed multi-GPU step (dd.py).  Vectors are
 * 4-wide (x,y,z,pad) in the context's precision and internal node order (free nodes, then the
 * pinned list); work runs on the context stream.
 *   dev_residual: r_free = b - K x on free rows (local step + deterministic gather + inertia),
 *                 the residual of pd_step's global solve (pdsolver.py:292-298)
 *   dev_apply_K:  Y_free = K_ff X_free + K_fp X_pinned (pdsolver.py:227-229)            */
int vkpd_dev_residual(vkpd_ctx* ctx, const void* x_int, const void* xhat_int, void* r_free);
int vkpd_dev_apply_K(vkpd_ctx* ctx, const void* X_int, void* Y_free);
int vkpd_dev_inv_diag(vkpd_ctx* ctx, void* out_free);
/*   dev_cheb_step: one step of the distributed Chebyshev solve (dd.py) on the free rows, fused:
 *                 q = K_ff d_free + K_fp d_pinned (the pinned slots carry the halo), y += d,
 *                 res -= q, dnext_free = c1 d + c2 D^-1 res (pdsolver.py:225-236 as an
 *                 iteration; the rank's share of GlobalSolver.solve)                       */
int vkpd_dev_cheb_step(vkpd_ctx* ctx, const void* d_int, void* res_free, void* y_free, void* dnext_int, double c1,
                       double c2);
/* Gershgorin bound of D^-1 K_ff (with_pinned_cols: rows of [K_ff K_fp], a rank's share of the
 * global bound when the pinned slots are its halo) */
int vkpd_get_gershgorin(vkpd_ctx* ctx, int with_pinned_cols, double* g);
int vkpd_get_node_order(vkpd_ctx* ctx, int64_t* int_of_orig);
int vkpd_get_sizes(vkpd_ctx* ctx, int64_t* n, int64_t* n_free, int64_t* n_pinned, int* precision);

/* a_jacobi_refine (pdsolver.py:632-703) on K_ff over free-node vectors (n_free, k), k <= 3:
 * aggregated weighted-Jacobi sweeps (or the Chebyshev variant with spectral radius rho),
 * best-iterate tracking and divergence stop.  hist: (k, steps+1) residual norms, row-major,
 * steps = sweeps (plain) or sweeps*aggregation (Chebyshev); n_hist/diverged: (k,). */
int vkpd_a_jacobi_refine(vkpd_ctx* ctx, const double* Bf, const double* X0f, int k, int sweeps, int aggregation,
                         double omega, int chebyshev, double rho, double* Xf, double* hist, int* n_hist,
                         int* diverged);
/* _power_rho (pdsolver.py:616-629): 30-ish power iterations of I - omega D^-1 K_ff from v0 (n_free) */
int vkpd_power_rho(vkpd_ctx* ctx, double omega, int iters, const double* v0, double* rho);
/* CmsSubspace (pdsolver.py:512-593): dense basis T (n_free x m, column-major) and K_red^-1 (m x m) */
int vkpd_cms_set_basis(vkpd_ctx* ctx, int m, const double* T, const double* Kred_inv);
/* The same subspace stored per domain (the zeros of the global T are neither stored nor streamed):
 * domain d holds A_d = [Phi_d | Psi_d on its adjacent boundary columns], n_d x c_d column-major,
 * concatenated in domain order in A; rows[row_ptr[d]..row_ptr[d+1]) are its interior free-node
 * indices and colmap[col_ptr[d]..col_ptr[d+1]) the global basis column of each local column
 * (modes first, then n_modes + j for boundary node boundary[j]); K_red^-1 is m x m with
 * m = n_modes + nb.  Replaces a dense basis set with vkpd_cms_set_basis. */
int vkpd_cms_set_blocks(vkpd_ctx* ctx, int n_dom, const int64_t* row_ptr, const int64_t* rows, const int64_t* col_ptr,
                        const int64_t* colmap, const double* A, int n_modes, int64_t nb, const int64_t* boundary,
                        const double* Kred_inv);
/* pd_step with GlobalSolver(mode="cms") (pdsolver.py:257-304, 237-246) as one device frame on a mesh
 * context whose subspace was set with vkpd_cms_set_blocks / vkpd_cms_set_basis: per PD round the local
 * step, b = rhs + (M/dt^2) xhat, x_f = a_jacobi_refine(K_ff, b_f - K_fp p, T K_red^-1 T^T (b_f - K_fp p)).
 * Same error contract as vkpd_step. */
int vkpd_step_cms(vkpd_ctx* ctx, int iterations, double damping, int sweeps, int aggregation, double omega,
                  int chebyshev, double rho, int* failed_iter);
/* device times (CUDA events) of the last vkpd_cms_solve's first column group: the subspace
 * apply x0 = T K_red^-1 T^T b and the a_jacobi_refine sweeps */
int vkpd_cms_timing(vkpd_ctx* ctx, double* apply_ms, double* sweeps_ms);
/* GlobalSolver.solve in "cms" mode (pdsolver.py:225-246): x0 = T K_red^-1 T^T (B_f - K_fp P), then
 * sweeps of a_jacobi_refine per column; B (nV,k), P (n_pins,k), X (nV,k) */
int vkpd_cms_solve(vkpd_ctx* ctx, const double* B, const double* P, int k, int sweeps, int aggregation, double omega,
                   int chebyshev, double rho, double* X);

int vkpd_batch_projections(int precision, int64_t n, const double* F, double* R, double* V,
                           unsigned int* n_robust, unsigned int* n_fallback);

/* projection_jacobians_batch (material.py:490-524): d vec(R)/d vec(F) and d vec(V)/d vec(F),
 * (n, 9, 9) each, row-major vec layout, float64 */
int vkpd_projection_jacobians(int64_t n, const double* F, double* JR, double* JV);

/* pd_equilibrium (pdsolver.py:315-338): `iterations` proximal local/global rounds solving
 * K x = (M/dt^2)(x_cur - a) + rhs from x0 with pinned rows = pin_vals (n_pins,3); the
 * simulation state is not touched.  VKPD_ENONFINITE with *failed_iter on non-finite x
 * ("quasi-static projection diverged at iteration {it}"). */
int vkpd_equilibrium(vkpd_ctx* ctx, const double* inertia_target, const double* x0, const double* pin_vals,
                     int iterations, double* x_out, int* failed_iter);

/* Per-frame output step (cli.py:628-656), on the device-resident state:
 *   vkpd_set_yarn_interp: the yarn embedding's interpolation matrix (transfer.py:26-28,
 *                         volmesh.py:401-419) in CSR, columns = caller node ids
 *   vkpd_frame_outputs:   yarn (n_yarn,3) = interp @ x and/or det_deviation =
 *                         max_e |det F_e - 1| (cli.py:639-640); either may be NULL
 *   vkpd_v2y:             transfer.v2y on host positions (float64, bit-identical to
 *                         scipy's CSR product) */
int vkpd_set_yarn_interp(vkpd_ctx* ctx, int64_t n_yarn, const int64_t* indptr, const int64_t* indices,
                         const double* data);
int vkpd_frame_outputs(vkpd_ctx* ctx, double* yarn, double* det_deviation);
int vkpd_v2y(int64_t n_yarn, const int64_t* indptr, const int64_t* indices, const double* data, int64_t n_nodes,
             const double* x, double* y);

/* Per-frame OBJ text of `volknit simulate` (cli.py:538-547, _write_obj): an optional "# comment"
 * line, "v x y z" per vertex with %.17g (Python's format(v, ".17g")), then "f a b c" per
 * triangle (1-based) and "l i j ..." per polyline (1-based; line_ptr has n_lines + 1 offsets
 * into line_idx).  Host code, no device needed.  Writes at most `cap` bytes into `out` and
 * returns the total length (call with out = NULL to size the buffer). */
int64_t vkpd_format_obj(const double* vertices, int64_t n_vertices, const int64_t* faces, int64_t n_faces,
                        const int64_t* line_ptr, const int64_t* line_idx, int64_t n_lines, const char* comment,
                        char* out, int64_t cap);

/* ---- fitting-side second order, float64, caller node order ----------------
 * One handle per (mesh, pins, dt); gammas refreshable.  Vectors are (nV,3) row-major doubles.
 *   vkpd_hess_energy_grad  elastic_energy (pdsolver.py:72-82) and elastic_gradient
 *                          (pdsolver.py:85-97) at x; either output may be NULL
 *   vkpd_hess_gamma_jt     out (2 nE) = gamma_jacobian(mesh, x)^T lam (fitting.py:172-190)
 *   vkpd_hess_linearize    keep the per-tet blocks 2V (gs (I - dR/dF) + gv (I - dV/dF)) at x
 *   vkpd_hess_csr          exact_elastic_hessian at the linearized x (pdsolver.py:100-118), CSR
 *                          3nV x 3nV with sorted columns; indptr = NULL queries *nnz
 *   vkpd_hess_apply        y = (H + mass_scale M/dt^2) p on all dofs
 *   vkpd_hess_solve        (H + mass_scale M/dt^2 + ridge I)_ff x_f = b_f by |diag|-preconditioned
 *                          MINRES (pinned dofs of b ignored, x = 0 there); *relres = the true
 *                          relative residual.  The caller decides what a non-converged solve
 *                          means (newton_polish falls back to the Gauss-Newton step, the adjoint
 *                          adds a ridge, as the reference does on a singular factorization). */
typedef struct vkpd_hess vkpd_hess;
int vkpd_hess_create(const vkpd_mesh_desc* mesh, int device, vkpd_hess** out);
void vkpd_hess_destroy(vkpd_hess* h);
int vkpd_hess_set_gammas(vkpd_hess* h, const double* gamma_s, const double* gamma_v);
int vkpd_hess_energy_grad(vkpd_hess* h, const double* x, double* energy, double* grad);
int vkpd_hess_gamma_jt(vkpd_hess* h, const double* x, const double* lam, double* out);
int vkpd_hess_linearize(vkpd_hess* h, const double* x);
int vkpd_hess_csr(vkpd_hess* h, int64_t* indptr, int64_t* indices, double* data, int64_t* nnz);
int vkpd_hess_apply(vkpd_hess* h, double mass_scale, const double* p, double* y);
int vkpd_hess_solve(vkpd_hess* h, double mass_scale, double ridge, const double* b, double* x, double tol,
                    int max_iters, int* iters, double* relres);

#ifdef __cplusplus
}
#endif
#endif /* VKPD_H */

// Global step (K1/K6/K7 of SURVEY.md section 2): matrix assembly, step
// prologue/epilogue and the persistent preconditioned-CG kernel.
//
// Node order on the device ("internal"): free nodes first, in the caller's
// order, then the pinned nodes in pin order.  The scalar global matrix
// K = M/dt^2 + sum_e 2V(gs+gv) G G^T (pdsolver.py:42-56) is kept as K_ff in
// column-major ELL over the free rows (free columns only), so pinned values
// are eliminated exactly as GlobalSolver does (pdsolver.py:210-229).
#pragma once

#include <cooperative_groups.h>

#include "vk_common.cuh"

namespace cg = cooperative_groups;

namespace vk {

// ---------------------------------------------------------------------------
// K_ff assembly, one thread per free row; deterministic (incidences in tet order).
template <typename T>
struct AssembleArgs {
    int nF, nE, ell_w;
    const int* inc_ptr;          // (n+1) per internal node
    const int* inc_code;         // a * nE + e, sorted by e
    const int4* tets;            // internal ids
    const double* G;             // (nE,4,3) float64 shape gradients (host layout)
    const double* wsum;          // (nE) 2 V (gs + gv)
    const double* m_dt2;         // (n) m / dt^2, internal order
    const int* ell_col;          // [s * nF + i], padded with the row's own index
    const int* ell_len;          // real entries per row
    T* ell_val;
    T* inv_diag;                 // (nF)
    double* diag64;              // (nF) float64 diagonal (A-Jacobi / reference-compat paths)
    // K_fp in CSR over free rows (columns are pin slots 0..nP-1)
    const int* fp_ptr;
    const int* fp_col;
    T* fp_val;
    int n_free_cols_base;        // = nF: internal id of the first pinned node
};

template <typename T>
__global__ void k_assemble(AssembleArgs<T> a) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.nF) return;
    const int b0 = a.inc_ptr[i], b1 = a.inc_ptr[i + 1];
    double diag = a.m_dt2[i];
    const int len = a.ell_len[i];
    for (int s = 0; s < a.ell_w; ++s) {
        const int col = a.ell_col[(size_t)s * a.nF + i];
        double v = 0.0;
        if (s < len) {
            for (int k = b0; k < b1; ++k) {
                const int code = a.inc_code[k];
                const int e = code % a.nE, an = code / a.nE;
                const int4 t = a.tets[e];
                const int nodes[4] = {t.x, t.y, t.z, t.w};
                for (int bn = 0; bn < 4; ++bn) {
                    if (nodes[bn] == col) {
                        const double* g = a.G + (size_t)e * 12;
                        v += a.wsum[e] * (g[an * 3 + 0] * g[bn * 3 + 0] + g[an * 3 + 1] * g[bn * 3 + 1] +
                                          g[an * 3 + 2] * g[bn * 3 + 2]);
                    }
                }
            }
            if (col == i) { v += diag; diag = v; }
        }
        a.ell_val[(size_t)s * a.nF + i] = (T)v;
    }
    a.inv_diag[i] = (T)(1.0 / diag);
    a.diag64[i] = diag;
    for (int k = a.fp_ptr[i]; k < a.fp_ptr[i + 1]; ++k) {
        const int col = a.n_free_cols_base + a.fp_col[k];
        double v = 0.0;
        for (int kk = b0; kk < b1; ++kk) {
            const int code = a.inc_code[kk];
            const int e = code % a.nE, an = code / a.nE;
            const int4 t = a.tets[e];
            const int nodes[4] = {t.x, t.y, t.z, t.w};
            for (int bn = 0; bn < 4; ++bn)
                if (nodes[bn] == col) {
                    const double* g = a.G + (size_t)e * 12;
                    v += a.wsum[e] * (g[an * 3 + 0] * g[bn * 3 + 0] + g[an * 3 + 1] * g[bn * 3 + 1] +
                                      g[an * 3 + 2] * g[bn * 3 + 2]);
                }
        }
        a.fp_val[k] = (T)v;
    }
}

// ---------------------------------------------------------------------------
// Step prologue (pdsolver.py:249-254, 283-289):
//   x_start = x, v_start = v, xhat = x + dt v + dt^2 m^-1 f (m^-1 := 0 where m = 0),
//   x = xhat on free nodes, x = pin target on pinned nodes.
template <typename T>
__global__ void k_prologue(int n, int nF, T dt, const T* __restrict__ dt2_inv_m, const vec4_t<T>* __restrict__ f,
                           const vec4_t<T>* __restrict__ pin_tgt, vec4_t<T>* x, vec4_t<T>* v,
                           vec4_t<T>* x_start, vec4_t<T>* v_start, vec4_t<T>* xhat, int* fail_iter,
                           int* zero2 = nullptr, int* zero1 = nullptr, unsigned* frame_ctr = nullptr) {
    pcg_mark(10);
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0) {
        *fail_iter = 0x7fffffff;
        if (zero2) { zero2[0] = 0; zero2[1] = 0; }     // suspicious-tet queue of the first local step
        if (zero1) *zero1 = 0;                          // PD-iteration counter of the loop node
        if (frame_ctr) *frame_ctr += 1u;                // warm-start ring index (cheb.cuh)
    }
    if (i >= n) return;
    const vec4_t<T> xi = x[i], vi = v[i];
    x_start[i] = xi;
    v_start[i] = vi;
    const T c = dt2_inv_m[i];
    vec4_t<T> fi = make4<T>(T(0), T(0), T(0), T(0));
    if (f != nullptr) fi = f[i];
    const vec4_t<T> xh = make4<T>(xi.x + dt * vi.x + c * fi.x, xi.y + dt * vi.y + c * fi.y,
                                  xi.z + dt * vi.z + c * fi.z, T(0));
    xhat[i] = xh;
    x[i] = (i < nF) ? xh : pin_tgt[i - nF];
}

// Step epilogue (pdsolver.py:302): v = damping (x - x_start) / dt.
template <typename T>
__global__ void k_epilogue(int n, T damp_over_dt, const vec4_t<T>* __restrict__ x,
                           const vec4_t<T>* __restrict__ x_start, vec4_t<T>* v) {
    pcg_mark(11);
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const vec4_t<T> a = x[i], b = x_start[i];
    v[i] = make4<T>(damp_over_dt * (a.x - b.x), damp_over_dt * (a.y - b.y), damp_over_dt * (a.z - b.z), T(0));
}

// pd_equilibrium round setup (pdsolver.py:330-333): xhat = x - a on free rows, so the
// residual-form solve targets K x = (M/dt^2)(x_cur - a) + rhs
template <typename T>
__global__ void k_eq_target(int nF, const vec4_t<T>* __restrict__ x, const vec4_t<T>* __restrict__ a,
                            vec4_t<T>* xhat) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nF) return;
    const vec4_t<T> xi = x[i], ai = a[i];
    xhat[i] = make4<T>(xi.x - ai.x, xi.y - ai.y, xi.z - ai.z, T(0));
}

// pinned rows (internal nF..n-1, pin order) := pin values
template <typename T>
__global__ void k_set_pinned(int n, int nF, const vec4_t<T>* __restrict__ pin_vals, vec4_t<T>* x) {
    const int i = nF + blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    x[i] = pin_vals[i - nF];
}

// Restore the step's input state after a non-finite abort.
template <typename T>
__global__ void k_restore(int n, vec4_t<T>* x, vec4_t<T>* v, const vec4_t<T>* x_start, const vec4_t<T>* v_start) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    x[i] = x_start[i];
    v[i] = v_start[i];
}

// Gershgorin bound of D^-1 K_ff: max_i sum_{j != i} |K_ij| / K_ii (the caller adds 1).
// Non-negative doubles order like their bit patterns, so an integer atomicMax works.
template <typename T>
__global__ void k_gershgorin(int nF, int ell_w, const int* __restrict__ ell_col, const T* __restrict__ ell_val,
                             const double* __restrict__ diag64, unsigned long long* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nF) return;
    double off = 0.0;
    for (int s = 0; s < ell_w; ++s)
        if (ell_col[(size_t)s * nF + i] != i) off += fabs((double)ell_val[(size_t)s * nF + i]);
    const double g = off / diag64[i];
    atomicMax(out, (unsigned long long)__double_as_longlong(g >= 0.0 ? g : 0.0));
}

// Same bound over the rows of [K_ff K_fp] (the pinned columns of a domain-decomposed rank hold
// its halo, dd.py): the rank's share of the global Gershgorin bound.
template <typename T>
__global__ void k_gershgorin_fp(int nF, int ell_w, const int* __restrict__ ell_col, const T* __restrict__ ell_val,
                                const int* __restrict__ fp_ptr, const T* __restrict__ fp_val,
                                const double* __restrict__ diag64, unsigned long long* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nF) return;
    double off = 0.0;
    for (int s = 0; s < ell_w; ++s)
        if (ell_col[(size_t)s * nF + i] != i) off += fabs((double)ell_val[(size_t)s * nF + i]);
    for (int k = fp_ptr[i]; k < fp_ptr[i + 1]; ++k) off += fabs((double)fp_val[k]);
    const double g = off / diag64[i];
    atomicMax(out, (unsigned long long)__double_as_longlong(g >= 0.0 ? g : 0.0));
}

// rhs_i = sum over incidences of corner contributions (tet order) -- the
// `np.add.at` of pdsolver.py:69-70, without atomics.  All n nodes.
template <typename T>
__global__ void k_gather(int n, const int* __restrict__ inc_ptr, const vec4_t<T>* __restrict__ corner,
                         vec4_t<T>* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    T sx = 0, sy = 0, sz = 0;
    for (int k = inc_ptr[i]; k < inc_ptr[i + 1]; ++k) {
        const vec4_t<T> c = ldg4(&corner[k]);
        sx += c.x; sy += c.y; sz += c.z;
    }
    out[i] = make4<T>(sx, sy, sz, T(0));
}

// ---------------------------------------------------------------------------
// Persistent Jacobi-preconditioned CG on K_ff for the three coordinate
// columns at once (one scalar recurrence per column), launched cooperatively
// with one grid barrier per half-iteration.  The search direction is double
// buffered so the "p = z + beta p" update fuses into the SpMV phase.
//
// init == INIT_PD:  r = sum_inc corner + (m/dt^2)(xhat - x)  (= b - K x at the
//                   current PD iterate, free rows), solve K_ff dx = r, x += dx.
// init == INIT_RHS: r = rhs (caller-assembled b_f - K_fp pins), x0 = 0, the
//                   solution is left in dx (GlobalSolver.solve drop-in).
// Stops when sum_c |r_c|^2 <= tol^2 * scale^2 (scale^2 = |M/dt^2 xhat|^2 for
// INIT_PD, |r0|^2 for INIT_RHS) or after max_iters.
enum PcgInit { INIT_PD = 0, INIT_RHS = 1 };
constexpr int kEllUnroll = 16;     // voxel meshes: <= 15 entries per row

template <typename T>
struct PcgArgs {
    int nF, ell_w;
    const int* ell_col;
    const T* ell_val;
    const T* inv_diag;
    const int* inc_ptr;
    const int* inc_code;
    const vec4_t<T>* corner;
    // optional (frame path): node partials of the local step's warp-segmented reduction
    // (part_ptr runs over wpart) plus, when robust_present[0] > 0, the corners of the tets the
    // robust pass finished (incidence flags robust_flag[k], cleared by the gather that reads them)
    const int* part_ptr;
    const vec4_t<T>* wpart;
    unsigned char* robust_flag;
    const int* robust_present;
    const T* m_dt2;
    const vec4_t<T>* xhat;
    const vec4_t<T>* rhs;
    vec4_t<T>* x;
    vec4_t<T>* r;
    vec4_t<T>* z;
    vec4_t<T>* p0;
    vec4_t<T>* p1;
    vec4_t<T>* q;
    vec4_t<T>* dx;
    double* partials;            // gridDim.x * 8
    double* scal;                // 16 published scalars
    GridBar* bar;
    int* iters_out;              // iteration count of this solve
    int* fail_iter;              // atomicMin'd with pd_iter on non-finite output
    int pd_iter;
    double tol;
    double tol_growth;           // > 1: PD round k of R solves to tol * tol_growth^(R-1-k) (experiment; 1 = off)
    int rounds_total;            // R (frame's PD rounds) for tol_growth
    int max_iters;
    int init;
    // colliders (pdsolver.py:271-297): extra diagonal m_i * k * K_ii and rhs weight k * K_ii
    const T* cdiag;              // null without colliders
    const T* cb;
    const double* coll;          // kCollStride doubles per collider
    int ncoll;
    int* reset_count;            // optional: the local step's suspicious-tet queue, zeroed on entry
    vec4_t<T>* h;                // POLY: h = K D^-1 r, updated with r
    double omega;                // POLY: polynomial preconditioner weight
    int poly_rounds;             // POLY kernel: PD rounds >= poly_rounds use plain Jacobi (<= 0: none)
    const T* ell_kd;             // POLY: ELL values of K_ff D^-1 (no contact diagonal), or null
    int* pd_iter_dev;            // optional: PD iteration index read on the device (graph loop body);
                                 // then fail_iter gets *pd_iter_dev and the count goes to iters_out[*pd_iter_dev]
    unsigned long long loop_handle;   // nonzero: conditional handle of the PD-iteration loop node
    unsigned long long robust_if;     // nonzero: the robust pass's IF node handle, cleared here
    int* first_stop;             // optional: min over this frame's rounds that met the exit condition (1-based)
    int loop_iterations;
    unsigned long long* rounds;  // optional: executed-PD-round counter
    vec4_t<T>* warm;             // POLY, optional: warm_rounds banks of nF; PD round k < warm_rounds starts
    int warm_rounds;             // from the previous frame's round-k correction and stores its own
    vec4_t<T>* warm_prev;        // optional: the correction before it; the guess is then the linear
                                 // extrapolation d_prev + beta (d_prev - d_prevprev)
    double warm_beta;
    vec4_t<T>* warm_prev2;       // optional (cheb.cuh): the frame before that; quadratic extrapolation
    vec4_t<T>* warm_prev3;       // ring mode: the fourth bank
    const unsigned* warm_ring;   // optional (cheb.cuh register path): frame counter; warm, warm_prev and
                                 // warm_prev2 are then a ring of the last three frames' corrections
    int warm_extrap_rounds;      // rounds < this extrapolate; later warm rounds reuse the last correction
    // Chebyshev solver (cheb.cuh)
    unsigned int* flags;         // per-CTA step counters (generic path) / tag base of the next launch
                                 // (register path), 128-B stride
    const int* cheb_nbr_ptr;     // CTAs whose rows a CTA's rows read (CSR over CTAs)
    const int* cheb_nbr;
    double cheb_lmin, cheb_lmax; // spectrum interval of D^-1 K_ff
    const unsigned* cheb_slot;   // register path, [h * nF + i]: direction-image byte offsets of off-diagonal
                                 //   entries 2h, 2h+1 of row i (16 bits each; pads: a read slot, value 0),
    const T* cheb_val;           //   [s * nF + i] the entry values, and the diagonal
    const T* cheb_kdiag;
    const int* cheb_nexp;        // per CTA: its leading rows that other CTAs read (register path)
    const int* cheb_halo_ptr;    // per CTA: rows of other CTAs its rows reference, grouped by owner CTA
    const int* cheb_halo;
    int cheb_halo_max;
    uint4* cheb_ll;              // REG: exported rows of d, flag-in-data, two step-parity buffers of nF rows
};

template <typename T>
__device__ __forceinline__ void pcg_exit(const PcgArgs<T>& a, bool bad, int it, bool moved = false) {
    const int pdi = a.pd_iter_dev != nullptr ? *a.pd_iter_dev : a.pd_iter;
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicMin(a.fail_iter, pdi);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *(a.pd_iter_dev != nullptr ? a.iters_out + pdi : a.iters_out) = it;
        if (a.rounds != nullptr) *a.rounds += 1ull;
        if (a.loop_handle != 0) {
            // PD-iteration loop node (graph WHILE): continue unless this was the last
            // round, or the solve took zero CG iterations -- x did not change, so every
            // remaining local step and solve would reproduce exactly this state (bit for
            // bit) -- or a round has failed (a failure in this very launch may only be
            // seen one round later; fail_iter keeps the earliest round either way).
            // Skipped rounds are recorded with 0 CG iterations.
            // (a zero-work round is only an exact repeat point when every round has the same tolerance)
            const bool stop = pdi + 1 >= a.loop_iterations || (it == 0 && !moved && !(a.tol_growth > 1.0)) ||
                              *(volatile int*)a.fail_iter != 0x7fffffff;
            if (stop) {
                for (int j = pdi + 1; j < a.loop_iterations; ++j) a.iters_out[j] = 0;
                if (a.first_stop != nullptr && pdi + 1 < *a.first_stop) *a.first_stop = pdi + 1;
            }
            *a.pd_iter_dev = pdi + 1;
            cudaGraphSetConditional((cudaGraphConditionalHandle)a.loop_handle, stop ? 0u : 1u);
            if (a.robust_if != 0) cudaGraphSetConditional((cudaGraphConditionalHandle)a.robust_if, 0u);
        }
    }
}

template <typename T>
__device__ __forceinline__ void pcg_entry(const PcgArgs<T>& a) {
    if (a.reset_count != nullptr && blockIdx.x == 0 && threadIdx.x == 0) {
        a.reset_count[0] = 0;
        a.reset_count[1] = 0;
    }
}

// ---------------------------------------------------------------------------
// Colliders: plane {0, p0, n_hat} and sphere {1, c, r} (pdsolver.py:125-163).
constexpr int kCollStride = 8;
constexpr int kMaxColliders = 16;

// Number of colliders x penetrates (the multiplicity of x in `collider_targets`).
__device__ __forceinline__ int collider_hits(const double* coll, int ncoll, double x, double y, double z) {
    int m = 0;
    for (int c = 0; c < ncoll; ++c) {
        const double* q = coll + c * kCollStride;
        if (q[0] == 0.0) {
            if ((x - q[1]) * q[4] + (y - q[2]) * q[5] + (z - q[3]) * q[6] < 0.0) ++m;
        } else {
            const double dx = x - q[1], dy = y - q[2], dz = z - q[3];
            if (sqrt(dx * dx + dy * dy + dz * dz) < q[4]) ++m;
        }
    }
    return m;
}

// `surface_targets` for one point: every collider is tested on the original
// point and a later penetrated collider overrides an earlier one.
__device__ __forceinline__ void collider_target(const double* coll, int ncoll, double x, double y, double z,
                                                double& tx, double& ty, double& tz) {
    tx = x; ty = y; tz = z;
    for (int c = 0; c < ncoll; ++c) {
        const double* q = coll + c * kCollStride;
        if (q[0] == 0.0) {
            const double depth = (x - q[1]) * q[4] + (y - q[2]) * q[5] + (z - q[3]) * q[6];
            if (depth < 0.0) { tx = x - depth * q[4]; ty = y - depth * q[5]; tz = z - depth * q[6]; }
        } else {
            const double dx = x - q[1], dy = y - q[2], dz = z - q[3];
            const double d = sqrt(dx * dx + dy * dy + dz * dz);
            if (d < q[4]) {
                const double f = q[4] / fmax(d, 1e-12);
                tx = q[1] + dx * f; ty = q[2] + dy * f; tz = q[3] + dz * f;
            }
        }
    }
}

// Per step: contact set from the prediction xhat (pdsolver.py:271, 277-280).
template <typename T>
__global__ void k_contact_setup(int nF, const vec4_t<T>* __restrict__ xhat, const double* __restrict__ diag64,
                                const double* __restrict__ coll, int ncoll, double kc, T* inv_diag_c, T* cdiag, T* cb) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nF) return;
    const vec4_t<T> xh = xhat[i];
    const int m = collider_hits(coll, ncoll, (double)xh.x, (double)xh.y, (double)xh.z);
    const double w = kc * diag64[i];
    cdiag[i] = (T)(m * w);
    cb[i] = (T)(m > 0 ? w : 0.0);
    inv_diag_c[i] = (T)(1.0 / (diag64[i] + m * w));
}


// Every CTA sums the per-CTA partials of the last phase in the same fixed
// order after the grid barrier, so all CTAs hold bit-identical scalars (no
// serial "last CTA" step, deterministic across runs).

template <int NV>
__device__ __forceinline__ void pcg_allreduce(cg::grid_group& grid, double* partials, int& parity, double (&acc)[NV],
                                              double* red, double* smem) {
    pcg_mark(1);
    block_sum<NV>(acc, smem);
    double* P = partials + (size_t)parity * gridDim.x * 8;
    if (threadIdx.x == 0)
#pragma unroll
        for (int k = 0; k < NV; ++k) P[blockIdx.x * 8 + k] = acc[k];
    pcg_mark(2);
    grid.sync();
    pcg_mark(3);
    reduce_partials_all<NV>(P, red, smem);
    pcg_mark(4);
    parity ^= 1;
}

// Right-hand side of row i of the global solve: the PD residual b - K x
// (deterministic gather of the node's corner run + inertia + contact terms,
// pdsolver.py:292-298) or the given rhs; adds |b|^2 of the reference rhs to bb.
template <typename T>
__device__ __forceinline__ void init_residual_row(const PcgArgs<T>& a, int i, bool coherent_corners, T& rx, T& ry,
                                                  T& rzv, double& bb) {
    if (a.init == INIT_PD) {
        rx = 0; ry = 0; rzv = 0;
        // the node's own loads first (independent of the gather; the sums keep their order)
        const T m = a.m_dt2[i];
        const vec4_t<T> xh = a.xhat[i], xi = a.x[i];
        if (a.part_ptr != nullptr) {
            const int p0 = __ldg(&a.part_ptr[i]), p1 = __ldg(&a.part_ptr[i + 1]);
#pragma unroll 4
            for (int k = p0; k < p1; ++k) {
                const vec4_t<T> c = ldg4(&a.wpart[k]);
                rx += c.x; ry += c.y; rzv += c.z;
            }
            if (*a.robust_present > 0) {
                const int k0 = a.inc_ptr[i], k1 = a.inc_ptr[i + 1];
                for (int k = k0; k < k1; ++k) {
                    if (!a.robust_flag[k]) continue;
                    a.robust_flag[k] = 0;
                    const vec4_t<T> c = ldg4(&a.corner[k]);
                    rx += c.x; ry += c.y; rzv += c.z;
                }
            }
        } else {
            const int k0 = a.inc_ptr[i], k1 = a.inc_ptr[i + 1];
#pragma unroll 4
            for (int k = k0; k < k1; ++k) {
                const vec4_t<T> c = coherent_corners ? ld4(&a.corner[k]) : ldg4(&a.corner[k]);
                rx += c.x; ry += c.y; rzv += c.z;
            }
        }
        rx += m * (xh.x - xi.x);
        ry += m * (xh.y - xi.y);
        rzv += m * (xh.z - xi.z);
        if (a.ncoll > 0) {
            // contact rows: b += cw * surface_target(x), K x += m cw x (pdsolver.py:294-297)
            const T w = a.cb[i];
            if (w != T(0)) {
                double tx, ty, tz;
                collider_target(a.coll, a.ncoll, (double)xi.x, (double)xi.y, (double)xi.z, tx, ty, tz);
                // cw (target - x) - (m - 1) cw x: the penetration vector is formed
                // before scaling by the (1e4 K_ii) weight, which keeps float32 exact enough
                const T extra = a.cdiag[i] - w;
                rx += w * (T)(tx - (double)xi.x) - extra * xi.x;
                ry += w * (T)(ty - (double)xi.y) - extra * xi.y;
                rzv += w * (T)(tz - (double)xi.z) - extra * xi.z;
            }
        }
        const double bx = (double)m * xh.x, by = (double)m * xh.y, bz = (double)m * xh.z;
        bb += bx * bx + by * by + bz * bz;
    } else {
        const vec4_t<T> b = a.rhs[i];
        rx = b.x; ry = b.y; rzv = b.z;
        bb += (double)rx * rx + (double)ry * ry + (double)rzv * rzv;
    }
}

// (K_ff v)_i, contact diagonal included
template <typename T>
__device__ __forceinline__ vec4_t<T> k_row(const PcgArgs<T>& a, const vec4_t<T>* v, int i) {
    const int nF = a.nF;
    T hx = 0, hy = 0, hz = 0;
    for (int s = 0; s < a.ell_w; ++s) {
        const int c = __ldg(&a.ell_col[(size_t)s * nF + i]);
        const T kv = __ldg(&a.ell_val[(size_t)s * nF + i]);
        const vec4_t<T> vc = ld4(&v[c]);
        hx += kv * vc.x; hy += kv * vc.y; hz += kv * vc.z;
    }
    if (a.cdiag != nullptr) {
        const vec4_t<T> vi = ld4(&v[i]);
        const T cd = a.cdiag[i];
        hx += cd * vi.x; hy += cd * vi.y; hz += cd * vi.z;
    }
    return make4<T>(hx, hy, hz, T(0));
}

// (K_ff D^-1 v)_i, contact diagonal included: one ELL row against D^-1 v
template <typename T>
__device__ __forceinline__ vec4_t<T> kdinv_row(const PcgArgs<T>& a, const vec4_t<T>* v, int i) {
    const int nF = a.nF;
    T hx = 0, hy = 0, hz = 0;
    if (a.ell_kd != nullptr && a.ell_w <= kEllUnroll) {
        // prescaled values K_ij / K_jj: same load pattern as the p-update SpMV
        int cols[kEllUnroll];
        T vals[kEllUnroll];
#pragma unroll
        for (int s = 0; s < kEllUnroll; ++s) {
            cols[s] = s < a.ell_w ? __ldg(&a.ell_col[(size_t)s * nF + i]) : i;
            vals[s] = s < a.ell_w ? __ldg(&a.ell_kd[(size_t)s * nF + i]) : T(0);
        }
#pragma unroll
        for (int s = 0; s < kEllUnroll; ++s) {
            if (s < a.ell_w) {
                const vec4_t<T> vc = ld4(&v[cols[s]]);
                hx += vals[s] * vc.x; hy += vals[s] * vc.y; hz += vals[s] * vc.z;
            }
        }
    } else {
        for (int s = 0; s < a.ell_w; ++s) {
            const int c = __ldg(&a.ell_col[(size_t)s * nF + i]);
            const T kd = __ldg(&a.ell_val[(size_t)s * nF + i]) * a.inv_diag[c];
            const vec4_t<T> vc = ld4(&v[c]);
            hx += kd * vc.x; hy += kd * vc.y; hz += kd * vc.z;
        }
    }
    if (a.cdiag != nullptr) {
        const vec4_t<T> vi = ld4(&v[i]);
        const T kd = a.cdiag[i] * a.inv_diag[i];
        hx += kd * vi.x; hy += kd * vi.y; hz += kd * vi.z;
    }
    return make4<T>(hx, hy, hz, T(0));
}

// K_ff D^-1 in ELL: kd[s][i] = K[s][i] / K_{col,col}
template <typename T>
__global__ void k_scale_ell(int nF, int ell_w, const int* __restrict__ ell_col, const T* __restrict__ ell_val,
                            const T* __restrict__ inv_diag, T* kd) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nF) return;
    for (int s = 0; s < ell_w; ++s) {
        const size_t k = (size_t)s * nF + i;
        kd[k] = ell_val[k] * inv_diag[ell_col[k]];
    }
}

// POLY = true: preconditioner M^-1 = w D^-1 (2 I - w K D^-1) (one Neumann step
// on weighted Jacobi; SPD while w lambda_max(D^-1 K) < 2, w set from the
// Gershgorin bound at assembly).  It roughly halves the CG iterations at C3.
// h = K D^-1 r is carried alongside r (h -= alpha K D^-1 q, with q read at
// the neighbour rows after the alpha barrier), so applying M^-1 costs one
// SpMV inside the existing update phase and no extra grid barrier; only the
// first application (h0 from r0) needs one more barrier, taken only when the
// initial residual is above tolerance.
template <typename T, bool POLY = false>
__device__ __forceinline__ void pcg_classic_body(const PcgArgs<T>& a, cg::grid_group& grid, double* smem,
                                                 double* red, bool coherent_corners) {
    pcg_mark(0);
    pcg_entry(a);
    const int nF = a.nF;
    const int chunk = (nF + gridDim.x - 1) / gridDim.x;
    const int row0 = blockIdx.x * chunk;
    const int row1 = min(nF, row0 + chunk);
    int parity = 0;
    double rz[3], rzp[3] = {1.0, 1.0, 1.0}, rr, bb;
    // warm start: PD round k of a frame begins from a guess of its correction, the linear
    // extrapolation of the previous two frames' round-k corrections (same solution to the
    // tolerance, fewer CG iterations)
    const int pdi_w = a.pd_iter_dev != nullptr ? *a.pd_iter_dev : a.pd_iter;
    const bool warm = POLY && a.warm != nullptr && a.init == INIT_PD && pdi_w < a.warm_rounds;
    const bool poly = POLY && (a.poly_rounds <= 0 || a.init != INIT_PD || pdi_w < a.poly_rounds);
    vec4_t<T>* const wb = warm ? a.warm + (size_t)pdi_w * nF : nullptr;

    // ---- init: residual, z = D^-1 r, p0 = 0, dx = 0
    if (!poly) {
        double acc[5] = {0, 0, 0, 0, 0};     // rz x3, rr, bb
        for (int i = row0 + threadIdx.x; i < row1; i += blockDim.x) {
            T rx, ry, rzv;
            init_residual_row(a, i, coherent_corners, rx, ry, rzv, acc[4]);
            if (warm) {
                const vec4_t<T> kw = k_row(a, wb, i);
                rx -= kw.x; ry -= kw.y; rzv -= kw.z;
            }
            const T d = a.inv_diag[i];
            const vec4_t<T> zi = make4<T>(d * rx, d * ry, d * rzv, T(0));
            a.r[i] = make4<T>(rx, ry, rzv, T(0));
            a.z[i] = zi;
            a.p0[i] = make4<T>(T(0), T(0), T(0), T(0));
            a.dx[i] = warm ? ld4(&wb[i]) : make4<T>(T(0), T(0), T(0), T(0));
            acc[0] += (double)rx * zi.x;
            acc[1] += (double)ry * zi.y;
            acc[2] += (double)rzv * zi.z;
            acc[3] += (double)rx * rx + (double)ry * ry + (double)rzv * rzv;
        }
        pcg_allreduce<5>(grid, a.partials, parity, acc, red, smem);
        for (int c = 0; c < 3; ++c) rz[c] = red[c];
        rr = red[3];
        bb = red[4];
    } else {
        {
            double acc[2] = {0, 0};          // rr, bb
            for (int i = row0 + threadIdx.x; i < row1; i += blockDim.x) {
                T rx, ry, rzv;
                init_residual_row(a, i, coherent_corners, rx, ry, rzv, acc[1]);
                vec4_t<T> d0 = make4<T>(T(0), T(0), T(0), T(0));
                if (warm) {
                    // start from the previous frame's first correction: r -= K dx0
                    d0 = ld4(&wb[i]);
                    const vec4_t<T> kw = k_row(a, wb, i);
                    rx -= kw.x; ry -= kw.y; rzv -= kw.z;
                }
                a.r[i] = make4<T>(rx, ry, rzv, T(0));
                a.p0[i] = make4<T>(T(0), T(0), T(0), T(0));
                a.dx[i] = d0;
                acc[0] += (double)rx * rx + (double)ry * ry + (double)rzv * rzv;
            }
            pcg_allreduce<2>(grid, a.partials, parity, acc, red, smem);
            rr = red[0];
            bb = red[1];
        }
        rz[0] = rz[1] = rz[2] = 0.0;
        if (rr > a.tol * a.tol * bb && a.max_iters > 0) {
            const T w = (T)a.omega;
            double acc[3] = {0, 0, 0};
            for (int i = row0 + threadIdx.x; i < row1; i += blockDim.x) {
                const vec4_t<T> hi = kdinv_row(a, a.r, i);
                const vec4_t<T> ri = ld4(&a.r[i]);
                const T wd = w * a.inv_diag[i];
                const vec4_t<T> zi = make4<T>(wd * (T(2) * ri.x - w * hi.x), wd * (T(2) * ri.y - w * hi.y),
                                              wd * (T(2) * ri.z - w * hi.z), T(0));
                a.h[i] = hi;
                a.z[i] = zi;
                acc[0] += (double)ri.x * zi.x;
                acc[1] += (double)ri.y * zi.y;
                acc[2] += (double)ri.z * zi.z;
            }
            pcg_allreduce<3>(grid, a.partials, parity, acc, red, smem);
            for (int c = 0; c < 3; ++c) rz[c] = red[c];
        }
    }

    int it = 0;
    for (;; ++it) {
        if (!(rr > a.tol * a.tol * bb) || it >= a.max_iters) break;   // also stops on NaN
        double beta[3];
        for (int c = 0; c < 3; ++c) beta[c] = (it == 0 || rzp[c] == 0.0) ? 0.0 : rz[c] / rzp[c];
        const T bx = (T)beta[0], by = (T)beta[1], bz = (T)beta[2];
        const vec4_t<T>* pold = (it & 1) ? a.p1 : a.p0;
        vec4_t<T>* pnew = (it & 1) ? a.p0 : a.p1;
        double pq[3];
        // ---- phase A: p_new = z + beta p_old; q = K_ff p_new
        {
            double acc[3] = {0, 0, 0};
            for (int i = row0 + threadIdx.x; i < row1; i += blockDim.x) {
                T qx = 0, qy = 0, qz = 0;
                // padded ELL (pad = own column, value 0): fixed trip count, all
                // column/value loads issued before the gathers
                if (a.ell_w <= kEllUnroll) {
                    int cols[kEllUnroll];
                    T vals[kEllUnroll];
#pragma unroll
                    for (int s = 0; s < kEllUnroll; ++s) {
                        cols[s] = s < a.ell_w ? __ldg(&a.ell_col[(size_t)s * nF + i]) : i;
                        vals[s] = s < a.ell_w ? __ldg(&a.ell_val[(size_t)s * nF + i]) : T(0);
                    }
#pragma unroll
                    for (int s = 0; s < kEllUnroll; ++s) {
                        if (s < a.ell_w) {
                            const vec4_t<T> zc = ld4(&a.z[cols[s]]);
                            const vec4_t<T> pc = ld4(&pold[cols[s]]);
                            qx += vals[s] * (zc.x + bx * pc.x);
                            qy += vals[s] * (zc.y + by * pc.y);
                            qz += vals[s] * (zc.z + bz * pc.z);
                        }
                    }
                } else {
                    for (int s = 0; s < a.ell_w; ++s) {
                        const int col = __ldg(&a.ell_col[(size_t)s * nF + i]);
                        const T kv = __ldg(&a.ell_val[(size_t)s * nF + i]);
                        const vec4_t<T> zc = ld4(&a.z[col]);
                        const vec4_t<T> pc = ld4(&pold[col]);
                        qx += kv * (zc.x + bx * pc.x);
                        qy += kv * (zc.y + by * pc.y);
                        qz += kv * (zc.z + bz * pc.z);
                    }
                }
                const vec4_t<T> zi = ld4(&a.z[i]);
                const vec4_t<T> pi = ld4(&pold[i]);
                const vec4_t<T> pn = make4<T>(zi.x + bx * pi.x, zi.y + by * pi.y, zi.z + bz * pi.z, T(0));
                if (a.cdiag != nullptr) {
                    const T cd = a.cdiag[i];
                    qx += cd * pn.x; qy += cd * pn.y; qz += cd * pn.z;
                }
                pnew[i] = pn;
                a.q[i] = make4<T>(qx, qy, qz, T(0));
                acc[0] += (double)pn.x * qx;
                acc[1] += (double)pn.y * qy;
                acc[2] += (double)pn.z * qz;
            }
            pcg_allreduce<3>(grid, a.partials, parity, acc, red, smem);
            for (int c = 0; c < 3; ++c) pq[c] = red[c];
        }
        // ---- phase B: dx += alpha p; r -= alpha q; z = D^-1 r
        {
            double alpha[3];
            for (int c = 0; c < 3; ++c) alpha[c] = pq[c] != 0.0 ? rz[c] / pq[c] : 0.0;
            const T ax = (T)alpha[0], ay = (T)alpha[1], az = (T)alpha[2];
            double acc[4] = {0, 0, 0, 0};
            for (int i = row0 + threadIdx.x; i < row1; i += blockDim.x) {
                const vec4_t<T> pn = ld4(&pnew[i]);
                const vec4_t<T> qi = ld4(&a.q[i]);
                vec4_t<T> d = ld4(&a.dx[i]);
                vec4_t<T> ri = ld4(&a.r[i]);
                d.x += ax * pn.x; d.y += ay * pn.y; d.z += az * pn.z;
                ri.x -= ax * qi.x; ri.y -= ay * qi.y; ri.z -= az * qi.z;
                const T dg = a.inv_diag[i];
                vec4_t<T> zi;
                if (poly) {
                    // h -= alpha K D^-1 q (q of the neighbour rows is complete after the alpha barrier)
                    const vec4_t<T> kq = kdinv_row(a, a.q, i);
                    vec4_t<T> hi = ld4(&a.h[i]);
                    hi.x -= ax * kq.x; hi.y -= ay * kq.y; hi.z -= az * kq.z;
                    a.h[i] = hi;
                    const T w = (T)a.omega, wd = w * dg;
                    zi = make4<T>(wd * (T(2) * ri.x - w * hi.x), wd * (T(2) * ri.y - w * hi.y),
                                  wd * (T(2) * ri.z - w * hi.z), T(0));
                } else {
                    zi = make4<T>(dg * ri.x, dg * ri.y, dg * ri.z, T(0));
                }
                a.dx[i] = d;
                a.r[i] = ri;
                a.z[i] = zi;
                acc[0] += (double)ri.x * zi.x;
                acc[1] += (double)ri.y * zi.y;
                acc[2] += (double)ri.z * zi.z;
                acc[3] += (double)ri.x * ri.x + (double)ri.y * ri.y + (double)ri.z * ri.z;
            }
            pcg_allreduce<4>(grid, a.partials, parity, acc, red, smem);
            for (int c = 0; c < 3; ++c) { rzp[c] = rz[c]; rz[c] = red[c]; }
            rr = red[3];
        }
    }
    // ---- finish: x += dx (PD mode), finite check.  Nothing to add after zero
    // iterations; a non-finite iterate then shows up as a non-finite residual.
    bool bad = a.init == INIT_PD && !(rr == rr && rr < INFINITY);
    if (it > 0 || bad || warm)
    for (int i = row0 + threadIdx.x; i < row1; i += blockDim.x) {
        const vec4_t<T> d = ld4(&a.dx[i]);
        if (a.init == INIT_PD) {
            vec4_t<T> xi = a.x[i];
            xi.x += d.x; xi.y += d.y; xi.z += d.z;
            a.x[i] = xi;
            if (warm) {
                if (a.warm_prev != nullptr && pdi_w < a.warm_extrap_rounds) {
                    vec4_t<T>* wp = a.warm_prev + (size_t)pdi_w * nF;
                    const vec4_t<T> dp = ld4(&wp[i]);
                    wp[i] = d;
                    const T be = (T)a.warm_beta;
                    wb[i] = make4<T>(d.x + be * (d.x - dp.x), d.y + be * (d.y - dp.y), d.z + be * (d.z - dp.z), T(0));
                } else {
                    wb[i] = d;
                }
            }
            bad |= !(isfinite(xi.x) && isfinite(xi.y) && isfinite(xi.z));
        } else {
            bad |= !(isfinite(d.x) && isfinite(d.y) && isfinite(d.z));
        }
    }
    pcg_mark(5);
    pcg_exit(a, bad, it, warm);
}

#ifndef VK_PCG_LB
#define VK_PCG_LB 768
#endif
template <typename T>
__global__ void __launch_bounds__(VK_PCG_LB) k_pcg_classic(PcgArgs<T> a) {
    cg::grid_group grid = cg::this_grid();
    __shared__ double smem[32 * 8];
    __shared__ double red[8];
    pcg_classic_body<T, false>(a, grid, smem, red, false);
}

#ifndef VK_POLY_MAXNREG
#define VK_POLY_MAXNREG 80     // 768 threads x 80 registers: one CTA per SM
#endif
template <typename T>
__global__ void __maxnreg__(VK_POLY_MAXNREG) k_pcg_poly(PcgArgs<T> a) {
    cg::grid_group grid = cg::this_grid();
    __shared__ double smem[32 * 8];
    __shared__ double red[8];
    pcg_classic_body<T, true>(a, grid, smem, red, false);
}

}  // namespace vk

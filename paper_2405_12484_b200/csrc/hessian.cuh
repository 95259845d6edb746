// Fitting-side second-order machinery, float64, caller node order.
//
//   k_hs_eval        per tet: F, (R, V), the elastic energy V (gs|F-R|^2 + gv|F-V|^2)
//                    (pdsolver.py:72-82), the gradient corners 2V P g_n with
//                    P = gs (F-R) + gv (F-V) (elastic_gradient, pdsolver.py:85-97), and
//                    optionally the coefficient-Jacobian products of gamma_jacobian^T lam
//                    (fitting.py:172-190): 2V <F-R, sum_n lam_n (x) g_n>, same with F-V.
//   k_hs_linearize   per tet: M_e = 2V (gs (I9 - dR/dF) + gv (I9 - dV/dF)) (pdsolver.py:100-118),
//                    9x9, stored as 81 planes; the exact element Hessian is D^T M_e D.
//   k_hs_apply       per tet: corners of D^T M_e D p (matrix-free exact Hessian product).
//   k_hs_block       per tet: the 12x12 D^T M_e D (for the assembled CSR).
//   k_hs_gather      per node: sum of its incidence run in tet order (np.add.at order),
//                    plus a diagonal shift; pinned dofs masked.
//   MINRES           preconditioned (|diag| Jacobi) Paige-Saunders MINRES on the free dofs,
//                    scalar recurrences on the device; every kernel of an iteration returns
//                    at once after convergence, so the host enqueues iterations in chunks.
// D[3i+j, 3n+i] = G[n,j] (volmesh.py:92-97): (D p)_{ij} = sum_n p_{n,i} G[n,j].
#pragma once

#include "jacobian.cuh"
#include "sl3.cuh"
#include "svd3.cuh"
#include "vk_common.cuh"

namespace vk {
namespace hs {

struct Args {
    int n, nE;
    const int4* tets;      // caller node ids
    const double* G;       // 12 planes of nE: G[(3n+j) nE + e] = shape_grad[e, n, j]
    const double* w;       // 2 planes: gs, gv
    const double* vol;     // V
    const int4* slot4;     // incidence-run position of each corner
    double* corner;        // 3 doubles per incidence, node-sorted runs
};

__device__ __forceinline__ void load_G(const Args& a, int e, double (&g)[4][3]) {
#pragma unroll
    for (int k = 0; k < 12; ++k) g[k / 3][k % 3] = __ldg(&a.G[(size_t)k * a.nE + e]);
}

__device__ __forceinline__ void grad_of(const double (&g)[4][3], const double* __restrict__ x, int4 t,
                                        double (&F)[3][3]) {
    const int id[4] = {t.x, t.y, t.z, t.w};
    double xs[4][3];
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int i = 0; i < 3; ++i) xs[m][i] = x[3 * (size_t)id[m] + i];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            F[i][j] = xs[0][i] * g[0][j] + xs[1][i] * g[1][j] + xs[2][i] * g[2][j] + xs[3][i] * g[3][j];
}

// corner_n = c * P g_n (the 2V factor is in c)
__device__ __forceinline__ void put_corners(const Args& a, int e, const double (&g)[4][3], const double (&P)[3][3],
                                            double c) {
    const int4 sl = __ldg(&a.slot4[e]);
    const int s4[4] = {sl.x, sl.y, sl.z, sl.w};
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int i = 0; i < 3; ++i)
            a.corner[3 * (size_t)s4[m] + i] = c * (P[i][0] * g[m][0] + P[i][1] * g[m][1] + P[i][2] * g[m][2]);
}

// R = U W^T, V = U diag(s) W^T of batch_projections (material.py:395-407)
__device__ __forceinline__ void rv_of(const double (&F)[3][3], double (&R)[3][3], double (&Vm)[3][3]) {
    double U[3][3], W[3][3], sg[3], s[3];
    svd3_rv(F, U, sg, W);
    sl3::project(sg, s, false);
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            R[i][j] = U[i][0] * W[j][0] + U[i][1] * W[j][1] + U[i][2] * W[j][2];
            Vm[i][j] = U[i][0] * s[0] * W[j][0] + U[i][1] * s[1] * W[j][1] + U[i][2] * s[2] * W[j][2];
        }
}

// energy (per tet), gradient corners (if want_grad) and J^T lam (if lam != nullptr: jt[e], jt[nE + e])
__global__ void __launch_bounds__(128) k_hs_eval(Args a, const double* __restrict__ x, int want_grad,
                                                 double* __restrict__ energy, const double* __restrict__ lam,
                                                 double* __restrict__ jt) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= a.nE) return;
    double g[4][3], F[3][3], R[3][3], Vm[3][3];
    load_G(a, e, g);
    const int4 t = __ldg(&a.tets[e]);
    grad_of(g, x, t, F);
    rv_of(F, R, Vm);
    const double vol = __ldg(&a.vol[e]);
    const double ws = __ldg(&a.w[e]), wv = __ldg(&a.w[(size_t)a.nE + e]);
    double ds = 0.0, dv = 0.0;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const double r = F[i][j] - R[i][j], v = F[i][j] - Vm[i][j];
            ds += r * r;
            dv += v * v;
        }
    if (energy) energy[e] = vol * (ws * ds + wv * dv);
    if (want_grad) {
        double P[3][3];
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) P[i][j] = ws * (F[i][j] - R[i][j]) + wv * (F[i][j] - Vm[i][j]);
        put_corners(a, e, g, P, 2.0 * vol);
    }
    if (lam) {
        double L[3][3];
        grad_of(g, lam, t, L);
        const double v2 = 2.0 * vol;
        double js = 0.0, jv = 0.0;
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                js += (F[i][j] - R[i][j]) * L[i][j];
                jv += (F[i][j] - Vm[i][j]) * L[i][j];
            }
        jt[e] = v2 * js;
        jt[(size_t)a.nE + e] = v2 * jv;
    }
}

// M_e = 2V (gs (I - LR) + gv (I - LV)), 81 planes (the 2V factor folded in)
__global__ void __launch_bounds__(64) k_hs_linearize(Args a, const double* __restrict__ x, double* __restrict__ M) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= a.nE) return;
    double g[4][3], F[3][3];
    load_G(a, e, g);
    grad_of(g, x, __ldg(&a.tets[e]), F);
    const double ws = __ldg(&a.w[e]), wv = __ldg(&a.w[(size_t)a.nE + e]);
    hessian_block9(F, ws, wv, 2.0 * __ldg(&a.vol[e]), M + e, (size_t)a.nE);
}

// corners of (D^T M D) p
__global__ void __launch_bounds__(128) k_hs_apply(Args a, const double* __restrict__ M, const double* __restrict__ p,
                                                  const int* __restrict__ done) {
    if (done && *done) return;
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= a.nE) return;
    double g[4][3], dF[3][3];
    load_G(a, e, g);
    grad_of(g, p, __ldg(&a.tets[e]), dF);
    double Y[3][3];
#pragma unroll
    for (int r = 0; r < 9; ++r) {
        double acc = 0.0;
#pragma unroll
        for (int c = 0; c < 9; ++c) acc += __ldg(&M[(size_t)(9 * r + c) * a.nE + e]) * dF[c / 3][c % 3];
        Y[r / 3][r % 3] = acc;
    }
    put_corners(a, e, g, Y, 1.0);
}

// He = D^T M D (12 x 12, row-major, dof order 3n+i), per tet
__global__ void __launch_bounds__(64) k_hs_block(Args a, const double* __restrict__ M, double* __restrict__ He) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= a.nE) return;
    double g[4][3];
    load_G(a, e, g);
    // (M D)[r, 3n+i] = sum_j M[r, 3i+j] G[n,j]; He[3m+k, 3n+i] = sum_l G[m,l] (M D)[3k+l, 3n+i]
    for (int n = 0; n < 4; ++n)
        for (int i = 0; i < 3; ++i) {
            double MD[9];
            for (int r = 0; r < 9; ++r) {
                double acc = 0.0;
                for (int j = 0; j < 3; ++j) acc += __ldg(&M[(size_t)(9 * r + 3 * i + j) * a.nE + e]) * g[n][j];
                MD[r] = acc;
            }
            for (int m = 0; m < 4; ++m)
                for (int k = 0; k < 3; ++k) {
                    double acc = 0.0;
                    for (int l = 0; l < 3; ++l) acc += g[m][l] * MD[3 * k + l];
                    He[(size_t)144 * e + 12 * (3 * m + k) + 3 * n + i] = acc;
                }
        }
}

// assembled CSR values: one thread per (node, component) row, incident tets in tet order;
// columns are the node's sorted neighbours x 3
__global__ void k_hs_csr_fill(int n, int nE, const int* __restrict__ inc_ptr, const int* __restrict__ inc_code,
                              const int4* __restrict__ tets, const int* __restrict__ nb_ptr,
                              const int* __restrict__ nb_col, const double* __restrict__ He,
                              const long long* __restrict__ row_ptr, double* __restrict__ data) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= 3 * n) return;
    const int i = r / 3, c = r % 3;
    const int nb0 = nb_ptr[i], deg = nb_ptr[i + 1] - nb0;
    double* row = data + row_ptr[r];
    for (int k = 0; k < 3 * deg; ++k) row[k] = 0.0;
    for (int k = inc_ptr[i]; k < inc_ptr[i + 1]; ++k) {
        const int code = inc_code[k];
        const int am = code / nE, e = code % nE;
        const int4 t = tets[e];
        const int id[4] = {t.x, t.y, t.z, t.w};
        for (int b = 0; b < 4; ++b) {
            int pos = 0;
            while (nb_col[nb0 + pos] != id[b]) ++pos;
            for (int d = 0; d < 3; ++d) row[3 * pos + d] += He[(size_t)144 * e + 12 * (3 * am + c) + 3 * b + d];
        }
    }
}

// y_i = sum of the node's corners (tet order) + shift_i p_i, zero on pinned nodes
__global__ void k_hs_gather(int n, const int* __restrict__ inc_ptr, const double* __restrict__ corner,
                            const unsigned char* __restrict__ pinned, const double* __restrict__ shift,
                            const double* __restrict__ p, double* __restrict__ y, const int* __restrict__ done) {
    if (done && *done) return;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int k = inc_ptr[i]; k < inc_ptr[i + 1]; ++k) {
        s0 += corner[3 * (size_t)k];
        s1 += corner[3 * (size_t)k + 1];
        s2 += corner[3 * (size_t)k + 2];
    }
    if (pinned && pinned[i]) s0 = s1 = s2 = 0.0;
    else if (shift) {
        const double sh = shift[i];
        s0 += sh * p[3 * (size_t)i];
        s1 += sh * p[3 * (size_t)i + 1];
        s2 += sh * p[3 * (size_t)i + 2];
    }
    y[3 * (size_t)i] = s0;
    y[3 * (size_t)i + 1] = s1;
    y[3 * (size_t)i + 2] = s2;
}

// exact-Hessian diagonal: per-tet corners of diag(D^T M D)
__global__ void __launch_bounds__(128) k_hs_diag(Args a, const double* __restrict__ M) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= a.nE) return;
    double g[4][3];
    load_G(a, e, g);
    const int4 sl = __ldg(&a.slot4[e]);
    const int s4[4] = {sl.x, sl.y, sl.z, sl.w};
    for (int m = 0; m < 4; ++m)
        for (int i = 0; i < 3; ++i) {
            double acc = 0.0;
            for (int j = 0; j < 3; ++j)
                for (int l = 0; l < 3; ++l)
                    acc += g[m][j] * __ldg(&M[(size_t)(9 * (3 * i + j) + 3 * i + l) * a.nE + e]) * g[m][l];
            a.corner[3 * (size_t)s4[m] + i] = acc;
        }
}

// deterministic block partial sums of a per-index array (fixed grid; thread 0 of the
// scalar kernel adds the partials in block order)
__global__ void k_hs_sum_partials(long long n, const double* __restrict__ v, double* __restrict__ partials) {
    __shared__ double sm[64];
    double acc[1] = {0.0};
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        acc[0] += v[i];
    block_sum<1>(acc, sm);
    if (threadIdx.x == 0) partials[blockIdx.x] = acc[0];
}

__global__ void k_hs_sum_final(int nb, const double* __restrict__ partials, double* out) {
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s += partials[b];
    *out = s;
}

// ---------------------------------------------------------------------------
// MINRES (Paige-Saunders, preconditioned), the scalar state lives on the device
struct MinresState {
    double beta1, beta, oldb, alfa, dbar, epsln, oldeps, phibar, phi, cs, sn, delta, denom, tol;
    int itn, done, last_s2, breakdown;
};

constexpr int kMrBlocks = 296;     // 2 x 148 SMs: fixed reduction grid

// dot partials of a.b over m entries
__device__ __forceinline__ void dot_partial(long long m, const double* __restrict__ a, const double* __restrict__ b,
                                            double* partials) {
    __shared__ double sm[64];
    double acc[1] = {0.0};
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x)
        acc[0] += a[i] * b[i];
    block_sum<1>(acc, sm);
    if (threadIdx.x == 0) partials[blockIdx.x] = acc[0];
}

__device__ __forceinline__ double sum_partials(const double* partials) {
    double s = 0.0;
    for (int b = 0; b < kMrBlocks; ++b) s += partials[b];
    return s;
}

// r1 = r2 = b (x0 = 0), y = Dinv b, partial b.y
__global__ void k_mr_init(long long m, const double* __restrict__ b, const double* __restrict__ dinv, double* r1,
                          double* r2, double* y, double* x, double* w, double* w2, double* partials) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x) {
        const double bi = b[i];
        r1[i] = bi;
        r2[i] = bi;
        y[i] = dinv[i] * bi;
        x[i] = 0.0;
        w[i] = 0.0;
        w2[i] = 0.0;
    }
    dot_partial(m, b, y, partials);
}

__global__ void k_mr_init_scalar(MinresState* st, const double* partials, double tol) {
    const double b2 = sum_partials(partials);
    MinresState s{};
    s.tol = tol;
    s.beta1 = b2 > 0.0 ? sqrt(b2) : 0.0;
    s.beta = s.beta1;
    s.oldb = 0.0;
    s.dbar = 0.0;
    s.epsln = 0.0;
    s.phibar = s.beta1;
    s.cs = -1.0;
    s.sn = 0.0;
    s.itn = 0;
    s.last_s2 = -1;
    s.done = (b2 <= 0.0) ? 1 : 0;       // b = 0: x = 0 exactly
    s.breakdown = (b2 < 0.0) ? 1 : 0;
    *st = s;
}

// v = y / beta
__global__ void k_mr_v(long long m, const MinresState* __restrict__ st, const double* __restrict__ y, double* v) {
    if (st->done) return;
    const double s = 1.0 / st->beta;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x)
        v[i] = s * y[i];
}

// y = A v - (beta/oldb) r1 (first iteration: A v); partial v.y
__global__ void k_mr_a(long long m, const MinresState* __restrict__ st, const double* __restrict__ Av,
                       const double* __restrict__ v, const double* __restrict__ r1, double* y, double* partials) {
    if (st->done) return;
    const double c = st->itn > 0 ? st->beta / st->oldb : 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x)
        y[i] = Av[i] - c * r1[i];
    __syncthreads();
    dot_partial(m, v, y, partials);
}

__global__ void k_mr_s1(MinresState* st, const double* partials) {
    if (st->done) return;
    st->alfa = sum_partials(partials);
}

// y -= (alfa/beta) r2; r1 = r2; r2 = y; y = Dinv r2; partial r2.y
__global__ void k_mr_b(long long m, const MinresState* __restrict__ st, double* y, double* r1, double* r2,
                       const double* __restrict__ dinv, double* partials) {
    if (st->done) return;
    const double c = st->alfa / st->beta;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x) {
        const double yi = y[i] - c * r2[i];
        r1[i] = r2[i];
        r2[i] = yi;
        y[i] = dinv[i] * yi;
    }
    __syncthreads();
    dot_partial(m, r2, y, partials);
}

__global__ void k_mr_s2(MinresState* st, const double* partials, int iter) {
    if (st->done) return;
    MinresState s = *st;
    const double b2 = sum_partials(partials);
    s.oldb = s.beta;
    if (b2 < 0.0) { s.breakdown = 1; s.done = 1; *st = s; return; }
    s.beta = sqrt(b2);
    s.oldeps = s.epsln;
    s.delta = s.cs * s.dbar + s.sn * s.alfa;
    const double gbar = s.sn * s.dbar - s.cs * s.alfa;
    s.epsln = s.sn * s.beta;
    s.dbar = -s.cs * s.beta;
    double gamma = sqrt(gbar * gbar + s.beta * s.beta);
    if (gamma < 2.220446049250313e-16) gamma = 2.220446049250313e-16;
    s.cs = gbar / gamma;
    s.sn = s.beta / gamma;
    s.phi = s.cs * s.phibar;
    s.phibar = s.sn * s.phibar;
    s.denom = 1.0 / gamma;
    s.itn = s.itn + 1;
    s.last_s2 = iter;
    // converged (preconditioned residual estimate) or Lanczos breakdown (exact solve)
    if (s.phibar <= s.tol * s.beta1 || s.beta == 0.0) s.done = 1;
    *st = s;
}

// w_new = (v - oldeps w2 - delta w) denom; w2 = w; w = w_new; x += phi w_new; v = y / beta
__global__ void k_mr_c(long long m, const MinresState* __restrict__ st, int iter, double* v, const double* __restrict__ y,
                       double* w, double* w2, double* x) {
    if (st->last_s2 != iter) return;
    const double oe = st->oldeps, de = st->delta, dn = st->denom, ph = st->phi;
    const double sb = st->beta > 0.0 ? 1.0 / st->beta : 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x) {
        const double wo = w[i];
        const double wn = (v[i] - oe * w2[i] - de * wo) * dn;
        w2[i] = wo;
        w[i] = wn;
        x[i] += ph * wn;
        v[i] = sb * y[i];
    }
}

}  // namespace hs
}  // namespace vk

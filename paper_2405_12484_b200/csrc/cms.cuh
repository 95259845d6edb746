// Reference-compatible domain-decomposed global solve:
// the component-mode-synthesis subspace apply x = T K_red^-1 T^T b and the
// aggregated / Chebyshev weighted-Jacobi refinement `a_jacobi_refine`
// (pdsolver.py:632-703), with the reference's control flow: recursive
// residual, per-column residual history, best-iterate tracking, divergence
// stop at 10x the best residual.  Up to three right-hand-side columns run in
// lockstep inside one persistent cooperative kernel; a diverged column freezes
// (the reference solves columns one by one and breaks that column's loop).
#pragma once

#include <cooperative_groups.h>

#include "vk_common.cuh"

namespace vk {

namespace cgr = cooperative_groups;

template <typename T>
struct AJArgs {
    int nF, ell_w;
    const int* ell_col;
    const T* ell_val;
    const double* diag;          // float64 diagonal of K_ff
    const vec4_t<T>* b;          // rhs (3 columns)
    vec4_t<T>* x;                // in: x0, out: result
    vec4_t<T>* r;                // residual (plain) / b - K x (Chebyshev)
    vec4_t<T>* s;
    vec4_t<T>* e;                // e (plain) / x_prev (Chebyshev)
    vec4_t<T>* cs0;
    vec4_t<T>* cs1;
    vec4_t<T>* best;
    double* partials;            // 2 * grid * 8
    double* hist;                // [(steps + 1) x 3] residual norms per column
    int* n_hist;                 // [3]
    int* diverged;               // [3]
    int sweeps, aggregation;
    double omega, rho;
    int ncols;                   // active columns (1..3)
};

template <typename T>
__device__ __forceinline__ vec4_t<T> spmv_row(const AJArgs<T>& a, const vec4_t<T>* v, int i) {
    T qx = 0, qy = 0, qz = 0;
    for (int sl = 0; sl < a.ell_w; ++sl) {
        const int col = __ldg(&a.ell_col[(size_t)sl * a.nF + i]);
        const T kv = __ldg(&a.ell_val[(size_t)sl * a.nF + i]);
        const vec4_t<T> c = ld4(&v[col]);
        qx += kv * c.x; qy += kv * c.y; qz += kv * c.z;
    }
    return make4<T>(qx, qy, qz, T(0));
}

template <int NV>
__device__ __forceinline__ void aj_allreduce(cgr::grid_group& grid, double* partials, int& parity, double (&acc)[NV],
                                             double* red, double* smem) {
    block_sum<NV>(acc, smem);
    double* P = partials + (size_t)parity * gridDim.x * 8;
    if (threadIdx.x == 0)
#pragma unroll
        for (int k = 0; k < NV; ++k) P[blockIdx.x * 8 + k] = acc[k];
    grid.sync();
    reduce_partials_all<NV>(P, red, smem);
    parity ^= 1;
}

// Per-column bookkeeping, identical in every thread of the grid.
struct AJState {
    double best[3], last[3];
    int nh[3];
    bool act[3], div[3];
};

__device__ __forceinline__ void aj_record(AJState& st, const double* red, double* hist, bool (&improve)[3],
                                          bool writer) {
    for (int c = 0; c < 3; ++c) {
        improve[c] = false;
        if (!st.act[c]) continue;
        const double rn = sqrt(red[c]);
        if (writer) hist[st.nh[c] * 3 + c] = rn;
        st.nh[c]++;
        st.last[c] = rn;
        if (rn < st.best[c]) { st.best[c] = rn; improve[c] = true; }
        if (rn > 10.0 * st.best[c]) { st.div[c] = true; st.act[c] = false; }
    }
}

template <typename T>
__device__ __forceinline__ void aj_save_best(const AJArgs<T>& a, const bool (&improve)[3], int tid, int stride) {
    if (!(improve[0] || improve[1] || improve[2])) return;
    for (int i = tid; i < a.nF; i += stride) {
        const vec4_t<T> xi = a.x[i];
        vec4_t<T> bi = a.best[i];
        if (improve[0]) bi.x = xi.x;
        if (improve[1]) bi.y = xi.y;
        if (improve[2]) bi.z = xi.z;
        a.best[i] = bi;
    }
}

template <typename T>
__device__ __forceinline__ void aj_finish(const AJArgs<T>& a, const AJState& st, int tid, int stride) {
    bool pick[3];
    for (int c = 0; c < 3; ++c) pick[c] = st.div[c] || st.last[c] > st.best[c];
    for (int i = tid; i < a.nF; i += stride) {
        vec4_t<T> xi = a.x[i];
        const vec4_t<T> bi = a.best[i];
        if (pick[0]) xi.x = bi.x;
        if (pick[1]) xi.y = bi.y;
        if (pick[2]) xi.z = bi.z;
        a.x[i] = xi;
    }
    if (tid == 0)
        for (int c = 0; c < 3; ++c) {
            a.diverged[c] = st.div[c] ? 1 : 0;
            a.n_hist[c] = st.nh[c];
        }
}

// r = b - K x, best = x, history[0]
template <typename T>
__device__ __forceinline__ void aj_start(const AJArgs<T>& a, AJState& st, cgr::grid_group& grid, int& parity,
                                         double* red, double* smem, int tid, int stride) {
    double acc[3] = {0, 0, 0};
    for (int i = tid; i < a.nF; i += stride) {
        const vec4_t<T> kx = spmv_row(a, a.x, i);
        const vec4_t<T> bi = a.b[i];
        const vec4_t<T> ri = make4<T>(bi.x - kx.x, bi.y - kx.y, bi.z - kx.z, T(0));
        a.r[i] = ri;
        a.best[i] = a.x[i];
        acc[0] += (double)ri.x * ri.x; acc[1] += (double)ri.y * ri.y; acc[2] += (double)ri.z * ri.z;
    }
    aj_allreduce<3>(grid, a.partials, parity, acc, red, smem);
    for (int c = 0; c < 3; ++c) {
        st.best[c] = sqrt(red[c]);
        st.last[c] = st.best[c];
        st.nh[c] = 1;
        st.act[c] = c < a.ncols;
        st.div[c] = false;
        if (tid == 0) a.hist[c] = st.best[c];
    }
}

// Plain aggregated sweeps (pdsolver.py:683-703).  Same arithmetic as the reference loop;
// two grid barriers per aggregated sweep at aggregation 2 (instead of three):
//  - the sweep's first correction cs = omega D^-1 r is formed in the previous sweep's
//    residual pass, unmasked, and masked per column (x 1 or x 0, exact) where it is read;
//  - the best-iterate copy of an improving sweep is deferred into the next sweep's first
//    pass (x is not touched there) or the final pass.
template <typename T>
__global__ void __launch_bounds__(256) k_ajacobi(AJArgs<T> a) {
    cgr::grid_group grid = cgr::this_grid();
    __shared__ double smem[32 * 8];
    __shared__ double red[8];
    const int nF = a.nF;
    const int stride = gridDim.x * blockDim.x;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    int parity = 0;
    AJState st;
    const T om = (T)a.omega;
    // r = b - K x, best = x, cs0 = omega D^-1 r, |r|
    {
        double acc[3] = {0, 0, 0};
        for (int i = tid; i < nF; i += stride) {
            const vec4_t<T> kx = spmv_row(a, a.x, i);
            const vec4_t<T> bi = a.b[i];
            const vec4_t<T> ri = make4<T>(bi.x - kx.x, bi.y - kx.y, bi.z - kx.z, T(0));
            a.r[i] = ri;
            a.best[i] = a.x[i];
            const T di = (T)(1.0 / a.diag[i]);
            a.cs0[i] = make4<T>(om * (di * ri.x), om * (di * ri.y), om * (di * ri.z), T(0));
            acc[0] += (double)ri.x * ri.x; acc[1] += (double)ri.y * ri.y; acc[2] += (double)ri.z * ri.z;
        }
        aj_allreduce<3>(grid, a.partials, parity, acc, red, smem);
        for (int c = 0; c < 3; ++c) {
            st.best[c] = sqrt(red[c]);
            st.last[c] = st.best[c];
            st.nh[c] = 1;
            st.act[c] = c < a.ncols;
            st.div[c] = false;
            if (tid == 0) a.hist[c] = st.best[c];
        }
    }
    bool pend[3] = {false, false, false};           // best = x still owed for these columns
    for (int sw = 0; sw < a.sweeps; ++sw) {
        if (!(st.act[0] || st.act[1] || st.act[2])) break;
        const T m0 = st.act[0] ? T(1) : T(0), m1 = st.act[1] ? T(1) : T(0), m2 = st.act[2] ? T(1) : T(0);
        const T w0 = st.act[0] ? om : T(0), w1 = st.act[1] ? om : T(0), w2 = st.act[2] ? om : T(0);
        const bool owe = pend[0] || pend[1] || pend[2];
        for (int ag = 0; ag < a.aggregation; ++ag) {
            const vec4_t<T>* cur = (ag & 1) ? a.cs1 : a.cs0;
            vec4_t<T>* nxt = (ag & 1) ? a.cs0 : a.cs1;
            const bool more = ag + 1 < a.aggregation;
            for (int i = tid; i < nF; i += stride) {
                vec4_t<T> kc = spmv_row(a, cur, i);
                vec4_t<T> si, ei;
                if (ag == 0) {
                    // s = r - K (mask cs0); e = mask cs0 (the reference's s = r, cs, e = cs)
                    kc.x *= m0; kc.y *= m1; kc.z *= m2;
                    const vec4_t<T> ri = a.r[i], c0 = a.cs0[i];
                    si = make4<T>(ri.x - kc.x, ri.y - kc.y, ri.z - kc.z, T(0));
                    ei = make4<T>(m0 * c0.x, m1 * c0.y, m2 * c0.z, T(0));
                    if (owe) {
                        const vec4_t<T> xi = a.x[i];
                        vec4_t<T> bi = a.best[i];
                        if (pend[0]) bi.x = xi.x;
                        if (pend[1]) bi.y = xi.y;
                        if (pend[2]) bi.z = xi.z;
                        a.best[i] = bi;
                    }
                } else {
                    si = a.s[i];
                    si.x -= kc.x; si.y -= kc.y; si.z -= kc.z;
                    ei = a.e[i];
                }
                a.s[i] = si;
                if (more) {
                    const T di = (T)(1.0 / a.diag[i]);
                    const vec4_t<T> c = make4<T>(w0 * (di * si.x), w1 * (di * si.y), w2 * (di * si.z), T(0));
                    nxt[i] = c;
                    ei.x += c.x; ei.y += c.y; ei.z += c.z;
                }
                a.e[i] = ei;
            }
            if (more) grid.sync();
        }
        pend[0] = pend[1] = pend[2] = false;
        // x += e; r = s; |r|; next sweep's cs0 = omega D^-1 r
        double acc[3] = {0, 0, 0};
        for (int i = tid; i < nF; i += stride) {
            vec4_t<T> xi = a.x[i];
            const vec4_t<T> ei = a.e[i];
            xi.x += ei.x; xi.y += ei.y; xi.z += ei.z;
            a.x[i] = xi;
            const vec4_t<T> si = a.s[i];
            a.r[i] = si;
            const T di = (T)(1.0 / a.diag[i]);
            a.cs0[i] = make4<T>(om * (di * si.x), om * (di * si.y), om * (di * si.z), T(0));
            acc[0] += (double)si.x * si.x; acc[1] += (double)si.y * si.y; acc[2] += (double)si.z * si.z;
        }
        aj_allreduce<3>(grid, a.partials, parity, acc, red, smem);
        bool improve[3];
        aj_record(st, red, a.hist, improve, tid == 0);
        for (int c = 0; c < 3; ++c) pend[c] = improve[c];
    }
    if (pend[0] || pend[1] || pend[2]) aj_save_best(a, pend, tid, stride);
    aj_finish(a, st, tid, stride);
}

// Chebyshev semi-iterative variant (pdsolver.py:657-681): sweeps * aggregation
// steps y = x + omega D^-1 (b - K x), x_new = w (y - x_prev) + x_prev; the
// residual b - K x_new of each step is reused by the next one (one SpMV/step).
template <typename T>
__global__ void __launch_bounds__(256) k_chebyshev(AJArgs<T> a) {
    cgr::grid_group grid = cgr::this_grid();
    __shared__ double smem[32 * 8];
    __shared__ double red[8];
    const int nF = a.nF;
    const int stride = gridDim.x * blockDim.x;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    int parity = 0;
    AJState st;
    aj_start(a, st, grid, parity, red, smem, tid, stride);     // a.r = b - K x0
    for (int i = tid; i < nF; i += stride) a.e[i] = a.x[i];    // x_prev
    const double rho2 = a.rho * a.rho;
    double w = 1.0;
    const int total = a.sweeps * a.aggregation;
    for (int k = 0; k < total; ++k) {
        if (!(st.act[0] || st.act[1] || st.act[2])) break;
        const T om = (T)a.omega;
        const T ww = (T)(k == 0 ? 1.0 : w);
        // new iterate (own rows)
        for (int i = tid; i < nF; i += stride) {
            const vec4_t<T> xi = a.x[i], xp = a.e[i], ri = a.r[i];
            const T di = (T)(1.0 / a.diag[i]);
            vec4_t<T> xn;
            const T yx = xi.x + om * (di * ri.x), yy = xi.y + om * (di * ri.y), yz = xi.z + om * (di * ri.z);
            if (k == 0) {
                xn = make4<T>(yx, yy, yz, T(0));
            } else {
                xn = make4<T>(ww * (yx - xp.x) + xp.x, ww * (yy - xp.y) + xp.y, ww * (yz - xp.z) + xp.z, T(0));
            }
            xn.x = st.act[0] ? xn.x : xi.x;
            xn.y = st.act[1] ? xn.y : xi.y;
            xn.z = st.act[2] ? xn.z : xi.z;
            a.e[i] = xi;
            a.s[i] = xn;
        }
        grid.sync();
        double acc[3] = {0, 0, 0};
        for (int i = tid; i < nF; i += stride) {
            const vec4_t<T> kx = spmv_row(a, a.s, i);
            const vec4_t<T> bi = a.b[i];
            const vec4_t<T> ri = make4<T>(bi.x - kx.x, bi.y - kx.y, bi.z - kx.z, T(0));
            a.r[i] = ri;
            acc[0] += (double)ri.x * ri.x; acc[1] += (double)ri.y * ri.y; acc[2] += (double)ri.z * ri.z;
        }
        aj_allreduce<3>(grid, a.partials, parity, acc, red, smem);
        for (int i = tid; i < nF; i += stride) a.x[i] = a.s[i];
        w = (k == 0) ? 2.0 / (2.0 - rho2) : 4.0 / (4.0 - rho2 * w);
        bool improve[3];
        aj_record(st, red, a.hist, improve, tid == 0);
        aj_save_best(a, improve, tid, stride);
    }
    aj_finish(a, st, tid, stride);
}

// Power iteration for the spectral radius of I - omega D^-1 K (pdsolver.py:616-629),
// 3 independent columns (column 0 is the reference's); v is the start vector.
template <typename T>
__global__ void __launch_bounds__(256) k_power_rho(AJArgs<T> a, int iters, double* rho_out) {
    cgr::grid_group grid = cgr::this_grid();
    __shared__ double smem[32 * 8];
    __shared__ double red[8];
    const int nF = a.nF;
    const int stride = gridDim.x * blockDim.x;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    int parity = 0;
    // normalise v (held in a.x)
    double acc[3] = {0, 0, 0};
    for (int i = tid; i < nF; i += stride) {
        const vec4_t<T> v = a.x[i];
        acc[0] += (double)v.x * v.x; acc[1] += (double)v.y * v.y; acc[2] += (double)v.z * v.z;
    }
    aj_allreduce<3>(grid, a.partials, parity, acc, red, smem);
    double nrm[3] = {sqrt(red[0]), sqrt(red[1]), sqrt(red[2])};
    for (int i = tid; i < nF; i += stride) {
        const vec4_t<T> v = a.x[i];
        a.s[i] = make4<T>((T)(v.x / nrm[0]), (T)(v.y / nrm[1]), (T)(v.z / nrm[2]), T(0));
    }
    double rho[3] = {0, 0, 0};
    bool stop[3] = {false, false, false};
    for (int k = 0; k < iters; ++k) {
        grid.sync();
        double ac2[3] = {0, 0, 0};
        for (int i = tid; i < nF; i += stride) {
            const vec4_t<T> kv = spmv_row(a, a.s, i);
            const vec4_t<T> v = a.s[i];
            const T di = (T)(1.0 / a.diag[i]);
            const T om = (T)a.omega;
            const vec4_t<T> u = make4<T>(v.x - om * (di * kv.x), v.y - om * (di * kv.y), v.z - om * (di * kv.z), T(0));
            a.r[i] = u;
            ac2[0] += (double)u.x * u.x; ac2[1] += (double)u.y * u.y; ac2[2] += (double)u.z * u.z;
        }
        aj_allreduce<3>(grid, a.partials, parity, ac2, red, smem);
        for (int c = 0; c < 3; ++c) {
            const double nv = sqrt(red[c]);
            if (stop[c]) continue;
            if (nv < 1e-300) { rho[c] = 0.0; stop[c] = true; continue; }
            rho[c] = nv;
            nrm[c] = nv;
        }
        for (int i = tid; i < nF; i += stride) {
            const vec4_t<T> u = a.r[i];
            a.s[i] = make4<T>((T)(u.x / nrm[0]), (T)(u.y / nrm[1]), (T)(u.z / nrm[2]), T(0));
        }
    }
    if (tid == 0)
        for (int c = 0; c < 3; ++c) rho_out[c] = fmin(rho[c], 0.9999);
}

// CMS subspace apply with a dense basis (column-major T: n x m) and a dense
// symmetric K_red^-1 (m x m):  y = T^T b  (one warp per basis column),
// z = K_red^-1 y, x = T z (one thread per row).
template <typename T>
__global__ void k_tmv(int n, int m, const double* __restrict__ Tb, const vec4_t<T>* __restrict__ b, double* y) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= m) return;
    const double* col = Tb + (size_t)warp * n;
    double s0 = 0, s1 = 0, s2 = 0;
    for (int i = lane; i < n; i += 32) {
        const double t = col[i];
        const vec4_t<T> v = b[i];
        s0 += t * v.x; s1 += t * v.y; s2 += t * v.z;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s0 += __shfl_xor_sync(0xffffffffu, s0, o);
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    }
    if (lane == 0) { y[3 * warp] = s0; y[3 * warp + 1] = s1; y[3 * warp + 2] = s2; }
}
__global__ void k_symv3(int m, const double* __restrict__ A, const double* __restrict__ y, double* z) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    double s0 = 0, s1 = 0, s2 = 0;
    for (int j = 0; j < m; ++j) {
        const double a = A[(size_t)j * m + i];
        s0 += a * y[3 * j]; s1 += a * y[3 * j + 1]; s2 += a * y[3 * j + 2];
    }
    z[3 * i] = s0; z[3 * i + 1] = s1; z[3 * i + 2] = s2;
}
template <typename T>
__global__ void k_tv(int n, int m, const double* __restrict__ Tb, const double* __restrict__ z, vec4_t<T>* x) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double s0 = 0, s1 = 0, s2 = 0;
    for (int j = 0; j < m; ++j) {
        const double t = Tb[(size_t)j * n + i];
        s0 += t * z[3 * j]; s1 += t * z[3 * j + 1]; s2 += t * z[3 * j + 2];
    }
    x[i] = make4<T>((T)s0, (T)s1, (T)s2, T(0));
}


// ---------------------------------------------------------------------------
// Blocked CMS apply (the same T = [Phi blocks | I_b + Psi blocks], stored per domain).
// Domain d keeps A_d = [Phi_d | Psi_d restricted to its adjacent boundary columns],
// n_d x c_d column-major (rows = its interior nodes), so the zeros of the global T
// (pdsolver.py:560-575 stores them) are neither stored nor streamed:
//   T^T b: per (domain, 8-column tile) CTA, partial y_d = A_d^T b_d; then per global
//          column the (<= 2 for slabs) domain contributions plus b on the boundary rows,
//          summed in domain order (deterministic);
//   T z:   per (domain, row chunk) CTA with the domain's z entries staged in shared
//          memory, one thread per interior row; boundary rows copy z.
struct CmsBlocks {
    int ndom, nmodes, nb, ntiles;
    const double* A;             // concatenated blocks
    const long long* a_off;      // per domain offset into A
    const int* row_ptr;          // per domain range into rows
    const int* rows;             // interior free-node rows (internal order)
    const int* col_ptr;          // per domain range into colmap / y_d
    const int* colmap;           // global column of each local column
    const int* tile_dom;         // per tile: domain, first local column
    const int* tile_c0;
    const int* bnd;              // boundary free-node rows (global column nmodes + j)
    const int* ysrc_ptr;         // per global column: contributions in y_d
    const int* ysrc;
};

constexpr int kCmsTile = 8;

template <typename T>
__global__ void __launch_bounds__(256) k_cms_tb(CmsBlocks c, const vec4_t<T>* __restrict__ b, double* __restrict__ yd) {
    __shared__ double smem[32 * 3 * kCmsTile];
    const int t = blockIdx.x;
    const int d = c.tile_dom[t], c0 = c.tile_c0[t];
    const int r0 = c.row_ptr[d], nd = c.row_ptr[d + 1] - r0;
    const int ncol = c.col_ptr[d + 1] - c.col_ptr[d];
    const int nc = min(kCmsTile, ncol - c0);
    const double* A = c.A + c.a_off[d] + (size_t)c0 * nd;
    double acc[3 * kCmsTile];
#pragma unroll
    for (int k = 0; k < 3 * kCmsTile; ++k) acc[k] = 0.0;
    // two rows per thread per step: 16 basis loads in flight (HBM latency)
    const int bd = blockDim.x;
    for (int r = threadIdx.x; r < nd; r += 2 * bd) {
        const int r2 = r + bd;
        const bool two = r2 < nd;
        const vec4_t<T> bv = b[c.rows[r0 + r]];
        const vec4_t<T> bw = two ? b[c.rows[r0 + r2]] : make4<T>(T(0), T(0), T(0), T(0));
        double av[kCmsTile], aw[kCmsTile];
#pragma unroll
        for (int k = 0; k < kCmsTile; ++k) {
            av[k] = k < nc ? __ldg(&A[(size_t)k * nd + r]) : 0.0;
            aw[k] = (k < nc && two) ? __ldg(&A[(size_t)k * nd + r2]) : 0.0;
        }
        const double bx = (double)bv.x, by = (double)bv.y, bz = (double)bv.z;
        const double cx = (double)bw.x, cy = (double)bw.y, cz = (double)bw.z;
#pragma unroll
        for (int k = 0; k < kCmsTile; ++k) {
            acc[3 * k] += av[k] * bx + aw[k] * cx;
            acc[3 * k + 1] += av[k] * by + aw[k] * cy;
            acc[3 * k + 2] += av[k] * bz + aw[k] * cz;
        }
    }
    block_sum<3 * kCmsTile>(acc, smem);
    if (threadIdx.x == 0) {
        const int base = c.col_ptr[d] + c0;
        for (int k = 0; k < nc; ++k) {
            yd[3 * (size_t)(base + k)] = acc[3 * k];
            yd[3 * (size_t)(base + k) + 1] = acc[3 * k + 1];
            yd[3 * (size_t)(base + k) + 2] = acc[3 * k + 2];
        }
    }
}

template <typename T>
__global__ void k_cms_y(CmsBlocks c, int m, const vec4_t<T>* __restrict__ b, const double* __restrict__ yd,
                        double* __restrict__ y) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= m) return;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    if (g >= c.nmodes) {
        const vec4_t<T> bv = b[c.bnd[g - c.nmodes]];
        s0 = (double)bv.x; s1 = (double)bv.y; s2 = (double)bv.z;
    }
    for (int k = c.ysrc_ptr[g]; k < c.ysrc_ptr[g + 1]; ++k) {
        const int q = c.ysrc[k];
        s0 += yd[3 * (size_t)q]; s1 += yd[3 * (size_t)q + 1]; s2 += yd[3 * (size_t)q + 2];
    }
    y[3 * (size_t)g] = s0; y[3 * (size_t)g + 1] = s1; y[3 * (size_t)g + 2] = s2;
}

// grid: (row chunks, domains, column groups); dynamic smem = 3 * (max columns per group) doubles.
// Group g covers columns [g ncol / G, (g + 1) ncol / G) of its domain and writes a partial row sum
// to part[g * total_rows + row]; k_cms_tz_sum adds the G partials in group order (deterministic).
// Splitting the columns gives G times the CTAs (a domain has only ~13K rows) for the same bytes.
constexpr int kCmsTzGroups = 4;
template <typename T>
__global__ void __launch_bounds__(256) k_cms_tz(CmsBlocks c, const double* __restrict__ z, double* __restrict__ part,
                                                int total_rows) {
    extern __shared__ double zs[];
    const int d = blockIdx.y, gi = blockIdx.z, G = gridDim.z;
    const int r0 = c.row_ptr[d], nd = c.row_ptr[d + 1] - r0;
    const int q0 = c.col_ptr[d], ncol = c.col_ptr[d + 1] - q0;
    const int c0 = (int)((long long)gi * ncol / G), c1 = (int)((long long)(gi + 1) * ncol / G);
    const int nc = c1 - c0;
    for (int k = threadIdx.x; k < nc; k += blockDim.x) {
        const int g = c.colmap[q0 + c0 + k];
        zs[3 * k] = z[3 * (size_t)g]; zs[3 * k + 1] = z[3 * (size_t)g + 1]; zs[3 * k + 2] = z[3 * (size_t)g + 2];
    }
    __syncthreads();
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nd) return;
    const double* A = c.A + c.a_off[d] + (size_t)c0 * nd + r;
    // two interleaved accumulator sets and 8 loads in flight per thread (HBM latency)
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, u0 = 0.0, u1 = 0.0, u2 = 0.0;
    int k = 0;
    for (; k + 8 <= nc; k += 8) {
        double av[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) av[q] = __ldg(&A[(size_t)(k + q) * nd]);
#pragma unroll
        for (int q = 0; q < 8; q += 2) {
            s0 += av[q] * zs[3 * (k + q)]; s1 += av[q] * zs[3 * (k + q) + 1]; s2 += av[q] * zs[3 * (k + q) + 2];
            u0 += av[q + 1] * zs[3 * (k + q + 1)]; u1 += av[q + 1] * zs[3 * (k + q + 1) + 1];
            u2 += av[q + 1] * zs[3 * (k + q + 1) + 2];
        }
    }
    for (; k < nc; ++k) {
        const double a = __ldg(&A[(size_t)k * nd]);
        s0 += a * zs[3 * k]; s1 += a * zs[3 * k + 1]; s2 += a * zs[3 * k + 2];
    }
    double* o = part + 3 * ((size_t)gi * total_rows + r0 + r);
    o[0] = s0 + u0; o[1] = s1 + u1; o[2] = s2 + u2;
}

template <typename T>
__global__ void k_cms_tz_sum(CmsBlocks c, int total_rows, int G, const double* __restrict__ part,
                             vec4_t<T>* __restrict__ x) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= total_rows) return;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int g = 0; g < G; ++g) {
        const double* o = part + 3 * ((size_t)g * total_rows + i);
        s0 += o[0]; s1 += o[1]; s2 += o[2];
    }
    x[c.rows[i]] = make4<T>((T)s0, (T)s1, (T)s2, T(0));
}

// z = K_red^-1 y for the symmetric K_red^-1: one warp per row (row i = column i, contiguous),
// lanes stride the columns, warp-shuffle reduction
__global__ void __launch_bounds__(256) k_symv3_warp(int m, const double* __restrict__ A, const double* __restrict__ y,
                                                    double* __restrict__ z) {
    const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (i >= m) return;
    const double* row = A + (size_t)i * m;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int j = lane; j < m; j += 32) {
        const double a = __ldg(&row[j]);
        s0 += a * y[3 * j]; s1 += a * y[3 * j + 1]; s2 += a * y[3 * j + 2];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s0 += __shfl_xor_sync(0xffffffffu, s0, o);
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    }
    if (lane == 0) { z[3 * i] = s0; z[3 * i + 1] = s1; z[3 * i + 2] = s2; }
}

template <typename T>
__global__ void k_cms_xb(CmsBlocks c, const double* __restrict__ z, vec4_t<T>* __restrict__ x) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= c.nb) return;
    const size_t g = (size_t)(c.nmodes + j);
    x[c.bnd[j]] = make4<T>((T)z[3 * g], (T)z[3 * g + 1], (T)z[3 * g + 2], T(0));
}

// ---------------------------------------------------------------------------
// Device frame in cms mode (pd_step with GlobalSolver(mode="cms"), pdsolver.py:283-300):
//   b_f = (sum of the node's rhs corners, tet order) + (m/dt^2) xhat   (pdsolver.py:292-293)
//   x_f = a_jacobi_refine(K_ff, b_f - K_fp p, T K_red^-1 T^T (b_f - K_fp p))
template <typename T>
__global__ void k_cms_b(int nF, const int* __restrict__ inc_ptr, const vec4_t<T>* __restrict__ corner,
                        const T* __restrict__ m_dt2, const vec4_t<T>* __restrict__ xhat, vec4_t<T>* __restrict__ B) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nF) return;
    T bx = 0, by = 0, bz = 0;
    for (int k = inc_ptr[i]; k < inc_ptr[i + 1]; ++k) {
        const vec4_t<T> c = corner[k];
        bx += c.x; by += c.y; bz += c.z;
    }
    const T mm = m_dt2[i];
    const vec4_t<T> xh = xhat[i];
    B[i] = make4<T>(mm * xh.x + bx, mm * xh.y + by, mm * xh.z + bz, T(0));
}

template <typename T>
__global__ void k_cms_set_x(int nF, const vec4_t<T>* __restrict__ X, vec4_t<T>* __restrict__ x, int* fail_iter, int it) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nF) return;
    const vec4_t<T> v = X[i];
    x[i] = v;
    if (!(isfinite(v.x) && isfinite(v.y) && isfinite(v.z))) atomicMin(fail_iter, it);
}

}  // namespace vk

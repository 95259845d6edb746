// PD local step (K2) and the projection kernel.
//
// One thread per tet: gather the four corner positions, F = Ds Dm^-1
// (volmesh.py:115-118), rotation-variant SVD (material.py:127-137), volume
// projection of the singular values (material.py:343-392, float64), then
//   P = gs R + gv V = U diag(gs + gv s) W^T                    (pdsolver.py:67)
// and the per-corner contributions 2 V P g_n                  (pdsolver.py:68)
// written into each node's incidence run (`corner[slot4[e].a]`); a
// deterministic node-centric gather (no float atomics) sums the run later, in
// tet order, like `np.add.at` (pdsolver.py:69-70).
//
// MODE_RESID writes 2V (P - (gs+gv) F) g_n instead: summed over a node and
// added to (m/dt^2)(xhat - x) it is exactly b - K x, the global-step residual
// at the current iterate (the `-K x` part is the frozen-projection Hessian
// applied to x).  That lets the global step solve for the correction in
// residual form, which is what makes float32 storage accurate enough.
#pragma once

#include "sl3.cuh"
#include "svd3.cuh"
#include "vk_common.cuh"

namespace vk {

enum LocalMode { MODE_RHS = 0, MODE_RESID = 1 };

#ifndef VK_LOCAL_MINB
#define VK_LOCAL_MINB 8        // resident 128-thread CTAs per SM the register budget targets
                               // (64 regs; measured faster than 4/6 despite small spills)
#endif

struct ProjStats {
    unsigned int robust;     // elements re-solved on the scalar path
    unsigned int fallback;   // robust path fell back to uniform scaling
    unsigned long long pd_rounds;   // PD rounds executed (solver launches in the PD loop)
};

__device__ __forceinline__ void count_path(ProjStats* st, int path) {
    if (st == nullptr) return;
    const unsigned int m1 = __ballot_sync(__activemask(), path >= 1);
    const unsigned int m2 = __ballot_sync(__activemask(), path == 2);
    const int lane = threadIdx.x & 31;
    const unsigned int lead = __ffs(__activemask()) - 1;
    if (lane == (int)lead) {
        if (m1) atomicAdd(&st->robust, (unsigned int)__popc(m1));
        if (m2) atomicAdd(&st->fallback, (unsigned int)__popc(m2));
    }
}

// F -> (U, d, W) with P = U diag(d_i) W^T for d_i = a + b * s_i.  Returns path id.
// pass: 0 = full per-element logic inline, 1 = defer suspicious elements
// (returns 3), 2 = robust scalar path only (for elements known suspicious).
template <typename T>
__device__ __forceinline__ int project_element(const T (&F)[3][3], T (&U)[3][3], T (&W)[3][3],
                                               T (&sig)[3], double (&s)[3], int pass = 0) {
#ifdef VK_EXP_NO_SVD          // cost-attribution experiments only (never in the product build)
    for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j) { U[i][j] = W[i][j] = (i == j); }
    sig[0] = F[0][0]; sig[1] = F[1][1]; sig[2] = F[2][2];
#else
    svd3_rv(F, U, sig, W);
#endif
    const double sd[3] = {(double)sig[0], (double)sig[1], (double)sig[2]};
#ifdef VK_EXP_NO_SL3
    s[0] = sd[0]; s[1] = sd[1]; s[2] = sd[2];
    return 0;
#else
    if (pass == 2) return sl3::project_robust(sd, s) ? 1 : 2;
    return sl3::project(sd, s, pass == 1);
#endif
}

// out = U diag(d) W^T
template <typename T>
__device__ __forceinline__ void udw(const T (&U)[3][3], const T (&d)[3], const T (&W)[3][3], T (&out)[3][3]) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            out[i][j] = U[i][0] * d[0] * W[j][0] + U[i][1] * d[1] * W[j][1] + U[i][2] * d[2] * W[j][2];
}

template <typename T>
struct LocalArgs {
    int nE;
    const int4* tets;            // internal node ids
    const T* G;                  // 9 planes of nE: rows 1..3 of the shape gradient (= Dm^-1 rows)
    const T* w;                  // 2 planes of nE: 2 V gs, 2 V gv
    const vec4_t<T>* x;          // positions, internal order
    const int4* slot4;           // position of (e, corner a) in its node's incidence run
    vec4_t<T>* corner;           // per-incidence contributions, node-sorted (tet order within a node)
    ProjStats* stats;
    int* robust_list;            // optional: suspicious elements are queued here (k_robust finishes them)
    int* robust_count;           // [0] queued elements, [1] chunk cursor of the robust pass
    unsigned long long robust_if;   // nonzero: graph IF-node handle set to 1 when anything is queued
                                    // (the robust pass is only launched then)
    T* robust_aux;               // optional, 24 per queue slot: the queued element's (sigma, U, W) from
                                 // the first pass, so the robust pass does not redo the SVD
    double* F_out;               // optional (nE,3,3) (RHS mode only)
    double* R_out;
    double* V_out;
    // optional (frame path, residual mode): warp-segmented node reduction.  The 32 tets of warp w
    // touch wr_ptr[w+1] - wr_ptr[w] distinct nodes; entry E sums the warp's staged corner values
    // wr_code[w*128 + wr_beg[E] ..] (lane*4 + corner) and writes node partial wpart[wr_slot[E]]
    // (node-sorted, warps in order).  Queued (robust) tets contribute zero there and write their
    // corners to `corner` later and mark their incidences in robust_flag (the gather clears them).
    const int* wr_ptr;
    const int* wr_slot;
    const unsigned char* wr_beg;
    const unsigned char* wr_code;
    vec4_t<T>* wpart;
    unsigned char* robust_flag;
};

// One tet of the local step.  COH selects coherent loads of x: required when
// x was written earlier in the same launch (the fused frame kernel).
// Load one tet: shape-gradient rows g, weights (2V gs, 2V gv) and F = Ds Dm^-1.
template <typename T, bool COH>
__device__ __forceinline__ void load_tet(const LocalArgs<T>& a, int e, T (&g)[3][3], T& ws, T& wv, T (&F)[3][3]) {
    const int nE = a.nE;
    const int4 t = __ldg(&a.tets[e]);
#pragma unroll
    for (int k = 0; k < 9; ++k) g[k / 3][k % 3] = __ldg(&a.G[(size_t)k * nE + e]);
    ws = __ldg(&a.w[e]);
    wv = __ldg(&a.w[(size_t)nE + e]);
    const vec4_t<T> x0 = COH ? ld4(&a.x[t.x]) : ldg4(&a.x[t.x]);
    const vec4_t<T> x1 = COH ? ld4(&a.x[t.y]) : ldg4(&a.x[t.y]);
    const vec4_t<T> x2 = COH ? ld4(&a.x[t.z]) : ldg4(&a.x[t.z]);
    const vec4_t<T> x3 = COH ? ld4(&a.x[t.w]) : ldg4(&a.x[t.w]);
    // edges x_n - x_0 (n = 1..3) as rows e[n-1][:]
    const T ed[3][3] = {{x1.x - x0.x, x1.y - x0.y, x1.z - x0.z},
                        {x2.x - x0.x, x2.y - x0.y, x2.z - x0.z},
                        {x3.x - x0.x, x3.y - x0.y, x3.z - x0.z}};
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            F[i][j] = ed[0][i] * g[0][j] + ed[1][i] * g[1][j] + ed[2][i] * g[2][j];
}

template <typename T, int MODE, bool WITH_FRV>
__device__ __forceinline__ void finish_tet(const LocalArgs<T>& a, int e, const T (&g)[3][3], T ws, T wv,
                                           const T (&F)[3][3], const T (&U)[3][3], const T (&W)[3][3],
                                           const double (&s)[3]);

template <typename T, int MODE, bool WITH_FRV, bool COH, int PASS = 0>
__device__ __forceinline__ void local_tet(const LocalArgs<T>& a, int e) {
    T g[3][3], F[3][3], ws, wv;
    load_tet<T, COH>(a, e, g, ws, wv, F);
    T U[3][3], W[3][3], sig[3];
    double s[3];
    const int path = project_element(F, U, W, sig, s, PASS);
    if (PASS == 1) {
        // queue suspicious elements (warp-aggregated); their corners are written by k_robust
        const unsigned int am = __activemask();
        const unsigned int m3 = __ballot_sync(am, path == 3);
        if (m3) {
            const int lane = threadIdx.x & 31;
            const int lead = __ffs(m3) - 1;
            int base = 0;
            if (lane == lead) {
                base = atomicAdd(a.robust_count, __popc(m3));
                if (a.robust_if != 0) cudaGraphSetConditional((cudaGraphConditionalHandle)a.robust_if, 1u);
            }
            base = __shfl_sync(am, base, lead);
            if (path == 3) {
                const int slot = base + __popc(m3 & ((1u << lane) - 1u));
                a.robust_list[slot] = e;
                if (a.robust_aux != nullptr) {
                    T* ax = a.robust_aux + (size_t)24 * slot;
                    ax[0] = sig[0]; ax[1] = sig[1]; ax[2] = sig[2];
#pragma unroll
                    for (int k = 0; k < 9; ++k) { ax[3 + k] = U[k / 3][k % 3]; ax[12 + k] = W[k / 3][k % 3]; }
                }
            }
        }
        if (path == 3) return;
    }
    if (PASS != 1) count_path(a.stats, path);
    finish_tet<T, MODE, WITH_FRV>(a, e, g, ws, wv, F, U, W, s);
}

template <typename T>
__device__ __forceinline__ void corner_forces(const T (&P)[3][3], const T (&g)[3][3], T (&f)[3][3]) {
#pragma unroll
    for (int n = 0; n < 3; ++n)
#pragma unroll
        for (int i = 0; i < 3; ++i) f[n][i] = P[i][0] * g[n][0] + P[i][1] * g[n][1] + P[i][2] * g[n][2];
}

// P = U diag(ws + wv s) W^T (minus (ws+wv) F in residual mode), optional
// (F, R, V) outputs, and the four corner contributions 2V P g_n.
template <typename T, int MODE, bool WITH_FRV>
__device__ __forceinline__ void finish_tet(const LocalArgs<T>& a, int e, const T (&g)[3][3], T ws, T wv,
                                           const T (&F)[3][3], const T (&U)[3][3], const T (&W)[3][3],
                                           const double (&s)[3]) {
    const T d[3] = {ws + wv * (T)s[0], ws + wv * (T)s[1], ws + wv * (T)s[2]};
    T P[3][3];
    udw(U, d, W, P);
    if (MODE == MODE_RESID) {
        const T c = ws + wv;
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) P[i][j] -= c * F[i][j];
    }
    if (WITH_FRV) {
        const T one[3] = {T(1), T(1), T(1)};
        const T sv[3] = {(T)s[0], (T)s[1], (T)s[2]};
        T R[3][3], V[3][3];
        udw(U, one, W, R);
        udw(U, sv, W, V);
#pragma unroll
        for (int k = 0; k < 9; ++k) {
            a.F_out[(size_t)e * 9 + k] = (double)F[k / 3][k % 3];
            a.R_out[(size_t)e * 9 + k] = (double)R[k / 3][k % 3];
            a.V_out[(size_t)e * 9 + k] = (double)V[k / 3][k % 3];
        }
    }
    // f_n = P g_n for n = 1..3, f_0 = -(f_1 + f_2 + f_3)
    T f[3][3];
    corner_forces(P, g, f);
    // scatter into each node's incidence run (slot precomputed): writes are
    // fire-and-forget, and the later per-node gather reads a contiguous run
    const int4 sl = __ldg(&a.slot4[e]);
    st4(&a.corner[sl.x], make4<T>(-(f[0][0] + f[1][0] + f[2][0]), -(f[0][1] + f[1][1] + f[2][1]),
                                  -(f[0][2] + f[1][2] + f[2][2]), T(0)));
    st4(&a.corner[sl.y], make4<T>(f[0][0], f[0][1], f[0][2], T(0)));
    st4(&a.corner[sl.z], make4<T>(f[1][0], f[1][1], f[1][2], T(0)));
    st4(&a.corner[sl.w], make4<T>(f[2][0], f[2][1], f[2][2], T(0)));
}

#ifndef VK_LOCAL_MINB64
#define VK_LOCAL_MINB64 6      // float64 build: 80 registers (warp-reduced pass: C3 4.74 -> 4.66 ms/frame vs 64)
#endif
// Residual-mode first pass with the warp-segmented node reduction (north_star (a)): every lane
// stages its tet's four corner vectors in shared memory, then lane j of the warp sums the
// contributions of the warp's j-th distinct node in a fixed (lane, corner) order and writes one
// partial per (warp, node).  At C3 a warp's 32 tets touch ~26 nodes and a node gets ~3 partials
// instead of ~15 corner vectors.  Deterministic: fixed orders everywhere, no atomics.
template <typename T>
__device__ __forceinline__ void local_wred(const LocalArgs<T>& a, T (*stage)[128], unsigned* scode) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    if ((e & ~31) >= a.nE) return;                 // a warp past the last tet (warp-uniform)
    const bool valid = e < a.nE;
    T f4[4][3] = {};
    bool queued = false;
    int path = 0;
    T g[3][3], F[3][3], ws = 0, wv = 0, U[3][3], W[3][3], sig[3];
    double s[3];
    if (valid) {
        load_tet<T, false>(a, e, g, ws, wv, F);
        path = project_element(F, U, W, sig, s, 1);
    }
    const unsigned int m3 = __ballot_sync(0xffffffffu, valid && path == 3);
    if (m3) {
        const int lead = __ffs(m3) - 1;
        int base = 0;
        if (lane == lead) {
            base = atomicAdd(a.robust_count, __popc(m3));
            if (a.robust_if != 0) cudaGraphSetConditional((cudaGraphConditionalHandle)a.robust_if, 1u);
        }
        base = __shfl_sync(0xffffffffu, base, lead);
        if (valid && path == 3) {
            queued = true;
            const int slot = base + __popc(m3 & ((1u << lane) - 1u));
            a.robust_list[slot] = e;
            if (a.robust_aux != nullptr) {
                T* ax = a.robust_aux + (size_t)24 * slot;
                ax[0] = sig[0]; ax[1] = sig[1]; ax[2] = sig[2];
#pragma unroll
                for (int k = 0; k < 9; ++k) { ax[3 + k] = U[k / 3][k % 3]; ax[12 + k] = W[k / 3][k % 3]; }
            }
        }
    }
    if (valid && !queued) {
        const T d[3] = {ws + wv * (T)s[0], ws + wv * (T)s[1], ws + wv * (T)s[2]};
        T P[3][3];
        udw(U, d, W, P);
        const T c = ws + wv;
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) P[i][j] -= c * F[i][j];
        T f[3][3];
        corner_forces(P, g, f);
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            f4[0][i] = -(f[0][i] + f[1][i] + f[2][i]);
            f4[1][i] = f[0][i]; f4[2][i] = f[1][i]; f4[3][i] = f[2][i];
        }
    }
    const int w = e >> 5;
    const int e0 = w << 5;
    const int cnt = 4 * min(32, a.nE - e0);
    // the warp's 128 codes into shared memory (one coalesced load) next to the staged values
    scode[lane] = __ldg(reinterpret_cast<const unsigned*>(a.wr_code + (size_t)w * 128) + lane);
#pragma unroll
    for (int n = 0; n < 4; ++n)
#pragma unroll
        for (int i = 0; i < 3; ++i) stage[i][lane * 4 + n] = f4[n][i];
    const int E0 = __ldg(&a.wr_ptr[w]), m = __ldg(&a.wr_ptr[w + 1]) - E0;
    __syncwarp();
    const unsigned char* code = reinterpret_cast<const unsigned char*>(scode);
    for (int j = lane; j < m; j += 32) {
        const int b = a.wr_beg[E0 + j], en = j + 1 < m ? a.wr_beg[E0 + j + 1] : cnt;
        T sx = 0, sy = 0, sz = 0;
        for (int k = b; k < en; ++k) {
            const int c = code[k];
            sx += stage[0][c]; sy += stage[1][c]; sz += stage[2][c];
        }
        st4(&a.wpart[__ldg(&a.wr_slot[E0 + j])], make4<T>(sx, sy, sz, T(0)));
    }
}

template <typename T>
__global__ void __launch_bounds__(128, sizeof(T) == 8 ? VK_LOCAL_MINB64 : VK_LOCAL_MINB) k_local_wred(LocalArgs<T> a) {
    pcg_mark(8);
    __shared__ T stage[4][3][128];
    __shared__ unsigned scode[4][32];
    local_wred<T>(a, stage[threadIdx.x >> 5], scode[threadIdx.x >> 5]);
}

template <typename T, int MODE, bool WITH_FRV, int PASS = 0>
__global__ void __launch_bounds__(128, sizeof(T) == 8 ? VK_LOCAL_MINB64 : VK_LOCAL_MINB) k_local(LocalArgs<T> a) {
    if (PASS == 1) pcg_mark(8);
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= a.nE) return;
    local_tet<T, MODE, WITH_FRV, false, PASS>(a, e);
}

// Robust pass as independent (chunk, start) tasks (needs the first pass's SVD hand-off).
// A warp takes one task = one Newton start (material.py:251-263) for 32 queued elements and
// writes (s, obj, ok) per (start, slot); no CTA barrier couples the fast starts to the slow
// one.  Tasks are handed out start-major with the usually-stalling sigma/cbrt start (2) first,
// then 3, 0, 1 (longest first).  The warp that completes a chunk's fourth start (per-chunk
// arrival counter, reset by that warp) picks the winner per element in the reference's start
// order with its strict comparison (material.py:264-280) and writes the corners.
// res: 4 doubles per (start, slot), ok: one int per (start, slot); cap = nE.
template <typename T, int MODE>
__device__ __forceinline__ void robust_select_one(const LocalArgs<T>& a, const double* __restrict__ res,
                                                  const int* __restrict__ okf, int cap, int i) {
    bool have = false;
    double best = 0.0, s[3] = {0, 0, 0};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const size_t r = (size_t)k * cap + i;
        const double ob = __ldcg(&res[4 * r + 3]);
        if (__ldcg(&okf[r]) && (!have || ob < best - 1e-15)) {
            have = true;
            best = ob;
            s[0] = __ldcg(&res[4 * r]); s[1] = __ldcg(&res[4 * r + 1]); s[2] = __ldcg(&res[4 * r + 2]);
        }
    }
    const T* ax = a.robust_aux + (size_t)24 * i;
    if (!have) {
        const double sd[3] = {(double)ax[0], (double)ax[1], (double)ax[2]};
        sl3::robust_fallback(sd, s);
    }
    if (a.stats) {
        atomicAdd(&a.stats->robust, 1u);
        if (!have) atomicAdd(&a.stats->fallback, 1u);
    }
    const int e = a.robust_list[i];
    T g[3][3], F[3][3], ws, wv, U[3][3], W[3][3];
    load_tet<T, false>(a, e, g, ws, wv, F);
#pragma unroll
    for (int k = 0; k < 9; ++k) { U[k / 3][k % 3] = ax[3 + k]; W[k / 3][k % 3] = ax[12 + k]; }
    finish_tet<T, MODE, false>(a, e, g, ws, wv, F, U, W, s);
    if (a.wpart != nullptr) {                      // warp-reduced first pass: flag the 4 incidences
        const int4 sl = __ldg(&a.slot4[e]);
        a.robust_flag[sl.x] = 1; a.robust_flag[sl.y] = 1; a.robust_flag[sl.z] = 1; a.robust_flag[sl.w] = 1;
    }
}

#ifndef VK_RTASK_MINB
#define VK_RTASK_MINB 5        // 96 registers, 5 CTAs per SM: fold frame 10.0 -> 9.65 ms (1: 116 registers; 6: 80 + spills, 9.85)
#endif
template <typename T, int MODE>
__global__ void __launch_bounds__(128, VK_RTASK_MINB) k_robust_tasks(LocalArgs<T> a, double* __restrict__ res,
                                                      int* __restrict__ okf, int* __restrict__ arrivals, int cap) {
    const int cnt = *a.robust_count;
    if (blockIdx.x == 0 && threadIdx.x == 0) a.robust_count[2] = cnt;   // for the solver's gather (kept)
    if (cnt == 0) return;
    const int nch = (cnt + 31) >> 5;
    const int lane = threadIdx.x & 31;
    const int order[4] = {2, 3, 0, 1};
    for (;;) {
        int task = 0;
        if (lane == 0) task = atomicAdd(a.robust_count + 1, 1);
        task = __shfl_sync(0xffffffffu, task, 0);
        if (task >= 4 * nch) break;
        const int k = order[task / nch];
        const int chunk = task % nch;
        const int i = chunk * 32 + lane;
        if (i < cnt) {
            const T* ax = a.robust_aux + (size_t)24 * i;
            const double sd[3] = {(double)ax[0], (double)ax[1], (double)ax[2]};
            double st[3], sk[3] = {0, 0, 0}, obj = 0.0;
            const bool ok = sl3::robust_start(sd, k, st) && sl3::robust_try(sd, st, sk, obj);
            const size_t r = (size_t)k * cap + i;
            okf[r] = ok;
            res[4 * r] = sk[0];
            res[4 * r + 1] = sk[1];
            res[4 * r + 2] = sk[2];
            res[4 * r + 3] = obj;
        }
        __threadfence();
        __syncwarp();
        int prev = 0;
        if (lane == 0) prev = atomicAdd(&arrivals[chunk], 1);
        prev = __shfl_sync(0xffffffffu, prev, 0);
        if (prev == 3) {                       // last start of this chunk: select and finish
            __threadfence();
            if (i < cnt) robust_select_one<T, MODE>(a, res, okf, cap, i);
            if (lane == 0) arrivals[chunk] = 0;
        }
    }
}

// Stateless projections of a batch of F (material.py:395-407): (R, V).
template <typename T>
__global__ void __launch_bounds__(128) k_project(int n, const double* __restrict__ Fin, double* R, double* V,
                                                 ProjStats* stats) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n) return;
    T F[3][3];
#pragma unroll
    for (int k = 0; k < 9; ++k) F[k / 3][k % 3] = (T)Fin[(size_t)e * 9 + k];
    T U[3][3], W[3][3], sig[3];
    double s[3];
    const int path = project_element(F, U, W, sig, s);
    count_path(stats, path);
    const T one[3] = {T(1), T(1), T(1)};
    const T sv[3] = {(T)s[0], (T)s[1], (T)s[2]};
    T Rm[3][3], Vm[3][3];
    udw(U, one, W, Rm);
    udw(U, sv, W, Vm);
#pragma unroll
    for (int k = 0; k < 9; ++k) {
        R[(size_t)e * 9 + k] = (double)Rm[k / 3][k % 3];
        V[(size_t)e * 9 + k] = (double)Vm[k / 3][k % 3];
    }
}

}  // namespace vk

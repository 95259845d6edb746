// Projection derivatives and the exact elastic Hessian (SURVEY.md 8f rank 2,
// fitting side), float64, one thread per tet.
//
//   d vec(R) / d vec(F) and d vec(V) / d vec(F), 9x9 in the row-major vec layout
//   (material.py:490-524, projection_jacobians_batch): in the singular-vector frame
//   the rotation part couples each pair (ij, ji) with 1/(s_i + s_j); the volume part
//   takes ds/dsigma from differentiating the constrained stationarity system
//   (material.py:420-440, clamped entries insensitive) on the diagonal and the
//   divided differences (s_i - s_j)/(sigma_i - sigma_j) (confluent form at ties) and
//   (s_i + s_j)/(sigma_i + sigma_j) on the pairs; both are conjugated by
//   Q = kron(U, W).
#pragma once

#include "sl3.cuh"
#include "svd3.cuh"

namespace vk {

// L (9x9) conjugated by Q = kron(U, W): J[(9r + c) * stride] = (Q L Q^T)[r][c].
// J is a global pointer on every call site: with a thread-local J the sm_100a build
// produced wrong values (tests/native/hess_probe.cu), so outputs always go to memory.
__device__ __forceinline__ void conjugate9(const double (&U)[3][3], const double (&W)[3][3], const double* L,
                                           double* J, size_t stride = 1) {
    double Q[9][9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
#pragma unroll
            for (int k = 0; k < 3; ++k)
#pragma unroll
                for (int l = 0; l < 3; ++l) Q[3 * i + j][3 * k + l] = U[i][k] * W[j][l];
    double Tm[9][9];
    for (int r = 0; r < 9; ++r)
        for (int c = 0; c < 9; ++c) {
            double acc = 0.0;
            for (int m = 0; m < 9; ++m) acc += Q[r][m] * L[9 * m + c];
            Tm[r][c] = acc;
        }
    for (int r = 0; r < 9; ++r)
        for (int c = 0; c < 9; ++c) {
            double acc = 0.0;
            for (int m = 0; m < 9; ++m) acc += Tm[r][m] * Q[c][m];
            J[(size_t)(9 * r + c) * stride] = acc;
        }
}

// ds/dsigma of the (clamped) constrained singular-value solve (material.py:420-440)
__device__ __forceinline__ void sl3_ds_dsigma(const double (&s)[3], double lam, const bool (&cl)[3],
                                              double (&D)[3][3]) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) D[i][j] = 0.0;
    double p[3];
    sl3::pairprod(s, p);
    for (int col = 0; col < 3; ++col) {
        if (cl[col]) continue;
        // frozen entries: identity row/column and zero right-hand side (same solution on
        // the free block as the reference's reduced (nf+1) system)
        double J[4][4], b[4] = {0.0, 0.0, 0.0, 0.0};
        for (int i = 0; i < 3; ++i) {
            for (int j = 0; j < 3; ++j) {
                const double v = (i == j) ? 1.0 : lam * s[3 - i - j];
                J[i][j] = (!cl[i] && !cl[j]) ? v : (i == j ? 1.0 : 0.0);
            }
            J[i][3] = cl[i] ? 0.0 : p[i];
            J[3][i] = cl[i] ? 0.0 : p[i];
        }
        J[3][3] = 0.0;
        b[col] = 1.0;
        if (!sl3::gesv4(J, b)) continue;
        for (int i = 0; i < 3; ++i) D[i][col] = cl[i] ? 0.0 : b[i];
    }
}

// the singular-value-frame derivatives LR, LV (material.py:490-524) and the SVD frame
__device__ __forceinline__ void projection_frame(const double (&F)[3][3], double (&U)[3][3], double (&W)[3][3],
                                                 double* LR, double* LV) {
    double sg[3];
    svd3_rv(F, U, sg, W);
    double s[3], lam = 0.0;
    bool cl[3] = {false, false, false};
    sl3::project(sg, s, false, &lam, cl);
    double ds[3][3];
    sl3_ds_dsigma(s, lam, cl, ds);
    for (int k = 0; k < 81; ++k) LR[k] = LV[k] = 0.0;
    const int dia[3] = {0, 4, 8};
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) LV[9 * dia[i] + dia[j]] = ds[i][j];
    const int PI[3] = {0, 0, 1}, PJ[3] = {1, 2, 2};
    for (int q = 0; q < 3; ++q) {
        const int i = PI[q], j = PJ[q], a = 3 * i + j, b = 3 * j + i;
        double den = sg[i] + sg[j];
        if (fabs(den) < 1e-8) den = copysign(1e-8, den != 0.0 ? den : 1.0);
        const double c = 1.0 / den;
        LR[9 * a + a] = LR[9 * b + b] = c;
        LR[9 * a + b] = LR[9 * b + a] = -c;
        const double dd = sg[i] - sg[j];
        const double scale = fmax(1.0, fmax(fabs(sg[i]), fabs(sg[j])));
        const double cs = fabs(dd) > 1e-7 * scale ? (s[i] - s[j]) / dd : ds[i][i] - ds[i][j];
        const double ca = (s[i] + s[j]) / den;
        LV[9 * a + a] = LV[9 * b + b] = 0.5 * (cs + ca);
        LV[9 * a + b] = LV[9 * b + a] = 0.5 * (cs - ca);
    }
}

// JR, JV: global memory, 81 entries each
__device__ __forceinline__ void projection_jacobians(const double (&F)[3][3], double* JR, double* JV) {
    double U[3][3], W[3][3], LR[81], LV[81];
    projection_frame(F, U, W, LR, LV);
    conjugate9(U, W, LR, JR);
    conjugate9(U, W, LV, JV);
}

// M = c (ws (I - JR) + wv (I - JV)) = c (ws + wv) I - Q (c (ws LR + wv LV)) Q^T: the 9x9
// block of the exact Hessian (pdsolver.py:109-112), written with stride (global memory)
__device__ __forceinline__ void hessian_block9(const double (&F)[3][3], double ws, double wv, double c, double* M,
                                               size_t stride) {
    double U[3][3], W[3][3], LR[81], LV[81];
    projection_frame(F, U, W, LR, LV);
    for (int k = 0; k < 81; ++k) LR[k] = -c * (ws * LR[k] + wv * LV[k]);
    conjugate9(U, W, LR, M, stride);
    const double d = c * (ws + wv);
    for (int k = 0; k < 9; ++k) M[(size_t)(10 * k) * stride] += d;
}

__global__ void __launch_bounds__(128) k_proj_jacobians(int n, const double* __restrict__ Fin, double* JR,
                                                        double* JV) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n) return;
    double F[3][3];
    for (int k = 0; k < 9; ++k) F[k / 3][k % 3] = Fin[(size_t)9 * e + k];
    projection_jacobians(F, JR + (size_t)81 * e, JV + (size_t)81 * e);
}

}  // namespace vk

// Rotation-variant 3x3 SVD, F = U diag(sigma) W^T with U, W in SO(3).
//
// Convention of the reference `svd_rv_batch` (material.py:127-137):
// sigma0 >= sigma1 >= |sigma2|, sigma0, sigma1 >= 0, and sigma2 < 0 exactly
// when det F < 0 (the reflection is pushed into the last singular value).
//
// Method (branch-light, per thread): cyclic Jacobi eigen-decomposition of the
// symmetric A = F^T F gives W; columns sorted by eigenvalue; then a Givens QR
// of B = F W gives U (a product of rotations, so det U = +1) and the
// diagonal of R as sigma, which keeps small singular values accurate (they do
// not come from sqrt(eigenvalue)).
#pragma once

#include "vk_common.cuh"

namespace vk {

template <typename T>
VK_HD void jacobi_rotate(T (&a)[3][3], T (&W)[3][3], int p, int q) {
    const T apq = a[p][q];
    if (apq == T(0)) return;
    T t;
    if constexpr (sizeof(T) == 8) {
        // t = sgn(theta) / (|theta| + sqrt(theta^2 + 1)), theta = tau / b (tau = a_qq - a_pp,
        // b = 2 a_pq) multiplied through by |b|: one division instead of two.  The sign rule keeps
        // theta = -0 -> t = +1; if the squares underflow (|tau|, |b| < 1e-154) and tau = 0 the
        // denominator is 0 and t = 1 is theta = 0's value.
        const T tau = a[q][q] - a[p][p], b = T(2) * apq;
        const T ab = fabs(b), at = fabs(tau), den = at + sqrt(at * at + ab * ab);
        t = den > T(0) ? ab / den : T(1);
        t = (tau != T(0) && ((tau < T(0)) != (b < T(0)))) ? -t : t;
    } else {
        const T theta = (a[q][q] - a[p][p]) / (T(2) * apq);
        const T at = fabs(theta);
        if (at > T(1e15)) {
            t = T(0.5) / theta;
        } else {
            t = T(1) / (at + sqrt(at * at + T(1)));
            t = theta < T(0) ? -t : t;
        }
    }
    const T c = rsqrt_(t * t + T(1));
    const T s = t * c;
    const int r = 3 - p - q;
    const T arp = a[r][p], arq = a[r][q];
    a[p][p] -= t * apq;
    a[q][q] += t * apq;
    a[p][q] = a[q][p] = T(0);
    const T nrp = c * arp - s * arq;
    const T nrq = s * arp + c * arq;
    a[r][p] = a[p][r] = nrp;
    a[r][q] = a[q][r] = nrq;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const T wp = W[k][p], wq = W[k][q];
        W[k][p] = c * wp - s * wq;
        W[k][q] = s * wp + c * wq;
    }
}

template <typename T>
VK_HD void givens_rows(T (&B)[3][3], T (&Qt)[3][3], int i, int j) {
    // rotate rows (i, j) so that B[j][i] becomes 0 and B[i][i] = hypot >= 0
    const T a = B[i][i], b = B[j][i];
    const T rr = a * a + b * b;
    T c = T(1), s = T(0);
    if (b == T(0)) {
        c = a < T(0) ? T(-1) : T(1);      // exact: keeps already-triangular (e.g. diagonal) F exact
    } else if (rr > T(0)) {
        const T inv = rsqrt_(rr);
        c = a * inv;
        s = b * inv;
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const T bi = B[i][k], bj = B[j][k];
        B[i][k] = c * bi + s * bj;
        B[j][k] = -s * bi + c * bj;
        const T qi = Qt[i][k], qj = Qt[j][k];
        Qt[i][k] = c * qi + s * qj;
        Qt[j][k] = -s * qi + c * qj;
    }
}

template <typename T>
VK_HD void swap_cols(T (&W)[3][3], T (&lam)[3], int i, int j) {
    const T tl = lam[i]; lam[i] = lam[j]; lam[j] = tl;
#pragma unroll
    for (int k = 0; k < 3; ++k) { const T t = W[k][i]; W[k][i] = W[k][j]; W[k][j] = t; }
}

template <typename T>
VK_HD void svd3_rv(const T (&F)[3][3], T (&U)[3][3], T (&sig)[3], T (&W)[3][3]) {
    // A = F^T F
    T a[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = i; j < 3; ++j) {
            const T v = F[0][i] * F[0][j] + F[1][i] * F[1][j] + F[2][i] * F[2][j];
            a[i][j] = v; a[j][i] = v;
        }
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) W[i][j] = (i == j) ? T(1) : T(0);

    constexpr int kMaxSweeps = sizeof(T) == 4 ? 5 : 8;
    for (int sweep = 0; sweep < kMaxSweeps; ++sweep) {
        const T off = a[0][1] * a[0][1] + a[0][2] * a[0][2] + a[1][2] * a[1][2];
        const T dia = a[0][0] * a[0][0] + a[1][1] * a[1][1] + a[2][2] * a[2][2];
        if (!(off > Eps<T>::v * Eps<T>::v * T(1e-2) * dia)) break;
        jacobi_rotate(a, W, 0, 1);
        jacobi_rotate(a, W, 0, 2);
        jacobi_rotate(a, W, 1, 2);
    }
    T lam[3] = {a[0][0], a[1][1], a[2][2]};
    // sort descending (three compare-swaps)
    if (lam[0] < lam[1]) swap_cols(W, lam, 0, 1);
    if (lam[0] < lam[2]) swap_cols(W, lam, 0, 2);
    if (lam[1] < lam[2]) swap_cols(W, lam, 1, 2);
    // make W proper
    const T detW = W[0][0] * (W[1][1] * W[2][2] - W[1][2] * W[2][1])
                 - W[0][1] * (W[1][0] * W[2][2] - W[1][2] * W[2][0])
                 + W[0][2] * (W[1][0] * W[2][1] - W[1][1] * W[2][0]);
    if (detW < T(0)) {
#pragma unroll
        for (int k = 0; k < 3; ++k) W[k][2] = -W[k][2];
    }
    // B = F W, then Givens QR: Qt B = R, U = Qt^T
    T B[3][3], Qt[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            B[i][j] = F[i][0] * W[0][j] + F[i][1] * W[1][j] + F[i][2] * W[2][j];
            Qt[i][j] = (i == j) ? T(1) : T(0);
        }
    givens_rows(B, Qt, 0, 1);
    givens_rows(B, Qt, 0, 2);
    givens_rows(B, Qt, 1, 2);
    sig[0] = B[0][0];
    sig[1] = B[1][1];
    sig[2] = B[2][2];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) U[i][j] = Qt[j][i];
}

}  // namespace vk

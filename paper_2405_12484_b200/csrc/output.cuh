// Per-frame output step, run on the device after the step:
//   v2y          yarn vertex positions = interp @ x (transfer.py:26-28), one thread per
//                yarn vertex summing its CSR row in stored order with separately rounded
//                multiply and add -- the order and rounding of scipy's csr_matvecs, so the
//                float64 result is bit-identical to the reference's sparse product;
//   det deviation max_e |det F_e - 1| (cli.py:639-640), F = Ds Dm^-1 per tet in float64,
//                a max reduction through the bit pattern (non-negative doubles and NaN
//                order like unsigned integers, so NaN propagates as in numpy's max).
#pragma once

#include "vk_common.cuh"

namespace vk {

template <typename T>
__global__ void k_v2y(int n_yarn, const long long* __restrict__ indptr, const int* __restrict__ col_int,
                      const double* __restrict__ w, const vec4_t<T>* __restrict__ x, double* __restrict__ y) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n_yarn) return;
    double sx = 0.0, sy = 0.0, sz = 0.0;
    for (long long j = indptr[k]; j < indptr[k + 1]; ++j) {
        const vec4_t<T> p = x[col_int[j]];
        const double a = w[j];
        sx = __dadd_rn(sx, __dmul_rn(a, (double)p.x));
        sy = __dadd_rn(sy, __dmul_rn(a, (double)p.y));
        sz = __dadd_rn(sz, __dmul_rn(a, (double)p.z));
    }
    y[3 * k + 0] = sx;
    y[3 * k + 1] = sy;
    y[3 * k + 2] = sz;
}

// standalone variant on caller-order float64 positions (transfer.v2y drop-in)
__global__ void k_v2y_host_order(int n_yarn, const long long* __restrict__ indptr,
                                 const long long* __restrict__ col, const double* __restrict__ w,
                                 const double* __restrict__ x, double* __restrict__ y) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n_yarn) return;
    double sx = 0.0, sy = 0.0, sz = 0.0;
    for (long long j = indptr[k]; j < indptr[k + 1]; ++j) {
        const double* p = x + 3 * col[j];
        const double a = w[j];
        sx = __dadd_rn(sx, __dmul_rn(a, p[0]));
        sy = __dadd_rn(sy, __dmul_rn(a, p[1]));
        sz = __dadd_rn(sz, __dmul_rn(a, p[2]));
    }
    y[3 * k + 0] = sx;
    y[3 * k + 1] = sy;
    y[3 * k + 2] = sz;
}

// max_e |det(F_e) - 1| with F = sum_n x_n (x) g_n (g_0 = -(g_1 + g_2 + g_3)), float64
template <typename T>
__global__ void __launch_bounds__(256) k_det_deviation(int nE, const int4* __restrict__ tets,
                                                       const double* __restrict__ G64,
                                                       const vec4_t<T>* __restrict__ x,
                                                       unsigned long long* out) {
    __shared__ unsigned long long red[8];
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long mine = 0ull;
    if (e < nE) {
        const int4 t = tets[e];
        const int nd[4] = {t.x, t.y, t.z, t.w};
        const double* g = G64 + (size_t)12 * e;   // (4, 3) shape gradients, host layout
        double F[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            const vec4_t<T> p = x[nd[a]];
            const double xa[3] = {(double)p.x, (double)p.y, (double)p.z};
#pragma unroll
            for (int i = 0; i < 3; ++i)
#pragma unroll
                for (int j = 0; j < 3; ++j) F[i][j] += xa[i] * g[3 * a + j];
        }
        const double det = F[0][0] * (F[1][1] * F[2][2] - F[1][2] * F[2][1]) -
                           F[0][1] * (F[1][0] * F[2][2] - F[1][2] * F[2][0]) +
                           F[0][2] * (F[1][0] * F[2][1] - F[1][1] * F[2][0]);
        mine = (unsigned long long)__double_as_longlong(fabs(det - 1.0));
    }
    // warp max, then block max, then one atomic per CTA
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long v = __shfl_xor_sync(0xffffffffu, mine, o);
        mine = v > mine ? v : mine;
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) red[wid] = mine;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long m = 0ull;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) m = red[k] > m ? red[k] : m;
        atomicMax(out, m);
    }
}

}  // namespace vk

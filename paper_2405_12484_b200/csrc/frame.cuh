// One whole PD frame in a single persistent cooperative kernel:
//   prologue -> iterations x [local step over all tets | grid sync | CG solve
//   (residual gather, Jacobi-PCG, x += dx) | grid sync] -> epilogue.
// Same arithmetic as the per-phase kernels (k_prologue, k_local<MODE_RESID>,
// k_pcg_classic, k_epilogue) -- they share the device functions -- but 1
// launch per frame instead of 2 per PD iteration: no launch gaps, no wave
// tails between phases, and the CG scalars never leave the SMs.
#pragma once

#include <climits>

#include "local_step.cuh"
#include "solver.cuh"

namespace vk {

template <typename T>
struct FrameArgs {
    LocalArgs<T> la;
    PcgArgs<T> pa;                 // pd_iter / iters_out set per PD iteration
    int n, nF, iterations;
    T dt, damp_over_dt;
    const T* dt2_inv_m;
    const vec4_t<T>* f;            // may be null
    const vec4_t<T>* pin_tgt;
    vec4_t<T>* x;
    vec4_t<T>* v;
    vec4_t<T>* x_start;
    vec4_t<T>* v_start;
    vec4_t<T>* xhat;
    int* fail_iter;
    int* iters;                    // CG iterations per PD iteration
};

#ifndef VK_FRAME_MINB
#define VK_FRAME_MINB 2
#endif

template <typename T>
__global__ void __launch_bounds__(512, VK_FRAME_MINB) k_frame(FrameArgs<T> fa) {
    cg::grid_group grid = cg::this_grid();
    __shared__ double smem[32 * 8];
    __shared__ double red[8];
    const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const int gstride = gridDim.x * blockDim.x;
    // ---- prologue (pdsolver.py:249-254, 283-289)
    if (gtid == 0) *fa.fail_iter = INT_MAX;
    for (int i = gtid; i < fa.n; i += gstride) {
        const vec4_t<T> xi = fa.x[i], vi = fa.v[i];
        fa.x_start[i] = xi;
        fa.v_start[i] = vi;
        const T c = fa.dt2_inv_m[i];
        vec4_t<T> fi = make4<T>(T(0), T(0), T(0), T(0));
        if (fa.f != nullptr) fi = fa.f[i];
        const vec4_t<T> xh = make4<T>(xi.x + fa.dt * vi.x + c * fi.x, xi.y + fa.dt * vi.y + c * fi.y,
                                      xi.z + fa.dt * vi.z + c * fi.z, T(0));
        fa.xhat[i] = xh;
        fa.x[i] = (i < fa.nF) ? xh : fa.pin_tgt[i - fa.nF];
    }
    grid.sync();
    // ---- PD iterations (pdsolver.py:291-300)
    for (int it = 0; it < fa.iterations; ++it) {
        for (int e = gtid; e < fa.la.nE; e += gstride) local_tet<T, MODE_RESID, false, true>(fa.la, e);
        grid.sync();
        PcgArgs<T> pa = fa.pa;
        pa.pd_iter = it;
        pa.iters_out = fa.iters + it;
        pcg_classic_body(pa, grid, smem, red, true);
        grid.sync();
    }
    // ---- epilogue (pdsolver.py:302)
    for (int i = gtid; i < fa.n; i += gstride) {
        const vec4_t<T> a = fa.x[i], b = fa.x_start[i];
        fa.v[i] = make4<T>(fa.damp_over_dt * (a.x - b.x), fa.damp_over_dt * (a.y - b.y),
                           fa.damp_over_dt * (a.z - b.z), T(0));
    }
}

}  // namespace vk

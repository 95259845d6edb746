// Global step as a Chebyshev semi-iteration on the Jacobi-scaled K_ff with
// neighbour-only synchronisation (the fp64 solver of the frame graph).
//
// The reference solves K_ff x = b exactly per PD round (SuperLU,
// pdsolver.py:201-236).  The persistent CG (solver.cuh) needs two grid-wide
// reductions per iteration; at fp64 tolerance (1e-12 of |M/dt^2 xhat|) a PD
// round takes ~20 CG iterations, and each reduction is a grid barrier, so
// the solve is bound by barrier latency.  Chebyshev acceleration of Jacobi
// needs no inner products at all: every step is y += d, res -= K d,
// d = c1 d + c2 D^-1 res with scalar coefficients fixed by the spectrum
// interval [lmin, lmax] of D^-1 K_ff.  Its only data dependence is the SpMV,
// i.e. the rows a CTA reads from the CTAs that own its columns, so a step
// waits for those rows only (register path: each row carries its step tag,
// below; generic path: per-CTA release flags) instead of a grid barrier.  The
// residual norm is reduced (one grid barrier) only at the predicted step count
// and then until it meets the same tolerance the CG uses
// (|r| <= tol |M/dt^2 xhat|).
//
// Spectrum: lmax is the Gershgorin bound of D^-1 K_ff (rigorous), lmin a
// Lanczos estimate of the smallest eigenvalue of D^-1/2 K_ff D^-1/2 computed
// once per assembly (never below the rigorous bound min_i (m_i/dt^2)/K_ii:
// K - M/dt^2 is positive semidefinite).  An optimistic lmin only slows the
// lowest modes (|p_k| < 1 still holds on (0, lmin)); the residual check keeps
// the stopping rule exact either way.  Contact rows (pdsolver.py:271-297) add
// c_i to both K_ii and the mass term, which keeps both bounds valid.
//
// When a CTA owns at most one row per thread (the C3 case) the row state
// lives in registers (residual, direction d, packed column offsets), the
// row's ELL values and accumulated correction in shared memory, and the SpMV
// reads a 32-bit image of d from shared memory over the CTA's own rows plus
// its halo (the rows of other CTAs its rows reference, loaded from L2 once per
// step): each neighbour value crosses L2 once per CTA instead of once per
// reference.  Only the exported rows' d crosses CTAs (flag-in-data rows,
// double-buffered by step parity).  All arithmetic has a fixed order, so
// results are bit-reproducible run to run.
#pragma once

#include "solver.cuh"

namespace vk {

__device__ __forceinline__ void cheb_wait(const unsigned int* flags, const int* nbr, int nn, unsigned int target) {
    // one lane per neighbour CTA polls its flag (acquire): the neighbour's d for
    // this step is then visible to the whole CTA after the barrier below
    if (threadIdx.x < 32) {
        for (int j = threadIdx.x; j < nn; j += 32) {
            const unsigned int* f = flags + (size_t)nbr[j] * 32;
            unsigned long long spins = 0;
            while ((int)(ld_acquire_gpu(f) - target) < 0) {
                if (++spins > (1ull << 33)) __trap();
            }
        }
    }
    __syncthreads();
}

#ifndef VK_CHEB_FENCE
#define VK_CHEB_FENCE 0    // st.release after the CTA barrier orders the CTA's stores (cumulativity)
#endif
__device__ __forceinline__ void cheb_publish(unsigned int* flags, unsigned int value) {
    __syncthreads();
    if (threadIdx.x == 0) {
#if VK_CHEB_FENCE
        __threadfence();
#endif
        st_release_gpu(flags + (size_t)blockIdx.x * 32, value);
    }
}

// x, y, z of a vec4 row through L2 only (rows written by other CTAs in this launch)
__device__ __forceinline__ void ldcg3(const float4* p, float& x, float& y, float& z) {
    const float4 v = __ldcg(p);
    x = v.x; y = v.y; z = v.z;
}
__device__ __forceinline__ void ldcg3(const double4* p, double& x, double& y, double& z) {
    const double2 v = __ldcg(reinterpret_cast<const double2*>(p));
    x = v.x; y = v.y;
    z = __ldcg(reinterpret_cast<const double*>(p) + 2);
}

// Exported rows cross CTAs in a flag-in-data format (the LL idea of NCCL's low-latency protocol):
// every 8-byte word carries 4 bytes of d and the 4-byte step tag, written and read as 16-byte
// vectors of two 64-bit elements with relaxed gpu-scope accesses.  Each naturally aligned 64-bit
// element access is single-copy atomic, so a consumer that sees the tag in every word of a row
// has that row's d of that step: no separate flag, no release barrier after the stores, no
// acquire round trip before the loads.  Row
// layout: fp64 3 x {lo, tag, hi, tag}; fp32 {x, tag, y, tag}, {z, tag, 0, tag}.
template <typename T> struct LLRow;
template <> struct LLRow<double> { static constexpr int W = 3; };
template <> struct LLRow<float> { static constexpr int W = 2; };
template <> struct LLRow<unsigned> { static constexpr int W = 2; };

// words (a | b << 32), (c | d << 32): the same bytes as {a, b, c, d}
__device__ __forceinline__ void ll_st(uint4* p, unsigned a, unsigned b, unsigned c, unsigned d) {
    const unsigned long long w0 = (unsigned long long)a | ((unsigned long long)b << 32);
    const unsigned long long w1 = (unsigned long long)c | ((unsigned long long)d << 32);
    asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1,%2};" :: "l"(p), "l"(w0), "l"(w1) : "memory");
}
__device__ __forceinline__ uint4 ll_ld(const uint4* p) {
    unsigned long long w0, w1;
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0,%1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(p) : "memory");
    return make_uint4((unsigned)w0, (unsigned)(w0 >> 32), (unsigned)w1, (unsigned)(w1 >> 32));
}
__device__ __forceinline__ void ll_store(uint4* p, double x, double y, double z, unsigned tag) {
    const unsigned long long a = __double_as_longlong(x), b = __double_as_longlong(y), c = __double_as_longlong(z);
    ll_st(p, (unsigned)a, tag, (unsigned)(a >> 32), tag);
    ll_st(p + 1, (unsigned)b, tag, (unsigned)(b >> 32), tag);
    ll_st(p + 2, (unsigned)c, tag, (unsigned)(c >> 32), tag);
}
__device__ __forceinline__ void ll_store(uint4* p, float x, float y, float z, unsigned tag) {
    ll_st(p, __float_as_uint(x), tag, __float_as_uint(y), tag);
    ll_st(p + 1, __float_as_uint(z), tag, 0u, tag);
}
__device__ __forceinline__ void ll_store(uint4* p, unsigned x, unsigned y, unsigned z, unsigned tag) {
    ll_st(p, x, tag, y, tag);
    ll_st(p + 1, z, tag, 0u, tag);
}
__device__ __forceinline__ bool ll_ok(const uint4& v, unsigned tag) { return v.y == tag && v.w == tag; }
// spin until the row carries `tag` (traps after ~2^33 polls: a lost producer)
__device__ __forceinline__ void ll_load(const uint4* p, unsigned tag, double& x, double& y, double& z) {
    uint4 a = ll_ld(p), b = ll_ld(p + 1), c = ll_ld(p + 2);
    unsigned long long spins = 0;
    while (!(ll_ok(a, tag) && ll_ok(b, tag) && ll_ok(c, tag))) {
        if (++spins > (1ull << 33)) __trap();
        a = ll_ld(p); b = ll_ld(p + 1); c = ll_ld(p + 2);
    }
    x = __longlong_as_double(((unsigned long long)a.z << 32) | a.x);
    y = __longlong_as_double(((unsigned long long)b.z << 32) | b.x);
    z = __longlong_as_double(((unsigned long long)c.z << 32) | c.x);
}
__device__ __forceinline__ void ll_load(const uint4* p, unsigned tag, float& x, float& y, float& z) {
    uint4 a = ll_ld(p), b = ll_ld(p + 1);
    unsigned long long spins = 0;
    while (!(ll_ok(a, tag) && ll_ok(b, tag))) {
        if (++spins > (1ull << 33)) __trap();
        a = ll_ld(p); b = ll_ld(p + 1);
    }
    x = __uint_as_float(a.x); y = __uint_as_float(a.z); z = __uint_as_float(b.x);
}
__device__ __forceinline__ void ll_load(const uint4* p, unsigned tag, unsigned& x, unsigned& y, unsigned& z) {
    float fx, fy, fz;
    ll_load(p, tag, fx, fy, fz);
    x = __float_as_uint(fx); y = __float_as_uint(fy); z = __float_as_uint(fz);
}

// Register path: a row keeps the shared-memory byte offsets of its kChebOff off-diagonal
// entries in registers (two 16-bit offsets per register, positions bank-conflict-free per warp,
// vkpd.cu conflict_free_positions) and the diagonal.  Shared memory (compile-time strides, so
// every access is one address register plus an immediate offset): two step-parity buffers of
// the x / y / z planes of the image of d over kChebSlots slots (own rows: slot = tid; halo row
// j: slot = blockDim.x + j), the x / y / z planes of the accumulated correction y, the 14 planes
// of the rows' ELL values (thread-indexed: conflict-free), then the halo rows' global indices.
//
// Exported rows first: the rows other CTAs read (a CTA's exported rows lead its row range,
// vkpd.cu patch_order) are computed by the leading warps, which also load the halo rows (one
// per thread) and store their new d in the flag-in-data format as soon as it is computed; the
// interior rows (read by nobody else, kept in shared memory only) are computed by the other
// warps while the exported warps wait for the halo.
constexpr int kChebMaxThreads = 768;
constexpr int kChebSlots = 2048;
constexpr int kChebOff = 14;       // voxel enclosures: <= 15 entries per row, one of them diagonal
// Type of the shared-memory / cross-CTA image of the direction d.  float64 solves apply a
// 32-bit rounding of the direction, the upper word of the double (sign, 11-bit exponent, 20-bit
// mantissa, rounded to nearest): y += h(d) and r -= K h(d) (K, r, y in float64), so y and r stay
// consistent (r is the residual of y to float64 rounding) and the stopping test is unchanged;
// only the Chebyshev direction carries a 5e-7 relative perturbation, which the recurrence damps
// like any other.  Halves the SpMV's shared-memory wavefronts and the halo bytes, and decoding
// is a register pair {0, h}: no F2F conversion (a quarter-rate pipe) per gathered value.
#ifndef VK_CHEB_D32
#define VK_CHEB_D32 1
#endif
template <typename T> struct ChebImage { using type = T; };
#if VK_CHEB_D32
template <> struct ChebImage<double> { using type = unsigned; };
#endif
__device__ __forceinline__ float img_enc(float x) { return x; }
__device__ __forceinline__ float img_dec(float x) { return x; }
__device__ __forceinline__ double img_dec(double x) { return x; }
__device__ __forceinline__ double img_dec(unsigned h) { return __hiloint2double((int)h, 0); }
template <typename DS> __device__ __forceinline__ DS img_enc64(double x);
template <> __device__ __forceinline__ double img_enc64<double>(double x) { return x; }
template <> __device__ __forceinline__ unsigned img_enc64<unsigned>(double x) {
    return (unsigned)(((unsigned long long)__double_as_longlong(x) + 0x80000000ull) >> 32);
}
template <typename DS, typename T> __device__ __forceinline__ DS img_enc(T x) {
    if constexpr (sizeof(T) == 4) return x;
    else return img_enc64<DS>(x);
}
template <typename T>
constexpr size_t cheb_smem_bytes() {
    return sizeof(typename ChebImage<T>::type) * 6 * (size_t)kChebSlots +
           sizeof(T) * (3 + kChebOff) * (size_t)kChebMaxThreads + sizeof(int) * kChebSlots;
}

// Shared-memory loads at an absolute shared-window address plus a compile-time offset (the
// plane and step-parity offsets of the direction image): one LDS per value, no address math.
template <int OFF> __device__ __forceinline__ float lds_img(unsigned addr, float*) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1+%2];" : "=f"(v) : "r"(addr), "n"(OFF));
    return v;
}
template <int OFF> __device__ __forceinline__ unsigned lds_img(unsigned addr, unsigned*) {
    unsigned v;
    asm volatile("ld.shared.u32 %0, [%1+%2];" : "=r"(v) : "r"(addr), "n"(OFF));
    return v;
}
template <int OFF> __device__ __forceinline__ double lds_img(unsigned addr, double*) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1+%2];" : "=d"(v) : "r"(addr), "n"(OFF));
    return v;
}
// q += sum_s vals[s] d[slot_s] over the image buffer P (x / y / z planes), one sum per component.
// colp: two 16-bit byte offsets (into the buffer-0 x plane) per register.  Plain shared loads,
// so the compiler can keep several in flight.
template <int P, typename DS, typename T>
__device__ __forceinline__ void spmv_img(const DS* sd, const unsigned (&colp)[(kChebOff + 1) / 2],
                                         const T* sv, T& qx, T& qy, T& qz) {
    const char* const b = reinterpret_cast<const char*>(sd + P * 3 * kChebSlots);
#pragma unroll
    for (int h = 0; h < (kChebOff + 1) / 2; ++h) {
        const DS* d0 = reinterpret_cast<const DS*>(b + (colp[h] & 0xffffu));
        const T v0 = sv[(2 * h) * kChebMaxThreads];
        qx += v0 * (T)img_dec(d0[0]);
        qy += v0 * (T)img_dec(d0[kChebSlots]);
        qz += v0 * (T)img_dec(d0[2 * kChebSlots]);
        if (2 * h + 1 < kChebOff) {
            const DS* d1 = reinterpret_cast<const DS*>(b + (colp[h] >> 16));
            const T v1 = sv[(2 * h + 1) * kChebMaxThreads];
            qx += v1 * (T)img_dec(d1[0]);
            qy += v1 * (T)img_dec(d1[kChebSlots]);
            qz += v1 * (T)img_dec(d1[2 * kChebSlots]);
        }
    }
}

// Steps needed for a residual reduction by `ratio` at Chebyshev parameter sigma
// (|p_k| <= 1 / T_k(sigma) on the interval).
__device__ __forceinline__ int cheb_steps_for(double ratio, double acosh_sigma) {
    if (!(ratio > 1.0)) return 1;
    const double k = acosh(ratio) / acosh_sigma;
    return k < 1e6 ? max(1, (int)ceil(k)) : 1000000;
}

// REG = true: one row per thread, row state in registers (requires chunk <= blockDim.x
// and ell_w <= kEllUnroll); REG = false: any size, row state in a.r / a.dx, ELL from L1/L2.
template <typename T, bool REG>
__device__ __forceinline__ void cheb_body(const PcgArgs<T>& a, cg::grid_group& grid, double* smem, double* red) {
    pcg_entry(a);
    pcg_mark(15);
    const int nF = a.nF;
    const int chunk = (nF + gridDim.x - 1) / gridDim.x;
    const int row0 = blockIdx.x * chunk;
    const int row1 = min(nF, row0 + chunk);
    int parity = 0;
    __shared__ unsigned int s_base;
    if (threadIdx.x == 0) s_base = ld_acquire_gpu(a.flags + (size_t)blockIdx.x * 32);
    const int pdi_w = a.pd_iter_dev != nullptr ? *a.pd_iter_dev : a.pd_iter;
    const bool warm = a.warm != nullptr && a.init == INIT_PD && pdi_w < a.warm_rounds;
    vec4_t<T>* const wb = warm ? a.warm + (size_t)pdi_w * nF : nullptr;
    // ring of the last three frames' round corrections (frame f writes bank f % 3): the guess
    // 3 d_{f-1} - 3 d_{f-2} + d_{f-3} is formed where it is read, and the finish stores one bank
    const bool ring = REG && warm && a.warm_ring != nullptr;
    const vec4_t<T>* g1 = nullptr;
    const vec4_t<T>* g2 = nullptr;
    const vec4_t<T>* g3 = nullptr;
    vec4_t<T>* gw = nullptr;
    if (ring) {
        const unsigned f = *a.warm_ring;
        vec4_t<T>* const R[4] = {a.warm, a.warm_prev, a.warm_prev2, a.warm_prev3};
        gw = R[f % 4u] + (size_t)pdi_w * nF;          // d_{f-4}, overwritten by this frame's finish
        g1 = R[(f + 3u) % 4u] + (size_t)pdi_w * nF;
        g2 = R[(f + 2u) % 4u] + (size_t)pdi_w * nF;
        g3 = R[(f + 1u) % 4u] + (size_t)pdi_w * nF;
    }
    // cubic extrapolation 4 d1 - 6 d2 + 4 d3 - d4 while the motion is smooth (no tet took the
    // robust SL(3) path this round), the last frame's correction d1 otherwise (C3 210-frame
    // series, steps per steady / fold frame: quadratic 1,070 / 1,920, cubic 971 / 2,006, linear in
    // the fold 1,844, constant 1,793)
    const bool smooth = ring && *a.robust_present == 0;
    const T w1 = smooth ? T(4) : T(1), w2 = smooth ? T(-6) : T(0), w3 = smooth ? T(4) : T(0),
            w4 = smooth ? T(-1) : T(0);
    auto guess_at = [&](int j) -> vec4_t<T> {
        if (!ring) return ld4(&wb[j]);
        const vec4_t<T> p = ld4(&g1[j]), q = ld4(&g2[j]), o = ld4(&g3[j]), u = ld4(&gw[j]);
        return make4<T>(w1 * p.x + w2 * q.x + w3 * o.x + w4 * u.x, w1 * p.y + w2 * q.y + w3 * o.y + w4 * u.y,
                        w1 * p.z + w2 * q.z + w3 * o.z + w4 * u.z, T(0));
    };

    const double lmin = a.cheb_lmin, lmax = a.cheb_lmax;
    const double theta = 0.5 * (lmax + lmin), delta = 0.5 * (lmax - lmin);
    const double sigma = theta / delta;
    const double acosh_sigma = acosh(sigma);
    double tol_k = a.tol;
    if (a.tol_growth > 1.0 && a.init == INIT_PD && a.rounds_total > 0)
        tol_k *= pow(a.tol_growth, (double)max(0, a.rounds_total - 1 - pdi_w));

    // ---- init: res = b - K x (PD residual form) minus K * warm guess; y = guess; d0 = D^-1 res / theta
    const int i = row0 + threadIdx.x;              // REG path: this thread's row
    const bool own = REG && i < row1;
    unsigned colp[(kChebOff + 1) / 2];             // REG: image byte offsets of the off-diagonal columns
                                                   //      (two 16-bit per register)
    T kdiag = 0;
    extern __shared__ __align__(16) unsigned char cheb_smem[];
    using DS = typename ChebImage<T>::type;
    DS* const sd = reinterpret_cast<DS*>(cheb_smem);   // REG: d planes, buffer p at sd + 3 p kChebSlots
    T* const yv0 = reinterpret_cast<T*>(sd + 6 * kChebSlots);
    T* yv = yv0 + threadIdx.x;                     // REG: this row's y, planes kChebMaxThreads apart
    T* const sv = yv0 + 3 * kChebMaxThreads + threadIdx.x;   // REG: this row's ELL values, planes apart
    int* hidx = reinterpret_cast<int*>(yv0 + (3 + kChebOff) * kChebMaxThreads);   // REG: halo rows
    // exported rows [row0, row0 + nexp) belong to the leading warps
    const int nexp = REG ? a.cheb_nexp[blockIdx.x] : 0;
    // the exported-warp group also covers the halo rows: one halo row per thread, one L2 round trip
    const int nh = REG ? a.cheb_halo_ptr[blockIdx.x + 1] - a.cheb_halo_ptr[blockIdx.x] : 0;
    const int exp_threads = min((int)blockDim.x, max(32, (max(nexp, nh) + 31) & ~31));
    const bool exp_warp = (int)threadIdx.x < exp_threads;
    if (REG) {
        const int* halo = a.cheb_halo + a.cheb_halo_ptr[blockIdx.x];
        for (int j = threadIdx.x; j < nh; j += blockDim.x) hidx[j] = __ldg(&halo[j]);
    }
    T rx = 0, ry = 0, rzz = 0, dxv = 0, dyv = 0, dzv = 0, dg = 0;
    double acc[2] = {0, 0};                        // rr, bb
    if (REG) {
        // the residual's corner gather, then the row's ELL (loading it first, live across the
        // gather, measured slower: 25 vs 21 us per launch)
        if (own) {
            init_residual_row(a, i, false, rx, ry, rzz, acc[1]);
#pragma unroll
            for (int h = 0; h < (kChebOff + 1) / 2; ++h) colp[h] = __ldg(&a.cheb_slot[(size_t)h * nF + i]);
#pragma unroll
            for (int s = 0; s < kChebOff; ++s) sv[s * kChebMaxThreads] = __ldg(&a.cheb_val[(size_t)s * nF + i]);
            kdiag = __ldg(&a.cheb_kdiag[i]);
            dg = a.inv_diag[i];
        }
        pcg_mark(16);
        if (warm) {
            // K * guess from shared memory like a step: own rows' guesses and the halo rows'
            // (written by the previous frame's launch: plain loads) into buffer 1's planes
            DS* const sg = sd + 3 * kChebSlots;
            T gx = 0, gy = 0, gz = 0;
            __syncthreads();                       // hidx
            if (own) {
                const vec4_t<T> g = guess_at(i);
                gx = (T)img_dec(img_enc<DS>(g.x)); gy = (T)img_dec(img_enc<DS>(g.y));   // the guess as applied
                gz = (T)img_dec(img_enc<DS>(g.z));
                sg[threadIdx.x] = img_enc<DS>(gx); sg[kChebSlots + threadIdx.x] = img_enc<DS>(gy);
                sg[2 * kChebSlots + threadIdx.x] = img_enc<DS>(gz);
            }
            for (int j = threadIdx.x; j < nh; j += blockDim.x) {
                const vec4_t<T> g = guess_at(hidx[j]);
                const int sl = blockDim.x + j;
                sg[sl] = img_enc<DS>(g.x); sg[kChebSlots + sl] = img_enc<DS>(g.y); sg[2 * kChebSlots + sl] = img_enc<DS>(g.z);
            }
            __syncthreads();
            if (own) {
                T qx = kdiag * gx, qy = kdiag * gy, qz = kdiag * gz;
                spmv_img<1, DS>(sd, colp, sv, qx, qy, qz);
                if (a.cdiag != nullptr) {
                    const T cd = a.cdiag[i];
                    qx += cd * gx; qy += cd * gy; qz += cd * gz;
                }
                rx -= qx; ry -= qy; rzz -= qz;
            }
            yv[0] = gx; yv[kChebMaxThreads] = gy; yv[2 * kChebMaxThreads] = gz;
        } else {
            yv[0] = T(0); yv[kChebMaxThreads] = T(0); yv[2 * kChebMaxThreads] = T(0);
        }
        pcg_mark(17);
        if (own) {
            const T c0 = (T)(1.0 / theta) * dg;
            dxv = c0 * rx; dyv = c0 * ry; dzv = c0 * rzz;
            sd[threadIdx.x] = img_enc<DS>(dxv); sd[kChebSlots + threadIdx.x] = img_enc<DS>(dyv);
            sd[2 * kChebSlots + threadIdx.x] = img_enc<DS>(dzv);
            acc[0] = (double)rx * rx + (double)ry * ry + (double)rzz * rzz;
        }
    } else {
        for (int j = row0 + threadIdx.x; j < row1; j += blockDim.x) {
            T ax, ay, az;
            init_residual_row(a, j, false, ax, ay, az, acc[1]);
            vec4_t<T> y0 = make4<T>(T(0), T(0), T(0), T(0));
            if (warm) {
                y0 = ld4(&wb[j]);
                const vec4_t<T> kw = k_row(a, wb, j);
                ax -= kw.x; ay -= kw.y; az -= kw.z;
            }
            const T c0 = (T)(1.0 / theta) * a.inv_diag[j];
            a.r[j] = make4<T>(ax, ay, az, T(0));
            a.dx[j] = y0;
            a.p0[j] = make4<T>(c0 * ax, c0 * ay, c0 * az, T(0));
            acc[0] += (double)ax * ax + (double)ay * ay + (double)az * az;
        }
    }
    pcg_allreduce<2>(grid, a.partials, parity, acc, red, smem);
    double rr = red[0];
    const double bb = red[1];
    const double thr = tol_k * tol_k * bb;
    const unsigned int base = s_base;
    const int* nbr = a.cheb_nbr + a.cheb_nbr_ptr[blockIdx.x];
    const int nn = a.cheb_nbr_ptr[blockIdx.x + 1] - a.cheb_nbr_ptr[blockIdx.x];

    int k = 0;
    double rho = 1.0 / sigma;
    const double two_over_delta = 2.0 / delta;
    constexpr int LLW = LLRow<DS>::W;
    if (rr > thr && a.max_iters > 0) {
        int target = min(a.max_iters, cheb_steps_for(sqrt(rr / thr), acosh_sigma));
        if (REG && own && (int)threadIdx.x < nexp)
            ll_store(a.cheb_ll + (size_t)i * LLW, img_enc<DS>(dxv), img_enc<DS>(dyv), img_enc<DS>(dzv), base);
        for (;;) {
            for (; k < target; ++k) {
                pcg_mark(10);
                if (!REG && k > 0) cheb_wait(a.flags, nbr, nn, base + (unsigned)k);
                const vec4_t<T>* dcur = (k & 1) ? a.p1 : a.p0;
                vec4_t<T>* dnext = (k & 1) ? a.p0 : a.p1;
                const double rho_n = 1.0 / (2.0 * sigma - rho);
                const T c1 = (T)(rho_n * rho), c2 = (T)(rho_n * two_over_delta);
                rho = rho_n;
                if (REG) {
                    DS* const sx = sd + (k & 1) * 3 * kChebSlots;         // d_k
                    DS* const sn = sd + ((k + 1) & 1) * 3 * kChebSlots;   // d_{k+1} (own rows)
                    // every own row's d_k is in shared memory (written by step k-1)
                    if (k > 0) __syncthreads();
                    if (exp_warp) {
                        // exported warps: the halo rows of d_k (flag-in-data, each row spins on its
                        // own tag), then the exported rows.  (Doing the own-column part of the
                        // exported rows before the halo and only the halo columns after it measured
                        // slower: 12.9 vs 9.0 ms/frame at C3 fp64, per-entry predicates diverge.)
                        pcg_mark(11);
                        const uint4* src = a.cheb_ll + (size_t)(k & 1) * nF * LLW;
                        for (int j = threadIdx.x; j < nh; j += exp_threads) {
                            DS hx, hy, hz;
                            ll_load(src + (size_t)hidx[j] * LLW, base + (unsigned)k, hx, hy, hz);
                            const int sl = blockDim.x + j;
                            sx[sl] = hx; sx[kChebSlots + sl] = hy; sx[2 * kChebSlots + sl] = hz;
                        }
                        // non-.aligned barrier: the halo loop before it leaves the warp's lanes diverged
                        asm volatile("barrier.sync 1, %0;" ::"r"(exp_threads) : "memory");
                        pcg_mark(12);
                    }
                    // interior warps run their rows meanwhile: they read own rows only
                    // the applied direction (own row): the image's rounding of d_k
                    const DS ex = img_enc<DS>(dxv), ey = img_enc<DS>(dyv), ez = img_enc<DS>(dzv);
                    const T ax = (T)img_dec(ex), ay = (T)img_dec(ey), az = (T)img_dec(ez);
                    T qx = kdiag * ax, qy = kdiag * ay, qz = kdiag * az;
                    if (own) {
                        if (k & 1) spmv_img<1, DS>(sd, colp, sv, qx, qy, qz);
                        else spmv_img<0, DS>(sd, colp, sv, qx, qy, qz);
                        if (a.cdiag != nullptr) {
                            const T cd = a.cdiag[i];
                            qx += cd * ax; qy += cd * ay; qz += cd * az;
                        }
                        yv[0] += ax; yv[kChebMaxThreads] += ay; yv[2 * kChebMaxThreads] += az;
                        rx -= qx; ry -= qy; rzz -= qz;
                        const T e = c2 * dg;
                        dxv = c1 * dxv + e * rx;
                        dyv = c1 * dyv + e * ry;
                        dzv = c1 * dzv + e * rzz;
                        const DS nx = img_enc<DS>(dxv), ny = img_enc<DS>(dyv), nz = img_enc<DS>(dzv);
                        sn[threadIdx.x] = nx; sn[kChebSlots + threadIdx.x] = ny; sn[2 * kChebSlots + threadIdx.x] = nz;
                        if ((int)threadIdx.x < nexp)
                            ll_store(a.cheb_ll + (size_t)((k + 1) & 1) * nF * LLW + (size_t)i * LLW, nx, ny, nz,
                                     base + (unsigned)(k + 1));
                    }
                    pcg_mark(13);
                } else {
                    for (int j = row0 + threadIdx.x; j < row1; j += blockDim.x) {
                        T qx = 0, qy = 0, qz = 0;
                        for (int s = 0; s < a.ell_w; ++s) {
                            const int c = __ldg(&a.ell_col[(size_t)s * nF + j]);
                            const T kv = __ldg(&a.ell_val[(size_t)s * nF + j]);
                            T vx, vy, vz;
                            ldcg3(&dcur[c], vx, vy, vz);
                            qx += kv * vx; qy += kv * vy; qz += kv * vz;
                        }
                        vec4_t<T> dj;
                        ldcg3(&dcur[j], dj.x, dj.y, dj.z);
                        if (a.cdiag != nullptr) {
                            const T cd = a.cdiag[j];
                            qx += cd * dj.x; qy += cd * dj.y; qz += cd * dj.z;
                        }
                        vec4_t<T> y = a.dx[j], r = a.r[j];
                        y.x += dj.x; y.y += dj.y; y.z += dj.z;
                        r.x -= qx; r.y -= qy; r.z -= qz;
                        const T e = c2 * a.inv_diag[j];
                        a.dx[j] = y;
                        a.r[j] = r;
                        st4(&dnext[j], make4<T>(c1 * dj.x + e * r.x, c1 * dj.y + e * r.y, c1 * dj.z + e * r.z, T(0)));
                    }
                }
                if (!REG) cheb_publish(a.flags, base + (unsigned)(k + 1));
            }
            // residual check (one grid barrier): the same rule as the CG
            double acc1[1] = {0.0};
            if (REG) {
                if (own) acc1[0] = (double)rx * rx + (double)ry * ry + (double)rzz * rzz;
            } else {
                for (int j = row0 + threadIdx.x; j < row1; j += blockDim.x) {
                    const vec4_t<T> r = a.r[j];
                    acc1[0] += (double)r.x * r.x + (double)r.y * r.y + (double)r.z * r.z;
                }
            }
            pcg_allreduce<1>(grid, a.partials, parity, acc1, red, smem);
            rr = red[0];
            if (!(rr > thr) || k >= a.max_iters) break;      // also stops on NaN
            target = min(a.max_iters, k + 1 + cheb_steps_for(sqrt(rr / thr), acosh_sigma));
        }
    }
    // REG: the next launch's tags start above every tag this one wrote
    if (REG && threadIdx.x == 0) a.flags[(size_t)blockIdx.x * 32] = base + (unsigned)k + 1u;
    // ---- finish: x += y (PD mode), warm-start bank, finite check
    bool bad = a.init == INIT_PD && !(rr == rr && rr < INFINITY);
    auto finish_row = [&](int j, vec4_t<T> d) {
        vec4_t<T> xi = a.x[j];
        xi.x += d.x; xi.y += d.y; xi.z += d.z;
        a.x[j] = xi;
        if (ring) {
            gw[j] = d;
        } else if (warm) {
            if (a.warm_prev != nullptr && pdi_w < a.warm_extrap_rounds) {
                vec4_t<T>* wp = a.warm_prev + (size_t)pdi_w * nF;
                const vec4_t<T> dp = ld4(&wp[j]);
                wp[j] = d;
                if (a.warm_prev2 != nullptr) {          // quadratic: 3 d - 3 d' + d''
                    vec4_t<T>* wq = a.warm_prev2 + (size_t)pdi_w * nF;
                    const vec4_t<T> dq = ld4(&wq[j]);
                    wq[j] = dp;
                    wb[j] = make4<T>(T(3) * (d.x - dp.x) + dq.x, T(3) * (d.y - dp.y) + dq.y,
                                     T(3) * (d.z - dp.z) + dq.z, T(0));
                } else {
                    const T be = (T)a.warm_beta;
                    wb[j] = make4<T>(d.x + be * (d.x - dp.x), d.y + be * (d.y - dp.y), d.z + be * (d.z - dp.z), T(0));
                }
            } else {
                wb[j] = d;
            }
        }
        bad |= !(isfinite(xi.x) && isfinite(xi.y) && isfinite(xi.z));
    };
    if (k > 0 || bad || warm) {
        if (REG) {
            if (own) finish_row(i, make4<T>(yv[0], yv[kChebMaxThreads], yv[2 * kChebMaxThreads], T(0)));
        } else {
            for (int j = row0 + threadIdx.x; j < row1; j += blockDim.x) finish_row(j, a.dx[j]);
        }
    }
    pcg_mark(19);
    pcg_exit(a, bad, k, warm);
    pcg_mark(20);
}

#ifndef VK_CHEB_THREADS
#define VK_CHEB_THREADS 768
#endif
template <typename T>
// (80 registers: up to 6 warps per SM sub-partition of 16K registers; 88 would need <= 20 warps)
__global__ void __launch_bounds__(VK_CHEB_THREADS, 1) k_cheb_reg(PcgArgs<T> a) {
    cg::grid_group grid = cg::this_grid();
    __shared__ double smem[32 * 8];
    __shared__ double red[8];
    cheb_body<T, true>(a, grid, smem, red);
}
template <typename T>
__global__ void __launch_bounds__(VK_CHEB_THREADS, 1) k_cheb(PcgArgs<T> a) {
    cg::grid_group grid = cg::this_grid();
    __shared__ double smem[32 * 8];
    __shared__ double red[8];
    cheb_body<T, false>(a, grid, smem, red);
}

// ---------------------------------------------------------------------------
// Lanczos on D^-1/2 K_ff D^-1/2 (no reorthogonalisation: only the extreme Ritz
// values are used), one cooperative launch, deterministic reductions.
// alpha[j], beta[j+1] for j < m; v0 from a fixed hash (reproducible).
template <typename T>
struct LanczosArgs {
    int nF, ell_w, m;
    const int* ell_col;
    const T* ell_val;
    const double* diag64;
    double* v0;       // 3 vectors of nF: v_{j-1}, v_j, w
    double* v1;
    double* w;
    double* partials;
    double* alpha;
    double* beta;
};

__device__ __forceinline__ double lanczos_start(int i) {
    unsigned int h = (unsigned int)i * 2654435761u + 0x9e3779b9u;
    h ^= h >> 16; h *= 0x85ebca6bu; h ^= h >> 13; h *= 0xc2b2ae35u; h ^= h >> 16;
    return (double)(h & 0xffffff) / 16777216.0 - 0.5;
}

template <typename T>
__global__ void __launch_bounds__(512) k_lanczos(LanczosArgs<T> a) {
    cg::grid_group grid = cg::this_grid();
    __shared__ double smem[32 * 8];
    __shared__ double red[8];
    int parity = 0;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
    double acc[1] = {0.0};
    for (int i = tid; i < a.nF; i += nth) {
        const double s = lanczos_start(i);
        a.v1[i] = s;
        a.v0[i] = 0.0;
        acc[0] += s * s;
    }
    pcg_allreduce<1>(grid, a.partials, parity, acc, red, smem);
    double inv = 1.0 / sqrt(red[0]);
    for (int i = tid; i < a.nF; i += nth) a.v1[i] *= inv;
    grid.sync();
    double beta = 0.0;
    double* vp = a.v0;
    double* vc = a.v1;
    for (int j = 0; j < a.m; ++j) {
        // w = A v_j - beta_j v_{j-1};  alpha_j = w . v_j
        double ac[1] = {0.0};
        for (int i = tid; i < a.nF; i += nth) {
            const double si = rsqrt(a.diag64[i]);
            double h = 0.0;
            for (int s = 0; s < a.ell_w; ++s) {
                const int c = a.ell_col[(size_t)s * a.nF + i];
                h += (double)a.ell_val[(size_t)s * a.nF + i] * rsqrt(a.diag64[c]) * __ldcg(&vc[c]);
            }
            const double wi = si * h - beta * __ldcg(&vp[i]);
            a.w[i] = wi;
            ac[0] += wi * __ldcg(&vc[i]);
        }
        pcg_allreduce<1>(grid, a.partials, parity, ac, red, smem);
        const double alpha = red[0];
        double bc[1] = {0.0};
        for (int i = tid; i < a.nF; i += nth) {
            const double wi = a.w[i] - alpha * __ldcg(&vc[i]);
            a.w[i] = wi;
            bc[0] += wi * wi;
        }
        pcg_allreduce<1>(grid, a.partials, parity, bc, red, smem);
        const double bn = sqrt(red[0]);
        if (blockIdx.x == 0 && threadIdx.x == 0) { a.alpha[j] = alpha; a.beta[j + 1] = bn; }
        if (!(bn > 0.0)) break;
        const double ib = 1.0 / bn;
        for (int i = tid; i < a.nF; i += nth) vp[i] = a.w[i] * ib;     // v_{j+1} into the old v_{j-1}
        grid.sync();
        double* t = vp; vp = vc; vc = t;
        beta = bn;
    }
}

}  // namespace vk

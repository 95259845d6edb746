// Common device helpers for the PD step library (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cuda/atomic>

namespace vk {

template <typename T> struct Vec4;
template <> struct Vec4<float> { using type = float4; };
template <> struct Vec4<double> { using type = double4; };
template <typename T> using vec4_t = typename Vec4<T>::type;

template <typename T> __device__ __forceinline__ vec4_t<T> make4(T a, T b, T c, T d);
template <> __device__ __forceinline__ float4 make4<float>(float a, float b, float c, float d) {
    return make_float4(a, b, c, d);
}
template <> __device__ __forceinline__ double4 make4<double>(double a, double b, double c, double d) {
    return make_double4(a, b, c, d);
}

// 16-B (float4) / 32-B (double4) vector load through the read-only path.
__device__ __forceinline__ float4 ldg4(const float4* p) { return __ldg(p); }
__device__ __forceinline__ double4 ldg4(const double4* p) {
    double4 r;
    asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w) : "l"(p));
    return r;
}
// plain (coherent) vector load for data written earlier in the same kernel
__device__ __forceinline__ float4 ld4(const float4* p) { return *p; }
__device__ __forceinline__ double4 ld4(const double4* p) {
    double4 r;
    asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w) : "l"(p) : "memory");
    return r;
}
__device__ __forceinline__ void st4(float4* p, float4 v) { *p = v; }
__device__ __forceinline__ void st4(double4* p, double4 v) {
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};"
                 :: "l"(p), "d"(v.x), "d"(v.y), "d"(v.z), "d"(v.w) : "memory");
}

#define VK_HD __host__ __device__ __forceinline__
#define VK_HDNI __host__ __device__ __noinline__

template <typename T> VK_HD T rsqrt_(T x);
template <> VK_HD float rsqrt_<float>(float x) {
#ifdef __CUDA_ARCH__
    return rsqrtf(x);
#else
    return 1.0f / sqrtf(x);
#endif
}
template <> VK_HD double rsqrt_<double>(double x) {
#ifdef __CUDA_ARCH__
    return rsqrt(x);
#else
    return 1.0 / sqrt(x);
#endif
}

template <typename T> struct Eps;
template <> struct Eps<float> { static constexpr float v = 1.1920929e-7f; };
template <> struct Eps<double> { static constexpr double v = 2.220446049250313e-16; };

// ---------------------------------------------------------------------------
// Grid-wide barrier for a cooperatively launched (co-resident) grid.
//
// Sense-reversing counter + generation word.  The last CTA to arrive runs
// `on_last` (a deterministic grid reduction over per-CTA partials, fixed
// order) before releasing everyone, so the reduced scalars are published by
// the barrier itself.  A bounded spin turns a lost CTA into a trap instead
// of a hang.
struct GridBar {
    unsigned int count;
    unsigned int gen;
};

template <typename OnLast>
__device__ __forceinline__ void grid_sync(GridBar* bar, OnLast on_last) {
    __syncthreads();
    __shared__ int s_last;
    if (threadIdx.x == 0) {
        cuda::atomic_ref<unsigned int, cuda::thread_scope_device> gen(bar->gen);
        cuda::atomic_ref<unsigned int, cuda::thread_scope_device> cnt(bar->count);
        unsigned int g = gen.load(cuda::memory_order_relaxed);
        __threadfence();
        unsigned int arrived = cnt.fetch_add(1u, cuda::memory_order_acq_rel);
        s_last = (arrived == gridDim.x - 1) ? 1 : 0;
        if (!s_last) {
            unsigned long long spins = 0;
            while (gen.load(cuda::memory_order_acquire) == g) {
                if (++spins > (1ull << 31)) __trap();
                if (spins > 64) __nanosleep(20);
            }
        }
        __threadfence();
    }
    __syncthreads();
    if (s_last) {
        on_last();                    // whole CTA participates
        __syncthreads();
        if (threadIdx.x == 0) {
            cuda::atomic_ref<unsigned int, cuda::thread_scope_device> gen(bar->gen);
            cuda::atomic_ref<unsigned int, cuda::thread_scope_device> cnt(bar->count);
            __threadfence();
            cnt.store(0u, cuda::memory_order_relaxed);
            gen.fetch_add(1u, cuda::memory_order_release);
        }
        __syncthreads();
    }
}

struct NoOp { __device__ void operator()() const {} };

// Lean grid barrier: one release-add per CTA, tight acquire-poll on the
// generation word (no sleep), no serial reduction step.  Callers that need
// grid-wide sums write per-CTA partials before the barrier and every CTA
// reduces them afterwards in the same fixed order (identical results).
__device__ __forceinline__ unsigned int ld_acquire_gpu(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned int atom_add_acqrel_gpu(unsigned int* p, unsigned int v) {
    unsigned int old;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ void st_release_gpu(unsigned int* p, unsigned int v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void grid_sync_lean(GridBar* bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int g = ld_acquire_gpu(&bar->gen);
        const unsigned int arrived = atom_add_acqrel_gpu(&bar->count, 1u);
        if (arrived == gridDim.x - 1) {
            bar->count = 0;                      // ordered before the release below
            st_release_gpu(&bar->gen, g + 1u);
        } else {
            unsigned long long spins = 0;
            while (ld_acquire_gpu(&bar->gen) == g) {
                if (++spins > (1ull << 33)) __trap();
            }
        }
    }
    __syncthreads();
}

// Block-wide sum of NV doubles per thread; result valid in thread 0.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* smem /* >= 32*NV */) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
    }
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) smem[warp * NV + k] = v[k];
    }
    __syncthreads();
    // second level: warp 0 combines the per-warp sums with a shuffle tree
    // (a serial loop over warps in thread 0 cost ~1 us at 16 warps)
    if (warp == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            double a = lane < nw ? smem[lane * NV + k] : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
            v[k] = a;
        }
    }
    __syncthreads();
}

// After grid_sync_lean: sum NV per-CTA partials (stride 8 doubles) in fixed
// order; every CTA gets the same bits.  Result broadcast through `out` (smem).
template <int NV>
__device__ __forceinline__ void reduce_partials_all(const double* partials, double* out, double* smem) {
    double v[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
#pragma unroll
        for (int k = 0; k < NV; ++k) v[k] += __ldcg(&partials[b * 8 + k]);
    }
    block_sum<NV>(v, smem);
    if (threadIdx.x == 0)
#pragma unroll
        for (int k = 0; k < NV; ++k) out[k] = v[k];
    __syncthreads();
}

// ---------------------------------------------------------------------------
// All-to-all flag barrier with a fused, deterministic all-reduce.
//
// Every CTA owns one 64-byte slot {7 doubles, epoch}.  To cross a barrier a
// CTA publishes its partial sums and the new epoch (release store after a
// __syncthreads, so all of the CTA's earlier global writes are ordered before
// it); then thread t polls slot t with acquire loads until its epoch arrives
// and the CTA sums the slots in index order.  No atomics, no serial "last
// CTA" step, and the reduction rides on the barrier's own traffic.  Every CTA
// adds the same values in the same order, so all get identical bits.
// Requires gridDim.x <= blockDim.x.  Epochs increase monotonically across
// launches (the caller persists the base), so slots never need resetting.
struct alignas(64) FlagSlot {
    double v[7];
    unsigned long long epoch;
};

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}

// `part` holds this CTA's NV partials in thread 0 (e.g. from block_sum); on
// return `out[0..NV)` (shared memory) holds the grid-wide sums in every CTA.
template <int NV>
__device__ __forceinline__ void grid_allreduce(FlagSlot* slots, unsigned long long epoch, const double (&part)[NV],
                                               double* out, double* smem) {
    static_assert(NV <= 7, "at most 7 values per slot");
    // two slot banks by epoch parity: a CTA can only reuse a bank after every
    // CTA has published the next epoch, i.e. finished reading this one
    slots += (epoch & 1ull) * gridDim.x;
    if (threadIdx.x == 0) {
        FlagSlot* me = &slots[blockIdx.x];
#pragma unroll
        for (int k = 0; k < NV; ++k) me->v[k] = part[k];
        st_release_u64(&me->epoch, epoch);
    }
    double v[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = 0.0;
    if (threadIdx.x < gridDim.x) {
        const FlagSlot* sl = &slots[threadIdx.x];
        unsigned long long spins = 0;
        while (ld_acquire_u64(&sl->epoch) < epoch) {
            if (++spins > (1ull << 33)) __trap();
        }
#pragma unroll
        for (int k = 0; k < NV; ++k) v[k] = __ldcg(&sl->v[k]);
    }
    block_sum<NV>(v, smem);
    if (threadIdx.x == 0)
#pragma unroll
        for (int k = 0; k < NV; ++k) out[k] = v[k];
    __syncthreads();
}

// Phase timeline (globaltimer marks of block 0, thread 0): experiment build only.
#ifdef VK_PCG_TRACE               // phase-timing experiment build only
__device__ unsigned long long g_pcg_trace[8192];
__device__ int g_pcg_trace_n;
__device__ __forceinline__ void pcg_mark(int tag) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        const int k = g_pcg_trace_n;
        if (k < 8190) { g_pcg_trace[k] = ((unsigned long long)tag << 56) | (t & 0xffffffffffffffull); g_pcg_trace_n = k + 1; }
    }
}
#else
__device__ __forceinline__ void pcg_mark(int) {}
#endif

}  // namespace vk

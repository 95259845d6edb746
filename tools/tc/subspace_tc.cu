// Tensor-core probe for the subspace contraction of the paper's domain-decomposed solve
// (north_star (b): U^T r with per-domain bases, pdsolver.py:546-593; SURVEY 8d "CMS apply"):
//   Y (m x 3) = U^T R,  U: m = 128 basis vectors over n = 105,560 free nodes (C3), R: n x 3.
// Three kernels, same data:
//   tc    tcgen05.mma (kind::f16, BF16 x BF16 -> FP32 in TMEM), M = 128 modes, N = 16 (3 columns
//         + zero padding), K split across 148 CTAs; operands pre-tiled in global memory in the
//         canonical K-major no-swizzle core-matrix layout and streamed by 1-D bulk copies
//         (cp.async.bulk, mbarrier complete_tx) through a 4-stage shared-memory ring; one thread
//         issues the MMAs and commits them to the ring's "empty" barriers; tcgen05.ld epilogue.
//   cc16  CUDA cores, the same BF16 U, FP32 accumulation (same bytes as tc).
//   cc64  CUDA cores, FP64 U and R (the precision the solver needs).
// Each is timed per launch with CUDA events after an L2 flush (256 MB write), 50 launches; the
// results are checked against a float64 host product.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -o subspace_tc subspace_tc.cu
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) {                                                           \
            std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            std::exit(1);                                                                  \
        }                                                                                  \
    } while (0)

constexpr int M = 128;          // basis vectors (UMMA M)
constexpr int NN = 16;          // UMMA N: 3 residual columns + 13 zeros
constexpr int KT = 64;          // nodes per stage (4 UMMA K-steps of 16)
constexpr int STAGES = 4;
constexpr int A_TILE = M * KT * 2;      // 16 KB
constexpr int B_TILE = NN * KT * 2;     // 2 KB

// ---- PTX helpers ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(b)), "r"(phase) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// K-major, no swizzle: core matrix = 8 rows x 16 B contiguous; LBO = K-half stride, SBO = 8-row stride
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;                         // descriptor version (sm_100)
    return d;                                       // base offset 0, layout SWIZZLE_NONE
}
// BF16 x BF16 -> F32, K-major A and B, M = 128, N = 16
constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(NN >> 3) << 17) | ((uint32_t)(M >> 4) << 24);

__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d), "l"(da), "l"(db),
        "r"(IDESC), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

// ---- tensor-core kernel ----------------------------------------------------------------------
// A_t: [tile][s(4)][g(16)][h(2)][r8(8)][8] bf16 (U, 16 KB per tile); B_t: [tile][s][g(2)][h][r8][8] (R^T).
__global__ void __launch_bounds__(128, 1) k_tc(const __nv_bfloat16* __restrict__ A_t, const __nv_bfloat16* __restrict__ B_t,
                                             int n_tiles, float* __restrict__ partial) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES], done;
    __shared__ uint32_t tmem_base;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int per = (n_tiles + gridDim.x - 1) / gridDim.x;
    const int t0 = blockIdx.x * per, t1 = min(n_tiles, t0 + per);
    const int nt = max(0, t1 - t0);
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        mbar_init(&done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base;
    unsigned char* As = sm;
    unsigned char* Bs = sm + STAGES * A_TILE;
    if (threadIdx.x == 0) {                           // producer: bulk copies into the ring
        for (int i = 0; i < nt; ++i) {
            const int s = i % STAGES;
            if (i >= STAGES) mbar_wait(&empty[s], ((i / STAGES) - 1) & 1);
            mbar_expect_tx(&full[s], A_TILE + B_TILE);
            bulk_g2s(As + s * A_TILE, A_t + (size_t)(t0 + i) * (A_TILE / 2), A_TILE, &full[s]);
            bulk_g2s(Bs + s * B_TILE, B_t + (size_t)(t0 + i) * (B_TILE / 2), B_TILE, &full[s]);
        }
    } else if (threadIdx.x == 32) {                   // MMA issuer
        for (int i = 0; i < nt; ++i) {
            const int s = i % STAGES;
            mbar_wait(&full[s], (i / STAGES) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint32_t a0 = smem_u32(As + s * A_TILE), b0 = smem_u32(Bs + s * B_TILE);
#pragma unroll
            for (int k = 0; k < KT / 16; ++k)
                umma(tmem, umma_desc(a0 + k * (M * 32), 128, 256), umma_desc(b0 + k * (NN * 32), 128, 256),
                     (i > 0 || k > 0) ? 1u : 0u);
            umma_commit(&empty[s]);                   // the slot is free once these MMAs have read it
        }
        umma_commit(&done);
    }
    __syncwarp();
    // epilogue: accumulator lanes = modes, columns = residual columns
    if (nt > 0) mbar_wait(&done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t r[16];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    const int mode = warp * 32 + lane;
    float* out = partial + ((size_t)blockIdx.x * M + mode) * 3;
    for (int c = 0; c < 3; ++c) out[c] = nt > 0 ? __uint_as_float(r[c]) : 0.f;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}

// fixed-order sum of the per-CTA partials
__global__ void k_sum_partials(const float* __restrict__ partial, int nb, float* __restrict__ y) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= M * 3) return;
    float s = 0.f;
    for (int b = 0; b < nb; ++b) s += partial[(size_t)b * M * 3 + i];
    y[i] = s;
}

// ---- CUDA-core kernels: one warp per (mode, node chunk), row-major U -------------------------
template <typename TU, typename TA>
__global__ void k_cc(const TU* __restrict__ U, const TA* __restrict__ R3, int n, int chunk, TA* __restrict__ partial) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int nchunks = (n + chunk - 1) / chunk;
    if (warp >= M * nchunks) return;
    const int mode = warp / nchunks, c = warp % nchunks;
    const int k0 = c * chunk, k1 = min(n, k0 + chunk);
    TA a0 = 0, a1 = 0, a2 = 0;
    for (int k = k0 + lane; k < k1; k += 32) {
        const TA u = (TA)U[(size_t)mode * n + k];
        a0 += u * R3[3 * (size_t)k]; a1 += u * R3[3 * (size_t)k + 1]; a2 += u * R3[3 * (size_t)k + 2];
    }
    for (int o = 16; o > 0; o >>= 1) {
        a0 += __shfl_xor_sync(0xffffffffu, a0, o);
        a1 += __shfl_xor_sync(0xffffffffu, a1, o);
        a2 += __shfl_xor_sync(0xffffffffu, a2, o);
    }
    if (lane == 0) {
        TA* o = partial + ((size_t)c * M + mode) * 3;
        o[0] = a0; o[1] = a1; o[2] = a2;
    }
}
template <typename TA>
__global__ void k_cc_sum(const TA* __restrict__ partial, int nb, TA* __restrict__ y) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= M * 3) return;
    TA s = 0;
    for (int b = 0; b < nb; ++b) s += partial[(size_t)b * M * 3 + i];
    y[i] = s;
}
__global__ void k_flush(float* f, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) f[i] = 0.f;
}

int main(int argc, char** argv) {
    const int n = argc > 1 ? std::atoi(argv[1]) : 105560;
    const int reps = 50;
    const int n_tiles = (n + KT - 1) / KT, np = n_tiles * KT;
    // deterministic data: smooth-ish modes and a residual
    std::vector<float> Uf((size_t)M * np, 0.f), Rf((size_t)np * 3, 0.f);
    uint64_t st = 0x9e3779b97f4a7c15ull;
    auto rnd = [&]() { st ^= st << 13; st ^= st >> 7; st ^= st << 17; return (double)(st >> 11) / 9007199254740992.0 - 0.5; };
    for (int m = 0; m < M; ++m)
        for (int k = 0; k < n; ++k) Uf[(size_t)m * np + k] = (float)(std::sin(0.001 * (m + 1) * k) + 0.1 * rnd());
    for (int k = 0; k < n; ++k)
        for (int c = 0; c < 3; ++c) Rf[(size_t)k * 3 + c] = (float)rnd();
    // bf16 copies (the tc and cc16 operands) and the float64 references
    std::vector<__nv_bfloat16> Ub((size_t)M * np), Rb((size_t)np * 3);
    for (size_t i = 0; i < Ub.size(); ++i) Ub[i] = __float2bfloat16(Uf[i]);
    for (size_t i = 0; i < Rb.size(); ++i) Rb[i] = __float2bfloat16(Rf[i]);
    std::vector<double> y_b(M * 3, 0.0), y_f(M * 3, 0.0);
    for (int m = 0; m < M; ++m)
        for (int k = 0; k < n; ++k)
            for (int c = 0; c < 3; ++c) {
                y_b[m * 3 + c] += (double)__bfloat162float(Ub[(size_t)m * np + k]) * (double)__bfloat162float(Rb[(size_t)k * 3 + c]);
                y_f[m * 3 + c] += (double)Uf[(size_t)m * np + k] * (double)Rf[(size_t)k * 3 + c];
            }
    // tiled operands for tc
    std::vector<__nv_bfloat16> At((size_t)n_tiles * M * KT), Bt((size_t)n_tiles * NN * KT, __float2bfloat16(0.f));
    for (int t = 0; t < n_tiles; ++t)
        for (int kk = 0; kk < KT; ++kk) {
            const int k = t * KT + kk, s = kk / 16, h = (kk % 16) / 8, e = kk % 8;
            for (int m = 0; m < M; ++m) {
                const size_t off = (size_t)t * M * KT + (size_t)s * M * 16 + (size_t)(m / 8) * 128 + h * 64 + (m % 8) * 8 + e;
                At[off] = Ub[(size_t)m * np + k];
            }
            for (int c = 0; c < 3; ++c) {
                const size_t off = (size_t)t * NN * KT + (size_t)s * NN * 16 + (size_t)(c / 8) * 128 + h * 64 + (c % 8) * 8 + e;
                Bt[off] = Rb[(size_t)k * 3 + c];
            }
        }
    __nv_bfloat16 *dA, *dB, *dUb, *dRb;
    float *dpart, *dy, *dflush, *dR3f, *dpart16, *dy16;
    double *dU64, *dR64, *dpart64, *dy64;
    const int nb = 148;
    CK(cudaMalloc(&dA, At.size() * 2)); CK(cudaMemcpy(dA, At.data(), At.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&dB, Bt.size() * 2)); CK(cudaMemcpy(dB, Bt.data(), Bt.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&dpart, (size_t)nb * M * 3 * 4)); CK(cudaMalloc(&dy, M * 3 * 4));
    const size_t nflush = 64ull << 20;
    CK(cudaMalloc(&dflush, nflush * 4));
    // cc16: row-major bf16 U and float R
    std::vector<float> R3f((size_t)n * 3);
    for (size_t i = 0; i < R3f.size(); ++i) R3f[i] = __bfloat162float(Rb[i]);
    std::vector<__nv_bfloat16> Ubn((size_t)M * n);
    for (int m = 0; m < M; ++m) std::memcpy(&Ubn[(size_t)m * n], &Ub[(size_t)m * np], (size_t)n * 2);
    CK(cudaMalloc(&dUb, Ubn.size() * 2)); CK(cudaMemcpy(dUb, Ubn.data(), Ubn.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&dR3f, R3f.size() * 4)); CK(cudaMemcpy(dR3f, R3f.data(), R3f.size() * 4, cudaMemcpyHostToDevice));
    const int chunk = 4096, nch = (n + chunk - 1) / chunk;
    CK(cudaMalloc(&dpart16, (size_t)nch * M * 3 * 4)); CK(cudaMalloc(&dy16, M * 3 * 4));
    // cc64
    std::vector<double> U64((size_t)M * n), R64((size_t)n * 3);
    for (int m = 0; m < M; ++m) for (int k = 0; k < n; ++k) U64[(size_t)m * n + k] = Uf[(size_t)m * np + k];
    for (size_t i = 0; i < R64.size(); ++i) R64[i] = Rf[i];
    CK(cudaMalloc(&dU64, U64.size() * 8)); CK(cudaMemcpy(dU64, U64.data(), U64.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&dR64, R64.size() * 8)); CK(cudaMemcpy(dR64, R64.data(), R64.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&dpart64, (size_t)nch * M * 3 * 8)); CK(cudaMalloc(&dy64, M * 3 * 8));
    (void)dRb;

    const int smem = STAGES * (A_TILE + B_TILE);
    CK(cudaFuncSetAttribute(k_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    auto timeit = [&](auto launch) {
        std::vector<float> ms;
        for (int r = 0; r < reps + 3; ++r) {
            k_flush<<<4 * 148, 256>>>(dflush, nflush);
            CK(cudaEventRecord(e0));
            launch();
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float t = 0;
            CK(cudaEventElapsedTime(&t, e0, e1));
            if (r >= 3) ms.push_back(t);
        }
        std::sort(ms.begin(), ms.end());
        return ms[ms.size() / 2];
    };
    const float t_tc = timeit([&] {
        k_tc<<<nb, 128, smem>>>(dA, dB, n_tiles, dpart);
        k_sum_partials<<<3, 128>>>(dpart, nb, dy);
    });
    CK(cudaGetLastError());
    const int warps = M * nch, thr = 256;
    const float t_16 = timeit([&] {
        k_cc<__nv_bfloat16, float><<<(warps * 32 + thr - 1) / thr, thr>>>(dUb, dR3f, n, chunk, dpart16);
        k_cc_sum<float><<<3, 128>>>(dpart16, nch, dy16);
    });
    const float t_64 = timeit([&] {
        k_cc<double, double><<<(warps * 32 + thr - 1) / thr, thr>>>(dU64, dR64, n, chunk, dpart64);
        k_cc_sum<double><<<3, 128>>>(dpart64, nch, dy64);
    });
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<float> y_tc(M * 3), y16(M * 3);
    std::vector<double> y64(M * 3);
    CK(cudaMemcpy(y_tc.data(), dy, M * 3 * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(y16.data(), dy16, M * 3 * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(y64.data(), dy64, M * 3 * 8, cudaMemcpyDeviceToHost));
    auto rel = [&](auto& a, std::vector<double>& b) {
        double num = 0, den = 0;
        for (int i = 0; i < M * 3; ++i) { num += (a[i] - b[i]) * (a[i] - b[i]); den += b[i] * b[i]; }
        return std::sqrt(num / den);
    };
    const double bytes16 = (double)M * n * 2 + (double)n * 3 * 2, bytes64 = (double)M * n * 8 + (double)n * 3 * 8;
    std::printf("{\"n\": %d, \"modes\": %d, \"tc_ms\": %.5f, \"cc16_ms\": %.5f, \"cc64_ms\": %.5f, "
                "\"tc_GBs\": %.1f, \"cc16_GBs\": %.1f, \"cc64_GBs\": %.1f, "
                "\"tc_rel_err_vs_bf16_exact\": %.3e, \"cc16_rel_err_vs_bf16_exact\": %.3e, "
                "\"bf16_rel_err_vs_fp64\": %.3e, \"cc64_rel_err_vs_fp64\": %.3e, "
                "\"tc_tflops\": %.4f}\n",
                n, M, t_tc, t_16, t_64, bytes16 / t_tc / 1e6, bytes16 / t_16 / 1e6, bytes64 / t_64 / 1e6,
                rel(y_tc, y_b), rel(y16, y_b), rel(y_b, y_f), rel(y64, y_f), 2.0 * M * NN * np / t_tc / 1e9);
    return 0;
}

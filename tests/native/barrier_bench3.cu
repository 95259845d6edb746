// Test-only microbenchmark of vk::grid_allreduce (flag barrier with fused reduction).
#include <cstdio>
#include "../../paper_2405_12484_b200/csrc/vk_common.cuh"

__global__ void bars(vk::FlagSlot* slots, unsigned long long* base, int n, double* out) {
    __shared__ double smem[256];
    __shared__ double res[8];
    const unsigned long long e0 = *base;
    double acc = 0;
    for (int k = 0; k < n; ++k) {
        double part[3] = {1.0, (double)blockIdx.x, (double)k};
        vk::grid_allreduce<3>(slots, e0 + 1 + k, part, res, smem);
        acc += res[0];
    }
    if (threadIdx.x == 0 && blockIdx.x == 0) { *out = acc; }
    // next launch's base: written after the last barrier by CTA 0 only
    if (threadIdx.x == 0 && blockIdx.x == 0) *base = e0 + n;
}

int main() {
    vk::FlagSlot* s; unsigned long long* base; double* o;
    cudaMalloc(&s, sizeof(vk::FlagSlot) * 2 * 1024); cudaMemset(s, 0, sizeof(vk::FlagSlot) * 2 * 1024);
    cudaMalloc(&base, 8); cudaMemset(base, 0, 8); cudaMalloc(&o, 8);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int thr : {256, 512, 1024}) for (int g : {148, 296}) {
        if (g > thr) continue;
        if (thr == 1024 && g > 148) continue;
        for (int n : {0, 100}) {
            void* args[] = {&s, &base, &n, &o};
            cudaLaunchCooperativeKernel((void*)bars, g, thr, args, 0, 0);
            cudaDeviceSynchronize();
            cudaEventRecord(a);
            for (int rep = 0; rep < 10; ++rep) cudaLaunchCooperativeKernel((void*)bars, g, thr, args, 0, 0);
            cudaEventRecord(b);
            cudaError_t e = cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            double h; cudaMemcpy(&h, o, 8, cudaMemcpyDeviceToHost);
            printf("threads=%d grid=%d barriers=%d  us/launch=%.2f  check=%g (expect %d) err=%s\n", thr, g, n, ms * 100, h, n * g, cudaGetErrorString(e));
        }
    }
    return 0;
}

// Test-only microbenchmark of vk::grid_sync_lean + reduce_partials_all.
#include <cstdio>
#include "../../paper_2405_12484_b200/csrc/vk_common.cuh"

__global__ void bars(vk::GridBar* bar, int n, double* partials, double* out) {
    __shared__ double smem[256];
    __shared__ double res[8];
    for (int k = 0; k < n; ++k) {
        double* P = partials + (k & 1) * 8 * 4096;
        if (threadIdx.x == 0) P[blockIdx.x * 8] = k;
        vk::grid_sync_lean(bar);
        vk::reduce_partials_all<3>(P, res, smem);
    }
    if (threadIdx.x == 0 && blockIdx.x == 0) *out = res[0];
}

int main() {
    vk::GridBar* bar; double *p, *o;
    cudaMalloc(&bar, sizeof(vk::GridBar)); cudaMemset(bar, 0, sizeof(vk::GridBar));
    cudaMalloc(&p, 8 * 8 * 4096 * 2); cudaMemset(p, 0, 8 * 8 * 4096 * 2); cudaMalloc(&o, 8);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int thr : {256, 512, 1024}) for (int g : {148, 296, 413}) {
        if (thr == 1024 && g > 148) continue;
        for (int n : {0, 100}) {
            void* args[] = {&bar, &n, &p, &o};
            cudaLaunchCooperativeKernel((void*)bars, g, thr, args, 0, 0);
            cudaDeviceSynchronize();
            cudaEventRecord(a);
            for (int rep = 0; rep < 10; ++rep) cudaLaunchCooperativeKernel((void*)bars, g, thr, args, 0, 0);
            cudaEventRecord(b);
            cudaError_t e = cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            printf("threads=%d grid=%d barriers=%d  us/launch=%.2f  err=%s\n", thr, g, n, ms * 100, cudaGetErrorString(e));
        }
    }
    return 0;
}

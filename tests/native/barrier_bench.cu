// Test-only microbenchmark of vk::grid_sync (cooperative launch), reports us/barrier.
#include <cstdio>
#include "../../paper_2405_12484_b200/csrc/vk_common.cuh"

__global__ void bars(vk::GridBar* bar, int n, double* partials, double* out) {
    __shared__ double smem[256];
    for (int k = 0; k < n; ++k) {
        if (threadIdx.x == 0) partials[blockIdx.x] = k;
        vk::grid_sync(bar, [&]() {
            double v = 0;
            for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) v += partials[b];
            double arr[1] = {v};
            vk::block_sum<1>(arr, smem);
            if (threadIdx.x == 0) *out = arr[0];
        });
    }
}
__global__ void empty_k() {}

int main() {
    vk::GridBar* bar; double *p, *o;
    cudaMalloc(&bar, sizeof(vk::GridBar)); cudaMemset(bar, 0, sizeof(vk::GridBar));
    cudaMalloc(&p, 8 * 4096); cudaMalloc(&o, 8);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    int grids[] = {148, 296, 413, 592};
    for (int g : grids) {
        for (int n : {0, 1, 100}) {
            void* args[] = {&bar, &n, &p, &o};
            cudaLaunchCooperativeKernel((void*)bars, g, 256, args, 0, 0);
            cudaDeviceSynchronize();
            cudaEventRecord(a);
            for (int rep = 0; rep < 10; ++rep) cudaLaunchCooperativeKernel((void*)bars, g, 256, args, 0, 0);
            cudaEventRecord(b);
            cudaError_t e = cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            printf("grid=%d barriers=%d  us/launch=%.2f  err=%s\n", g, n, ms * 100, cudaGetErrorString(e));
        }
    }
    cudaEventRecord(a);
    for (int rep = 0; rep < 100; ++rep) empty_k<<<148, 256>>>();
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("empty normal launch us=%.2f\n", ms * 10);
    return 0;
}

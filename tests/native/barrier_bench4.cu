// Test-only: barrier implementation variants, us per barrier.
#include <cstdio>
#include <cooperative_groups.h>
#include "../../paper_2405_12484_b200/csrc/vk_common.cuh"
namespace cg = cooperative_groups;

template <int V>
__global__ void bars(unsigned int* cnt, unsigned int* gen, int n) {
    unsigned int g0 = 0;
    if (threadIdx.x == 0) g0 = *((volatile unsigned int*)gen);
    for (int k = 0; k < n; ++k) {
        if (V == 4) { cg::this_grid().sync(); continue; }
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned int want = g0 + 1;
            if (V == 2) __threadfence();
            unsigned int arrived;
            if (V == 1) arrived = vk::atom_add_acqrel_gpu(cnt, 1u);
            else arrived = atomicAdd(cnt, 1u);
            if (arrived == gridDim.x - 1) {
                *((volatile unsigned int*)cnt) = 0;
                if (V == 1) vk::st_release_gpu(gen, want);
                else { if (V == 2) __threadfence(); *((volatile unsigned int*)gen) = want; }
            } else {
                if (V == 1) { while (vk::ld_acquire_gpu(gen) != want) {} }
                else { while (*((volatile unsigned int*)gen) != want) {} }
            }
            g0 = want;
        }
        __syncthreads();
    }
}

int main() {
    unsigned int *c, *g;
    cudaMalloc(&c, 4); cudaMalloc(&g, 4); cudaMemset(c, 0, 4); cudaMemset(g, 0, 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    void* ks[] = {(void*)bars<1>, (void*)bars<2>, (void*)bars<3>, (void*)bars<4>};
    const char* names[] = {"acqrel", "fence+relaxed", "nofence(unsafe)", "cg.grid.sync"};
    for (int v = 0; v < 4; ++v) for (int grid : {148, 296}) {
        int n = 200;
        void* args[] = {&c, &g, &n};
        cudaMemset(c, 0, 4); cudaMemset(g, 0, 4);
        cudaLaunchCooperativeKernel(ks[v], grid, 256, args, 0, 0);
        cudaDeviceSynchronize();
        cudaMemset(c, 0, 4); cudaMemset(g, 0, 4);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel(ks[v], grid, 256, args, 0, 0);
        cudaEventRecord(b);
        cudaError_t e = cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("%-16s grid=%d  us/barrier=%.3f err=%s\n", names[v], grid, ms * 1000 / n, cudaGetErrorString(e));
    }
    return 0;
}

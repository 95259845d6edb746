// Probe: cost profile of the batched SL(3) path (sl3::project, defer mode) on
// all sigma triples of a frame (tools/dbg/dump_robust_sigma.py ... all).
#include <cstdio>
#include <vector>
#include <algorithm>
__device__ int* g_probe;
#ifndef NO_COUNTERS
#define VK_SL3_PROBE(k) (g_probe[(blockIdx.x * blockDim.x + threadIdx.x) * 4 + (k)]++)
#endif
#include "../../paper_2405_12484_b200/csrc/sl3.cuh"
using namespace vk;
__global__ void set_probe(int* p) { g_probe = p; }
__global__ void k_batch(int n, const double* sig, int* path, long long* cyc) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    double sd[3] = {sig[3 * t], sig[3 * t + 1], sig[3 * t + 2]}, s[3];
    long long c0 = clock64();
    path[t] = sl3::project(sd, s, true);
    cyc[t] = clock64() - c0 + (long long)(s[0] * 0);
}
int main(int argc, char** argv) {
    FILE* f = fopen(argv[1], "rb");
    fseek(f, 0, SEEK_END); long sz = ftell(f); fseek(f, 0, SEEK_SET);
    int n = (int)(sz / 24);
    std::vector<double> h(3 * (size_t)n);
    if (fread(h.data(), 8, 3 * (size_t)n, f) != 3 * (size_t)n) return 1;
    fclose(f);
    double* d; int *pr, *path; long long* cyc;
    cudaMalloc(&d, 24 * (size_t)n); cudaMemcpy(d, h.data(), 24 * (size_t)n, cudaMemcpyHostToDevice);
    cudaMalloc(&pr, 16 * (size_t)n); cudaMemset(pr, 0, 16 * (size_t)n);
    cudaMalloc(&path, 4 * (size_t)n); cudaMalloc(&cyc, 8 * (size_t)n);
    set_probe<<<1, 1>>>(pr);
    k_batch<<<(n + 127) / 128, 128>>>(n, d, path, cyc);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_batch<<<(n + 127) / 128, 128>>>(n, d, path, cyc);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    std::vector<int> hp(4 * (size_t)n), hpath(n); std::vector<long long> hc(n);
    cudaMemcpy(hp.data(), pr, 16 * (size_t)n, cudaMemcpyDeviceToHost);
    cudaMemcpy(hpath.data(), path, 4 * (size_t)n, cudaMemcpyDeviceToHost);
    cudaMemcpy(hc.data(), cyc, 8 * (size_t)n, cudaMemcpyDeviceToHost);
    long long it = 0, sec = 0, defer = 0; std::vector<int> hist(32, 0);
    double cs = 0;
    for (int i = 0; i < n; ++i) {
        int k = hp[4 * i + 3] / 2;   // two launches
        it += k; sec += hp[4 * i + 2] / 2; defer += hpath[i] == 3; hist[std::min(k, 31)]++; cs += hc[i];
    }
    printf("n=%d kernel %.1f us | batch newton iters mean %.2f | second start %.3f | deferred %.4f | cycles/thread mean %.0f\n",
           n, ms * 1e3, (double)it / n, (double)sec / n, (double)defer / n, cs / n);
    printf("newton-iteration histogram:");
    for (int k = 0; k < 32; ++k) if (hist[k]) printf(" %d:%d", k, hist[k]);
    printf("\n");
}

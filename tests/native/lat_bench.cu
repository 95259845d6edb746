// Dependent-chain latency of FP64 / FP32 ops on this GPU (one thread, clock64).
#include <cstdio>
__global__ void k(double* out, float* outf, long long* cyc, double a, double b, float af, float bf) {
    double x = a; float y = af;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1000; ++i) { x = fma(x, b, a); }
    long long t1 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1000; ++i) { x = a / x + b; }
    long long t2 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1000; ++i) { y = fmaf(y, bf, af); }
    long long t3 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1000; ++i) { x = sqrt(x) + b; }
    long long t4 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1000; ++i) { x = fabs(x) > b ? x * a : x + b; }
    long long t5 = clock64();
    out[0] = x; outf[0] = y;
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4;
}
int main() {
    double* o; float* of; long long* c;
    cudaMalloc(&o, 8); cudaMalloc(&of, 4); cudaMalloc(&c, 40);
    for (int r = 0; r < 2; ++r) k<<<1, 1>>>(o, of, c, 0.999, 0.5, 0.999f, 0.5f);
    cudaDeviceSynchronize();
    long long h[5];
    cudaMemcpy(h, c, 40, cudaMemcpyDeviceToHost);
    printf("per-op cycles (incl. loop overhead): dfma %.1f  ddiv+dadd %.1f  ffma %.1f  dsqrt+dadd %.1f  dcmp/select/dmul %.1f\n",
           h[0] / 1000.0, h[1] / 1000.0, h[2] / 1000.0, h[3] / 1000.0, h[4] / 1000.0);
}

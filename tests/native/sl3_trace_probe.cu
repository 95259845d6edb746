// Test-only probe: traces the KKT Newton + 4x4 solve on the device.
#include <cstdio>
#include "../../paper_2405_12484_b200/csrc/sl3.cuh"

__global__ void trace(double* out) {
    const double sig[3] = {2.5, 2.5, 2.5};
    double s[3] = {0.16, 2.5, 2.5};
    double p[3];
    vk::sl3::pairprod(s, p);
    const double denom = fmax(p[0] * p[0] + p[1] * p[1] + p[2] * p[2], 1e-300);
    double lam = (s[0] * s[1] * s[2] - 1.0) / denom;
    int o = 0;
    for (int it = 0; it < 6; ++it) {
        vk::sl3::pairprod(s, p);
        double r[4];
        for (int i = 0; i < 3; ++i) r[i] = s[i] - sig[i] + lam * p[i];
        r[3] = s[0] * s[1] * s[2] - 1.0;
        double J[4][4] = {{1.0, lam * s[2], lam * s[1], p[0]},
                          {lam * s[2], 1.0, lam * s[0], p[1]},
                          {lam * s[1], lam * s[0], 1.0, p[2]},
                          {p[0], p[1], p[2], 0.0}};
        double d[4] = {-r[0], -r[1], -r[2], -r[3]};
        bool ok = vk::sl3::gesv(J, d, 4);
        out[o++] = it; out[o++] = s[0]; out[o++] = s[1]; out[o++] = s[2]; out[o++] = lam;
        out[o++] = r[0]; out[o++] = r[3]; out[o++] = ok; out[o++] = d[0]; out[o++] = d[3];
        s[0] += d[0]; s[1] += d[1]; s[2] += d[2]; lam += d[3];
    }
    double s2[3] = {0.16, 2.5, 2.5}, l2;
    out[60] = vk::sl3::kkt_newton(sig, s2, l2);
    out[61] = s2[0]; out[62] = s2[1]; out[63] = l2;
}

int main() {
    double* d; double h[64];
    cudaMalloc(&d, sizeof h);
    cudaMemset(d, 0, sizeof h);
    trace<<<1, 1>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("err=%s\n", cudaGetErrorString(e));
    for (int it = 0; it < 6; ++it) {
        double* q = h + 10 * it;
        printf("it=%g s=%.6g %.6g %.6g lam=%.6g r0=%.3g r3=%.3g ok=%g d0=%.3g d3=%.3g\n", q[0], q[1], q[2], q[3], q[4], q[5], q[6], q[7], q[8], q[9]);
    }
    printf("kkt_newton ok=%g s=%g %g lam=%g\n", h[60], h[61], h[62], h[63]);
    return 0;
}

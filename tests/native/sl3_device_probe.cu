// Test-only probe: runs the SVD + SL(3) device code on the GPU for a few F and
// prints sigma, s and the path (used to debug device/host differences).
#include <cstdio>
#include "../../paper_2405_12484_b200/csrc/sl3.cuh"
#include "../../paper_2405_12484_b200/csrc/svd3.cuh"

__global__ void probe(const double* Fin, double* out, int n) {
    int e = threadIdx.x;
    if (e >= n) return;
    double F[3][3], U[3][3], W[3][3], sg[3];
    for (int k = 0; k < 9; ++k) F[k / 3][k % 3] = Fin[9 * e + k];
    vk::svd3_rv(F, U, sg, W);
    const double sd[3] = {sg[0], sg[1], sg[2]};
    double s[3];
    int path = vk::sl3::project(sd, s);
    double s2[3] = {fmax(sd[0], 0.01), fmax(sd[1], 0.01), fmax(sd[2], 0.01)};
    double lam;
    int j = vk::sl3::argmin3(sd);
    double prod = sd[0] * sd[1] * sd[2];
    s2[j] = fmax(1.0 / fmax(prod / fmax(sd[j], 1e-300), 1e-12), 0.01);
    bool ok2 = vk::sl3::kkt_newton(sd, s2, lam);
    double* o = out + 16 * e;
    o[0] = sd[0]; o[1] = sd[1]; o[2] = sd[2]; o[3] = s[0]; o[4] = s[1]; o[5] = s[2]; o[6] = path;
    o[7] = ok2; o[8] = s2[0]; o[9] = s2[1]; o[10] = s2[2]; o[11] = lam; o[12] = j;
}

int main() {
    const int n = 4;
    double ts[n] = {1.95, 2.0, 2.5, 1.5};
    double hF[9 * n] = {0};
    for (int e = 0; e < n; ++e) for (int i = 0; i < 3; ++i) hF[9 * e + 4 * i] = ts[e];
    double *dF, *dO, hO[16 * n];
    cudaMalloc(&dF, sizeof hF); cudaMalloc(&dO, sizeof hO);
    cudaMemcpy(dF, hF, sizeof hF, cudaMemcpyHostToDevice);
    probe<<<1, 32>>>(dF, dO, n);
    cudaMemcpy(hO, dO, sizeof hO, cudaMemcpyDeviceToHost);
    for (int e = 0; e < n; ++e) {
        double* o = hO + 16 * e;
        printf("t=%g sig=%.17g %.17g %.17g s=%.6f %.6f %.6f path=%g | 2nd ok=%g s=%.6f %.6f %.6f lam=%g j=%g\n",
               ts[e], o[0], o[1], o[2], o[3], o[4], o[5], o[6], o[7], o[8], o[9], o[10], o[11], o[12]);
    }
    return 0;
}

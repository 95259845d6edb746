// Test-only probe: k_project-like kernel with sigma / s / path outputs, built with
// the library's flags; runs the golden t*I and random cases.
#include <cstdio>
#include <vector>
#include "../../paper_2405_12484_b200/csrc/local_step.cuh"

template <typename T>
__global__ void __launch_bounds__(128) kp(int n, const double* Fin, double* out) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n) return;
    T F[3][3];
    for (int k = 0; k < 9; ++k) F[k / 3][k % 3] = (T)Fin[(size_t)e * 9 + k];
    T U[3][3], W[3][3], sig[3];
    double s[3];
    const int path = vk::project_element(F, U, W, sig, s);
    double* o = out + 8 * e;
    o[0] = sig[0]; o[1] = sig[1]; o[2] = sig[2]; o[3] = s[0]; o[4] = s[1]; o[5] = s[2]; o[6] = path;
}

int main() {
    std::vector<double> F;
    double ts[] = {0.5, 1.0, 1.5, 1.8, 1.95, 2.0, 2.5};
    for (double t : ts) for (int k = 0; k < 9; ++k) F.push_back(k % 4 == 0 ? t : 0.0);
    int n = (int)(F.size() / 9);
    double *dF, *dO;
    cudaMalloc(&dF, F.size() * 8); cudaMalloc(&dO, n * 64);
    cudaMemcpy(dF, F.data(), F.size() * 8, cudaMemcpyHostToDevice);
    std::vector<double> h(8 * n);
    kp<double><<<1, 128>>>(n, dF, dO);
    printf("sync=%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    cudaMemcpy(h.data(), dO, n * 64, cudaMemcpyDeviceToHost);
    for (int e = 0; e < n; ++e)
        printf("t=%g sig=%.17g %.17g %.17g s=%.6f %.6f %.6f path=%g\n", ts[e], h[8*e], h[8*e+1], h[8*e+2], h[8*e+3], h[8*e+4], h[8*e+5], h[8*e+6]);
    return 0;
}

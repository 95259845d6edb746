// Probe: k_hs_linearize's M vs 2V(gs(I-JR)+gv(I-JV)) from k_proj_jacobians on random tets.
// (Found: projection_jacobians with thread-local output arrays gave wrong values on sm_100a;
// k_local_copy below reproduces that variant.)
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "../../paper_2405_12484_b200/csrc/hessian.cuh"

__global__ void k_local_copy(int n, const double* Fin, double* JRo, double* JVo) {
    const int e = threadIdx.x;
    if (e >= n) return;
    double F[3][3];
    for (int k = 0; k < 9; ++k) F[k / 3][k % 3] = Fin[9 * e + k];
    double JR[81], JV[81];
    vk::projection_jacobians(F, JR, JV);
    for (int k = 0; k < 81; ++k) { JRo[81 * e + k] = JR[k]; JVo[81 * e + k] = JV[k]; }
}
__global__ void k_gradof(vk::hs::Args a, const double* x, double* Fo) {
    const int e = threadIdx.x;
    if (e >= a.nE) return;
    double g[4][3], F[3][3];
    vk::hs::load_G(a, e, g);
    vk::hs::grad_of(g, x, a.tets[e], F);
    for (int k = 0; k < 9; ++k) Fo[9 * e + k] = F[k / 3][k % 3];
}

int main() {
    const int nE = 4;
    std::vector<double> Gp(12 * nE), w(2 * nE), vol(nE), x(12 * nE), F(9 * nE);
    srand(1);
    auto rnd = [] { return (rand() / (double)RAND_MAX - 0.5); };
    std::vector<int4> tets(nE);
    for (int e = 0; e < nE; ++e) {
        tets[e] = make_int4(4 * e, 4 * e + 1, 4 * e + 2, 4 * e + 3);
        double g[4][3] = {{-1, -1, -1}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
        for (int k = 0; k < 12; ++k) Gp[k * nE + e] = g[k / 3][k % 3];
        w[e] = 2.0; w[nE + e] = 1.0; vol[e] = 1.0 / 6.0;
        double X[4][3] = {{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
        for (int m = 0; m < 4; ++m) for (int i = 0; i < 3; ++i) x[12 * e + 3 * m + i] = X[m][i] + 0.1 * rnd();
        for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j) {
            double s = 0; for (int m = 0; m < 4; ++m) s += x[12 * e + 3 * m + i] * g[m][j];
            F[9 * e + 3 * i + j] = s;
        }
    }
    double *dG, *dw, *dv, *dx, *dF, *dJR, *dJV, *dM;
    int4* dt;
    cudaMalloc(&dG, 8 * Gp.size()); cudaMalloc(&dw, 8 * w.size()); cudaMalloc(&dv, 8 * nE); cudaMalloc(&dx, 8 * x.size());
    cudaMalloc(&dF, 8 * F.size()); cudaMalloc(&dJR, 8 * 81 * nE); cudaMalloc(&dJV, 8 * 81 * nE); cudaMalloc(&dM, 8 * 81 * nE);
    cudaMalloc(&dt, 16 * nE);
    cudaMemcpy(dG, Gp.data(), 8 * Gp.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dw, w.data(), 8 * w.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dv, vol.data(), 8 * nE, cudaMemcpyHostToDevice);
    cudaMemcpy(dx, x.data(), 8 * x.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dF, F.data(), 8 * F.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dt, tets.data(), 16 * nE, cudaMemcpyHostToDevice);
    vk::k_proj_jacobians<<<1, 128>>>(nE, dF, dJR, dJV);
    vk::hs::Args a{};
    a.n = 4 * nE; a.nE = nE; a.tets = dt; a.G = dG; a.w = dw; a.vol = dv;
    vk::hs::k_hs_linearize<<<1, 64>>>(a, dx, dM);
    printf("err %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    std::vector<double> JR(81 * nE), JV(81 * nE), M(81 * nE);
    cudaMemcpy(JR.data(), dJR, 8 * JR.size(), cudaMemcpyDeviceToHost);
    cudaMemcpy(JV.data(), dJV, 8 * JV.size(), cudaMemcpyDeviceToHost);
    cudaMemcpy(M.data(), dM, 8 * M.size(), cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int e = 0; e < nE; ++e)
        for (int k = 0; k < 81; ++k) {
            const double id = k % 10 == 0 ? 1.0 : 0.0;
            const double ref = 2 * vol[e] * (w[e] * (id - JR[81 * e + k]) + w[nE + e] * (id - JV[81 * e + k]));
            mx = fmax(mx, fabs(ref - M[k * nE + e]));
            if (e == 0 && k < 12) printf("k=%d ref %.6f M %.6f\n", k, ref, M[k * nE + e]);
        }
    printf("max |M - ref| = %.3e\n", mx);
    double *dJR2, *dJV2, *dF2;
    cudaMalloc(&dJR2, 8 * 81 * nE); cudaMalloc(&dJV2, 8 * 81 * nE); cudaMalloc(&dF2, 8 * 9 * nE);
    k_local_copy<<<1, 32>>>(nE, dF, dJR2, dJV2);
    k_gradof<<<1, 32>>>(a, dx, dF2);
    std::vector<double> JR2(81 * nE), F2(9 * nE);
    cudaMemcpy(JR2.data(), dJR2, 8 * JR2.size(), cudaMemcpyDeviceToHost);
    cudaMemcpy(F2.data(), dF2, 8 * F2.size(), cudaMemcpyDeviceToHost);
    double m2 = 0, m3 = 0;
    for (int k = 0; k < 81 * nE; ++k) m2 = fmax(m2, fabs(JR2[k] - JR[k]));
    for (int k = 0; k < 9 * nE; ++k) m3 = fmax(m3, fabs(F2[k] - F[k]));
    printf("local-array JR vs global JR: %.3e ; grad_of F vs host F: %.3e\n", m2, m3);
    for (int k = 0; k < 9; ++k) printf("F %d host %.6f dev %.6f\n", k, F[k], F2[k]);
    return 0;
}

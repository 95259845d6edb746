// Test-only harness: runs the device projection math (__host__ __device__)
// on the host over a binary file of F matrices; writes R, V (float64).
// Built by tests/test_native_host.py; never part of the product library.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../../paper_2405_12484_b200/csrc/sl3.cuh"
#include "../../paper_2405_12484_b200/csrc/svd3.cuh"

template <typename T>
static void run(const std::vector<double>& F, std::vector<double>& R, std::vector<double>& V, int n) {
    for (int e = 0; e < n; ++e) {
        T f[3][3], U[3][3], W[3][3], sg[3];
        for (int k = 0; k < 9; ++k) f[k / 3][k % 3] = (T)F[9 * e + k];
        vk::svd3_rv(f, U, sg, W);
        const double sd[3] = {(double)sg[0], (double)sg[1], (double)sg[2]};
        double s[3];
        vk::sl3::project(sd, s);
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) {
                double r = 0, v = 0;
                for (int k = 0; k < 3; ++k) {
                    r += (double)U[i][k] * (double)W[j][k];
                    v += (double)U[i][k] * s[k] * (double)W[j][k];
                }
                R[9 * e + 3 * i + j] = r;
                V[9 * e + 3 * i + j] = v;
            }
    }
}

int main(int argc, char** argv) {
    if (argc < 4) return 2;
    const int prec = atoi(argv[1]);
    FILE* f = fopen(argv[2], "rb");
    std::vector<double> F;
    double buf[9];
    while (fread(buf, sizeof(double), 9, f) == 9) F.insert(F.end(), buf, buf + 9);
    fclose(f);
    const int n = (int)(F.size() / 9);
    std::vector<double> R(F.size()), V(F.size());
    if (prec == 32) run<float>(F, R, V, n); else run<double>(F, R, V, n);
    FILE* o = fopen(argv[3], "wb");
    fwrite(R.data(), sizeof(double), R.size(), o);
    fwrite(V.data(), sizeof(double), V.size(), o);
    fclose(o);
    return 0;
}

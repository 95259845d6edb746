// Probe: per-start cost of the robust SL(3) path on sigma triples dumped from a
// simulation (tools/dbg/dump_robust_sigma.py).  Prints, per start, the
// distribution of Newton iterations, line-search evaluations, clamp rounds and
// clock64 cycles; and the per-element critical path (max over starts).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
__device__ int* g_probe;
#ifndef NO_COUNTERS
#define VK_SL3_PROBE(k) (g_probe[(blockIdx.x * blockDim.x + threadIdx.x) * 4 + (k)]++)
#endif
#include "../../paper_2405_12484_b200/csrc/sl3.cuh"
using namespace vk;

__global__ void k_probe(int n, const double* sig, long long* cyc, int* okv) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n * 4) return;
    int e = t >> 2, q = t & 3;
    double sd[3] = {sig[3 * e], sig[3 * e + 1], sig[3 * e + 2]};
    double st[3], sk[3], obj = 0;
    long long c0 = clock64();
    bool use = sl3::robust_start(sd, q, st);
    bool ok = use && sl3::robust_try(sd, st, sk, obj);
    long long c1 = clock64();
    cyc[t] = c1 - c0;
    okv[t] = use ? (ok ? 1 : 0) : -1;
}
__global__ void set_probe(int* p) { g_probe = p; }

// pure single-lane latency: one thread per warp, start q of element e
__global__ void k_lat(int n, const double* sig, int q, long long* cyc, int* its) {
    if (threadIdx.x != 0) return;
    int e = blockIdx.x;
    if (e >= n) return;
    double sd[3] = {sig[3 * e], sig[3 * e + 1], sig[3 * e + 2]};
    double st[3], sk[3], obj = 0;
    int base = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
    int i0 = g_probe[base], l0 = g_probe[base + 1];
    long long c0 = clock64();
    bool use = sl3::robust_start(sd, q, st);
    bool ok = use && sl3::robust_try(sd, st, sk, obj);
    long long c1 = clock64();
    cyc[e] = (c1 - c0) + (ok ? 0 : 0);
    its[2 * e] = g_probe[base] - i0;
    its[2 * e + 1] = g_probe[base + 1] - l0;
}

template <typename V>
static double pct(V v, double p) {
    std::sort(v.begin(), v.end());
    return (double)v[(size_t)(p * (v.size() - 1))];
}
template <typename V>
static double mean(const V& v) {
    double s = 0;
    for (auto x : v) s += x;
    return s / v.size();
}

int main(int argc, char** argv) {
    FILE* f = fopen(argv[1], "rb");
    fseek(f, 0, SEEK_END);
    long sz = ftell(f);
    fseek(f, 0, SEEK_SET);
    int n = (int)(sz / 24);
    std::vector<double> h(3 * n);
    if (fread(h.data(), 8, 3 * n, f) != (size_t)(3 * n)) return 1;
    fclose(f);
    double* d;
    int *probe, *okv;
    long long* cyc;
    cudaMalloc(&d, 24 * n);
    cudaMemcpy(d, h.data(), 24 * n, cudaMemcpyHostToDevice);
    cudaMalloc(&probe, 16 * 4 * n);
    cudaMemset(probe, 0, 16 * 4 * n);
    cudaMalloc(&cyc, 8 * 4 * n);
    cudaMalloc(&okv, 4 * 4 * n);
    set_probe<<<1, 1>>>(probe);
    k_probe<<<(4 * n + 127) / 128, 128>>>(n, d, cyc, okv);
    cudaError_t err = cudaDeviceSynchronize();
    if (err) {
        printf("err %s\n", cudaGetErrorString(err));
        return 1;
    }
    std::vector<int> hp(16 * n), ho(4 * n);
    std::vector<long long> hc(4 * n);
    cudaMemcpy(hp.data(), probe, 16 * 4 * n, cudaMemcpyDeviceToHost);
    cudaMemcpy(hc.data(), cyc, 8 * 4 * n, cudaMemcpyDeviceToHost);
    cudaMemcpy(ho.data(), okv, 4 * 4 * n, cudaMemcpyDeviceToHost);
    printf("n=%d elements\n", n);
    for (int q = 0; q < 4; ++q) {
        std::vector<int> it, ls, rd;
        std::vector<long long> cy;
        int used = 0, okc = 0;
        for (int e = 0; e < n; ++e) {
            int t = 4 * e + q;
            if (ho[t] < 0) continue;
            ++used;
            okc += ho[t];
            it.push_back(hp[4 * t]);
            ls.push_back(hp[4 * t + 1]);
            rd.push_back(hp[4 * t + 2]);
            cy.push_back(hc[t]);
        }
        if (!used) {
            printf("start %d unused\n", q);
            continue;
        }
        printf("start %d used %d ok %d | newton mean %.1f p50 %.0f p99 %.0f max %.0f | ls mean %.1f p99 %.0f | "
               "rounds mean %.2f | cycles mean %.0f p50 %.0f p99 %.0f max %.0f\n",
               q, used, okc, mean(it), pct(it, .5), pct(it, .99), pct(it, 1.0), mean(ls), pct(ls, .99), mean(rd),
               mean(cy), pct(cy, .5), pct(cy, .99), pct(cy, 1.0));
    }
    {
        int m = std::min(n, 64);
        long long* lc; int* li; int* pr2;
        cudaMalloc(&lc, 8 * m); cudaMalloc(&li, 8 * m); cudaMalloc(&pr2, 16 * 32 * m);
        cudaMemset(pr2, 0, 16 * 32 * m);
        set_probe<<<1, 1>>>(pr2);
        for (int q = 0; q < 4; ++q) {
            k_lat<<<m, 32>>>(m, d, q, lc, li);
            cudaDeviceSynchronize();
            std::vector<long long> c(m); std::vector<int> it(2 * m);
            cudaMemcpy(c.data(), lc, 8 * m, cudaMemcpyDeviceToHost);
            cudaMemcpy(it.data(), li, 8 * m, cudaMemcpyDeviceToHost);
            double sc = 0, si = 0, sl = 0;
            for (int e = 0; e < m; ++e) { sc += c[e]; si += it[2 * e]; sl += it[2 * e + 1]; }
            printf("latency start %d: mean cycles %.0f, newton %.1f, ls %.1f -> cycles per (newton+ls) %.0f\n", q, sc / m,
                   si / m, sl / m, sc / std::max(1.0, si + sl));
        }
    }
    std::vector<long long> crit(n);
    for (int e = 0; e < n; ++e) {
        long long m = 0;
        for (int q = 0; q < 4; ++q) m = std::max(m, hc[4 * e + q]);
        crit[e] = m;
    }
    std::sort(crit.begin(), crit.end());
    printf("critical path cycles p50 %lld p90 %lld p99 %lld max %lld\n", crit[n / 2], crit[(size_t)(0.9 * (n - 1))],
           crit[(size_t)(0.99 * (n - 1))], crit[n - 1]);
    return 0;
}

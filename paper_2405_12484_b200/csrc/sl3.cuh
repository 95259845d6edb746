// Volume (SL(3)) projection in singular-value space, per thread, in float64.
//
//   min |s - sigma|^2  s.t.  s0 s1 s2 = 1,  s_i >= 0.01
//
// Restates, per element, the reference's batched solve
// `sl3_sigma_project_batch` (material.py:343-392) with its KKT Newton
// `_sl3_batch_newton` (309-340), and the robust multi-start scalar path
// `sl3_sigma_project` (242-287) with `_sl3_solve_clamping` (217-239) and
// `_sl3_newton_free` (171-214).  All thresholds are the reference's, verbatim;
// the arithmetic is always float64 (also in the fp32 build), so the branch
// decisions (second start, "suspicious" re-solve, clamping) are the
// reference's decisions for the same sigma.
//
// Deviation (documented in DESIGN.md): a singular 4x4 KKT Jacobian fails only
// that element's Newton (ok = false); the reference's batched
// `np.linalg.solve` raises for the whole batch and re-solves every element on
// the scalar path.
#pragma once

#include <math.h>

#include "vk_common.cuh"

namespace vk {
namespace sl3 {

constexpr double kFloor = 0.01;     // material.py:25
constexpr double kTol = 1e-12;      // material.py:30
constexpr int kIters = 20;          // material.py:29

// instrumentation hook for tests/native probes (iteration / line-search / round counters)
#ifndef VK_SL3_PROBE
#define VK_SL3_PROBE(k)
#endif

VK_HD double nanmax(double m, double a) { return (a > m || a != a) ? a : m; }

VK_HD void pairprod(const double (&s)[3], double (&p)[3]) {
    p[0] = s[1] * s[2];
    p[1] = s[0] * s[2];
    p[2] = s[0] * s[1];
}

// Fixed-size 4x4 solve with partial pivoting, fully unrolled so the matrix
// stays in registers (row exchanges are conditional moves, pivot = first
// largest magnitude as in LAPACK idamax).  false on an exactly zero pivot.
VK_HD bool gesv4(double (&A)[4][4], double (&b)[4]) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
#pragma unroll
        for (int i = k + 1; i < 4; ++i) {
            const bool sw = fabs(A[i][k]) > fabs(A[k][k]);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const double a = A[k][j], c = A[i][j];
                A[k][j] = sw ? c : a;
                A[i][j] = sw ? a : c;
            }
            const double a = b[k], c = b[i];
            b[k] = sw ? c : a;
            b[i] = sw ? a : c;
        }
        if (A[k][k] == 0.0) return false;
        const double inv = 1.0 / A[k][k];
#pragma unroll
        for (int i = k + 1; i < 4; ++i) {
            const double f = A[i][k] * inv;
#pragma unroll
            for (int j = k + 1; j < 4; ++j) A[i][j] -= f * A[k][j];
            b[i] -= f * b[k];
        }
    }
#pragma unroll
    for (int k = 3; k >= 0; --k) {
        double v = b[k];
#pragma unroll
        for (int j = k + 1; j < 4; ++j) v -= A[k][j] * b[j];
        b[k] = v / A[k][k];
    }
    return true;
}

// One KKT Newton update on (s, lam) in precision R (material.py:322-335):
// bordered solve of [[A, p], [p^T, 0]] [ds; dl] = -[r; r4] with
// A = I + lam * offdiag(s2, s1, s0) through the adjugate of A.  Returns
// false when A is near singular (the caller then uses the pivoted 4x4
// elimination in float64, or gives the step to the float64 phase).
template <typename R>
VK_HD bool kkt_bordered_step(const R (&r)[4], const R (&p)[3], R (&s)[3], R& lam) {
    const R a = lam * s[2], b = lam * s[1], c = lam * s[0];
    const R c00 = R(1) - c * c, c11 = R(1) - b * b, c22 = R(1) - a * a;
    const R c01 = b * c - a, c02 = a * c - b, c12 = a * b - c;
    const R det = c00 + a * c01 + b * c02;
    const R ar0 = c00 * r[0] + c01 * r[1] + c02 * r[2];
    const R ar1 = c01 * r[0] + c11 * r[1] + c12 * r[2];
    const R ar2 = c02 * r[0] + c12 * r[1] + c22 * r[2];
    const R ap0 = c00 * p[0] + c01 * p[1] + c02 * p[2];
    const R ap1 = c01 * p[0] + c11 * p[1] + c12 * p[2];
    const R ap2 = c02 * p[0] + c12 * p[1] + c22 * p[2];
    const R pap = p[0] * ap0 + p[1] * ap1 + p[2] * ap2;
    const R par = p[0] * ar0 + p[1] * ar1 + p[2] * ar2;
    if (!(fabs(det) > R(1e-6) && fabs(pap) > R(1e-12) * fabs(det) * (p[0] * p[0] + p[1] * p[1] + p[2] * p[2])))
        return false;
    // one reciprocal for both divisions: 1/pap = det q, 1/det = pap q
    const R q = R(1) / (det * pap);
    const R dl = (r[3] * det - par) * (det * q);
    const R idet = pap * q;
    s[0] -= (ar0 + ap0 * dl) * idet;
    s[1] -= (ar1 + ap1 * dl) * idet;
    s[2] -= (ar2 + ap2 * dl) * idet;
    lam += dl;
    return true;
}

template <typename R>
VK_HD R kkt_residual(const R (&sig)[3], const R (&s)[3], R lam, R (&r)[4], R (&p)[3]) {
    p[0] = s[1] * s[2];
    p[1] = s[0] * s[2];
    p[2] = s[0] * s[1];
    for (int i = 0; i < 3; ++i) r[i] = s[i] - sig[i] + lam * p[i];
    r[3] = s[0] * s[1] * s[2] - R(1);
    R rn = R(0);
    for (int i = 0; i < 4; ++i) rn = (fabs(r[i]) > rn || r[i] != r[i]) ? fabs(r[i]) : rn;
    return rn;
}

// float64 Newton loop of `_sl3_batch_newton` from (s, lam) with an iteration
// budget; returns the reference's ok flag (material.py:336-340).
VK_HD bool kkt_newton_f64(const double (&sig)[3], double (&s)[3], double& lam, int budget) {
    double r[4], p[3];
    for (int it = 0; it < budget; ++it) {
        const double rn = kkt_residual(sig, s, lam, r, p);
        if (rn < kTol) break;
        VK_SL3_PROBE(3);
        if (!kkt_bordered_step(r, p, s, lam)) {
            const double a = lam * s[2], b = lam * s[1], c = lam * s[0];
            double J[4][4] = {{1.0, a, b, p[0]}, {a, 1.0, c, p[1]}, {b, c, 1.0, p[2]}, {p[0], p[1], p[2], 0.0}};
            double d[4] = {-r[0], -r[1], -r[2], -r[3]};
            if (!gesv4(J, d)) return false;
            s[0] += d[0]; s[1] += d[1]; s[2] += d[2];
            lam += d[3];
        }
    }
    pairprod(s, p);
    double r3 = 0.0;
    for (int i = 0; i < 3; ++i) r3 = nanmax(r3, fabs(s[i] - sig[i] + lam * p[i]));
    const double rc = fabs(s[0] * s[1] * s[2] - 1.0);
    const bool fin = isfinite(s[0]) && isfinite(s[1]) && isfinite(s[2]);
    return (nanmax(r3, rc) < 1e-10) && fin;
}

// One element of `_sl3_batch_newton` (material.py:309-340): unclamped KKT
// Newton on (s, lam) from start s (lam0 = (prod s - 1)/|p|^2); returns ok.
// (A float32-first variant was measured: no gain, the loop is latency-bound.)
VK_HD bool kkt_newton(const double (&sig)[3], double (&s)[3], double& lam) {
    double p[3];
    pairprod(s, p);
    const double denom = fmax(p[0] * p[0] + p[1] * p[1] + p[2] * p[2], 1e-300);
    lam = (s[0] * s[1] * s[2] - 1.0) / denom;
    return kkt_newton_f64(sig, s, lam, kIters);
}

VK_HD double sq3(const double (&a)[3], const double (&b)[3]) {
    const double d0 = a[0] - b[0], d1 = a[1] - b[1], d2 = a[2] - b[2];
    return d0 * d0 + d1 * d1 + d2 * d2;
}
VK_HD double nanmin3(const double (&a)[3]) {
    double m = a[0];
    for (int i = 1; i < 3; ++i) m = (a[i] < m || a[i] != a[i]) ? a[i] : m;
    return m;
}
VK_HD int argmin3(const double (&a)[3]) {
    int j = 0;
    if (a[1] < a[j]) j = 1;
    if (a[2] < a[j]) j = 2;
    return j;
}

// Residual of the frozen-entry system (material.py:163-168), max-norm over free + constraint,
// compared with the line search's bar: rnorm < rn || rnorm < kTol, decided without forming the norm: the
// NaN-propagating max is below thr = fmax(rn, kTol) iff every entry is (a NaN entry fails its
// comparison; fmax(NaN, kTol) = kTol keeps the `< kTol` branch when rn is NaN).  The line search's
// candidate steps only need this decision; it halves their FP64 compare/select work.
VK_HD bool free_accept(const double (&sig)[3], const double (&s)[3], double lam, const bool (&fr)[3], double thr) {
    double p[3];
    pairprod(s, p);
    bool ok = fabs(s[0] * s[1] * s[2] - 1.0) < thr;     // (bitwise: no branches)
    for (int i = 0; i < 3; ++i)
        ok &= !fr[i] || fabs(s[i] - sig[i] + lam * p[i]) < thr;
    return ok;
}

// same residual, also returning the masked residual vector and the pair products
VK_HD double free_res(const double (&sig)[3], const double (&s)[3], double lam, const bool (&fr)[3],
                      double (&rr)[4], double (&p)[3]) {
    pairprod(s, p);
    rr[3] = s[0] * s[1] * s[2] - 1.0;
    double rn = fabs(rr[3]);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        rr[i] = fr[i] ? (s[i] - sig[i] + lam * p[i]) : 0.0;
        if (fr[i]) rn = nanmax(rn, fabs(rr[i]));
    }
    return rn;
}

// `_sl3_newton_free` (material.py:171-214).  The reduced (nf+1) system is
// solved embedded in the 4x4 one: frozen entries get an identity row/column
// and a zero right-hand side, so their update is exactly zero.
//
// Same iterates as the reference loop, shorter dependency chain:
//  - the residual of the accepted line-search point is the next iteration's
//    residual (the reference recomputes the same value);
//  - the damped line search (step 1, 1/2, ..., 1/32; first step whose residual
//    drops, else the last) tries the full step first and, when that fails,
//    evaluates the five shorter steps independently (steps are exact powers of
//    two, so every candidate is the value the sequential halving produces) and
//    takes the first acceptable one.  A stalled start (the usual fate of the
//    sigma/cbrt start on strongly stretched tets) then costs two residual
//    latencies per iteration instead of up to six.
VK_HD bool newton_free(const double (&sig)[3], double (&s)[3], double& lam, const bool (&fr)[3]) {
    const int nf = (int)fr[0] + (int)fr[1] + (int)fr[2];
    if (nf == 0) return false;
    double rr[4], p[3];
    double rn = free_res(sig, s, lam, fr, rr, p);
    for (int it = 0; it < kIters; ++it) {
        if (rn < kTol) return true;
        VK_SL3_PROBE(0);
        double d[4];
        {
            // masked bordered system: frozen entries get identity rows/cols, zero p and rhs;
            // solved through the adjugate (kkt_bordered_step), pivoted elimination if A is near singular
            double pm[3], sd[3] = {0.0, 0.0, 0.0}, ld = 0.0;
#pragma unroll
            for (int i = 0; i < 3; ++i) pm[i] = fr[i] ? p[i] : 0.0;
            const double a = (fr[0] && fr[1]) ? lam * s[2] : 0.0;
            const double b = (fr[0] && fr[2]) ? lam * s[1] : 0.0;
            const double c = (fr[1] && fr[2]) ? lam * s[0] : 0.0;
            const double c00 = 1.0 - c * c, c11 = 1.0 - b * b, c22 = 1.0 - a * a;
            const double c01 = b * c - a, c02 = a * c - b, c12 = a * b - c;
            const double det = c00 + a * c01 + b * c02;
            const double ar0 = c00 * rr[0] + c01 * rr[1] + c02 * rr[2];
            const double ar1 = c01 * rr[0] + c11 * rr[1] + c12 * rr[2];
            const double ar2 = c02 * rr[0] + c12 * rr[1] + c22 * rr[2];
            const double ap0 = c00 * pm[0] + c01 * pm[1] + c02 * pm[2];
            const double ap1 = c01 * pm[0] + c11 * pm[1] + c12 * pm[2];
            const double ap2 = c02 * pm[0] + c12 * pm[1] + c22 * pm[2];
            const double pap = pm[0] * ap0 + pm[1] * ap1 + pm[2] * ap2;
            const double par = pm[0] * ar0 + pm[1] * ar1 + pm[2] * ar2;
            const double pp = pm[0] * pm[0] + pm[1] * pm[1] + pm[2] * pm[2];
            if (fabs(det) > 1e-6 && fabs(pap) > 1e-12 * fabs(det) * pp) {
                const double q = 1.0 / (det * pap);
                ld = (rr[3] * det - par) * (det * q);
                const double idet = pap * q;
                sd[0] = -(ar0 + ap0 * ld) * idet;
                sd[1] = -(ar1 + ap1 * ld) * idet;
                sd[2] = -(ar2 + ap2 * ld) * idet;
                d[0] = fr[0] ? sd[0] : 0.0; d[1] = fr[1] ? sd[1] : 0.0; d[2] = fr[2] ? sd[2] : 0.0;
                d[3] = ld;
            } else {
                double J[4][4];
#pragma unroll
                for (int i = 0; i < 3; ++i) {
#pragma unroll
                    for (int j = 0; j < 3; ++j) {
                        const double v = (i == j) ? 1.0 : lam * s[3 - i - j];
                        J[i][j] = (fr[i] && fr[j]) ? v : (i == j ? 1.0 : 0.0);
                    }
                    J[i][3] = pm[i];
                    J[3][i] = pm[i];
                    d[i] = -rr[i];
                }
                J[3][3] = 0.0;
                d[3] = -rr[3];
                if (!gesv4(J, d)) return false;
            }
        }
        double sn[3], ln, rrn[4], pn[3];
#pragma unroll
        for (int i = 0; i < 3; ++i) sn[i] = fr[i] ? s[i] + d[i] : s[i];
        ln = lam + d[3];
        VK_SL3_PROBE(1);
        double rn_new = free_res(sig, sn, ln, fr, rrn, pn);
        if (!(rn_new < rn || rn_new < kTol)) {
            // steps 1/2 .. 1/32 (material.py:203-211), evaluated independently
            double step = 0.5;
            int take = 5;
            const double thr = fmax(rn, kTol);
#pragma unroll
            for (int t = 1; t < 6; ++t) {
                double st[3];
#pragma unroll
                for (int i = 0; i < 3; ++i) st[i] = fr[i] ? s[i] + step * d[i] : s[i];
                if (take == 5 && free_accept(sig, st, lam + step * d[3], fr, thr)) take = t;
                step *= 0.5;
            }
#ifdef __CUDA_ARCH__
            step = __longlong_as_double((long long)(1023 - take) << 52);   // 2^-take, exact
#else
            step = ldexp(1.0, -take);
#endif
#pragma unroll
            for (int i = 0; i < 3; ++i) sn[i] = fr[i] ? s[i] + step * d[i] : s[i];
            ln = lam + step * d[3];
            VK_SL3_PROBE(1);
            rn_new = free_res(sig, sn, ln, fr, rrn, pn);
        }
        s[0] = sn[0]; s[1] = sn[1]; s[2] = sn[2];
        lam = ln;
        rr[0] = rrn[0]; rr[1] = rrn[1]; rr[2] = rrn[2]; rr[3] = rrn[3];
        p[0] = pn[0]; p[1] = pn[1]; p[2] = pn[2];
        rn = rn_new;
    }
    return rn < 1e-10;
}

// `_sl3_solve_clamping` (material.py:217-239); returns false for "None"
// `clamped` (optional, 3 entries): the frozen pattern of the returned solution (~free).
VK_HD bool solve_clamping(const double (&sig)[3], double (&s)[3], double& lam, bool* clamped = nullptr) {
    bool fr[3] = {true, true, true};
    for (int round = 0; round < 3; ++round) {
        VK_SL3_PROBE(2);
        for (int i = 0; i < 3; ++i) if (!fr[i]) s[i] = kFloor;
        if (!newton_free(sig, s, lam, fr)) return false;
        bool viol[3], any = false;
        for (int i = 0; i < 3; ++i) { viol[i] = fr[i] && (s[i] < kFloor - 1e-12); any |= viol[i]; }
        if (!any) {
            if (clamped) for (int i = 0; i < 3; ++i) clamped[i] = !fr[i];
            return true;
        }
        int nfree = 0, last = -1;
        for (int i = 0; i < 3; ++i) { fr[i] = fr[i] && !viol[i]; if (fr[i]) { ++nfree; last = i; } }
        if (nfree == 1) {
            s[0] = s[1] = s[2] = kFloor;
            s[last] = 1.0 / (kFloor * kFloor);
            double p[3];
            pairprod(s, p);
            lam = (sig[last] - s[last]) / p[last];
            if (clamped) for (int i = 0; i < 3; ++i) clamped[i] = !fr[i];
            return true;
        }
    }
    return false;
}

// `sl3_sigma_project` (material.py:242-287); returns ok (false = uniform-scaling fallback)
// Start k (0..3) of the multi-start list (material.py:251-263); false if the
// reference would not use start k for this sigma.
VK_HD bool robust_start(const double (&sig)[3], int k, double (&st)[3]) {
    const double prod = sig[0] * sig[1] * sig[2];
    int idx = 0;
    for (int i = 0; i < 3; ++i) st[i] = fmax(sig[i], kFloor);
    if (k == idx++) return true;
    st[0] = st[1] = st[2] = 1.0;
    if (k == idx++) return true;
    if (prod > 1e-12) {
        const double c = cbrt(prod);
        for (int i = 0; i < 3; ++i) st[i] = fmax(sig[i] / c, kFloor);
        if (k == idx++) return true;
    }
    if (prod > 1.0) {
        const int j = argmin3(sig);
        double others = 1.0;
        for (int i = 0; i < 3; ++i) if (i != j) others *= sig[i];
        if (others > 1e-12) {
            for (int i = 0; i < 3; ++i) st[i] = fmax(sig[i], kFloor);
            st[j] = fmax(1.0 / others, kFloor);
            if (k == idx++) return true;
        }
    }
    return false;
}

// One start of `sl3_sigma_project` (material.py:265-277): clamped Newton and the
// acceptance test; returns true with (s, obj) when the start is admissible.
VK_HD bool robust_try(const double (&sig)[3], const double (&st)[3], double (&s)[3], double& obj) {
    s[0] = st[0]; s[1] = st[1]; s[2] = st[2];
    double p[3];
    pairprod(s, p);
    const double den = p[0] * p[0] + p[1] * p[1] + p[2] * p[2];
    double lam = den > 1e-300 ? (s[0] * s[1] * s[2] - 1.0) / den : 0.0;
    if (!solve_clamping(sig, s, lam)) return false;
    if (nanmin3(s) < kFloor - 1e-9 || fabs(s[0] * s[1] * s[2] - 1.0) > 1e-8) return false;
    obj = sq3(s, sig);
    return true;
}

// Uniform-scaling fallback with its warning (material.py:281-287).
VK_HD void robust_fallback(const double (&sig)[3], double (&out)[3]) {
    double s[3];
    for (int i = 0; i < 3; ++i) s[i] = fmax(fabs(sig[i]), kFloor);
    for (int r = 0; r < 3; ++r) {
        const double c = cbrt(s[0] * s[1] * s[2]);
        for (int i = 0; i < 3; ++i) s[i] = fmax(s[i] / c, kFloor);
    }
    out[0] = s[0]; out[1] = s[1]; out[2] = s[2];
}

// lam_out / cl_out (optional): multiplier and clamp pattern of the returned solution
// (the fallback reports lam = 0 and clamped = s <= floor, material.py:281-287)
VK_HD bool project_robust(const double (&sig)[3], double (&out)[3], double* lam_out = nullptr,
                          bool* cl_out = nullptr) {
    double starts[4][3];
    int ns = 0;
    for (int i = 0; i < 3; ++i) starts[0][i] = fmax(sig[i], kFloor);
    starts[1][0] = starts[1][1] = starts[1][2] = 1.0;
    ns = 2;
    const double prod = sig[0] * sig[1] * sig[2];
    if (prod > 1e-12) {
        const double c = cbrt(prod);
        for (int i = 0; i < 3; ++i) starts[ns][i] = fmax(sig[i] / c, kFloor);
        ++ns;
    }
    if (prod > 1.0) {
        const int j = argmin3(sig);
        double others = 1.0;
        for (int i = 0; i < 3; ++i) if (i != j) others *= sig[i];
        if (others > 1e-12) {
            for (int i = 0; i < 3; ++i) starts[ns][i] = fmax(sig[i], kFloor);
            starts[ns][j] = fmax(1.0 / others, kFloor);
            ++ns;
        }
    }
    bool have = false;
    double best = 0.0;
    for (int k = 0; k < ns; ++k) {
        double s[3] = {starts[k][0], starts[k][1], starts[k][2]};
        double p[3];
        pairprod(s, p);
        const double den = p[0] * p[0] + p[1] * p[1] + p[2] * p[2];
        double lam = den > 1e-300 ? (s[0] * s[1] * s[2] - 1.0) / den : 0.0;
        bool cl[3] = {false, false, false};
        if (!solve_clamping(sig, s, lam, cl)) continue;
        if (nanmin3(s) < kFloor - 1e-9 || fabs(s[0] * s[1] * s[2] - 1.0) > 1e-8) continue;
        const double obj = sq3(s, sig);
        if (!have || obj < best - 1e-15) {
            have = true;
            best = obj;
            out[0] = s[0]; out[1] = s[1]; out[2] = s[2];
            if (lam_out) *lam_out = lam;
            if (cl_out) for (int i = 0; i < 3; ++i) cl_out[i] = cl[i];
        }
    }
    if (have) return true;
    double s[3];
    for (int i = 0; i < 3; ++i) s[i] = fmax(fabs(sig[i]), kFloor);
    for (int r = 0; r < 3; ++r) {
        const double c = cbrt(s[0] * s[1] * s[2]);
        for (int i = 0; i < 3; ++i) s[i] = fmax(s[i] / c, kFloor);
    }
    out[0] = s[0]; out[1] = s[1]; out[2] = s[2];
    if (lam_out) *lam_out = 0.0;
    if (cl_out) for (int i = 0; i < 3; ++i) cl_out[i] = s[i] <= kFloor;
    return false;
}

// Per-element `sl3_sigma_project_batch` (material.py:343-392).
// Returns 0 = batch Newton result, 1 = robust path, 2 = robust path fell back
// to uniform scaling (the reference logs a warning).
// defer = true: a "suspicious" element returns 3 without running the robust
// scalar path; the caller queues it for a separate dense pass (no warp
// divergence between the cheap batch path and the expensive robust one).
VK_HD int project(const double (&sig)[3], double (&s)[3], bool defer = false, double* lam_out = nullptr,
                  bool* cl_out = nullptr) {
    // Elements outside [0.2, 5] are "suspicious" whatever the batch Newton
    // returns, and the reference overwrites their batch result with the robust
    // scalar solve (material.py:377-391) -- so the batch solves are skipped.
    {
        const double mn = nanmin3(sig);
        const double mx = fmax(fmax(fabs(sig[0]), fabs(sig[1])), fabs(sig[2]));
        if (mn < 0.2 || mx > 5.0) {
            if (defer) return 3;
            return project_robust(sig, s, lam_out, cl_out) ? 1 : 2;
        }
    }
    for (int i = 0; i < 3; ++i) s[i] = fmax(sig[i], kFloor);
    double lam;
    const bool ok = kkt_newton(sig, s, lam);
    bool feas = ok && (nanmin3(s) >= kFloor - 1e-12);
    double obj = feas ? sq3(s, sig) : INFINITY;
    const double prod = sig[0] * sig[1] * sig[2];
    // The second start can only be taken if it lands on a strictly better
    // stationary point.  Any stationary point that uses the smaller root of
    // s_j^2 - sigma_j s_j + lam = 0 for some j has (s_j - sigma_j)^2 >=
    // sigma_j^2 / 4; so when the first start found the all-larger-root point
    // with an objective below min_j sigma_j^2 / 4 it is the global stationary
    // minimum and the reference's second Newton cannot replace it (it would
    // reproduce it or land higher).  Skipping it is exact.
    bool need_second = prod > 1.0;
    if (need_second && feas) {
        const double mn = fmin(fmin(sig[0], sig[1]), sig[2]);
        const bool plus_root = s[0] >= 0.5 * sig[0] && s[1] >= 0.5 * sig[1] && s[2] >= 0.5 * sig[2];
        // margin 1e-8 covers the 1e-10 KKT residual the reference accepts as "ok"
        if (plus_root && mn > 0.0 && obj < 0.25 * mn * mn - 1e-8) need_second = false;
    }
    if (need_second) {
        const int j = argmin3(sig);
        const double others = prod / fmax(sig[j], 1e-300);
        double s2[3];
        for (int i = 0; i < 3; ++i) s2[i] = fmax(sig[i], kFloor);
        s2[j] = fmax(1.0 / fmax(others, 1e-12), kFloor);
        double lam2;
        VK_SL3_PROBE(2);
        const bool ok2 = kkt_newton(sig, s2, lam2);
        const double obj2 = sq3(s2, sig);
        if (ok2 && nanmin3(s2) >= kFloor - 1e-12 && obj2 < obj - 1e-15) {
            s[0] = s2[0]; s[1] = s2[1]; s[2] = s2[2];
            obj = obj2;
            lam = lam2;
            feas = true;
        }
    }
    double mn = nanmin3(sig);
    double mx = fmax(fmax(fabs(sig[0]), fabs(sig[1])), fabs(sig[2]));
    bool odd = !feas || (mn < 0.2) || (mx > 5.0);
    if (!odd && prod > 1e-12) {
        const double c = cbrt(fmax(prod, 1e-300));
        const double r0 = sig[0] / c, r1 = sig[1] / c, r2 = sig[2] / c;
        if (fmin(fmin(r0, r1), r2) >= kFloor) {
            const double oref = (r0 - sig[0]) * (r0 - sig[0]) + (r1 - sig[1]) * (r1 - sig[1]) +
                                (r2 - sig[2]) * (r2 - sig[2]);
            odd = obj > oref + 1e-12;
        }
    }
    if (!odd) {
        if (lam_out) *lam_out = lam;
        if (cl_out) cl_out[0] = cl_out[1] = cl_out[2] = false;
        return 0;
    }
    if (defer) return 3;
    return project_robust(sig, s, lam_out, cl_out) ? 1 : 2;
}

}  // namespace sl3
}  // namespace vk

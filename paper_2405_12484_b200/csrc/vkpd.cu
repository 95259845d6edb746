// vkpd: C-ABI host runtime of the B200 projective-dynamics step.
//
// Owns the device-resident mesh, material, matrix and state of one scene and
// drives a frame as  prologue -> iterations x (local step, persistent CG) ->
// epilogue,  captured once into a CUDA graph and replayed per frame.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>
#include <atomic>
#include <thread>
#include <functional>

#include "../../include/vkpd.h"
#include "local_step.cuh"
#include "solver.cuh"
#include "cms.cuh"
#include "cheb.cuh"
#include "output.cuh"
#include "jacobian.cuh"
#include "hessian.cuh"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define CK(call)                                                                                   \
    do {                                                                                           \
        cudaError_t e__ = (call);                                                                  \
        if (e__ != cudaSuccess)                                                                    \
            return fail(VKPD_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e__));           \
    } while (0)

template <typename X>
struct DBuf {
    X* p = nullptr;
    size_t n = 0;
    ~DBuf() { if (p) cudaFree(p); }
    cudaError_t alloc(size_t count) {
        if (p) { cudaFree(p); p = nullptr; }
        n = count;
        if (count == 0) return cudaSuccess;
        return cudaMalloc(&p, count * sizeof(X));
    }
    cudaError_t upload(const X* h, size_t count, cudaStream_t s) {
        return cudaMemcpyAsync(p, h, count * sizeof(X), cudaMemcpyHostToDevice, s);
    }
};

inline int cdiv(long long a, long long b) { return (int)((a + b - 1) / b); }

// Selects the context's device for the call and restores the caller's current device after it
// (a torch caller working on another GPU keeps its device).
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};


// ---------------------------------------------------------------------------
// layout conversion kernels: host (nV,3) float64 in caller order <-> device vec4 internal order
template <typename T>
__global__ void k_scatter_in(int n, const double* __restrict__ src, const int* __restrict__ int_of_orig,
                             vk::vec4_t<T>* dst) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    dst[int_of_orig[j]] = vk::make4<T>((T)src[3 * j], (T)src[3 * j + 1], (T)src[3 * j + 2], T(0));
}
// between two frames of vkpd_simulate, one launch: frame i's positions out (caller order, f64),
// its failure slot, and frame i+1's inputs in (forces, pin targets) when given
template <typename T>
__global__ void k_sim_between(int n, int nP, const vk::vec4_t<T>* __restrict__ x, const int* __restrict__ int_of_orig,
                              double* __restrict__ out, const int* __restrict__ fail_iter, int* fail_slot,
                              const double* __restrict__ fin, vk::vec4_t<T>* f, const double* __restrict__ pin,
                              vk::vec4_t<T>* pin_tgt) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j == 0 && fail_slot) *fail_slot = *fail_iter;
    if (j < nP && pin) pin_tgt[j] = vk::make4<T>((T)pin[3 * j], (T)pin[3 * j + 1], (T)pin[3 * j + 2], T(0));
    if (j >= n) return;
    const int k = int_of_orig[j];
    if (out) {
        const vk::vec4_t<T> v = x[k];
        out[3 * j] = (double)v.x;
        out[3 * j + 1] = (double)v.y;
        out[3 * j + 2] = (double)v.z;
    }
    if (fin) f[k] = vk::make4<T>((T)fin[3 * j], (T)fin[3 * j + 1], (T)fin[3 * j + 2], T(0));
}
// New state (caller order, float64) into the device state: flags a change (bit pattern) against
// the current contents, so a caller that feeds back the state it received keeps the solver's warm
// start (pd_step called frame by frame behaves like simulate_mesh); zero v when src is null.
template <typename T>
__global__ void k_state_in(int n, const double* __restrict__ src, const int* __restrict__ int_of_orig,
                           vk::vec4_t<T>* dst, int* changed) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const vk::vec4_t<T> nv = src ? vk::make4<T>((T)src[3 * j], (T)src[3 * j + 1], (T)src[3 * j + 2], T(0))
                                 : vk::make4<T>(T(0), T(0), T(0), T(0));
    const int i = int_of_orig[j];
    const vk::vec4_t<T> ov = dst[i];
    if (nv.x != ov.x || nv.y != ov.y || nv.z != ov.z) *changed = 1;
    dst[i] = nv;
}
template <typename T>
__global__ void k_zero_if(size_t n, vk::vec4_t<T>* a, const int* __restrict__ flag) {
    if (*flag == 0) return;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        a[i] = vk::make4<T>(T(0), T(0), T(0), T(0));
}
template <typename T>
__global__ void k_gather_out(int n, const vk::vec4_t<T>* __restrict__ src, const int* __restrict__ int_of_orig,
                             double* dst) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const vk::vec4_t<T> v = src[int_of_orig[j]];
    dst[3 * j] = (double)v.x;
    dst[3 * j + 1] = (double)v.y;
    dst[3 * j + 2] = (double)v.z;
}
// plain vec4 rows (first m rows) from (m, 3) float64
template <typename T>
__global__ void k_rows_in(int m, const double* __restrict__ src, vk::vec4_t<T>* dst) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= m) return;
    dst[j] = vk::make4<T>((T)src[3 * j], (T)src[3 * j + 1], (T)src[3 * j + 2], T(0));
}
// out_f = B_f - K_fp P  (columns are packed 3-wide)
template <typename T>
__global__ void k_rhs_minus_fp(int nF, const vk::vec4_t<T>* __restrict__ Bint, const int* __restrict__ fp_ptr,
                               const int* __restrict__ fp_col, const T* __restrict__ fp_val,
                               const vk::vec4_t<T>* __restrict__ P, vk::vec4_t<T>* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nF) return;
    vk::vec4_t<T> b = Bint[i];
    for (int k = fp_ptr[i]; k < fp_ptr[i + 1]; ++k) {
        const T v = fp_val[k];
        const vk::vec4_t<T> p = P[fp_col[k]];
        b.x -= v * p.x; b.y -= v * p.y; b.z -= v * p.z;
    }
    out[i] = b;
}
// Y_f = K_ff X_f + K_fp X_p (free rows), Y_p = 0
template <typename T>
__global__ void k_apply_K(int n, int nF, const int* __restrict__ ell_len, const int* __restrict__ ell_col,
                          const T* __restrict__ ell_val,
                          const int* __restrict__ fp_ptr, const int* __restrict__ fp_col, const T* __restrict__ fp_val,
                          const vk::vec4_t<T>* __restrict__ X, vk::vec4_t<T>* Y) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (i >= nF) { Y[i] = vk::make4<T>(T(0), T(0), T(0), T(0)); return; }
    T a = 0, b = 0, c = 0;
    for (int s = 0; s < ell_len[i]; ++s) {
        const int col = ell_col[(size_t)s * nF + i];
        const T v = ell_val[(size_t)s * nF + i];
        const vk::vec4_t<T> x = X[col];
        a += v * x.x; b += v * x.y; c += v * x.z;
    }
    for (int k = fp_ptr[i]; k < fp_ptr[i + 1]; ++k) {
        const T v = fp_val[k];
        const vk::vec4_t<T> x = X[nF + fp_col[k]];
        a += v * x.x; b += v * x.y; c += v * x.z;
    }
    Y[i] = vk::make4<T>(a, b, c, T(0));
}

// One Chebyshev step of the domain-decomposed solve on a rank's free rows (dd.py): q = K_ff d_f +
// K_fp d_p (the pinned columns hold the halo: the neighbours' d of this step), y += d,
// res -= q, d_next = c1 d + c2 D^-1 res.  d / d_next are full internal vectors (free, pinned,
// halo); only the free rows of d_next are written.
template <typename T>
__global__ void k_dd_cheb_step(int nF, const int* __restrict__ ell_len, const int* __restrict__ ell_col,
                               const T* __restrict__ ell_val, const int* __restrict__ fp_ptr,
                               const int* __restrict__ fp_col, const T* __restrict__ fp_val,
                               const T* __restrict__ inv_diag, const vk::vec4_t<T>* __restrict__ d,
                               vk::vec4_t<T>* __restrict__ res, vk::vec4_t<T>* __restrict__ y,
                               vk::vec4_t<T>* __restrict__ dnext, T c1, T c2) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nF) return;
    T a = 0, b = 0, c = 0;
    for (int s = 0; s < ell_len[i]; ++s) {
        const vk::vec4_t<T> x = d[ell_col[(size_t)s * nF + i]];
        const T v = ell_val[(size_t)s * nF + i];
        a += v * x.x; b += v * x.y; c += v * x.z;
    }
    for (int k = fp_ptr[i]; k < fp_ptr[i + 1]; ++k) {
        const vk::vec4_t<T> x = d[nF + fp_col[k]];
        const T v = fp_val[k];
        a += v * x.x; b += v * x.y; c += v * x.z;
    }
    const vk::vec4_t<T> di = d[i];
    vk::vec4_t<T> yi = y[i], ri = res[i];
    yi.x += di.x; yi.y += di.y; yi.z += di.z;
    ri.x -= a; ri.y -= b; ri.z -= c;
    y[i] = yi;
    res[i] = ri;
    const T e = c2 * inv_diag[i];
    dnext[i] = vk::make4<T>(c1 * di.x + e * ri.x, c1 * di.y + e * ri.y, c1 * di.z + e * ri.z, T(0));
}

// r_i = sum of corner contributions + (m/dt^2)(xhat_i - x_i) on free rows (= b - K x)
template <typename T>
__global__ void k_resid_free(int nF, const int* __restrict__ inc_ptr, const vk::vec4_t<T>* __restrict__ corner,
                             const T* __restrict__ m_dt2, const vk::vec4_t<T>* __restrict__ x,
                             const vk::vec4_t<T>* __restrict__ xhat, vk::vec4_t<T>* r) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nF) return;
    T a = 0, b = 0, c = 0;
    for (int k = inc_ptr[i]; k < inc_ptr[i + 1]; ++k) {
        const vk::vec4_t<T> v = corner[k];
        a += v.x; b += v.y; c += v.z;
    }
    const T m = m_dt2[i];
    const vk::vec4_t<T> xh = xhat[i], xi = x[i];
    r[i] = vk::make4<T>(a + m * (xh.x - xi.x), b + m * (xh.y - xi.y), c + m * (xh.z - xi.z), T(0));
}

// ---------------------------------------------------------------------------
struct CtxBase {
    virtual ~CtxBase() {}
    virtual int init(const vkpd_mesh_desc* d, const vkpd_config* c) = 0;
    virtual int set_state(const double* x, const double* v) = 0;
    virtual int get_state(double* x, double* v) = 0;
    virtual int set_state_dev(const void* x, const void* v) = 0;
    virtual int get_state_dev(void* x, void* v) = 0;
    virtual int set_forces_dev(const void* f) = 0;
    virtual int set_pin_targets_dev(const void* t) = 0;
    virtual int set_pin_targets(const double* t) = 0;
    virtual int set_forces(const double* f) = 0;
    virtual int set_gammas(const double* gs, const double* gv) = 0;
    virtual int set_yarn_interp(int64_t n_yarn, const int64_t* indptr, const int64_t* indices, const double* data) = 0;
    virtual int frame_outputs(double* yarn, double* det_dev) = 0;
    virtual int equilibrium(const double* a, const double* x0, const double* pin_vals, int iterations, double* x_out,
                            int* failed) = 0;
    virtual int set_colliders(int n, const int* kinds, const double* params, double kc) = 0;
    virtual int step_async(int iterations, double damping) = 0;
    virtual int simulate(int steps, int iterations, double damping, const double* forces, int forces_per_step,
                         const double* pin_path, double* frames, int* failed_frame, int* failed_iter) = 0;
    virtual int sync(int* failed) = 0;
    virtual int profile(int iterations, double damping, double* lms, double* gms, double* fms) = 0;
    virtual int elastic_rhs(const double* x, double* rhs, double* F, double* R, double* V) = 0;
    virtual int global_solve(const double* B, const double* P, double* X, int k) = 0;
    virtual int apply_K(const double* X, double* Y) = 0;
    virtual int stats(vkpd_stats* st) = 0;
    virtual int init_matrix(int64_t n, const int64_t* indptr, const int64_t* indices, const double* data,
                            const int64_t* pins, int64_t npins, const vkpd_config* c) = 0;
    virtual int get_csr(int64_t* indptr, int64_t* indices, double* data, int64_t* nnz) = 0;
    virtual int aj_refine(const double* Bf, const double* X0f, int k, int sweeps, int agg, double omega, int cheb,
                          double rho, double* Xf, double* hist, int* nhist, int* diverged) = 0;
    virtual int power_rho(double omega, int iters, const double* v0, double* rho) = 0;
    virtual int cms_set_basis(int m, const double* T, const double* Kinv) = 0;
    virtual int cms_set_blocks(int ndom, const int64_t* row_ptr, const int64_t* rows, const int64_t* col_ptr,
                               const int64_t* colmap, const double* A, int nmodes, int64_t nb, const int64_t* bnd,
                               const double* Kinv) = 0;
    virtual int cms_timing(double* apply_ms, double* sweeps_ms) = 0;
    virtual int time_local(int reps, double* local_ms, double* pass_ms) = 0;
    virtual int step_cms(int iterations, double damping, int sweeps, int agg, double omega, int cheb, double rho,
                         int* failed) = 0;
    virtual int dev_residual(const void* x, const void* xhat, void* r) = 0;
    virtual int dev_apply_K(const void* X, void* Y) = 0;
    virtual int dev_inv_diag(void* out) = 0;
    virtual int dev_cheb_step(const void* d, void* res, void* y, void* dnext, double c1, double c2) = 0;
    virtual int gershgorin(int with_pinned, double* g) = 0;
    virtual int node_order(int64_t* ioo) = 0;
    virtual void sizes(int64_t* n, int64_t* nfree, int64_t* npinned, int* prec) = 0;
    virtual int cms_solve(const double* B, const double* P, int k, int sweeps, int agg, double omega, int cheb,
                          double rho, double* X) = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t own_stream = nullptr;
    int device = 0;
};

template <typename T>
struct Ctx : CtxBase {
    using V4 = vk::vec4_t<T>;
    int n = 0, nE = 0, nF = 0, nP = 0, ell_w = 0;
    double dt = 0, tol = 0;
    int max_iters = 1000;
    int pcg_blocks = 0;
    bool use_graph = true;
    bool has_forces = false;
    int n_sms = 0;
    std::vector<int> int_of_orig_h;
    std::vector<int> free_perm;          // caller's free-row rank (free nodes in caller order) -> internal row
    void set_free_perm() {
        free_perm.clear();
        for (int j = 0; j < n; ++j)
            if (int_of_orig_h[j] < nF) free_perm.push_back(int_of_orig_h[j]);
    }

    // topology / material
    DBuf<int4> tets;
    DBuf<T> G, w, inv_diag, ell_val, fp_val, m_dt2, dt2_inv_m;
    DBuf<int> ell_col, ell_len, fp_ptr, fp_col, inc_ptr, inc_code, int_of_orig;
    DBuf<int4> slot4;
    // warp-segmented reduction of the local step's corner vectors (frame path, local_step.cuh)
    DBuf<int> wr_ptr, wr_slot, part_ptr;
    DBuf<unsigned char> wr_beg, wr_code, robust_flag;
    DBuf<V4> wpart;
    DBuf<double> diag64;
    DBuf<double> G64k, md64k;            // float64 shape gradients and m/dt^2 (re-assembly)
    std::vector<double> vol2_h;          // 2 V per tet (host)
    DBuf<T> ell_kd;                      // K_ff D^-1 (polynomial preconditioner)
    DBuf<V4> warm0;                      // per-round corrections of the previous frame (solver warm start)
    DBuf<V4> warm1;                      // the frame before: the guess is the linear extrapolation
    DBuf<V4> warm2;                      // the frame before that (warm_order 2): quadratic extrapolation
    DBuf<V4> warm3;                      // register-path ring: the fourth bank
    DBuf<unsigned> warm_ctr;             // frames started (k_prologue): index of the register path's ring
#ifndef VK_WARM_ORDER64
#define VK_WARM_ORDER64 2
#endif
    int warm_order = sizeof(T) == 8 ? VK_WARM_ORDER64 : 1;   // fp64 C3: 8.03 -> 7.69 ms/frame steady; fp32 unchanged
    bool warm_extrap = true;             // d + beta (d - d_before), beta = 1
    double warm_beta = 1.0;
    int warm_extrap_rounds = sizeof(T) == 8 ? 32 : 1;   // fp32 extrapolates round 0 only (later rounds'
                                         // corrections are noise-level: C3 0.88 ms, C5 2.76 ms; all three
                                         // rounds: 0.885 / 3.37 ms)
    bool warm_start = true;              // vkpd_config.warm_rounds = 0: off
    int warm_rounds = sizeof(T) == 8 ? 32 : 3;   // fp64 runs every round (no early exit), where all rounds
                                         // gain (C3: 19.3 -> 15.9 ms/frame); fp32 only the first 3
    // state
    DBuf<V4> x, v, x_start, v_start, xhat, f, pin_tgt, corner, r, z, p0, p1, q, dx, rhs, tmp4a, tmp4b;
    DBuf<V4> hh;                         // polynomial preconditioner: h = K D^-1 r
    int pcg_threads = 512;               // CTA size of the persistent solver
    int solver_kind = VKPD_SOLVER_PCG_POLY;   // resolved vkpd_config.solver
    double tol_growth = 1.0;             // vkpd_config.tol_growth (experiment)
    bool solver_auto = true;
    bool pcg_poly = true;                // Neumann-1 polynomial preconditioner (CG kinds)
    bool cheb = false;                   // Chebyshev semi-iteration with neighbour flags (cheb.cuh)
    bool cheb_reg = false;               // ... with the row state in registers (one row per thread)
    double poly_omega = 1.0;             // min(1, 1.9 / Gershgorin bound of D^-1 K_ff)
    double gersh = 2.0;                  // Gershgorin bound of D^-1 K_ff
    double lam_min = 0.0, lam_min_bound = 0.0;   // Lanczos estimate / rigorous bound of lambda_min(D^-1 K_ff)
    DBuf<unsigned int> cheb_flags;
    DBuf<uint4> cheb_ll;
    DBuf<int> cheb_nbr_ptr, cheb_nbr;
    DBuf<double> partials, scal, stage;
    DBuf<vk::GridBar> bar;
    DBuf<int> iters, fail_iter, robust_list, robust_count;
    DBuf<T> robust_aux;                  // (sigma, U, W) of each queued element (24 per slot)
    int robust_task_blocks = 4;
    DBuf<double> robust_res;
    DBuf<int> robust_ok, robust_arrivals;
    DBuf<vk::ProjStats> pstats;
    int* h_fail = nullptr;
    int last_iterations = 0;
    std::vector<double> prof_local, prof_global;

    // graph cache
    cudaGraphExec_t graph_exec = nullptr;
    int graph_iters = -1;
    double graph_damp = 0;
    bool graph_forces = false;
    bool graph_broken = false;
    bool pd_early_exit = true;           // loop node with the zero-work exit (vkpd_config.pd_early_exit)
    int last_exec_rounds = 0;            // PD rounds of the last directly launched frame
    cudaStream_t body_stream = nullptr;  // captures the loop body
    int unroll_rounds = 0;               // PD rounds captured ahead of the WHILE node (see step_async)
    int unroll_cfg = -1;                 // vkpd_config.unroll_rounds: fixed count (-1: adaptive)
    int graph_unroll = 0;
    DBuf<int> first_stop;                // rounds the last frame needed (device), mirrored to h_stop
    int* h_stop = nullptr;
    int stop_hist[32];
    int stop_n = 0, stop_pos = 0, stop_fill = 0;
    DBuf<int> pd_it;                     // device PD-iteration counter of the loop node
    int graph_ncoll = 0;
    // colliders (pdsolver.py:125-173, 271-297)
    int ncoll = 0;
    double contact_k = 1e4;
    DBuf<double> coll_d;
    DBuf<T> inv_diag_c, cdiag, cb;

    ~Ctx() override {
        if (graph_exec) cudaGraphExecDestroy(graph_exec);
        if (h_fail) cudaFreeHost(h_fail);
        if (h_stop) cudaFreeHost(h_stop);
        if (sim_hin) cudaFreeHost(sim_hin);
        if (sim_hout) cudaFreeHost(sim_hout);
        for (int k = 0; k < 2; ++k)
            for (cudaEvent_t e : {ev_h2d[k], ev_scat[k]})
                if (e) cudaEventDestroy(e);
        for (int k = 0; k < kOutSlots; ++k)
            for (cudaEvent_t e : {ev_out[k], ev_d2h[k]})
                if (e) cudaEventDestroy(e);
        if (copy_stream) cudaStreamDestroy(copy_stream);
        if (in_stream) cudaStreamDestroy(in_stream);
        if (own_stream) cudaStreamDestroy(own_stream);
        if (body_stream) cudaStreamDestroy(body_stream);
        for (auto& ev : cms_ev)
            if (ev) cudaEventDestroy(ev);
    }

    // Recursive coordinate bisection of the free nodes into `parts` patches of ceil(nF/parts)
    // nodes (the solver CTAs' row ranges), split across the longest extent of each box.  Inside
    // a patch the nodes that share a tet with another patch's node come first (the rows other
    // CTAs read: the Chebyshev solver publishes them ahead of the interior), each group in
    // caller order.
    int part_blocks = 0;
    static void patch_order(const double* X, const int64_t* tets, int64_t n_tets, int n_nodes, std::vector<int>& ids,
                            int parts) {
        const int nf = (int)ids.size();
        const int chunk = cdiv(nf, parts);
        parts = cdiv(nf, chunk);
        std::function<void(int, int, int, int)> split = [&](int lo, int hi, int p0, int p1) {
            if (p1 - p0 <= 1 || hi - lo <= 1) {
                std::sort(ids.begin() + lo, ids.begin() + hi);
                return;
            }
            double mn[3] = {1e300, 1e300, 1e300}, mx[3] = {-1e300, -1e300, -1e300};
            for (int k = lo; k < hi; ++k)
                for (int c = 0; c < 3; ++c) {
                    mn[c] = std::min(mn[c], X[3 * (size_t)ids[k] + c]);
                    mx[c] = std::max(mx[c], X[3 * (size_t)ids[k] + c]);
                }
            int ax = 0;
            for (int c = 1; c < 3; ++c) if (mx[c] - mn[c] > mx[ax] - mn[ax]) ax = c;
            const int pm = (p0 + p1) / 2;
            const int mid = std::min(hi, lo + (pm - p0) * chunk);
            std::nth_element(ids.begin() + lo, ids.begin() + mid, ids.begin() + hi, [&](int a, int b) {
                const double xa = X[3 * (size_t)a + ax], xb = X[3 * (size_t)b + ax];
                return xa < xb || (xa == xb && a < b);
            });
            split(lo, mid, p0, pm);
            split(mid, hi, pm, p1);
        };
        split(0, nf, 0, parts);
        std::vector<int> patch(n_nodes, -1);
        for (int k = 0; k < nf; ++k) patch[ids[k]] = k / chunk;
        std::vector<char> exported(n_nodes, 0);
        for (int64_t e = 0; e < n_tets; ++e) {
            const int64_t* t = tets + 4 * e;
            for (int a = 0; a < 4; ++a)
                for (int b = 0; b < 4; ++b) {
                    const int pa = patch[t[a]], pb = patch[t[b]];
                    if (pa >= 0 && pb >= 0 && pa != pb) exported[t[a]] = 1;
                }
        }
        for (int p = 0; p < parts; ++p) {
            const int lo = p * chunk, hi = std::min(nf, lo + chunk);
            std::stable_partition(ids.begin() + lo, ids.begin() + hi, [&](int v) { return exported[v] != 0; });
        }
    }

    int init(const vkpd_mesh_desc* d, const vkpd_config* c) override {
        n = (int)d->n_nodes;
        nE = (int)d->n_tets;
        nP = (int)d->n_pins;
        dt = d->dt;
        tol = c->tol > 0 ? c->tol : (sizeof(T) == 4 ? 2e-6 : 1e-12);
        max_iters = c->max_iters > 0 ? c->max_iters : 1000;
        use_graph = c->use_graph != 0;
        if (n <= 0 || nE <= 0) return fail(VKPD_EINVAL, "empty mesh");
        if (d->n_nodes > (1ll << 30) || 4ll * d->n_tets > (1ll << 31) - 1)
            return fail(VKPD_EINVAL, "mesh too large for 32-bit indexing");
        if (!(dt > 0.0)) return fail(VKPD_EINVAL, "dt must be positive");
        if (d->node_mass == nullptr) return fail(VKPD_EINVAL, "mesh node masses not lumped yet");
        for (int e = 0; e < nE; ++e) {
            if (d->gamma_s[e] < 0.0 || d->gamma_v[e] < 0.0)
                return fail(VKPD_EINVAL, "negative material coefficient");
            if (!(d->volume[e] > 0.0)) return fail(VKPD_EINVAL, "non-positive element volume");
            for (int k = 0; k < 4; ++k) {
                const int64_t id = d->tets[4 * (size_t)e + k];
                if (id < 0 || id >= n) return fail(VKPD_EINVAL, "tet node index out of range");
            }
        }
        // internal order: free nodes, then pins (pin order).  With rest positions the free
        // nodes are grouped into compact patches by recursive coordinate bisection, one patch
        // per solver CTA (its rows' neighbours then mostly live in the same CTA); without,
        // caller order.
        std::vector<int> ioo(n, -1);
        std::vector<char> pinned(n, 0);
        for (int k = 0; k < nP; ++k) {
            const int64_t id = d->pins[k];
            if (id < 0 || id >= n) return fail(VKPD_EINVAL, "pin index out of range");
            if (pinned[id]) return fail(VKPD_EINVAL, "duplicate pin index");
            pinned[id] = 1;
        }
        CK(cudaSetDevice(device));
        CK(cudaDeviceGetAttribute(&n_sms, cudaDevAttrMultiProcessorCount, device));
        nF = 0;
        std::vector<int> free_ids;
        for (int j = 0; j < n; ++j) if (!pinned[j]) free_ids.push_back(j);
        nF = (int)free_ids.size();
        part_blocks = c->pcg_blocks > 0 ? c->pcg_blocks : std::min(n_sms, std::max(1, cdiv(nF, 32)));
        if (d->nodes != nullptr && nF > 0) patch_order(d->nodes, d->tets, d->n_tets, n, free_ids, part_blocks);
        for (int k = 0; k < nF; ++k) ioo[free_ids[k]] = k;
        for (int k = 0; k < nP; ++k) ioo[d->pins[k]] = nF + k;
        int_of_orig_h = ioo;
        set_free_perm();
        std::vector<int4> tets_h(nE);
        for (int e = 0; e < nE; ++e)
            tets_h[e] = make_int4(ioo[d->tets[4 * (size_t)e]], ioo[d->tets[4 * (size_t)e + 1]],
                                  ioo[d->tets[4 * (size_t)e + 2]], ioo[d->tets[4 * (size_t)e + 3]]);
        // incidences per internal node, tet order
        std::vector<int> iptr(n + 1, 0);
        for (int e = 0; e < nE; ++e) {
            const int* t = &tets_h[e].x;
            for (int a = 0; a < 4; ++a) iptr[t[a] + 1]++;
        }
        for (int i = 0; i < n; ++i) iptr[i + 1] += iptr[i];
        std::vector<int> icode(iptr[n]), fillp(iptr.begin(), iptr.end() - 1);
        std::vector<int4> slot_h(nE);
        for (int e = 0; e < nE; ++e) {
            const int* t = &tets_h[e].x;
            int* sl = &slot_h[e].x;
            for (int a = 0; a < 4; ++a) {
                sl[a] = fillp[t[a]];
                icode[fillp[t[a]]++] = a * nE + e;
            }
        }
        // warp-segmented reduction tables: the 32 tets of warp w (internal order) and their 128
        // corners grouped by node (ascending node, then lane*4 + corner); node partial slots in
        // warp order (part_ptr over nodes)
        const int nW = cdiv(std::max(1, nE), 32);
        std::vector<int> wrp(nW + 1, 0), pcount(n + 1, 0);
        std::vector<std::pair<int, int>> pr;
        auto warp_pairs = [&](int wq) {
            pr.clear();
            for (int l = 0; l < 32; ++l) {
                const int e = wq * 32 + l;
                if (e >= nE) break;
                const int* t = &tets_h[e].x;
                for (int c = 0; c < 4; ++c) pr.push_back({t[c], l * 4 + c});
            }
            std::sort(pr.begin(), pr.end());
        };
        for (int wq = 0; wq < nW; ++wq) {
            warp_pairs(wq);
            int m = 0;
            for (size_t k = 0; k < pr.size(); ++k)
                if (k == 0 || pr[k].first != pr[k - 1].first) { ++m; pcount[pr[k].first + 1]++; }
            wrp[wq + 1] = wrp[wq] + m;
        }
        for (int i = 0; i < n; ++i) pcount[i + 1] += pcount[i];
        std::vector<int> wslot(std::max(1, wrp[nW])), pfill(pcount.begin(), pcount.end() - 1);
        std::vector<unsigned char> wbeg(std::max(1, wrp[nW])), wcode((size_t)nW * 128, 0);
        for (int wq = 0; wq < nW; ++wq) {
            warp_pairs(wq);
            int E = wrp[wq];
            for (size_t k = 0; k < pr.size(); ++k) {
                wcode[(size_t)wq * 128 + k] = (unsigned char)pr[k].second;
                if (k == 0 || pr[k].first != pr[k - 1].first) {
                    wbeg[E] = (unsigned char)k;
                    wslot[E] = pfill[pr[k].first]++;
                    ++E;
                }
            }
        }
        // neighbour sets of free rows -> ELL (free cols) + K_fp CSR (pin slots)
        std::vector<std::vector<int>> nb(nF);
        ell_w = 0;
        std::vector<int> fptr(nF + 1, 0), fcol;
        for (int i = 0; i < nF; ++i) {
            std::vector<int>& s = nb[i];
            s.push_back(i);
            for (int k = iptr[i]; k < iptr[i + 1]; ++k) {
                const int e = icode[k] % nE;
                const int* t = &tets_h[e].x;
                for (int a = 0; a < 4; ++a) s.push_back(t[a]);
            }
            std::sort(s.begin(), s.end());
            s.erase(std::unique(s.begin(), s.end()), s.end());
            int nfree = 0;
            for (int col : s) {
                if (col < nF) ++nfree;
                else fcol.push_back(col - nF);
            }
            fptr[i + 1] = (int)fcol.size();
            ell_w = std::max(ell_w, nfree);
        }
        std::vector<int> ecol((size_t)ell_w * nF), elen(nF);
        for (int i = 0; i < nF; ++i) {
            int s = 0;
            for (int col : nb[i])
                if (col < nF) ecol[(size_t)s++ * nF + i] = col;
            elen[i] = s;
            for (; s < ell_w; ++s) ecol[(size_t)s * nF + i] = i;     // pad: own column, value 0
        }
        // per-node arrays in internal order
        std::vector<double> mdt2(n);
        std::vector<T> mdt2_t(n), dt2im(n);
        for (int j = 0; j < n; ++j) {
            const double m = d->node_mass[j];
            mdt2[ioo[j]] = m / (dt * dt);
            mdt2_t[ioo[j]] = (T)(m / (dt * dt));
            dt2im[ioo[j]] = (T)(m > 0.0 ? dt * dt / m : 0.0);
        }
        // per-tet planes
        std::vector<T> Gp((size_t)9 * nE), wp((size_t)2 * nE);
        std::vector<double> wsum(nE);
        for (int e = 0; e < nE; ++e) {
            const double* g = d->shape_grad + (size_t)12 * e;
            for (int k = 0; k < 9; ++k) Gp[(size_t)k * nE + e] = (T)g[3 + k];
            const double vv = 2.0 * d->volume[e];
            wp[e] = (T)(vv * d->gamma_s[e]);
            wp[(size_t)nE + e] = (T)(vv * d->gamma_v[e]);
            wsum[e] = vv * (d->gamma_s[e] + d->gamma_v[e]);
        }

        CK(cudaStreamCreateWithFlags(&own_stream, cudaStreamNonBlocking));
        stream = own_stream;
        cudaStream_t s = stream;
        CK(tets.alloc(nE)); CK(tets.upload(tets_h.data(), nE, s));
        CK(slot4.alloc(nE)); CK(slot4.upload(slot_h.data(), nE, s));
        CK(ell_len.alloc(nF)); CK(ell_len.upload(elen.data(), nF, s));
        CK(G.alloc((size_t)9 * nE)); CK(G.upload(Gp.data(), Gp.size(), s));
        CK(w.alloc((size_t)2 * nE)); CK(w.upload(wp.data(), wp.size(), s));
        CK(inc_ptr.alloc(n + 1)); CK(inc_ptr.upload(iptr.data(), n + 1, s));
        CK(inc_code.alloc(icode.size())); CK(inc_code.upload(icode.data(), icode.size(), s));
        CK(wr_ptr.alloc(wrp.size())); CK(wr_ptr.upload(wrp.data(), wrp.size(), s));
        CK(wr_slot.alloc(wslot.size())); CK(wr_slot.upload(wslot.data(), wslot.size(), s));
        CK(wr_beg.alloc(wbeg.size())); CK(wr_beg.upload(wbeg.data(), wbeg.size(), s));
        CK(wr_code.alloc(wcode.size())); CK(wr_code.upload(wcode.data(), wcode.size(), s));
        CK(part_ptr.alloc(pcount.size())); CK(part_ptr.upload(pcount.data(), pcount.size(), s));
        CK(wpart.alloc(std::max(1, pcount[n])));
        CK(robust_flag.alloc(std::max<size_t>(1, icode.size())));
        CK(cudaMemsetAsync(robust_flag.p, 0, std::max<size_t>(1, icode.size()), s));
        CK(int_of_orig.alloc(n)); CK(int_of_orig.upload(ioo.data(), n, s));
        CK(ell_col.alloc(ecol.size())); CK(ell_col.upload(ecol.data(), ecol.size(), s));
        CK(ell_val.alloc(ecol.size()));
        CK(fp_ptr.alloc(nF + 1)); CK(fp_ptr.upload(fptr.data(), nF + 1, s));
        CK(fp_col.alloc(std::max<size_t>(1, fcol.size())));
        if (!fcol.empty()) CK(fp_col.upload(fcol.data(), fcol.size(), s));
        CK(fp_val.alloc(std::max<size_t>(1, fcol.size())));
        CK(inv_diag.alloc(nF));
        CK(diag64.alloc(nF));
        CK(m_dt2.alloc(n)); CK(m_dt2.upload(mdt2_t.data(), n, s));
        CK(dt2_inv_m.alloc(n)); CK(dt2_inv_m.upload(dt2im.data(), n, s));
        // assembly inputs (float64), kept for re-assembly when the material changes
        CK(G64k.alloc((size_t)12 * nE)); CK(G64k.upload(d->shape_grad, (size_t)12 * nE, s));
        CK(md64k.alloc(n)); CK(md64k.upload(mdt2.data(), n, s));
        vol2_h.resize(nE);
        for (int e = 0; e < nE; ++e) vol2_h[e] = 2.0 * d->volume[e];
        if (int rc = assemble(wsum)) return rc;
        return alloc_work(c);
    }

    // pd_equilibrium (pdsolver.py:315-338): proximal local/global rounds on the quasi-static
    // objective; the simulation state is untouched (own iterate buffers).  A round whose
    // solve needs zero CG iterations leaves x unchanged, so the rest would repeat it: stop.
    int equilibrium(const double* ha, const double* hx0, const double* hpins, int iterations, double* x_out,
                    int* failed) override {
        if (!G64k.p) return fail(VKPD_EINVAL, "pd_equilibrium needs a mesh context");
        if (iterations < 0 || iterations > 100000) return fail(VKPD_EINVAL, "bad iteration count");
        if (nP > 0 && !hpins) return fail(VKPD_EINVAL, "pin values required");
        if (failed) *failed = -1;
        DBuf<V4> a4;
        CK(a4.alloc(n));
        if (int rc = upload_nodes(ha, a4.p)) return rc;
        if (int rc = upload_nodes(hx0, tmp4a.p)) return rc;
        DBuf<V4> p4;
        if (nP > 0) {
            CK(p4.alloc(nP));
            CK(cudaMemcpyAsync(stage.p, hpins, sizeof(double) * 3 * nP, cudaMemcpyHostToDevice, stream));
            k_rows_in<T><<<cdiv(nP, 256), 256, 0, stream>>>(nP, stage.p, p4.p);
            CK(cudaGetLastError());
            vk::k_set_pinned<T><<<cdiv(nP, 256), 256, 0, stream>>>(n, nF, p4.p, tmp4a.p);
            CK(cudaGetLastError());
        }
        CK(cudaMemsetAsync(fail_iter.p, 0x7f, sizeof(int), stream));     // 0x7f7f7f7f: no failure
        const vk::LocalArgs<T> la = local_args(tmp4a.p);
        for (int it = 0; it < iterations && nF > 0; ++it) {
            vk::k_eq_target<T><<<cdiv(nF, 256), 256, 0, stream>>>(nF, tmp4a.p, a4.p, tmp4b.p);
            CK(cudaGetLastError());
            if (int rc = launch_local_resid(la)) return rc;
            vk::PcgArgs<T> pa = pcg_args(vk::INIT_PD, it, iters.p);
            pa.x = tmp4a.p; pa.xhat = tmp4b.p;
            pa.warm = nullptr; pa.rounds = nullptr;
            pa.inv_diag = inv_diag.p; pa.cdiag = nullptr; pa.cb = nullptr; pa.coll = nullptr; pa.ncoll = 0;
            pa.ell_kd = ell_kd.p;
            CK(launch_pcg(pa));
            int cgi = -1, fi = 0;
            CK(cudaMemcpyAsync(&cgi, iters.p, sizeof(int), cudaMemcpyDeviceToHost, stream));
            CK(cudaMemcpyAsync(&fi, fail_iter.p, sizeof(int), cudaMemcpyDeviceToHost, stream));
            CK(cudaStreamSynchronize(stream));
            if (fi != 0x7f7f7f7f) {
                if (failed) *failed = fi;
                return fail(VKPD_ENONFINITE, "quasi-static projection diverged at iteration " + std::to_string(fi));
            }
            if (cgi == 0) break;
        }
        return download_nodes(tmp4a.p, x_out);
    }

    // per-frame output step (transfer.py:26-28, cli.py:639-640)
    DBuf<long long> y_ptr;
    DBuf<int> y_col;
    DBuf<double> y_w, y_out;
    int64_t n_yarn = 0;
    int set_yarn_interp(int64_t ny, const int64_t* indptr, const int64_t* indices, const double* data) override {
        if (ny < 0 || (ny > 0 && (!indptr || !indices || !data))) return fail(VKPD_EINVAL, "bad interpolation matrix");
        if (int_of_orig_h.empty()) return fail(VKPD_EINVAL, "no mesh in this context");
        const int64_t nnz = ny > 0 ? indptr[ny] : 0;
        std::vector<int> ci(std::max<int64_t>(1, nnz));
        for (int64_t k = 0; k < ny; ++k)
            if (indptr[k + 1] < indptr[k]) return fail(VKPD_EINVAL, "interpolation indptr not monotone");
        for (int64_t j = 0; j < nnz; ++j) {
            if (indices[j] < 0 || indices[j] >= n) return fail(VKPD_EINVAL, "interpolation column out of range");
            ci[j] = int_of_orig_h[indices[j]];
        }
        n_yarn = ny;
        CK(y_ptr.alloc(ny + 1));
        CK(y_ptr.upload((const long long*)indptr, ny + 1, stream));
        CK(y_col.alloc(std::max<int64_t>(1, nnz)));
        CK(y_w.alloc(std::max<int64_t>(1, nnz)));
        if (nnz > 0) { CK(y_col.upload(ci.data(), nnz, stream)); CK(y_w.upload(data, nnz, stream)); }
        CK(y_out.alloc((size_t)3 * std::max<int64_t>(1, ny)));
        CK(cudaStreamSynchronize(stream));
        return VKPD_OK;
    }
    int frame_outputs(double* yarn, double* det_dev) override {
        if (yarn) {
            if (n_yarn <= 0 && !y_ptr.p) return fail(VKPD_EINVAL, "no yarn interpolation set (vkpd_set_yarn_interp)");
            if (n_yarn > 0) {
                vk::k_v2y<T><<<cdiv((int)n_yarn, 256), 256, 0, stream>>>((int)n_yarn, y_ptr.p, y_col.p, y_w.p, x.p,
                                                                          y_out.p);
                CK(cudaGetLastError());
                CK(cudaMemcpyAsync(yarn, y_out.p, sizeof(double) * 3 * n_yarn, cudaMemcpyDeviceToHost, stream));
            }
        }
        if (det_dev) {
            if (!G64k.p) return fail(VKPD_EINVAL, "det deviation needs a mesh context");
            DBuf<unsigned long long> m;
            CK(m.alloc(1));
            CK(cudaMemsetAsync(m.p, 0, sizeof(unsigned long long), stream));
            if (nE > 0)
                vk::k_det_deviation<T><<<cdiv(nE, 256), 256, 0, stream>>>(nE, tets.p, G64k.p, x.p, m.p);
            CK(cudaGetLastError());
            unsigned long long b = 0;
            CK(cudaMemcpyAsync(&b, m.p, sizeof b, cudaMemcpyDeviceToHost, stream));
            CK(cudaStreamSynchronize(stream));
            std::memcpy(det_dev, &b, sizeof b);
        }
        CK(cudaStreamSynchronize(stream));
        return VKPD_OK;
    }

    // K_ff / K_fp from the per-tet weights 2V(gs+gv) (pdsolver.py:42-56), deterministic
    int assemble(const std::vector<double>& wsum) {
        cudaStream_t s = stream;
        DBuf<double> ws64;
        CK(ws64.alloc(nE)); CK(ws64.upload(wsum.data(), nE, s));
        vk::AssembleArgs<T> aa;
        aa.nF = nF; aa.nE = nE; aa.ell_w = ell_w;
        aa.inc_ptr = inc_ptr.p; aa.inc_code = inc_code.p; aa.tets = tets.p; aa.G = G64k.p; aa.wsum = ws64.p;
        aa.m_dt2 = md64k.p; aa.ell_col = ell_col.p; aa.ell_len = ell_len.p; aa.ell_val = ell_val.p;
        aa.inv_diag = inv_diag.p;
        aa.diag64 = diag64.p; aa.fp_ptr = fp_ptr.p; aa.fp_col = fp_col.p; aa.fp_val = fp_val.p;
        aa.n_free_cols_base = nF;
        if (nF > 0) vk::k_assemble<T><<<cdiv(nF, 128), 128, 0, s>>>(aa);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(s));
        return VKPD_OK;
    }
    // polynomial preconditioner: Gershgorin weight and the prescaled K D^-1
    int refresh_precond() {
        if (nF <= 0) return VKPD_OK;
        cudaStream_t s = stream;
        // Gershgorin bound G >= lambda_max(D^-1 K_ff); w = min(1, 1.9 / G) keeps
        // w D^-1 (2 - w K D^-1) SPD with margin
        DBuf<unsigned long long> gmax;
        CK(gmax.alloc(1));
        CK(cudaMemsetAsync(gmax.p, 0, sizeof(unsigned long long), s));
        vk::k_gershgorin<T><<<cdiv(nF, 256), 256, 0, s>>>(nF, ell_w, ell_col.p, ell_val.p, diag64.p, gmax.p);
        CK(cudaGetLastError());
        unsigned long long gb = 0;
        CK(cudaMemcpyAsync(&gb, gmax.p, sizeof gb, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        double g = 1.0;
        std::memcpy(&g, &gb, sizeof g);
        g += 1.0;
        gersh = (g > 0.0 && std::isfinite(g)) ? g : 2.0;
        poly_omega = (g > 0.0 && std::isfinite(g)) ? std::min(1.0, 1.9 / g) : 0.5;
        if (ell_kd.n != (size_t)std::max(1, ell_w) * nF) CK(ell_kd.alloc((size_t)std::max(1, ell_w) * nF));
        vk::k_scale_ell<T><<<cdiv(nF, 256), 256, 0, s>>>(nF, ell_w, ell_col.p, ell_val.p, inv_diag.p, ell_kd.p);
        CK(cudaGetLastError());
        if (cheb) if (int rc = spectrum_low()) return rc;
        if (cheb && pcg_blocks > 0) {
            if (int rc = build_cheb_neighbours()) return rc;
            if (solver_auto && !cheb_reg) {
                cheb = false;
                pcg_poly = true;
                solver_kind = VKPD_SOLVER_PCG_POLY;
            }
        }
        return VKPD_OK;
    }

    // lambda_min of D^-1 K_ff for the Chebyshev solver: rigorous lower bound min_i (m_i/dt^2)/K_ii
    // (K - M/dt^2 is PSD), and the smallest Ritz value of 80 Lanczos steps on D^-1/2 K_ff D^-1/2
    // (an upper estimate that converges fast at the spectrum's end); the solver uses
    // max(bound, 0.97 * Ritz).  Its residual check keeps the stopping rule exact either way.
    int spectrum_low() {
        cudaStream_t s = stream;
        std::vector<double> dg(nF), md(n);
        CK(cudaMemcpyAsync(dg.data(), diag64.p, sizeof(double) * nF, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(md.data(), md64k.p, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        double lb = 1.0;
        for (int i = 0; i < nF; ++i) lb = std::min(lb, md[i] / dg[i]);
        lam_min_bound = std::max(0.0, lb);
        const int m = std::min(80, nF);
        DBuf<double> v0, v1, w, al, be;
        CK(v0.alloc(nF)); CK(v1.alloc(nF)); CK(w.alloc(nF)); CK(al.alloc(m + 1)); CK(be.alloc(m + 2));
        CK(cudaMemsetAsync(al.p, 0, sizeof(double) * (m + 1), s));
        CK(cudaMemsetAsync(be.p, 0, sizeof(double) * (m + 2), s));
        vk::LanczosArgs<T> la;
        la.nF = nF; la.ell_w = ell_w; la.m = m; la.ell_col = ell_col.p; la.ell_val = ell_val.p;
        la.diag64 = diag64.p; la.v0 = v0.p; la.v1 = v1.p; la.w = w.p; la.partials = partials.p;
        la.alpha = al.p; la.beta = be.p;
        int occ = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, vk::k_lanczos<T>, 512, 0));
        const int blocks = std::max(1, std::min(occ * n_sms, std::min(pcg_blocks, cdiv(nF, 512))));
        void* args[] = {&la};
        CK(cudaLaunchCooperativeKernel((const void*)vk::k_lanczos<T>, dim3(blocks), dim3(512), args, 0, s));
        std::vector<double> a(m + 1), b(m + 2);
        CK(cudaMemcpyAsync(a.data(), al.p, sizeof(double) * (m + 1), cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(b.data(), be.p, sizeof(double) * (m + 2), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        int mm = m;
        for (int j = 0; j < m; ++j)
            if (!(b[j + 1] > 0.0)) { mm = j + 1; break; }
        const double ritz = tridiag_min_eig(a.data(), b.data() + 1, mm);
        lam_min = std::max(lam_min_bound, 0.97 * ritz);
        if (!(lam_min > 0.0) || !(lam_min < gersh)) lam_min = std::max(lam_min_bound, 1e-6);
        return VKPD_OK;
    }
    // smallest eigenvalue of the symmetric tridiagonal (diag a[0..m), off-diag b[0..m-1)) by bisection
    // on the Sturm count
    static double tridiag_min_eig(const double* a, const double* b, int m) {
        double lo = a[0], hi = a[0];
        for (int i = 0; i < m; ++i) {
            const double r = (i > 0 ? std::fabs(b[i - 1]) : 0.0) + (i + 1 < m ? std::fabs(b[i]) : 0.0);
            lo = std::min(lo, a[i] - r);
            hi = std::max(hi, a[i] + r);
        }
        auto count_below = [&](double x) {
            int c = 0;
            double q = a[0] - x;
            if (q < 0) ++c;
            for (int i = 1; i < m; ++i) {
                if (q == 0.0) q = 1e-300;
                q = a[i] - x - b[i - 1] * b[i - 1] / q;
                if (q < 0) ++c;
            }
            return c;
        };
        for (int it = 0; it < 200; ++it) {
            const double mid = 0.5 * (lo + hi);
            if (count_below(mid) >= 1) hi = mid; else lo = mid;
        }
        return 0.5 * (lo + hi);
    }

    size_t cheb_smem_bytes() const { return vk::cheb_smem_bytes<T>(); }
    // Per CTA (rows [b*chunk, (b+1)*chunk)): the CTAs owning the columns its rows read (the
    // neighbour flags it waits on), its halo (those rows themselves, staged in shared memory
    // each step) and every ELL column's shared-memory slot.  The register path needs one row
    // per thread and the staged image within the shared-memory limit.
    int cheb_halo_max = 0;
    DBuf<unsigned> cheb_slot;
    DBuf<int> cheb_halo_ptr, cheb_halo;
    DBuf<T> cheb_val, cheb_kdiag;
    DBuf<int> cheb_nexp;
    // Entry positions of one wavefront group's rows without shared-memory bank conflicts.
    // k_cheb_reg's SpMV loads d[slot[o]] for o = 0..13 at once across a warp; a 32-bit load is
    // served per warp (32 lanes, bank = slot mod 32), a 64-bit one per half-warp (16 lanes, bank
    // pair = slot mod 16), and costs as many wavefronts as the most distinct slots that share a
    // bank (C = number of banks).  The rows' entries form a bipartite multigraph
    // lanes x bank pairs; an edge colouring with D = max(14, max degree) colours (Konig:
    // alternating-path recolouring) puts distinct bank pairs at each position.  Colours >= 14
    // (an overloaded bank pair) fold into a lane's free position where they add the least; pad
    // positions (value 0) read a slot another lane already reads there (broadcast).  C3 fp64:
    // 3.6 -> 2.1 wavefronts per gather (tools/dbg/bank_model.py).
    static void conflict_free_positions(int lanes, int C, const int* ent_n, const int (*ent_slot)[vk::kChebOff],
                                        const int* own_slot, int (*pos_of)[vk::kChebOff],
                                        int (*pad_slot)[vk::kChebOff]) {
        constexpr int K = vk::kChebOff;
        int deg[32] = {0};
        int ne = 0;
        for (int u = 0; u < lanes; ++u)
            for (int t = 0; t < ent_n[u]; ++t) { ++deg[ent_slot[u][t] % C]; ++ne; }
        int D = K;
        for (int b = 0; b < C; ++b) D = std::max(D, deg[b]);
        std::vector<int> eu(ne), ev(ne), et(ne), ec(ne, -1);
        std::vector<int> U((size_t)32 * D, -1), V((size_t)C * D, -1);
        int id = 0;
        for (int u = 0; u < lanes; ++u)
            for (int t = 0; t < ent_n[u]; ++t) { eu[id] = u; ev[id] = ent_slot[u][t] % C; et[id] = t; ++id; }
        std::vector<int> path;
        for (int e = 0; e < ne; ++e) {
            const int u = eu[e], v = ev[e];
            int a = 0, b = 0;
            while (U[(size_t)u * D + a] >= 0) ++a;
            while (V[(size_t)v * D + b] >= 0) ++b;
            if (V[(size_t)v * D + a] >= 0) {
                // flip the a/b alternating path that starts at v with colour a
                path.clear();
                bool at_v = true;
                int node = v, col = a;
                for (;;) {
                    const int f = at_v ? V[(size_t)node * D + col] : U[(size_t)node * D + col];
                    if (f < 0) break;
                    path.push_back(f);
                    node = at_v ? eu[f] : ev[f];
                    at_v = !at_v;
                    col = col == a ? b : a;
                }
                for (int f : path) { U[(size_t)eu[f] * D + ec[f]] = -1; V[(size_t)ev[f] * D + ec[f]] = -1; }
                for (int f : path) {
                    ec[f] = ec[f] == a ? b : a;
                    U[(size_t)eu[f] * D + ec[f]] = f; V[(size_t)ev[f] * D + ec[f]] = f;
                }
            }
            ec[e] = a; U[(size_t)u * D + a] = e; V[(size_t)v * D + a] = e;
        }
        // positions: colour c < K is position c; later colours fold into free positions
        std::vector<std::vector<int>> at((size_t)K * C);       // (position, bank) -> slots
        for (int u = 0; u < lanes; ++u) for (int o = 0; o < K; ++o) pos_of[u][o] = -1;
        auto add = [&](int o, int sl) {
            auto& L = at[(size_t)o * C + sl % C];
            if (std::find(L.begin(), L.end(), sl) == L.end()) L.push_back(sl);
        };
        for (int e = 0; e < ne; ++e)
            if (ec[e] < K) { pos_of[eu[e]][ec[e]] = et[e]; add(ec[e], ent_slot[eu[e]][et[e]]); }
        for (int e = 0; e < ne; ++e) {
            if (ec[e] < K) continue;
            const int u = eu[e], sl = ent_slot[u][et[e]];
            int best = -1;
            size_t bc = 0;
            for (int o = 0; o < K; ++o) {
                if (pos_of[u][o] >= 0) continue;
                const auto& L = at[(size_t)o * C + sl % C];
                const size_t c = std::find(L.begin(), L.end(), sl) != L.end() ? 0 : L.size();
                if (best < 0 || c < bc) { best = o; bc = c; }
            }
            pos_of[u][best] = et[e];
            add(best, sl);
        }
        for (int u = 0; u < lanes; ++u)
            for (int o = 0; o < K; ++o) {
                pad_slot[u][o] = own_slot[u];
                if (pos_of[u][o] >= 0) continue;
                for (int b = 0; b < C; ++b)
                    if (!at[(size_t)o * C + b].empty()) { pad_slot[u][o] = at[(size_t)o * C + b][0]; break; }
                if (at[(size_t)o * C + pad_slot[u][o] % C].empty()) add(o, pad_slot[u][o]);
            }
    }
    int build_cheb_neighbours() {
        const int chunk = cdiv(std::max(1, nF), pcg_blocks);
        std::vector<int> ecol((size_t)ell_w * nF);
        std::vector<T> evals((size_t)ell_w * nF);
        if (nF > 0) {
            CK(cudaMemcpy(ecol.data(), ell_col.p, ecol.size() * sizeof(int), cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(evals.data(), ell_val.p, evals.size() * sizeof(T), cudaMemcpyDeviceToHost));
        }
        // per row: the off-diagonal entries in a canonical order (by caller-order index offset,
        // so the rows of a warp, which are neighbours in the mesh, take the same direction at the
        // same position and hit consecutive shared-memory slots), and the diagonal
        std::vector<int> orig_of_int(n);
        for (int j = 0; j < n; ++j) orig_of_int[int_of_orig_h[j]] = j;
        const size_t nn1 = std::max(1, nF);
        std::vector<int> ocol((size_t)vk::kChebOff * nn1, -1);
        std::vector<T> oval((size_t)vk::kChebOff * nn1, T(0));
        std::vector<T> kd(nn1, T(0));
        bool fits = true;
        {
            std::vector<std::pair<long long, int>> ent;
            for (int i = 0; i < nF; ++i) {
                ent.clear();
                for (int sl = 0; sl < ell_w; ++sl) {
                    const size_t e = (size_t)sl * nF + i;
                    if (ecol[e] == i) { kd[i] += evals[e]; continue; }
                    ent.push_back({(long long)orig_of_int[ecol[e]] - orig_of_int[i], sl});
                }
                if ((int)ent.size() > vk::kChebOff) { fits = false; continue; }
                std::sort(ent.begin(), ent.end());
                for (size_t o = 0; o < ent.size(); ++o) {
                    const size_t e = (size_t)ent[o].second * nF + i;
                    ocol[o * nF + i] = ecol[e];
                    oval[o * nF + i] = evals[e];
                }
            }
        }
        // per CTA: neighbour CTAs and halo rows, grouped by owner CTA (in neighbour order: the
        // kernel loads each neighbour's rows as soon as its flag arrives); within a group in
        // first-use order over (position, row), so a warp's halo reads are consecutive too
        std::vector<int> ptr(pcg_blocks + 1, 0), lst, hptr(pcg_blocks + 1, 0), hl;
        std::vector<int> oslot((size_t)vk::kChebOff * nn1);
        std::vector<int> nbr_pos(pcg_blocks, -1);
        std::vector<int> hslot(nn1, -1);
        cheb_halo_max = 0;
        for (int b = 0; b < pcg_blocks; ++b) {
            const int r0 = b * chunk, r1 = std::min(nF, r0 + chunk);
            std::vector<int> first;                     // halo rows in first-use order
            const int n0 = (int)lst.size();
            auto note = [&](int c) {
                const int ow = c / chunk;
                if (nbr_pos[ow] < 0) { nbr_pos[ow] = (int)lst.size() - n0; lst.push_back(ow); }
            };
            for (int o = 0; o < vk::kChebOff; ++o)
                for (int i = r0; i < r1; ++i) {
                    const int c = ocol[(size_t)o * nF + i];
                    if (c < 0 || (c >= r0 && c < r1)) continue;
                    note(c);
                    if (hslot[c] < 0) { hslot[c] = 0; first.push_back(c); }
                }
            if (!fits)
                for (int sl = 0; sl < ell_w; ++sl)
                    for (int i = r0; i < r1; ++i) {
                        const int c = ecol[(size_t)sl * nF + i];
                        if (c < r0 || c >= r1) note(c);
                    }
            std::stable_sort(first.begin(), first.end(),
                             [&](int x, int y) { return nbr_pos[x / chunk] < nbr_pos[y / chunk]; });
            const int h0 = (int)hl.size();
            for (size_t j = 0; j < first.size(); ++j) { hslot[first[j]] = (int)j; hl.push_back(first[j]); }
            for (int o = 0; o < vk::kChebOff; ++o)
                for (int i = r0; i < r1; ++i) {
                    const int c = ocol[(size_t)o * nF + i];
                    if (c < 0) oslot[(size_t)o * nF + i] = i - r0;                 // pad: own row, value 0
                    else if (c >= r0 && c < r1) oslot[(size_t)o * nF + i] = c - r0;
                    else oslot[(size_t)o * nF + i] = pcg_threads + hslot[c];
                }
            // wavefront group: 32 lanes for a 4-byte direction image, 16 for an 8-byte one
            constexpr int G = sizeof(typename vk::ChebImage<T>::type) == 4 ? 32 : 16;
            if (fits)
                for (int h0 = r0; h0 < r1; h0 += G) {
                    const int lanes = std::min(G, r1 - h0);
                    int en[32], es[32][vk::kChebOff], own_s[32], pos[32][vk::kChebOff], pad[32][vk::kChebOff];
                    T ev[32][vk::kChebOff];
                    for (int u = 0; u < lanes; ++u) {
                        const int i = h0 + u;
                        own_s[u] = i - r0;
                        en[u] = 0;
                        for (int o = 0; o < vk::kChebOff; ++o)
                            if (ocol[(size_t)o * nF + i] >= 0) {
                                es[u][en[u]] = oslot[(size_t)o * nF + i];
                                ev[u][en[u]] = oval[(size_t)o * nF + i];
                                ++en[u];
                            }
                    }
                    conflict_free_positions(lanes, G, en, es, own_s, pos, pad);
                    for (int u = 0; u < lanes; ++u)
                        for (int o = 0; o < vk::kChebOff; ++o) {
                            const size_t x = (size_t)o * nF + h0 + u;
                            const int t = pos[u][o];
                            oslot[x] = t >= 0 ? es[u][t] : pad[u][o];
                            oval[x] = t >= 0 ? ev[u][t] : T(0);
                        }
                }
            for (int j = h0; j < (int)hl.size(); ++j) hslot[hl[j]] = -1;
            for (int q = n0; q < (int)lst.size(); ++q) nbr_pos[lst[q]] = -1;
            ptr[b + 1] = (int)lst.size();
            hptr[b + 1] = (int)hl.size();
            cheb_halo_max = std::max(cheb_halo_max, (int)hl.size() - h0);
        }
        if (lst.empty()) lst.push_back(0);
        if (hl.empty()) hl.push_back(0);
        // exported rows (read by another CTA) must lead each CTA's range for the early publish;
        // otherwise the CTA treats all its rows as exported
        std::vector<char> exp_row(nn1, 0);
        for (int j = 0; j < hptr[pcg_blocks]; ++j) exp_row[hl[j]] = 1;
        std::vector<int> nexp(pcg_blocks, 0);
        for (int b = 0; b < pcg_blocks; ++b) {
            const int r0 = b * chunk, r1 = std::min(nF, r0 + chunk);
            int e = 0;
            while (r0 + e < r1 && exp_row[r0 + e]) ++e;
            for (int r = r0 + e; r < r1; ++r)
                if (exp_row[r]) { e = r1 - r0; break; }
            nexp[b] = std::max(0, e);
        }
        CK(cheb_nexp.alloc(pcg_blocks)); CK(cheb_nexp.upload(nexp.data(), nexp.size(), stream));
        int max_smem = 0;
        CK(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
        cheb_reg = fits && chunk <= pcg_threads && pcg_threads <= vk::kChebMaxThreads &&
                   pcg_threads + cheb_halo_max <= vk::kChebSlots && cheb_smem_bytes() + 4096 <= (size_t)max_smem;
        if (cheb_reg) {
            CK(cudaFuncSetAttribute(vk::k_cheb_reg<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)cheb_smem_bytes()));
            int o = 0;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, vk::k_cheb_reg<T>, pcg_threads, cheb_smem_bytes()));
            if (o * n_sms < pcg_blocks) cheb_reg = false;
        }
        CK(cheb_nbr_ptr.alloc(pcg_blocks + 1)); CK(cheb_nbr_ptr.upload(ptr.data(), ptr.size(), stream));
        CK(cheb_nbr.alloc(lst.size())); CK(cheb_nbr.upload(lst.data(), lst.size(), stream));
        CK(cheb_halo_ptr.alloc(pcg_blocks + 1)); CK(cheb_halo_ptr.upload(hptr.data(), hptr.size(), stream));
        CK(cheb_halo.alloc(hl.size())); CK(cheb_halo.upload(hl.data(), hl.size(), stream));
        // slots as packed byte offsets into the direction image (two 16-bit per word)
        constexpr unsigned kImg = (unsigned)sizeof(typename vk::ChebImage<T>::type);
        constexpr int kHalf = (vk::kChebOff + 1) / 2;
        std::vector<unsigned> opack((size_t)kHalf * nn1, 0u);
        for (int h = 0; h < kHalf; ++h)
            for (int i = 0; i < nF; ++i) {
                const unsigned c0 = kImg * (unsigned)oslot[(size_t)(2 * h) * nF + i];
                const unsigned c1 = 2 * h + 1 < vk::kChebOff ? kImg * (unsigned)oslot[(size_t)(2 * h + 1) * nF + i] : 0u;
                opack[(size_t)h * nF + i] = c0 | (c1 << 16);
            }
        CK(cheb_slot.alloc(opack.size())); CK(cheb_slot.upload(opack.data(), opack.size(), stream));
        CK(cheb_val.alloc(oval.size())); CK(cheb_val.upload(oval.data(), oval.size(), stream));
        CK(cheb_kdiag.alloc(kd.size())); CK(cheb_kdiag.upload(kd.data(), kd.size(), stream));
        CK(cheb_flags.alloc((size_t)32 * pcg_blocks));
        CK(cudaMemsetAsync(cheb_flags.p, 0, sizeof(unsigned int) * 32 * pcg_blocks, stream));
        // tags restart with the flags: no stale row may carry a tag the next launches wait for
        CK(cheb_ll.alloc((size_t)2 * vk::LLRow<typename vk::ChebImage<T>::type>::W * std::max(1, nF)));
        CK(cudaMemsetAsync(cheb_ll.p, 0xff, cheb_ll.n * sizeof(uint4), stream));
        CK(cudaStreamSynchronize(stream));
        return VKPD_OK;
    }
    // new per-tet material (MaterialField): weights of the local step, K re-assembled on the
    // device; the frame graph is rebuilt (its solver weight may change), warm starts dropped
    int set_gammas(const double* gs, const double* gv) override {
        if (!G64k.p) return fail(VKPD_EINVAL, "set_gammas needs a mesh context");
        std::vector<T> wp((size_t)2 * nE);
        std::vector<double> wsum(nE);
        for (int e = 0; e < nE; ++e) {
            if (!(gs[e] >= 0.0) || !(gv[e] >= 0.0)) return fail(VKPD_EINVAL, "gamma must be non-negative");
            wp[e] = (T)(vol2_h[e] * gs[e]);
            wp[(size_t)nE + e] = (T)(vol2_h[e] * gv[e]);
            wsum[e] = vol2_h[e] * (gs[e] + gv[e]);
        }
        CK(w.upload(wp.data(), wp.size(), stream));
        if (int rc = assemble(wsum)) return rc;
        if (int rc = refresh_precond()) return rc;
        if (warm0.p) CK(cudaMemsetAsync(warm0.p, 0, warm0.n * sizeof(V4), stream));
        if (warm1.p) CK(cudaMemsetAsync(warm1.p, 0, warm1.n * sizeof(V4), stream));
        if (warm2.p) CK(cudaMemsetAsync(warm2.p, 0, warm2.n * sizeof(V4), stream));
        if (warm3.p) CK(cudaMemsetAsync(warm3.p, 0, warm3.n * sizeof(V4), stream));
        if (graph_exec) { cudaGraphExecDestroy(graph_exec); graph_exec = nullptr; }
        CK(cudaStreamSynchronize(stream));
        return VKPD_OK;
    }

    int alloc_work(const vkpd_config* c) {
        cudaStream_t s = stream;
        for (DBuf<V4>* b : {&x, &v, &x_start, &v_start, &xhat, &tmp4a, &tmp4b}) {
            CK(b->alloc(n));
            CK(cudaMemsetAsync(b->p, 0, n * sizeof(V4), s));
        }
        CK(f.alloc(n));
        CK(cudaMemsetAsync(f.p, 0, n * sizeof(V4), s));
        CK(pin_tgt.alloc(std::max(1, nP)));
        CK(cudaMemsetAsync(pin_tgt.p, 0, std::max(1, nP) * sizeof(V4), s));
        CK(corner.alloc((size_t)4 * nE));
        for (DBuf<V4>* b : {&r, &z, &p0, &p1, &q, &dx, &rhs, &hh}) {
            CK(b->alloc(std::max(1, nF)));
            CK(cudaMemsetAsync(b->p, 0, std::max(1, nF) * sizeof(V4), s));
        }
        // one CTA per SM (fewer arrivals per grid barrier measured faster than 2 CTAs/SM at C3),
        // all SMs busy, one row per thread where possible (each extra row per thread adds a
        // full memory round trip to every solver phase): CTA size = rows per CTA rounded up to
        // a warp, <= 768
        pcg_blocks = c->pcg_blocks > 0 ? c->pcg_blocks
                   : part_blocks > 0 ? part_blocks : std::min(n_sms, std::max(1, cdiv(nF, 32)));
        pcg_threads = std::max(128, std::min(768, 32 * cdiv(cdiv(std::max(1, nF), pcg_blocks), 32)));
        // AUTO: the Chebyshev solver where its register path applies (one row per thread, the
        // CTA's rows + halo staged in shared memory: C3 0.89 / 8.9 ms per frame fp32 / fp64 vs
        // 0.62 / 16.1 for CG), else the polynomial CG (C5, 7K rows per CTA: the generic
        // Chebyshev path streams the ELL from HBM every step, 148 vs 122 ms per fp64 frame)
        solver_auto = c->solver == VKPD_SOLVER_AUTO;
        solver_kind = solver_auto ? VKPD_SOLVER_CHEBYSHEV : c->solver;
        if (solver_kind < VKPD_SOLVER_PCG_POLY || solver_kind > VKPD_SOLVER_PCG_JACOBI)
            return fail(VKPD_EINVAL, "unknown solver kind");
        pcg_poly = solver_kind == VKPD_SOLVER_PCG_POLY;
        cheb = solver_kind == VKPD_SOLVER_CHEBYSHEV && nE > 0;     // PD residual form only
        CK(robust_res.alloc((size_t)16 * std::max(1, nE)));
        CK(robust_ok.alloc((size_t)4 * std::max(1, nE)));
        CK(robust_arrivals.alloc((size_t)std::max(1, cdiv(nE, 32))));
        CK(cudaMemsetAsync(robust_arrivals.p, 0, sizeof(int) * std::max(1, cdiv(nE, 32)), stream));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&robust_task_blocks, vk::k_robust_tasks<T, vk::MODE_RESID>,
                                                         128, 0));
        robust_task_blocks = std::max(1, robust_task_blocks);
        int occ = 0, occ2 = 0, occ3 = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, vk::k_pcg_classic<T>, pcg_threads, 0));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ3, vk::k_pcg_poly<T>, pcg_threads, 0));
        // co-residency of every kernel that may be launched on this grid
        occ = std::min(occ2, occ3);
        if (cheb) {
            int o5 = 0;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o5, vk::k_cheb<T>, pcg_threads, 0));
            occ = std::min(occ, o5);
        }
        if (occ < 1) return fail(VKPD_ECUDA, "persistent solver kernel cannot be resident");
        pcg_blocks = std::max(1, std::min(pcg_blocks, occ * n_sms));
        CK(partials.alloc((size_t)16 * pcg_blocks));   // 2 parity banks x 8 doubles/CTA
        if (int rc = refresh_precond()) return rc;
        CK(scal.alloc(16));
        CK(bar.alloc(1));
        CK(cudaMemsetAsync(bar.p, 0, sizeof(vk::GridBar), s));
        CK(iters.alloc(1024));
        CK(cudaMemsetAsync(iters.p, 0, 1024 * sizeof(int), s));
        CK(fail_iter.alloc(1));
        CK(robust_list.alloc(std::max(1, nE)));
        CK(robust_aux.alloc((size_t)24 * std::max(1, nE)));
        CK(robust_count.alloc(3));   // [0] queued elements, [1] task cursor, [2] last pass's count
        CK(pd_it.alloc(1));
        if (c->warm_rounds >= 0) warm_rounds = std::min(32, c->warm_rounds);
        if (solver_kind == VKPD_SOLVER_PCG_JACOBI) warm_rounds = 0;
        warm_start = warm_rounds > 0;
        CK(warm0.alloc((size_t)std::max(1, warm_rounds) * std::max(1, nF)));
        CK(cudaMemsetAsync(warm0.p, 0, (size_t)std::max(1, warm_rounds) * std::max(1, nF) * sizeof(V4), s));
        unroll_cfg = c->unroll_rounds >= 0 ? std::min(64, c->unroll_rounds) : -1;
        unroll_rounds = unroll_cfg > 0 ? unroll_cfg : 0;
        pd_early_exit = c->pd_early_exit != 0;
        // per-round tolerance schedule: earlier PD rounds' solve errors are contracted by the later
        // rounds, so round k of R solves to tol * g^(R-1-k).  Default g = 1.15 in float64 (C2 after
        // 100 frames: 1.1e-11 vs the reference, bar 1e-10; C3 9.0 -> 7.9 ms/frame,
        // profiles/r02_tol_growth.json); float32 keeps g = 1 (its zero-work exit needs one tolerance)
        tol_growth = c->tol_growth > 1.0 ? c->tol_growth
                   : c->tol_growth < 0.0 ? (sizeof(T) == 8 ? 1.15 : 1.0) : 1.0;
        if (warm_extrap) {
            CK(warm1.alloc((size_t)std::max(1, warm_rounds) * std::max(1, nF)));
            CK(cudaMemsetAsync(warm1.p, 0, (size_t)std::max(1, warm_rounds) * std::max(1, nF) * sizeof(V4), s));
            CK(warm_ctr.alloc(1));
            CK(cudaMemsetAsync(warm_ctr.p, 0, sizeof(unsigned), s));
            if (warm_order == 2) {
                CK(warm2.alloc((size_t)std::max(1, warm_rounds) * std::max(1, nF)));
                CK(cudaMemsetAsync(warm2.p, 0, (size_t)std::max(1, warm_rounds) * std::max(1, nF) * sizeof(V4), s));
                CK(warm3.alloc((size_t)std::max(1, warm_rounds) * std::max(1, nF)));
                CK(cudaMemsetAsync(warm3.p, 0, (size_t)std::max(1, warm_rounds) * std::max(1, nF) * sizeof(V4), s));
            }
        }
        CK(cudaMemsetAsync(robust_count.p, 0, 3 * sizeof(int), s));
        CK(pstats.alloc(1));
        CK(cudaMemsetAsync(pstats.p, 0, sizeof(vk::ProjStats), s));
        CK(stage.alloc((size_t)3 * n));
        CK(cudaHostAlloc(&h_fail, sizeof(int), cudaHostAllocDefault));
        *h_fail = 0x7fffffff;
        CK(cudaHostAlloc(&h_stop, sizeof(int), cudaHostAllocDefault));
        *h_stop = 0;
        CK(first_stop.alloc(1));
        CK(cudaStreamSynchronize(s));
        return VKPD_OK;
    }


    // Matrix-only context (GlobalSolver drop-in, pdsolver.py:205-223): K given as CSR.
    int init_matrix(int64_t nn, const int64_t* indptr, const int64_t* indices, const double* data,
                    const int64_t* pins, int64_t npins, const vkpd_config* c) override {
        n = (int)nn;
        nE = 0;
        nP = (int)npins;
        dt = 1.0;
        tol = c->tol > 0 ? c->tol : (sizeof(T) == 4 ? 2e-6 : 1e-12);
        max_iters = c->max_iters > 0 ? c->max_iters : 1000;
        use_graph = false;
        if (n <= 0) return fail(VKPD_EINVAL, "empty matrix");
        std::vector<int> ioo(n, -1);
        std::vector<char> pinned(n, 0);
        for (int k = 0; k < nP; ++k) {
            if (pins[k] < 0 || pins[k] >= n) return fail(VKPD_EINVAL, "pin index out of range");
            if (pinned[pins[k]]) return fail(VKPD_EINVAL, "duplicate pin index");
            pinned[pins[k]] = 1;
        }
        nF = 0;
        for (int j = 0; j < n; ++j) if (!pinned[j]) ioo[j] = nF++;
        for (int k = 0; k < nP; ++k) ioo[pins[k]] = nF + k;
        int_of_orig_h = ioo;
        set_free_perm();
        std::vector<int> orig_of_int(n);
        for (int j = 0; j < n; ++j) orig_of_int[ioo[j]] = j;
        ell_w = 0;
        std::vector<int> fptr(nF + 1, 0), fcol;
        std::vector<T> fval;
        std::vector<double> dg(nF, 0.0);
        std::vector<std::vector<std::pair<int, double>>> rows(nF);
        for (int i = 0; i < nF; ++i) {
            const int j = orig_of_int[i];
            for (int64_t k = indptr[j]; k < indptr[j + 1]; ++k) {
                const int64_t cj = indices[k];
                if (cj < 0 || cj >= n) return fail(VKPD_EINVAL, "matrix column out of range");
                const int ci = ioo[cj];
                if (ci < nF) rows[i].push_back({ci, data[k]});
                else { fcol.push_back(ci - nF); fval.push_back((T)data[k]); }
                if (ci == i) dg[i] += data[k];
            }
            std::sort(rows[i].begin(), rows[i].end());
            fptr[i + 1] = (int)fcol.size();
            ell_w = std::max(ell_w, (int)rows[i].size());
            if (!(dg[i] > 0.0)) return fail(VKPD_EINVAL, "matrix diagonal must be positive");
        }
        std::vector<int> ecol((size_t)ell_w * nF), elen(nF);
        std::vector<T> evals((size_t)ell_w * nF, T(0)), idg(nF);
        for (int i = 0; i < nF; ++i) {
            for (size_t s2 = 0; s2 < (size_t)ell_w; ++s2) {
                const bool real = s2 < rows[i].size();
                ecol[s2 * nF + i] = real ? rows[i][s2].first : i;
                evals[s2 * nF + i] = real ? (T)rows[i][s2].second : T(0);
            }
            elen[i] = (int)rows[i].size();
            idg[i] = (T)(1.0 / dg[i]);
        }
        CK(cudaSetDevice(device));
        CK(cudaDeviceGetAttribute(&n_sms, cudaDevAttrMultiProcessorCount, device));
        CK(cudaStreamCreateWithFlags(&own_stream, cudaStreamNonBlocking));
        stream = own_stream;
        cudaStream_t s = stream;
        CK(int_of_orig.alloc(n)); CK(int_of_orig.upload(ioo.data(), n, s));
        CK(ell_col.alloc(ecol.size())); CK(ell_col.upload(ecol.data(), ecol.size(), s));
        CK(ell_val.alloc(evals.size())); CK(ell_val.upload(evals.data(), evals.size(), s));
        CK(ell_len.alloc(nF)); CK(ell_len.upload(elen.data(), nF, s));
        CK(fp_ptr.alloc(nF + 1)); CK(fp_ptr.upload(fptr.data(), nF + 1, s));
        CK(fp_col.alloc(std::max<size_t>(1, fcol.size())));
        CK(fp_val.alloc(std::max<size_t>(1, fcol.size())));
        if (!fcol.empty()) { CK(fp_col.upload(fcol.data(), fcol.size(), s)); CK(fp_val.upload(fval.data(), fval.size(), s)); }
        CK(inv_diag.alloc(nF)); CK(inv_diag.upload(idg.data(), nF, s));
        CK(diag64.alloc(nF)); CK(diag64.upload(dg.data(), nF, s));
        CK(m_dt2.alloc(n));
        CK(dt2_inv_m.alloc(n));
        CK(inc_ptr.alloc(n + 1));
        CK(cudaMemsetAsync(inc_ptr.p, 0, (n + 1) * sizeof(int), s));
        return alloc_work(c);
    }

    // K in CSR, caller node order, rows of free nodes only (all rows when there are no pins)
    int get_csr(int64_t* indptr, int64_t* indices, double* data, int64_t* nnz) override {
        std::vector<int> ecol((size_t)ell_w * nF), fptr(nF + 1), fcol(fp_col.n);
        std::vector<T> evals((size_t)ell_w * nF), fval(fp_val.n);
        CK(cudaStreamSynchronize(stream));
        std::vector<int> elen(nF);
        if (nF) {
            CK(cudaMemcpy(elen.data(), ell_len.p, nF * sizeof(int), cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(ecol.data(), ell_col.p, ecol.size() * sizeof(int), cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(evals.data(), ell_val.p, evals.size() * sizeof(T), cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(fptr.data(), fp_ptr.p, fptr.size() * sizeof(int), cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(fcol.data(), fp_col.p, fcol.size() * sizeof(int), cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(fval.data(), fp_val.p, fval.size() * sizeof(T), cudaMemcpyDeviceToHost));
        }
        std::vector<int> orig_of_int(n);
        for (int j = 0; j < n; ++j) orig_of_int[int_of_orig_h[j]] = j;
        // count
        int64_t total = 0;
        std::vector<std::vector<std::pair<int64_t, double>>> rows(n);
        for (int i = 0; i < nF; ++i) {
            auto& r = rows[orig_of_int[i]];
            for (int s2 = 0; s2 < elen[i]; ++s2) {
                const int col = ecol[(size_t)s2 * nF + i];
                r.push_back({orig_of_int[col], (double)evals[(size_t)s2 * nF + i]});
            }
            for (int k = fptr[i]; k < fptr[i + 1]; ++k) r.push_back({orig_of_int[nF + fcol[k]], (double)fval[k]});
            std::sort(r.begin(), r.end());
            total += (int64_t)r.size();
        }
        *nnz = total;
        if (!indptr) return VKPD_OK;     // size query
        int64_t pos = 0;
        indptr[0] = 0;
        for (int j = 0; j < n; ++j) {
            for (auto& kv : rows[j]) { indices[pos] = kv.first; data[pos] = kv.second; ++pos; }
            indptr[j + 1] = pos;
        }
        return VKPD_OK;
    }

    int upload_nodes(const double* h, V4* dst) {
        CK(cudaMemcpyAsync(stage.p, h, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, stream));
        k_scatter_in<T><<<cdiv(n, 256), 256, 0, stream>>>(n, stage.p, int_of_orig.p, dst);
        CK(cudaGetLastError());
        return VKPD_OK;
    }
    int download_nodes(const V4* src, double* h) {
        k_gather_out<T><<<cdiv(n, 256), 256, 0, stream>>>(n, src, int_of_orig.p, stage.p);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(h, stage.p, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        return VKPD_OK;
    }

    DBuf<int> state_changed;
    // x, v (caller order, float64) from host (dev = false) or device memory (dev = true, on the
    // context stream, no host synchronisation).  A state other than the one the context holds
    // starts a new trajectory: the warm-start banks are cleared (results depend on the state
    // only); the state it handed out last keeps them.
    int set_state_any(const double* sx, const double* sv, bool dev) {
        if (!state_changed.p) CK(state_changed.alloc(1));
        CK(cudaMemsetAsync(state_changed.p, 0, sizeof(int), stream));
        const double* px = sx;
        const double* pv = sv;
        if (!dev) {
            CK(cudaMemcpyAsync(stage.p, sx, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, stream));
            px = stage.p;
        }
        k_state_in<T><<<cdiv(n, 256), 256, 0, stream>>>(n, px, int_of_orig.p, x.p, state_changed.p);
        CK(cudaGetLastError());
        if (!dev && sv) {
            CK(cudaMemcpyAsync(stage.p, sv, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, stream));
            pv = stage.p;
        }
        k_state_in<T><<<cdiv(n, 256), 256, 0, stream>>>(n, pv, int_of_orig.p, v.p, state_changed.p);
        CK(cudaGetLastError());
        for (DBuf<V4>* b : {&warm0, &warm1, &warm2, &warm3})
            if (b->p) k_zero_if<T><<<2 * n_sms, 256, 0, stream>>>(b->n, b->p, state_changed.p);
        CK(cudaGetLastError());
        if (!dev) CK(cudaStreamSynchronize(stream));
        return VKPD_OK;
    }
    int set_state(const double* hx, const double* hv) override { return set_state_any(hx, hv, false); }
    int set_state_dev(const void* dx, const void* dv) override {
        return set_state_any((const double*)dx, (const double*)dv, true);
    }
    int get_state_dev(void* dx, void* dv) override {
        if (dx) k_gather_out<T><<<cdiv(n, 256), 256, 0, stream>>>(n, x.p, int_of_orig.p, (double*)dx);
        if (dv) k_gather_out<T><<<cdiv(n, 256), 256, 0, stream>>>(n, v.p, int_of_orig.p, (double*)dv);
        CK(cudaGetLastError());
        return VKPD_OK;
    }
    int set_forces_dev(const void* df) override {
        if (df == nullptr) { has_forces = false; return VKPD_OK; }
        has_forces = true;
        k_scatter_in<T><<<cdiv(n, 256), 256, 0, stream>>>(n, (const double*)df, int_of_orig.p, f.p);
        CK(cudaGetLastError());
        return VKPD_OK;
    }
    int set_pin_targets_dev(const void* dt_) override {
        if (nP == 0) return VKPD_OK;
        k_rows_in<T><<<cdiv(nP, 256), 256, 0, stream>>>(nP, (const double*)dt_, pin_tgt.p);
        CK(cudaGetLastError());
        return VKPD_OK;
    }
    int get_state(double* hx, double* hv) override {
        if (hx) { int rc = download_nodes(x.p, hx); if (rc) return rc; }
        if (hv) { int rc = download_nodes(v.p, hv); if (rc) return rc; }
        return VKPD_OK;
    }
    int set_pin_targets(const double* t) override {
        if (nP == 0) return VKPD_OK;
        CK(cudaMemcpyAsync(stage.p, t, sizeof(double) * 3 * nP, cudaMemcpyHostToDevice, stream));
        k_rows_in<T><<<cdiv(nP, 256), 256, 0, stream>>>(nP, stage.p, pin_tgt.p);
        CK(cudaGetLastError());
        return VKPD_OK;
    }
    int set_colliders(int nc, const int* kinds, const double* params, double kc) override {
        if (nc < 0 || nc > vk::kMaxColliders) return fail(VKPD_EINVAL, "at most 16 colliders");
        std::vector<double> h((size_t)vk::kCollStride * std::max(1, nc), 0.0);
        for (int c = 0; c < nc; ++c) {
            const double* p = params + 6 * c;
            double* q = h.data() + vk::kCollStride * c;
            if (kinds[c] == 0) {                      // plane: point, normal (normalised here)
                const double nn = std::sqrt(p[3] * p[3] + p[4] * p[4] + p[5] * p[5]);
                if (!(nn > 0.0)) return fail(VKPD_EINVAL, "plane normal must be non-zero");
                q[0] = 0.0; q[1] = p[0]; q[2] = p[1]; q[3] = p[2];
                q[4] = p[3] / nn; q[5] = p[4] / nn; q[6] = p[5] / nn;
            } else if (kinds[c] == 1) {               // sphere: centre, radius
                q[0] = 1.0; q[1] = p[0]; q[2] = p[1]; q[3] = p[2]; q[4] = p[3];
            } else {
                return fail(VKPD_EINVAL, "unknown collider kind");
            }
        }
        if (!coll_d.p) {
            CK(coll_d.alloc((size_t)vk::kCollStride * vk::kMaxColliders));
            CK(inv_diag_c.alloc(std::max(1, nF)));
            CK(cdiag.alloc(std::max(1, nF)));
            CK(cb.alloc(std::max(1, nF)));
        }
        if (nc > 0) CK(cudaMemcpyAsync(coll_d.p, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice, stream));
        CK(cudaStreamSynchronize(stream));
        ncoll = nc;
        contact_k = kc;
        return VKPD_OK;
    }
    int set_forces(const double* hf) override {
        if (hf == nullptr) { has_forces = false; return VKPD_OK; }
        has_forces = true;
        return upload_nodes(hf, f.p);
    }

    vk::LocalArgs<T> local_args(const V4* xin, bool wred = false) {
        vk::LocalArgs<T> la;
        la.wr_ptr = wred ? wr_ptr.p : nullptr; la.wr_slot = wr_slot.p; la.wr_beg = wr_beg.p;
        la.wr_code = wr_code.p; la.wpart = wred ? wpart.p : nullptr; la.robust_flag = robust_flag.p;
        la.nE = nE; la.tets = tets.p; la.G = G.p; la.w = w.p; la.x = xin; la.corner = corner.p;
        la.slot4 = slot4.p;
        la.stats = pstats.p; la.F_out = la.R_out = la.V_out = nullptr;
        la.robust_list = robust_list.p; la.robust_count = robust_count.p;
        la.robust_aux = robust_aux.p;
        la.robust_if = 0;
        return la;
    }
    // local step in residual form, suspicious elements compacted into a dense second pass
    // reset = false inside a frame: the previous PD iteration's solver kernel zeroed the queue
    int launch_local_resid(const vk::LocalArgs<T>& la, bool reset = true) {
        if (reset) CK(cudaMemsetAsync(robust_count.p, 0, 2 * sizeof(int), stream));
        if (la.wpart != nullptr) vk::k_local_wred<T><<<cdiv(nE, 128), 128, 0, stream>>>(la);
        else vk::k_local<T, vk::MODE_RESID, false, 1><<<cdiv(nE, 128), 128, 0, stream>>>(la);
        CK(cudaGetLastError());
        // one resident wave of (chunk, start) tasks: cheap when the queue is empty
        vk::k_robust_tasks<T, vk::MODE_RESID><<<robust_task_blocks * n_sms, 128, 0, stream>>>(
            la, robust_res.p, robust_ok.p, robust_arrivals.p, std::max(1, nE));
        CK(cudaGetLastError());
        return VKPD_OK;
    }
    vk::PcgArgs<T> pcg_args(int init, int pd_iter, int* iters_slot) {
        vk::PcgArgs<T> pa;
        pa.nF = nF; pa.ell_w = ell_w; pa.ell_col = ell_col.p; pa.ell_val = ell_val.p; pa.inv_diag = inv_diag.p;
        pa.inc_ptr = inc_ptr.p; pa.inc_code = inc_code.p; pa.corner = corner.p; pa.m_dt2 = m_dt2.p;
        pa.part_ptr = nullptr; pa.wpart = wpart.p; pa.robust_flag = robust_flag.p;
        pa.robust_present = robust_count.p + 2;
        pa.xhat = xhat.p; pa.rhs = rhs.p; pa.x = x.p; pa.r = r.p; pa.z = z.p; pa.p0 = p0.p; pa.p1 = p1.p;
        pa.q = q.p; pa.dx = dx.p; pa.partials = partials.p; pa.scal = scal.p; pa.bar = bar.p;
        pa.iters_out = iters_slot; pa.fail_iter = fail_iter.p; pa.pd_iter = pd_iter; pa.tol = tol;
        pa.max_iters = max_iters; pa.init = init;
        pa.tol_growth = tol_growth; pa.rounds_total = last_iterations;
        pa.cdiag = nullptr; pa.cb = nullptr; pa.coll = nullptr; pa.ncoll = 0;
        pa.reset_count = nullptr;
        pa.pd_iter_dev = nullptr; pa.loop_handle = 0; pa.loop_iterations = 0; pa.robust_if = 0;
        pa.first_stop = nullptr;
        pa.rounds = init == vk::INIT_PD ? &pstats.p->pd_rounds : nullptr;
        pa.warm = (init == vk::INIT_PD && (pcg_poly || cheb) && warm_start) ? warm0.p : nullptr;
        pa.warm_rounds = warm_rounds;
        pa.warm_prev = (pa.warm != nullptr && warm_extrap) ? warm1.p : nullptr;
        pa.warm_beta = warm_beta;
        pa.warm_prev2 = (pa.warm_prev != nullptr && cheb) ? warm2.p : nullptr;
        pa.warm_prev3 = pa.warm_prev2 != nullptr ? warm3.p : nullptr;
        pa.warm_ring = (pa.warm_prev3 != nullptr && cheb_reg && warm_extrap_rounds >= warm_rounds) ? warm_ctr.p
                                                                                                  : nullptr;
        pa.warm_extrap_rounds = warm_extrap_rounds;
        pa.poly_rounds = 0;
        pa.flags = cheb_flags.p; pa.cheb_nbr_ptr = cheb_nbr_ptr.p; pa.cheb_nbr = cheb_nbr.p;
        pa.cheb_ll = cheb_ll.p;
        pa.cheb_lmin = lam_min; pa.cheb_lmax = gersh;
        pa.cheb_slot = cheb_slot.p; pa.cheb_val = cheb_val.p; pa.cheb_kdiag = cheb_kdiag.p;
        pa.cheb_nexp = cheb_nexp.p;
        pa.cheb_halo_ptr = cheb_halo_ptr.p; pa.cheb_halo = cheb_halo.p;
        pa.cheb_halo_max = cheb_halo_max;
        pa.h = hh.p; pa.omega = poly_omega; pa.ell_kd = ell_kd.p;
        if (init == vk::INIT_PD && ncoll > 0) {
            pa.inv_diag = inv_diag_c.p; pa.cdiag = cdiag.p; pa.cb = cb.p; pa.coll = coll_d.p; pa.ncoll = ncoll;
            pa.ell_kd = nullptr;                  // D changes with the contact set: scale on the fly
        }
        return pa;
    }
    cudaError_t launch_pcg(const vk::PcgArgs<T>& pa) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(pcg_blocks);
        cfg.blockDim = dim3(pcg_threads);
        cfg.dynamicSmemBytes = 0;
        cfg.stream = stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeCooperative;
        attr[0].val.cooperative = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (cheb && pa.init == vk::INIT_PD) {
            if (!cheb_reg) return cudaLaunchKernelEx(&cfg, vk::k_cheb<T>, pa);
            cfg.dynamicSmemBytes = cheb_smem_bytes();
            return cudaLaunchKernelEx(&cfg, vk::k_cheb_reg<T>, pa);
        }
        if (pcg_poly) return cudaLaunchKernelEx(&cfg, vk::k_pcg_poly<T>, pa);
        return cudaLaunchKernelEx(&cfg, vk::k_pcg_classic<T>, pa);
    }

    // enqueue one frame on `stream`; events (optional) bracket local / global launches
    int enqueue_frame(int iterations, double damping, std::vector<cudaEvent_t>* ev) {
        const int nb = cdiv(n, 256);
        vk::k_prologue<T><<<nb, 256, 0, stream>>>(n, nF, (T)dt, dt2_inv_m.p, has_forces ? f.p : nullptr,
                                                  pin_tgt.p, x.p, v.p, x_start.p, v_start.p, xhat.p,
                                                  fail_iter.p, nullptr, nullptr, warm_ctr.p);
        CK(cudaGetLastError());
        if (ncoll > 0 && nF > 0) {
            vk::k_contact_setup<T><<<cdiv(nF, 256), 256, 0, stream>>>(nF, xhat.p, diag64.p, coll_d.p, ncoll,
                                                                      contact_k, inv_diag_c.p, cdiag.p, cb.p);
            CK(cudaGetLastError());
        }
        const vk::LocalArgs<T> la = local_args(x.p, true);
        cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
        CK(cudaStreamIsCapturing(stream, &cap));
        const bool host_exit = pd_early_exit && nF > 0 && cap == cudaStreamCaptureStatusNone;
        last_exec_rounds = iterations;
        for (int it = 0; it < iterations; ++it) {
            if (ev) CK(cudaEventRecord((*ev)[3 * it], stream));
            if (int rc = launch_local_resid(la, it == 0 || nF == 0)) return rc;
            if (ev) CK(cudaEventRecord((*ev)[3 * it + 1], stream));
            if (nF > 0) {
                vk::PcgArgs<T> pa = pcg_args(vk::INIT_PD, it, iters.p + it);
                pa.reset_count = robust_count.p;      // zero the suspicious-tet queue for the next local step
                pa.part_ptr = part_ptr.p;             // the local step's node partials
                CK(launch_pcg(pa));
            }
            if (ev) CK(cudaEventRecord((*ev)[3 * it + 2], stream));
            if (host_exit && it + 1 < iterations) {
                // same early exit as the graph's loop node, decided on the host (direct launches)
                int cgi = -1;
                CK(cudaMemcpyAsync(&cgi, iters.p + it, sizeof(int), cudaMemcpyDeviceToHost, stream));
                CK(cudaStreamSynchronize(stream));
                if (cgi == 0 && !(it < warm_rounds && warm_start && (pcg_poly || cheb))) {   // a warm round moves x
                    CK(cudaMemsetAsync(iters.p + it + 1, 0, sizeof(int) * (iterations - it - 1), stream));
                    last_exec_rounds = it + 1;
                    break;
                }
            }
        }
        vk::k_epilogue<T><<<nb, 256, 0, stream>>>(n, (T)(damping / dt), x.p, x_start.p, v.p);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(h_fail, fail_iter.p, sizeof(int), cudaMemcpyDeviceToHost, stream));
        return VKPD_OK;
    }

    // One frame for graph capture with the PD iterations in a conditional WHILE node:
    // body = local step, robust pass, solver (which sets the loop condition).  The body stops after
    // `iterations` rounds, on a non-finite solve, or as soon as a solve needs zero CG
    // iterations (x unchanged: the remaining rounds would be exact repeats).
    int enqueue_frame_loop(int iterations, double damping) {
        const int nb = cdiv(n, 256);
        vk::k_prologue<T><<<nb, 256, 0, stream>>>(n, nF, (T)dt, dt2_inv_m.p, has_forces ? f.p : nullptr,
                                                  pin_tgt.p, x.p, v.p, x_start.p, v_start.p, xhat.p,
                                                  fail_iter.p, robust_count.p, pd_it.p, warm_ctr.p);
        CK(cudaGetLastError());
        if (ncoll > 0) {
            vk::k_contact_setup<T><<<cdiv(nF, 256), 256, 0, stream>>>(nF, xhat.p, diag64.p, coll_d.p, ncoll,
                                                                      contact_k, inv_diag_c.p, cdiag.p, cb.p);
            CK(cudaGetLastError());
        }
        CK(cudaMemsetAsync(first_stop.p, 0x7f, sizeof(int), stream));      // 0x7f7f7f7f: no stop yet
        // conditional node after the captured prologue
        cudaStreamCaptureStatus st;
        cudaGraph_t g = nullptr;
        const cudaGraphNode_t* deps = nullptr;
        size_t ndeps = 0;
        CK(cudaStreamGetCaptureInfo(stream, &st, nullptr, &g, &deps, &ndeps));
        cudaGraphConditionalHandle h;
        CK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
        // the first `unroll_rounds` rounds as plain graph nodes (no conditional-node overhead);
        // their solves set the loop handle like the loop body's, and a round run after the exit
        // point is an exact repeat (x unchanged), so the frame's result is the same
        const int nun = std::min(unroll_rounds, iterations);
        for (int it = 0; it < nun; ++it) {
            const vk::LocalArgs<T> la = local_args(x.p, true);
            if (int rc = launch_local_resid(la, false)) return rc;
            vk::PcgArgs<T> pa = pcg_args(vk::INIT_PD, 0, iters.p);
            pa.reset_count = robust_count.p;
                pa.part_ptr = part_ptr.p;             // the local step's node partials
            pa.pd_iter_dev = pd_it.p;
            pa.loop_handle = (unsigned long long)h;
            pa.loop_iterations = iterations;
            pa.first_stop = first_stop.p;
            CK(launch_pcg(pa));
        }
        CK(cudaStreamGetCaptureInfo(stream, &st, nullptr, &g, &deps, &ndeps));
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t cnode;
        CK(cudaGraphAddNode(&cnode, g, deps, ndeps, &cp));
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        if (!body_stream) CK(cudaStreamCreateWithFlags(&body_stream, cudaStreamNonBlocking));
        CK(cudaStreamBeginCaptureToGraph(body_stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
        cudaStream_t outer = stream;
        stream = body_stream;
        int rc = VKPD_OK;
        {
            const vk::LocalArgs<T> la = local_args(x.p, true);
            rc = launch_local_resid(la, false);
            if (rc == VKPD_OK) {
                vk::PcgArgs<T> pa = pcg_args(vk::INIT_PD, 0, iters.p);
                pa.reset_count = robust_count.p;
                pa.part_ptr = part_ptr.p;             // the local step's node partials
                pa.pd_iter_dev = pd_it.p;
                pa.first_stop = first_stop.p;
                pa.loop_handle = (unsigned long long)h;
                pa.loop_iterations = iterations;
                cudaError_t e = launch_pcg(pa);
                if (e != cudaSuccess) rc = fail(VKPD_ECUDA, cudaGetErrorString(e));
            }
        }
        stream = outer;
        cudaGraph_t body_out = nullptr;
        cudaError_t e = cudaStreamEndCapture(body_stream, &body_out);
        if (rc) return rc;
        CK(e);
        CK(cudaStreamUpdateCaptureDependencies(stream, &cnode, 1, cudaStreamSetCaptureDependencies));
        vk::k_epilogue<T><<<nb, 256, 0, stream>>>(n, (T)(damping / dt), x.p, x_start.p, v.p);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(h_fail, fail_iter.p, sizeof(int), cudaMemcpyDeviceToHost, stream));
        CK(cudaMemcpyAsync(h_stop, first_stop.p, sizeof(int), cudaMemcpyDeviceToHost, stream));
        return VKPD_OK;
    }

    // Adaptive unrolling: the rounds a recent frame needed (its first round that met the exit
    // condition, read from pinned memory the graph writes; no synchronization) are sampled at
    // every launch; the unrolled count becomes the minimum of the last 32 samples (after 8
    // samples, then every 64), so unrolled rounds are almost never past the exit point (and when
    // they are, they are exact repeats).
    void adapt_unroll(int iterations) {
        if (unroll_cfg >= 0 || !pd_early_exit) return;
        const int need = *(volatile int*)h_stop;
        if (need <= 0) return;                                   // no frame finished yet
        stop_hist[stop_pos] = std::min(need, iterations);        // 0x7f7f7f7f: every round ran
        stop_pos = (stop_pos + 1) % 32;
        stop_fill = std::min(32, stop_fill + 1);
        ++stop_n;
        // first decision after 8 samples, then every 64 (a re-capture costs ~0.3 ms of host time)
        if (!(stop_n == 8 || (stop_n > 8 && (stop_n - 8) % 64 == 0))) return;
        int m = iterations;
        for (int k = 0; k < stop_fill; ++k) m = std::min(m, stop_hist[k]);
        unroll_rounds = m;
    }

    int build_graph(int iterations, double damping) {
        if (graph_exec) { cudaGraphExecDestroy(graph_exec); graph_exec = nullptr; }
        cudaGraph_t g = nullptr;
        CK(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
        const bool loop = pd_early_exit && iterations >= 2 && nF > 0;
        int rc = loop ? enqueue_frame_loop(iterations, damping) : enqueue_frame(iterations, damping, nullptr);
        cudaError_t e = cudaStreamEndCapture(stream, &g);
        if (rc != VKPD_OK || e != cudaSuccess) {
            if (g) cudaGraphDestroy(g);
            cudaGetLastError();
            if (loop) { pd_early_exit = false; return build_graph(iterations, damping); }   // plain unrolled frame
            graph_broken = true;
            return VKPD_OK;     // fall back to direct launches
        }
        e = cudaGraphInstantiate(&graph_exec, g, 0);
        cudaGraphDestroy(g);
        if (e != cudaSuccess) {
            cudaGetLastError();
            graph_exec = nullptr;
            if (loop) { pd_early_exit = false; return build_graph(iterations, damping); }
            graph_broken = true;
            return VKPD_OK;
        }
        graph_iters = iterations;
        graph_unroll = unroll_rounds;
        graph_damp = damping;
        graph_forces = has_forces;
        graph_ncoll = ncoll;
        return VKPD_OK;
    }

    int step_async(int iterations, double damping) override {
        if (iterations < 0 || iterations > 1024) return fail(VKPD_EINVAL, "iterations must be in [0, 1024]");
        last_iterations = iterations;
        if (use_graph && !graph_broken) {
            if (graph_exec && graph_iters == iterations) adapt_unroll(iterations);
            if (!graph_exec || graph_iters != iterations || graph_damp != damping || graph_forces != has_forces ||
                graph_ncoll != ncoll || graph_unroll != unroll_rounds) {
                int rc = build_graph(iterations, damping);
                if (rc) return rc;
            }
            if (graph_exec) {
                CK(cudaGraphLaunch(graph_exec, stream));
                return VKPD_OK;
            }
        }
        return enqueue_frame(iterations, damping, nullptr);
    }

    // simulate_mesh's frame loop (pdsolver.py:744-762) pipelined: per-step inputs go up and each
    // frame's positions come down on a copy stream through double-buffered pinned / device staging,
    // overlapping the next frame's compute; the host copies into `frames` while the GPU runs.
    // Failures are recorded per frame and reported for the first failing frame after the loop.
    cudaStream_t copy_stream = nullptr;     // device -> host (positions)
    cudaStream_t in_stream = nullptr;       // host -> device (per-step inputs); separate so an upload
                                            // never queues behind the previous frame's download
    DBuf<double> sim_din, sim_dout;
    double* sim_hin = nullptr;
    double* sim_hout = nullptr;
    size_t sim_cap = 0;
    // positions out: up to kOutSlots staging slots (<= 64 MB), so the host writer can fall a few
    // frames behind (fold frames are ~2x a steady frame) without stalling the enqueue loop
    static constexpr int kOutSlots = 8;
    int out_slots = 2;
    cudaEvent_t ev_h2d[2] = {nullptr, nullptr}, ev_scat[2] = {nullptr, nullptr}, ev_out[kOutSlots] = {},
                ev_d2h[kOutSlots] = {};
    DBuf<int> fail_hist;
    int simulate(int steps, int iterations, double damping, const double* forces, int forces_per_step,
                 const double* pin_path, double* frames, int* failed_frame, int* failed_iter) override {
        if (failed_frame) *failed_frame = -1;
        if (failed_iter) *failed_iter = -1;
        if (steps < 0 || !frames) return fail(VKPD_EINVAL, "bad simulate arguments");
        if (nE == 0) return fail(VKPD_EINVAL, "matrix-only context has no mesh");
        if (steps == 0) return VKPD_OK;
        const size_t n3 = (size_t)3 * n, p3 = (size_t)3 * nP;
        const size_t slot_in = n3 + p3;
        if (!copy_stream) {
            CK(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking));
            CK(cudaStreamCreateWithFlags(&in_stream, cudaStreamNonBlocking));
            for (int k = 0; k < 2; ++k) {
                CK(cudaEventCreateWithFlags(&ev_h2d[k], cudaEventDisableTiming));
                CK(cudaEventCreateWithFlags(&ev_scat[k], cudaEventDisableTiming));
            }
            for (int k = 0; k < kOutSlots; ++k) {
                CK(cudaEventCreateWithFlags(&ev_out[k], cudaEventDisableTiming));
                CK(cudaEventCreateWithFlags(&ev_d2h[k], cudaEventDisableTiming));
            }
        }
        if (sim_cap < slot_in) {
            if (sim_hin) cudaFreeHost(sim_hin);
            if (sim_hout) cudaFreeHost(sim_hout);
            sim_hin = sim_hout = nullptr;
            out_slots = (int)std::max<size_t>(2, std::min<size_t>(kOutSlots, (size_t(64) << 20) / (sizeof(double) * n3)));
            CK(cudaHostAlloc(&sim_hin, sizeof(double) * 2 * slot_in, cudaHostAllocDefault));
            CK(cudaHostAlloc(&sim_hout, sizeof(double) * out_slots * n3, cudaHostAllocDefault));
            CK(sim_din.alloc(2 * slot_in));
            CK(sim_dout.alloc((size_t)out_slots * n3));
            sim_cap = slot_in;
        }
        if (fail_hist.n < (size_t)steps) CK(fail_hist.alloc(steps));
        if (forces && !forces_per_step) { if (int rc = set_forces(forces)) return rc; }
        else if (!forces) has_forces = false;
        else has_forces = true;
        const bool up_f = forces && forces_per_step, up_p = pin_path && nP > 0;
        // positions are copied from pinned staging into `frames` by a helper thread, so writing
        // (and first-touching) the caller's array never delays enqueueing the next frame
        std::atomic<int> posted{-1}, copied{-1};
        std::atomic<bool> werr{false};
        std::thread writer([&] {
            cudaSetDevice(device);
            for (int j = 0; j < steps; ++j) {
                while (posted.load(std::memory_order_acquire) < j) std::this_thread::yield();
                const int so = j % out_slots;
                if (cudaEventSynchronize(ev_d2h[so]) != cudaSuccess) werr = true;
                std::memcpy(frames + (size_t)j * n3, sim_hout + so * n3, sizeof(double) * n3);
                copied.store(j, std::memory_order_release);
            }
        });
        int rc_loop = VKPD_OK;
        const bool up = up_f || up_p;
        // inputs of frame j: host staging slot j & 1 -> device slot j & 1 on in_stream
        auto upload = [&](int j) -> bool {
            const int sl = j & 1;
            if (j >= 2 && cudaEventSynchronize(ev_h2d[sl]) != cudaSuccess) return false;   // host slot free
            double* hin = sim_hin + sl * slot_in;
            if (up_f) std::memcpy(hin, forces + (size_t)j * n3, sizeof(double) * n3);
            if (up_p) std::memcpy(hin + n3, pin_path + (size_t)j * p3, sizeof(double) * p3);
            if (j >= 2) cudaStreamWaitEvent(in_stream, ev_scat[sl], 0);             // device slot consumed
            cudaMemcpyAsync(sim_din.p + sl * slot_in, hin, sizeof(double) * slot_in, cudaMemcpyHostToDevice,
                            in_stream);
            cudaEventRecord(ev_h2d[sl], in_stream);
            return true;
        };
        if (up) {
            if (!upload(0)) rc_loop = VKPD_ECUDA;
            cudaStreamWaitEvent(stream, ev_h2d[0], 0);
            k_sim_between<T><<<cdiv(std::max(n, nP), 256), 256, 0, stream>>>(
                n, nP, x.p, int_of_orig.p, nullptr, fail_iter.p, nullptr, up_f ? sim_din.p : nullptr, f.p,
                up_p ? sim_din.p + n3 : nullptr, pin_tgt.p);
            cudaEventRecord(ev_scat[0], stream);
        }
        for (int i = 0; i < steps && rc_loop == VKPD_OK; ++i) {
            const int sl = i % out_slots, nx = (i + 1) & 1;
            const bool next = up && i + 1 < steps;
            if (next && !upload(i + 1)) { rc_loop = VKPD_ECUDA; break; }          // overlaps frame i
            if ((rc_loop = step_async(iterations, damping)) != VKPD_OK) break;
            if (i >= out_slots) cudaStreamWaitEvent(stream, ev_d2h[sl], 0);      // device out slot free
            if (next) cudaStreamWaitEvent(stream, ev_h2d[nx], 0);
            k_sim_between<T><<<cdiv(std::max(n, nP), 256), 256, 0, stream>>>(
                n, nP, x.p, int_of_orig.p, sim_dout.p + sl * n3, fail_iter.p, fail_hist.p + i,
                (next && up_f) ? sim_din.p + nx * slot_in : nullptr, f.p,
                (next && up_p) ? sim_din.p + nx * slot_in + n3 : nullptr, pin_tgt.p);
            cudaEventRecord(ev_out[sl], stream);
            if (next) cudaEventRecord(ev_scat[nx], stream);
            cudaStreamWaitEvent(copy_stream, ev_out[sl], 0);
            // the pinned slot is reused by frame i: the writer must have copied frame i - out_slots out
            while (copied.load(std::memory_order_acquire) < i - out_slots) std::this_thread::yield();
            cudaMemcpyAsync(sim_hout + sl * n3, sim_dout.p + sl * n3, sizeof(double) * n3, cudaMemcpyDeviceToHost,
                            copy_stream);
            cudaEventRecord(ev_d2h[sl], copy_stream);
            posted.store(i, std::memory_order_release);
            if (cudaPeekAtLastError() != cudaSuccess) { rc_loop = VKPD_ECUDA; break; }
        }
        if (rc_loop != VKPD_OK) posted.store(steps, std::memory_order_release);   // let the writer drain
        // (on an early exit the writer may copy stale staging: frames are undefined after an error)
        writer.join();
        if (rc_loop != VKPD_OK) return rc_loop == VKPD_ECUDA ? fail(VKPD_ECUDA, cudaGetErrorString(cudaGetLastError()))
                                                            : rc_loop;
        if (werr) return fail(VKPD_ECUDA, "device-to-host copy failed");
        std::vector<int> fh(steps);
        CK(cudaMemcpyAsync(fh.data(), fail_hist.p, sizeof(int) * steps, cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        *h_fail = 0x7fffffff;
        for (int i = 0; i < steps; ++i)
            if (fh[i] != 0x7fffffff) {
                if (failed_frame) *failed_frame = i;
                if (failed_iter) *failed_iter = fh[i];
                char buf[128];
                snprintf(buf, sizeof buf, "projective step produced non-finite positions at iteration %d", fh[i]);
                return fail(VKPD_ENONFINITE, buf);
            }
        return VKPD_OK;
    }

    int sync(int* failed) override {
        CK(cudaStreamSynchronize(stream));
        const int fi = *h_fail;
        if (failed) *failed = fi == 0x7fffffff ? -1 : fi;
        if (fi != 0x7fffffff) {
            vk::k_restore<T><<<cdiv(n, 256), 256, 0, stream>>>(n, x.p, v.p, x_start.p, v_start.p);
            CK(cudaGetLastError());
            CK(cudaStreamSynchronize(stream));
            *h_fail = 0x7fffffff;
            char buf[128];
            snprintf(buf, sizeof buf, "projective step produced non-finite positions at iteration %d", fi);
            return fail(VKPD_ENONFINITE, buf);
        }
        return VKPD_OK;
    }

    // back-to-back launches of the local step on the current state (measurement only), each
    // bracketed by its own events (all enqueued ahead, so no host gap falls inside a pair):
    // k_local alone, and k_local + the robust pass (the frame's local phase)
    int time_local(int reps, double* local_ms, double* pass_ms) override {
        if (nE == 0) return fail(VKPD_EINVAL, "matrix-only context has no mesh");
        if (reps < 1 || reps > 1000) return fail(VKPD_EINVAL, "reps must be in [1, 1000]");
        const vk::LocalArgs<T> la = local_args(x.p, true);      // the frame's (warp-reduced) pass
        std::vector<cudaEvent_t> e(4 * reps);
        for (auto& ev : e) CK(cudaEventCreate(&ev));
        for (int r = 0; r < reps; ++r) {
            CK(cudaMemsetAsync(robust_count.p, 0, 2 * sizeof(int), stream));
            CK(cudaEventRecord(e[4 * r], stream));
            vk::k_local_wred<T><<<cdiv(nE, 128), 128, 0, stream>>>(la);
            CK(cudaEventRecord(e[4 * r + 1], stream));
            CK(cudaMemsetAsync(robust_count.p, 0, 2 * sizeof(int), stream));
            CK(cudaEventRecord(e[4 * r + 2], stream));
            if (int rc = launch_local_resid(la, false)) return rc;
            CK(cudaEventRecord(e[4 * r + 3], stream));
        }
        CK(cudaStreamSynchronize(stream));
        CK(cudaGetLastError());
        double a = 0.0, b = 0.0;
        for (int r = 0; r < reps; ++r) {
            float t1 = 0.f, t2 = 0.f;
            CK(cudaEventElapsedTime(&t1, e[4 * r], e[4 * r + 1]));
            CK(cudaEventElapsedTime(&t2, e[4 * r + 2], e[4 * r + 3]));
            a += t1;
            b += t2;
        }
        for (auto& ev : e) cudaEventDestroy(ev);
        CK(cudaMemsetAsync(robust_count.p, 0, 3 * sizeof(int), stream));
        CK(cudaMemsetAsync(robust_flag.p, 0, robust_flag.n, stream));   // no gather consumed these passes
        CK(cudaStreamSynchronize(stream));
        if (local_ms) *local_ms = a / reps;
        if (pass_ms) *pass_ms = b / reps;
        return VKPD_OK;
    }
    int profile(int iterations, double damping, double* lms, double* gms, double* fms) override {
        std::vector<cudaEvent_t> ev(3 * iterations + 2);
        for (auto& e : ev) CK(cudaEventCreate(&e));
        CK(cudaEventRecord(ev[3 * iterations], stream));
        int rc = enqueue_frame(iterations, damping, &ev);
        CK(cudaEventRecord(ev[3 * iterations + 1], stream));
        CK(cudaStreamSynchronize(stream));
        double lsum = 0, gsum = 0;
        prof_local.assign(iterations, 0.0);
        prof_global.assign(iterations, 0.0);
        const int nex = rc ? 0 : std::min(iterations, last_exec_rounds);   // rounds actually launched
        for (int it = 0; it < nex; ++it) {
            float a = 0, b = 0;
            CK(cudaEventElapsedTime(&a, ev[3 * it], ev[3 * it + 1]));
            CK(cudaEventElapsedTime(&b, ev[3 * it + 1], ev[3 * it + 2]));
            lsum += a; gsum += b;
            prof_local[it] = a;
            prof_global[it] = b;
        }
        float fr = 0;
        CK(cudaEventElapsedTime(&fr, ev[3 * iterations], ev[3 * iterations + 1]));
        for (auto& e : ev) cudaEventDestroy(e);
        if (lms) *lms = nex ? lsum / nex : 0;
        if (gms) *gms = nex ? gsum / nex : 0;
        if (fms) *fms = fr;
        if (rc) return rc;
        int failed = -1;
        return sync(&failed);
    }

    int elastic_rhs(const double* hx, double* hrhs, double* F, double* R, double* Vv) override {
        int rc = upload_nodes(hx, tmp4a.p);
        if (rc) return rc;
        vk::LocalArgs<T> la = local_args(tmp4a.p);
        DBuf<double> dF, dR, dV;
        const bool frv = F || R || Vv;
        if (frv) {
            CK(dF.alloc((size_t)9 * nE)); CK(dR.alloc((size_t)9 * nE)); CK(dV.alloc((size_t)9 * nE));
            la.F_out = dF.p; la.R_out = dR.p; la.V_out = dV.p;
            vk::k_local<T, vk::MODE_RHS, true><<<cdiv(nE, 128), 128, 0, stream>>>(la);
        } else {
            vk::k_local<T, vk::MODE_RHS, false><<<cdiv(nE, 128), 128, 0, stream>>>(la);
        }
        CK(cudaGetLastError());
        vk::k_gather<T><<<cdiv(n, 256), 256, 0, stream>>>(n, inc_ptr.p, corner.p, tmp4b.p);
        CK(cudaGetLastError());
        rc = download_nodes(tmp4b.p, hrhs);
        if (rc) return rc;
        const size_t bytes = sizeof(double) * 9 * nE;
        if (F) CK(cudaMemcpy(F, dF.p, bytes, cudaMemcpyDeviceToHost));
        if (R) CK(cudaMemcpy(R, dR.p, bytes, cudaMemcpyDeviceToHost));
        if (Vv) CK(cudaMemcpy(Vv, dV.p, bytes, cudaMemcpyDeviceToHost));
        return VKPD_OK;
    }

    int global_solve(const double* B, const double* P, double* X, int k) override {
        if (k <= 0) return fail(VKPD_EINVAL, "need at least one right-hand side column");
        std::vector<double> b3((size_t)3 * n), p3((size_t)3 * std::max(1, nP)), x3((size_t)3 * n);
        int bad = 0;
        for (int c0 = 0; c0 < k; c0 += 3) {
            const int kc = std::min(3, k - c0);
            std::fill(b3.begin(), b3.end(), 0.0);
            std::fill(p3.begin(), p3.end(), 0.0);
            for (int j = 0; j < n; ++j)
                for (int c = 0; c < kc; ++c) b3[3 * (size_t)j + c] = B[(size_t)j * k + c0 + c];
            for (int j = 0; j < nP; ++j)
                for (int c = 0; c < kc; ++c) p3[3 * (size_t)j + c] = P[(size_t)j * k + c0 + c];
            int rc = upload_nodes(b3.data(), tmp4a.p);
            if (rc) return rc;
            if (nP) {
                CK(cudaMemcpyAsync(stage.p, p3.data(), sizeof(double) * 3 * nP, cudaMemcpyHostToDevice, stream));
                k_rows_in<T><<<cdiv(nP, 256), 256, 0, stream>>>(nP, stage.p, tmp4b.p);
                CK(cudaGetLastError());
            }
            if (nF > 0) {
                k_rhs_minus_fp<T><<<cdiv(nF, 256), 256, 0, stream>>>(nF, tmp4a.p, fp_ptr.p, fp_col.p, fp_val.p,
                                                                    tmp4b.p, rhs.p);
                CK(cudaGetLastError());
                CK(launch_pcg(pcg_args(vk::INIT_RHS, 0, iters.p + 1023)));
                // assemble internal vector [dx (free) ; P (pinned)] in tmp4a
                CK(cudaMemcpyAsync(tmp4a.p, dx.p, sizeof(V4) * nF, cudaMemcpyDeviceToDevice, stream));
            }
            if (nP) CK(cudaMemcpyAsync(tmp4a.p + nF, tmp4b.p, sizeof(V4) * nP, cudaMemcpyDeviceToDevice, stream));
            rc = download_nodes(tmp4a.p, x3.data());
            if (rc) return rc;
            for (int j = 0; j < n; ++j)
                for (int c = 0; c < kc; ++c) {
                    const double vv = x3[3 * (size_t)j + c];
                    X[(size_t)j * k + c0 + c] = vv;
                    bad |= !std::isfinite(vv);
                }
        }
        (void)bad;
        return VKPD_OK;
    }

    // ---- reference-compatible CMS / A-Jacobi path (cms.cuh) ----------------
    DBuf<double> cmsT, cmsKinv, cms_y, cms_z, hist_d, rho_d;
    DBuf<V4> bestv;
    DBuf<int> nhist_d, div_d;
    int cms_m = 0;
    // blocked basis (cms.cuh CmsBlocks)
    bool cms_blocked = false;
    DBuf<double> cmsA, cms_yd, cms_part;
    int cms_total_rows = 0;
    DBuf<long long> cms_aoff;
    DBuf<int> cms_rowp, cms_rows, cms_colp, cms_colmap, cms_tdom, cms_tc0, cms_bnd, cms_ysp, cms_ys;
    vk::CmsBlocks cmsb{};
    int cms_max_rows = 0, cms_max_cols = 0;
    cudaEvent_t cms_ev[3] = {nullptr, nullptr, nullptr};
    float cms_apply_ms = 0.f, cms_sweeps_ms = 0.f;

    // rows [0, m) of a V4 buffer from an (m, k) float64 host array, columns c0..c0+2
    // rows in the caller's free order (m == nF) or pin order (m == nP) -> device rows
    int upload_rows(const double* h, int m, int k, int c0, V4* dst) {
        std::vector<double> pk((size_t)3 * std::max(1, m), 0.0);
        const int kc = std::min(3, k - c0);
        const bool perm = m == nF && (int)free_perm.size() == nF;
        for (int j = 0; j < m; ++j) {
            const size_t r = perm ? (size_t)free_perm[j] : (size_t)j;
            for (int c = 0; c < kc; ++c) pk[3 * r + c] = h[(size_t)j * k + c0 + c];
        }
        if (m == 0) return VKPD_OK;
        CK(cudaMemcpyAsync(stage.p, pk.data(), sizeof(double) * 3 * m, cudaMemcpyHostToDevice, stream));
        k_rows_in<T><<<cdiv(m, 256), 256, 0, stream>>>(m, stage.p, dst);
        CK(cudaGetLastError());
        // the pageable host buffer must outlive the copy
        CK(cudaStreamSynchronize(stream));
        return VKPD_OK;
    }
    int download_rows(const V4* src, int m, int k, int c0, double* h) {
        if (m == 0) return VKPD_OK;
        std::vector<V4> tmp(m);
        CK(cudaMemcpyAsync(tmp.data(), src, sizeof(V4) * m, cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        const int kc = std::min(3, k - c0);
        const bool perm = m == nF && (int)free_perm.size() == nF;
        for (int j = 0; j < m; ++j) {
            const V4 t = tmp[perm ? free_perm[j] : j];
            const double v[3] = {(double)t.x, (double)t.y, (double)t.z};
            for (int c = 0; c < kc; ++c) h[(size_t)j * k + c0 + c] = v[c];
        }
        return VKPD_OK;
    }
    int ensure_aj() {
        if (!bestv.p) CK(bestv.alloc(std::max(1, nF)));
        if (!nhist_d.p) { CK(nhist_d.alloc(3)); CK(div_d.alloc(3)); CK(rho_d.alloc(3)); }
        return VKPD_OK;
    }
    vk::AJArgs<T> aj_args(int sweeps, int agg, double omega, double rho, int ncols) {
        vk::AJArgs<T> a;
        a.nF = nF; a.ell_w = ell_w; a.ell_col = ell_col.p; a.ell_val = ell_val.p; a.diag = diag64.p;
        a.b = rhs.p; a.x = dx.p; a.r = r.p; a.s = z.p; a.e = p0.p; a.cs0 = p1.p; a.cs1 = q.p; a.best = bestv.p;
        a.partials = partials.p; a.hist = hist_d.p; a.n_hist = nhist_d.p; a.diverged = div_d.p;
        a.sweeps = sweeps; a.aggregation = agg; a.omega = omega; a.rho = rho; a.ncols = ncols;
        return a;
    }
    template <typename K>
    cudaError_t launch_coop(K kernel, void** args) {
        int occ = 0;
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, 256, 0);
        if (e != cudaSuccess) return e;
        const int blocks = std::max(1, std::min(std::min(occ * n_sms, pcg_blocks), cdiv(std::max(1, nF), 256)));
        return cudaLaunchCooperativeKernel((const void*)kernel, dim3(blocks), dim3(256), args, 0, stream);
    }
    // a_jacobi_refine on K_ff over free-node vectors (pdsolver.py:632-703)
    int run_aj(int ncols, int sweeps, int agg, double omega, int cheb, double rho) {
        const int steps = cheb ? sweeps * agg : sweeps;
        if (hist_d.n < (size_t)3 * (steps + 1)) CK(hist_d.alloc((size_t)3 * (steps + 1)));
        CK(cudaMemsetAsync(hist_d.p, 0, sizeof(double) * 3 * (steps + 1), stream));
        vk::AJArgs<T> a = aj_args(sweeps, agg, omega, rho, ncols);
        void* args[] = {&a};
        if (cheb) CK(launch_coop(vk::k_chebyshev<T>, args));
        else CK(launch_coop(vk::k_ajacobi<T>, args));
        return VKPD_OK;
    }
    int aj_refine(const double* Bf, const double* X0f, int k, int sweeps, int agg, double omega, int cheb,
                  double rho, double* Xf, double* hist, int* nhist, int* diverged) override {
        if (agg != 2 && agg != 3) return fail(VKPD_EINVAL, "aggregation must be 2 or 3");
        if (k < 1 || k > 3) return fail(VKPD_EINVAL, "a_jacobi_refine takes 1 to 3 columns");
        int rc = ensure_aj();
        if (rc) return rc;
        if (cheb && !(rho >= 0.0)) return fail(VKPD_EINVAL, "chebyshev needs rho (vkpd_power_rho)");
        if ((rc = upload_rows(Bf, nF, k, 0, rhs.p))) return rc;
        if ((rc = upload_rows(X0f, nF, k, 0, dx.p))) return rc;
        if ((rc = run_aj(k, sweeps, agg, omega, cheb, rho))) return rc;
        if ((rc = download_rows(dx.p, nF, k, 0, Xf))) return rc;
        const int steps = cheb ? sweeps * agg : sweeps;
        std::vector<double> hh((size_t)3 * (steps + 1));
        CK(cudaMemcpy(hh.data(), hist_d.p, sizeof(double) * hh.size(), cudaMemcpyDeviceToHost));
        int nh[3], dv[3];
        CK(cudaMemcpy(nh, nhist_d.p, sizeof nh, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(dv, div_d.p, sizeof dv, cudaMemcpyDeviceToHost));
        for (int c = 0; c < k; ++c) {
            if (nhist) nhist[c] = nh[c];
            if (diverged) diverged[c] = dv[c];
            if (hist)
                for (int j = 0; j < nh[c]; ++j) hist[(size_t)c * (steps + 1) + j] = hh[(size_t)j * 3 + c];
        }
        return VKPD_OK;
    }
    // reference start vector: default_rng(0).normal(size=n) supplied by the caller (v0, nF)
    int power_rho(double omega, int iters, const double* v0, double* rho) override {
        int rc = ensure_aj();
        if (rc) return rc;
        if (!v0) return fail(VKPD_EINVAL, "power iteration needs a start vector");
        {
            std::vector<double> v3((size_t)3 * nF);
            for (int j = 0; j < nF; ++j) v3[3 * j] = v3[3 * j + 1] = v3[3 * j + 2] = v0[j];
            if ((rc = upload_rows(v3.data(), nF, 3, 0, dx.p))) return rc;
        }
        vk::AJArgs<T> a = aj_args(0, 2, omega, 0.0, 3);
        double* out = rho_d.p;
        void* args[] = {&a, &iters, &out};
        CK(launch_coop(vk::k_power_rho<T>, args));
        CK(cudaStreamSynchronize(stream));            // non-blocking stream: no implicit sync with cudaMemcpy
        double hr[3];
        CK(cudaMemcpy(hr, rho_d.p, sizeof hr, cudaMemcpyDeviceToHost));
        *rho = hr[0];
        return VKPD_OK;
    }
    int cms_set_basis(int m, const double* Tb, const double* Kinv) override {
        if (m < 0) return fail(VKPD_EINVAL, "bad subspace size");
        cms_m = m;
        cms_blocked = false;
        CK(cmsT.alloc((size_t)std::max(1, nF) * std::max(1, m)));
        CK(cmsKinv.alloc((size_t)std::max(1, m) * std::max(1, m)));
        CK(cms_y.alloc((size_t)3 * std::max(1, m)));
        CK(cms_z.alloc((size_t)3 * std::max(1, m)));
        if (m > 0) {
            std::vector<double> Tp((size_t)nF * m);       // column-major, rows to internal order
            for (int c = 0; c < m; ++c)
                for (int j = 0; j < nF; ++j) Tp[(size_t)c * nF + free_perm[j]] = Tb[(size_t)c * nF + j];
            CK(cudaMemcpy(cmsT.p, Tp.data(), sizeof(double) * nF * (size_t)m, cudaMemcpyHostToDevice));
            CK(cudaMemcpy(cmsKinv.p, Kinv, sizeof(double) * (size_t)m * m, cudaMemcpyHostToDevice));
        }
        return VKPD_OK;
    }
    int cms_set_blocks(int ndom, const int64_t* row_ptr, const int64_t* rows, const int64_t* col_ptr,
                       const int64_t* colmap, const double* A, int nmodes, int64_t nb, const int64_t* bnd,
                       const double* Kinv) override {
        if (ndom < 0 || nmodes < 0 || nb < 0) return fail(VKPD_EINVAL, "bad block structure");
        const int m = nmodes + (int)nb;
        std::vector<int> rp(ndom + 1), cp(ndom + 1), rw, cm, tdom, tc0, bd(nb);
        std::vector<long long> aoff(std::max(1, ndom));
        long long atot = 0;
        cms_max_rows = cms_max_cols = 0;
        for (int d = 0; d <= ndom; ++d) { rp[d] = (int)row_ptr[d]; cp[d] = (int)col_ptr[d]; }
        for (int d = 0; d < ndom; ++d) {
            const int nd = rp[d + 1] - rp[d], nc = cp[d + 1] - cp[d];
            if (nd < 0 || nc < 0) return fail(VKPD_EINVAL, "block pointers not monotone");
            aoff[d] = atot;
            atot += (long long)nd * nc;
            cms_max_rows = std::max(cms_max_rows, nd);
            cms_max_cols = std::max(cms_max_cols, nc);
            for (int c0 = 0; c0 < nc; c0 += vk::kCmsTile) { tdom.push_back(d); tc0.push_back(c0); }
        }
        rw.resize(std::max(1, rp[ndom]));
        for (int k = 0; k < rp[ndom]; ++k) {
            if (rows[k] < 0 || rows[k] >= nF) return fail(VKPD_EINVAL, "block row out of range");
            rw[k] = free_perm[rows[k]];
        }
        cm.resize(std::max(1, cp[ndom]));
        std::vector<std::vector<int>> src(m);
        for (int k = 0; k < cp[ndom]; ++k) {
            if (colmap[k] < 0 || colmap[k] >= m) return fail(VKPD_EINVAL, "block column out of range");
            cm[k] = (int)colmap[k];
            src[cm[k]].push_back(k);           // domain order (k increases with d)
        }
        for (int64_t j = 0; j < nb; ++j) {
            if (bnd[j] < 0 || bnd[j] >= nF) return fail(VKPD_EINVAL, "boundary row out of range");
            bd[j] = free_perm[bnd[j]];
        }
        std::vector<int> ysp(m + 1, 0), ys;
        for (int g = 0; g < m; ++g) { ys.insert(ys.end(), src[g].begin(), src[g].end()); ysp[g + 1] = (int)ys.size(); }
        cudaStream_t st = stream;
        CK(cmsA.alloc(std::max<long long>(1, atot)));
        if (atot) CK(cmsA.upload(A, atot, st));
        CK(cms_aoff.alloc(aoff.size())); CK(cms_aoff.upload(aoff.data(), aoff.size(), st));
        CK(cms_rowp.alloc(rp.size())); CK(cms_rowp.upload(rp.data(), rp.size(), st));
        CK(cms_colp.alloc(cp.size())); CK(cms_colp.upload(cp.data(), cp.size(), st));
        CK(cms_rows.alloc(rw.size())); CK(cms_rows.upload(rw.data(), rw.size(), st));
        CK(cms_colmap.alloc(cm.size())); CK(cms_colmap.upload(cm.data(), cm.size(), st));
        tdom.push_back(0); tc0.push_back(0);      // keep the buffers non-empty
        CK(cms_tdom.alloc(tdom.size())); CK(cms_tdom.upload(tdom.data(), tdom.size(), st));
        CK(cms_tc0.alloc(tc0.size())); CK(cms_tc0.upload(tc0.data(), tc0.size(), st));
        bd.push_back(0);
        CK(cms_bnd.alloc(bd.size())); CK(cms_bnd.upload(bd.data(), bd.size(), st));
        CK(cms_ysp.alloc(ysp.size())); CK(cms_ysp.upload(ysp.data(), ysp.size(), st));
        ys.push_back(0);
        CK(cms_ys.alloc(ys.size())); CK(cms_ys.upload(ys.data(), ys.size(), st));
        CK(cms_yd.alloc((size_t)3 * std::max(1, cp[ndom])));
        CK(cmsKinv.alloc((size_t)std::max(1, m) * std::max(1, m)));
        if (m > 0) CK(cmsKinv.upload(Kinv, (size_t)m * m, st));
        CK(cms_y.alloc((size_t)3 * std::max(1, m)));
        CK(cms_z.alloc((size_t)3 * std::max(1, m)));
        CK(cudaStreamSynchronize(st));
        cmsb.ndom = ndom; cmsb.nmodes = nmodes; cmsb.nb = (int)nb; cmsb.ntiles = (int)tdom.size() - 1;
        cmsb.A = cmsA.p; cmsb.a_off = cms_aoff.p; cmsb.row_ptr = cms_rowp.p; cmsb.rows = cms_rows.p;
        cmsb.col_ptr = cms_colp.p; cmsb.colmap = cms_colmap.p; cmsb.tile_dom = cms_tdom.p; cmsb.tile_c0 = cms_tc0.p;
        cmsb.bnd = cms_bnd.p; cmsb.ysrc_ptr = cms_ysp.p; cmsb.ysrc = cms_ys.p;
        const size_t smem = sizeof(double) * 3 * std::max(1, cdiv(cms_max_cols, vk::kCmsTzGroups) + 1);
        if (smem > 48 * 1024) {
            if (smem > 200 * 1024) return fail(VKPD_EINVAL, "too many basis columns in one domain");
            CK(cudaFuncSetAttribute(vk::k_cms_tz<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        }
        CK(cms_part.alloc((size_t)3 * vk::kCmsTzGroups * std::max(1, rp[ndom])));
        cms_total_rows = rp[ndom];
        cms_m = m;
        cms_blocked = true;
        return VKPD_OK;
    }
    int cms_timing(double* apply_ms, double* sweeps_ms) override {
        if (apply_ms) *apply_ms = cms_apply_ms;
        if (sweeps_ms) *sweeps_ms = cms_sweeps_ms;
        return VKPD_OK;
    }
    // x0 = T K_red^-1 T^T rhs into dx (blocked or dense basis)
    int cms_apply() {
        if (cms_m <= 0) {
            CK(cudaMemsetAsync(dx.p, 0, sizeof(V4) * nF, stream));
            return VKPD_OK;
        }
        if (cms_blocked) {
            if (cmsb.ntiles > 0) vk::k_cms_tb<T><<<cmsb.ntiles, 256, 0, stream>>>(cmsb, rhs.p, cms_yd.p);
            vk::k_cms_y<T><<<cdiv(cms_m, 128), 128, 0, stream>>>(cmsb, cms_m, rhs.p, cms_yd.p, cms_y.p);
            vk::k_symv3_warp<<<cdiv((size_t)cms_m * 32, 256), 256, 0, stream>>>(cms_m, cmsKinv.p, cms_y.p, cms_z.p);
            CK(cudaMemsetAsync(dx.p, 0, sizeof(V4) * nF, stream));
            if (cmsb.ndom > 0 && cms_max_rows > 0) {
                const dim3 grid(cdiv(cms_max_rows, 256), cmsb.ndom, vk::kCmsTzGroups);
                const size_t zsm = sizeof(double) * 3 * std::max(1, cdiv(cms_max_cols, vk::kCmsTzGroups) + 1);
                vk::k_cms_tz<T><<<grid, 256, zsm, stream>>>(cmsb, cms_z.p, cms_part.p, cms_total_rows);
                vk::k_cms_tz_sum<T><<<cdiv(cms_total_rows, 256), 256, 0, stream>>>(cmsb, cms_total_rows,
                                                                                   vk::kCmsTzGroups, cms_part.p, dx.p);
            }
            if (cmsb.nb > 0) vk::k_cms_xb<T><<<cdiv(cmsb.nb, 256), 256, 0, stream>>>(cmsb, cms_z.p, dx.p);
        } else {
            vk::k_tmv<T><<<cdiv((size_t)cms_m * 32, 256), 256, 0, stream>>>(nF, cms_m, cmsT.p, rhs.p, cms_y.p);
            vk::k_symv3<<<cdiv(cms_m, 128), 128, 0, stream>>>(cms_m, cmsKinv.p, cms_y.p, cms_z.p);
            vk::k_tv<T><<<cdiv(nF, 256), 256, 0, stream>>>(nF, cms_m, cmsT.p, cms_z.p, dx.p);
        }
        CK(cudaGetLastError());
        return VKPD_OK;
    }
    // pd_step with GlobalSolver(mode="cms") as one device frame (pdsolver.py:257-304, 237-246): per
    // PD round the local step in rhs form (+ robust pass), b = rhs + (M/dt^2) xhat on the free rows,
    // b_f - K_fp p, the subspace apply and the A-Jacobi / Chebyshev sweeps; no host round trip
    int step_cms(int iterations, double damping, int sweeps, int agg, double omega, int cheb, double rho,
                 int* failed) override {
        if (nE == 0) return fail(VKPD_EINVAL, "cms frame needs a mesh context");
        if (!cms_blocked && cms_m <= 0) return fail(VKPD_EINVAL, "no CMS subspace set (vkpd_cms_set_blocks)");
        if (iterations < 0 || iterations > 1024) return fail(VKPD_EINVAL, "iterations must be in [0, 1024]");
        if (sweeps > 0 && agg != 2 && agg != 3) return fail(VKPD_EINVAL, "aggregation must be 2 or 3");
        if (cheb && sweeps > 0 && !(rho >= 0.0)) return fail(VKPD_EINVAL, "chebyshev needs rho (vkpd_power_rho)");
        if (int rc = ensure_aj()) return rc;
        if (failed) *failed = -1;
        const int nb = cdiv(n, 256);
        vk::k_prologue<T><<<nb, 256, 0, stream>>>(n, nF, (T)dt, dt2_inv_m.p, has_forces ? f.p : nullptr, pin_tgt.p,
                                                  x.p, v.p, x_start.p, v_start.p, xhat.p, fail_iter.p);
        CK(cudaGetLastError());
        const vk::LocalArgs<T> la = local_args(x.p);
        for (int it = 0; it < iterations && nF > 0; ++it) {
            CK(cudaMemsetAsync(robust_count.p, 0, 2 * sizeof(int), stream));
            vk::k_local<T, vk::MODE_RHS, false, 1><<<cdiv(nE, 128), 128, 0, stream>>>(la);
            vk::k_robust_tasks<T, vk::MODE_RHS><<<robust_task_blocks * n_sms, 128, 0, stream>>>(
                la, robust_res.p, robust_ok.p, robust_arrivals.p, std::max(1, nE));
            vk::k_cms_b<T><<<cdiv(nF, 256), 256, 0, stream>>>(nF, inc_ptr.p, corner.p, m_dt2.p, xhat.p, tmp4a.p);
            k_rhs_minus_fp<T><<<cdiv(nF, 256), 256, 0, stream>>>(nF, tmp4a.p, fp_ptr.p, fp_col.p, fp_val.p, x.p + nF,
                                                                rhs.p);
            CK(cudaGetLastError());
            if (int rc = cms_apply()) return rc;
            if (sweeps > 0)
                if (int rc = run_aj(3, sweeps, agg, omega, cheb, rho)) return rc;
            vk::k_cms_set_x<T><<<cdiv(nF, 256), 256, 0, stream>>>(nF, dx.p, x.p, fail_iter.p, it);
            CK(cudaGetLastError());
        }
        vk::k_epilogue<T><<<nb, 256, 0, stream>>>(n, (T)(damping / dt), x.p, x_start.p, v.p);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(h_fail, fail_iter.p, sizeof(int), cudaMemcpyDeviceToHost, stream));
        return sync(failed);
    }
    // GlobalSolver.solve in "cms" mode (pdsolver.py:237-246): per column
    // x0 = T K_red^-1 T^T b_f, then a_jacobi_refine(K_ff, b_f, x0, ...).
    int cms_solve(const double* B, const double* P, int k, int sweeps, int agg, double omega, int cheb, double rho,
                  double* X) override {
        if (sweeps > 0 && agg != 2 && agg != 3) return fail(VKPD_EINVAL, "aggregation must be 2 or 3");
        int rc = ensure_aj();
        if (rc) return rc;
        if (cheb && sweeps > 0 && !(rho >= 0.0)) return fail(VKPD_EINVAL, "chebyshev needs rho (vkpd_power_rho)");
        std::vector<double> xcol((size_t)nF * k);
        for (int c0 = 0; c0 < k; c0 += 3) {
            const int kc = std::min(3, k - c0);
            // b_f - K_fp P  -> rhs
            std::vector<double> b3((size_t)3 * n, 0.0), p3((size_t)3 * std::max(1, nP), 0.0);
            for (int j = 0; j < n; ++j)
                for (int c = 0; c < kc; ++c) b3[3 * (size_t)j + c] = B[(size_t)j * k + c0 + c];
            for (int j = 0; j < nP; ++j)
                for (int c = 0; c < kc; ++c) p3[3 * (size_t)j + c] = P[(size_t)j * k + c0 + c];
            if ((rc = upload_nodes(b3.data(), tmp4a.p))) return rc;
            if (nP) {
                CK(cudaMemcpyAsync(stage.p, p3.data(), sizeof(double) * 3 * nP, cudaMemcpyHostToDevice, stream));
                k_rows_in<T><<<cdiv(nP, 256), 256, 0, stream>>>(nP, stage.p, tmp4b.p);
                CK(cudaGetLastError());
            }
            if (nF > 0) {
                k_rhs_minus_fp<T><<<cdiv(nF, 256), 256, 0, stream>>>(nF, tmp4a.p, fp_ptr.p, fp_col.p, fp_val.p,
                                                                    tmp4b.p, rhs.p);
                CK(cudaGetLastError());
                if (!cms_ev[0])
                    for (auto& ev : cms_ev) CK(cudaEventCreate(&ev));
                CK(cudaEventRecord(cms_ev[0], stream));
                if ((rc = cms_apply())) return rc;
                CK(cudaEventRecord(cms_ev[1], stream));
                if (sweeps > 0 && (rc = run_aj(kc, sweeps, agg, omega, cheb, rho))) return rc;
                CK(cudaEventRecord(cms_ev[2], stream));
                if (c0 == 0) {
                    CK(cudaEventSynchronize(cms_ev[2]));
                    CK(cudaEventElapsedTime(&cms_apply_ms, cms_ev[0], cms_ev[1]));
                    CK(cudaEventElapsedTime(&cms_sweeps_ms, cms_ev[1], cms_ev[2]));
                }
                CK(cudaMemcpyAsync(tmp4a.p, dx.p, sizeof(V4) * nF, cudaMemcpyDeviceToDevice, stream));
            }
            if (nP) CK(cudaMemcpyAsync(tmp4a.p + nF, tmp4b.p, sizeof(V4) * nP, cudaMemcpyDeviceToDevice, stream));
            std::vector<double> x3((size_t)3 * n);
            if ((rc = download_nodes(tmp4a.p, x3.data()))) return rc;
            for (int j = 0; j < n; ++j)
                for (int c = 0; c < kc; ++c) X[(size_t)j * k + c0 + c] = x3[3 * (size_t)j + c];
        }
        return VKPD_OK;
    }

    // ---- device-pointer primitives for the domain-decomposed multi-GPU step (dd.py) ----
    int dev_residual(const void* x_int, const void* xhat_int, void* r_free) override {
        if (nE == 0) return fail(VKPD_EINVAL, "matrix-only context has no mesh");
        vk::LocalArgs<T> la = local_args((const V4*)x_int);
        if (int rc = launch_local_resid(la)) return rc;
        if (nF > 0) {
            k_resid_free<T><<<cdiv(nF, 256), 256, 0, stream>>>(nF, inc_ptr.p, corner.p, m_dt2.p, (const V4*)x_int,
                                                               (const V4*)xhat_int, (V4*)r_free);
            CK(cudaGetLastError());
        }
        return VKPD_OK;
    }
    int dev_apply_K(const void* X, void* Y) override {
        if (nF > 0) {
            k_apply_K<T><<<cdiv(nF, 256), 256, 0, stream>>>(nF, nF, ell_len.p, ell_col.p, ell_val.p, fp_ptr.p, fp_col.p,
                                                           fp_val.p, (const V4*)X, (V4*)Y);
            CK(cudaGetLastError());
        }
        return VKPD_OK;
    }
    int dev_cheb_step(const void* d, void* res, void* y, void* dnext, double c1, double c2) override {
        if (nF > 0) {
            k_dd_cheb_step<T><<<cdiv(nF, 256), 256, 0, stream>>>(nF, ell_len.p, ell_col.p, ell_val.p, fp_ptr.p,
                                                                fp_col.p, fp_val.p, inv_diag.p, (const V4*)d,
                                                                (V4*)res, (V4*)y, (V4*)dnext, (T)c1, (T)c2);
            CK(cudaGetLastError());
        }
        return VKPD_OK;
    }
    int gershgorin(int with_pinned, double* g) override {
        if (!with_pinned) { *g = gersh; return VKPD_OK; }
        DBuf<unsigned long long> gmax;
        CK(gmax.alloc(1));
        CK(cudaMemsetAsync(gmax.p, 0, sizeof(unsigned long long), stream));
        if (nF > 0)
            vk::k_gershgorin_fp<T><<<cdiv(nF, 256), 256, 0, stream>>>(nF, ell_w, ell_col.p, ell_val.p, fp_ptr.p,
                                                                      fp_val.p, diag64.p, gmax.p);
        CK(cudaGetLastError());
        unsigned long long b = 0;
        CK(cudaMemcpyAsync(&b, gmax.p, sizeof b, cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        double v = 0.0;
        std::memcpy(&v, &b, sizeof v);
        *g = v + 1.0;
        return VKPD_OK;
    }
    int dev_inv_diag(void* out) override {
        if (nF > 0) CK(cudaMemcpyAsync(out, inv_diag.p, sizeof(T) * nF, cudaMemcpyDeviceToDevice, stream));
        return VKPD_OK;
    }
    int node_order(int64_t* ioo) override {
        for (int j = 0; j < n; ++j) ioo[j] = int_of_orig_h[j];
        return VKPD_OK;
    }
    void sizes(int64_t* nn, int64_t* nfree, int64_t* npinned, int* prec) override {
        if (nn) *nn = n;
        if (nfree) *nfree = nF;
        if (npinned) *npinned = nP;
        if (prec) *prec = sizeof(T) == 4 ? VKPD_FP32 : VKPD_FP64;
    }

    int apply_K(const double* hX, double* hY) override {
        int rc = upload_nodes(hX, tmp4a.p);
        if (rc) return rc;
        k_apply_K<T><<<cdiv(n, 256), 256, 0, stream>>>(n, nF, ell_len.p, ell_col.p, ell_val.p, fp_ptr.p, fp_col.p,
                                                       fp_val.p, tmp4a.p, tmp4b.p);
        CK(cudaGetLastError());
        return download_nodes(tmp4b.p, hY);
    }

    int stats(vkpd_stats* st) override {
        std::memset(st, 0, sizeof(*st));
        CK(cudaStreamSynchronize(stream));
        const int ni = std::min(last_iterations, 256);
        st->n_pd_iters = ni;
        if (ni > 0) CK(cudaMemcpy(st->cg_iters, iters.p, sizeof(int) * ni, cudaMemcpyDeviceToHost));
        for (int i = 0; i < ni; ++i) st->cg_iters_total += st->cg_iters[i];
        vk::ProjStats ps;
        CK(cudaMemcpy(&ps, pstats.p, sizeof(ps), cudaMemcpyDeviceToHost));
        st->robust = ps.robust;
        st->fallback = ps.fallback;
        st->pd_rounds_total = ps.pd_rounds;
        st->solver = solver_kind;
        st->pcg_blocks = pcg_blocks;
        st->ell_width = ell_w;
        st->n_free = nF;
        for (size_t i = 0; i < prof_local.size() && i < 256; ++i) {
            st->local_ms[i] = prof_local[i];
            st->global_ms[i] = prof_global[i];
        }
        return VKPD_OK;
    }
};

#include "hess_ctx.cuh"

}  // namespace

struct vkpd_ctx {
    std::unique_ptr<CtxBase> impl;
};
struct vkpd_hess {
    HessCtx impl;
};

extern "C" {

const char* vkpd_last_error(void) { return g_err.c_str(); }

int vkpd_device_count(int* count) {
    int c = 0;
    cudaError_t e = cudaGetDeviceCount(&c);
    if (e != cudaSuccess) {
        cudaGetLastError();
        *count = 0;
        return fail(VKPD_ECUDA, std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e));
    }
    *count = c;
    return VKPD_OK;
}

int vkpd_create(const vkpd_mesh_desc* mesh, const vkpd_config* cfg, vkpd_ctx** out) {
    if (!mesh || !cfg || !out) return fail(VKPD_EINVAL, "null argument");
    if (!mesh->tets || !mesh->shape_grad || !mesh->volume || !mesh->gamma_s || !mesh->gamma_v)
        return fail(VKPD_EINVAL, "missing mesh array");
    if (mesh->n_pins > 0 && !mesh->pins) return fail(VKPD_EINVAL, "missing pin array");
    int count = 0;
    if (vkpd_device_count(&count) != VKPD_OK || count == 0)
        return fail(VKPD_ECUDA, "no CUDA device available (the vkpd library has no CPU path)");
    if (cfg->device < 0 || cfg->device >= count) return fail(VKPD_EINVAL, "bad device ordinal");
    std::unique_ptr<vkpd_ctx> c(new vkpd_ctx);
    if (cfg->precision == VKPD_FP32) c->impl.reset(new Ctx<float>());
    else if (cfg->precision == VKPD_FP64) c->impl.reset(new Ctx<double>());
    else return fail(VKPD_EINVAL, "precision must be 32 or 64");
    c->impl->device = cfg->device;
    DeviceGuard guard_(cfg->device);
    int rc = c->impl->init(mesh, cfg);
    if (rc != VKPD_OK) return rc;
    *out = c.release();
    return VKPD_OK;
}

int vkpd_create_matrix(int64_t n, const int64_t* indptr, const int64_t* indices, const double* data,
                       const int64_t* pins, int64_t n_pins, const vkpd_config* cfg, vkpd_ctx** out) {
    if (!indptr || !indices || !data || !cfg || !out || (n_pins > 0 && !pins))
        return fail(VKPD_EINVAL, "null argument");
    int count = 0;
    if (vkpd_device_count(&count) != VKPD_OK || count == 0)
        return fail(VKPD_ECUDA, "no CUDA device available (the vkpd library has no CPU path)");
    if (cfg->device < 0 || cfg->device >= count) return fail(VKPD_EINVAL, "bad device ordinal");
    std::unique_ptr<vkpd_ctx> c(new vkpd_ctx);
    if (cfg->precision == VKPD_FP32) c->impl.reset(new Ctx<float>());
    else if (cfg->precision == VKPD_FP64) c->impl.reset(new Ctx<double>());
    else return fail(VKPD_EINVAL, "precision must be 32 or 64");
    c->impl->device = cfg->device;
    DeviceGuard guard_(cfg->device);
    int rc = c->impl->init_matrix(n, indptr, indices, data, pins, n_pins, cfg);
    if (rc != VKPD_OK) return rc;
    *out = c.release();
    return VKPD_OK;
}

int vkpd_get_matrix_csr(vkpd_ctx* ctx, int64_t* indptr, int64_t* indices, double* data, int64_t* nnz) {
    if (!ctx || !nnz) return fail(VKPD_EINVAL, "null argument");
    DeviceGuard guard_(ctx->impl->device);
    return ctx->impl->get_csr(indptr, indices, data, nnz);
}

void vkpd_destroy(vkpd_ctx* ctx) {
    if (!ctx) return;
    DeviceGuard guard_(ctx->impl->device);
    delete ctx;
}

int vkpd_set_stream(vkpd_ctx* ctx, void* stream) {
    if (!ctx) return fail(VKPD_EINVAL, "null context");
    ctx->impl->stream = stream ? (cudaStream_t)stream : ctx->impl->own_stream;
    return VKPD_OK;
}
void* vkpd_get_stream(vkpd_ctx* ctx) { return ctx ? (void*)ctx->impl->stream : nullptr; }

#define CTX_CALL(expr)                                                                             \
    do {                                                                                           \
        if (!ctx) return fail(VKPD_EINVAL, "null context");                                       \
        DeviceGuard guard_(ctx->impl->device);                                                     \
        return ctx->impl->expr;                                                                    \
    } while (0)

int vkpd_set_state(vkpd_ctx* ctx, const double* x, const double* v) {
    if (!x) return fail(VKPD_EINVAL, "null positions");
    CTX_CALL(set_state(x, v));
}
int vkpd_get_state(vkpd_ctx* ctx, double* x, double* v) { CTX_CALL(get_state(x, v)); }
int vkpd_set_state_dev(vkpd_ctx* ctx, const void* x, const void* v) {
    if (!x) return fail(VKPD_EINVAL, "null positions");
    CTX_CALL(set_state_dev(x, v));
}
int vkpd_get_state_dev(vkpd_ctx* ctx, void* x, void* v) { CTX_CALL(get_state_dev(x, v)); }
int vkpd_set_forces_dev(vkpd_ctx* ctx, const void* f) { CTX_CALL(set_forces_dev(f)); }
int vkpd_set_pin_targets_dev(vkpd_ctx* ctx, const void* t) {
    if (!t) return fail(VKPD_EINVAL, "null pin targets");
    CTX_CALL(set_pin_targets_dev(t));
}
int vkpd_set_pin_targets(vkpd_ctx* ctx, const double* t) {
    if (!t) return fail(VKPD_EINVAL, "null pin targets");
    CTX_CALL(set_pin_targets(t));
}
int vkpd_set_forces(vkpd_ctx* ctx, const double* f) { CTX_CALL(set_forces(f)); }
int vkpd_set_yarn_interp(vkpd_ctx* ctx, int64_t n_yarn, const int64_t* indptr, const int64_t* indices,
                         const double* data) {
    CTX_CALL(set_yarn_interp(n_yarn, indptr, indices, data));
}
int vkpd_frame_outputs(vkpd_ctx* ctx, double* yarn, double* det_deviation) {
    CTX_CALL(frame_outputs(yarn, det_deviation));
}
int64_t vkpd_format_obj(const double* v, int64_t nv, const int64_t* faces, int64_t nf, const int64_t* line_ptr,
                        const int64_t* line_idx, int64_t nl, const char* comment, char* out, int64_t cap) {
    std::string s;
    s.reserve((size_t)nv * 72 + (size_t)nf * 24 + 64);
    char buf[128];
    if (comment && comment[0]) { s += "# "; s += comment; s += '\n'; }
    for (int64_t i = 0; i < nv; ++i) {
        const int m = std::snprintf(buf, sizeof buf, "v %.17g %.17g %.17g\n", v[3 * i], v[3 * i + 1], v[3 * i + 2]);
        s.append(buf, (size_t)m);
    }
    for (int64_t i = 0; i < nf; ++i) {
        const int m = std::snprintf(buf, sizeof buf, "f %lld %lld %lld\n", (long long)faces[3 * i] + 1,
                                    (long long)faces[3 * i + 1] + 1, (long long)faces[3 * i + 2] + 1);
        s.append(buf, (size_t)m);
    }
    for (int64_t l = 0; l < nl; ++l) {
        s += 'l';
        for (int64_t k = line_ptr[l]; k < line_ptr[l + 1]; ++k) {
            const int m = std::snprintf(buf, sizeof buf, " %lld", (long long)line_idx[k] + 1);
            s.append(buf, (size_t)m);
        }
        s += '\n';
    }
    if (out && cap > 0) std::memcpy(out, s.data(), (size_t)std::min<int64_t>(cap, (int64_t)s.size()));
    return (int64_t)s.size();
}
int vkpd_v2y(int64_t n_yarn, const int64_t* indptr, const int64_t* indices, const double* data, int64_t n_nodes,
             const double* x, double* y) {
    if (n_yarn < 0 || n_nodes < 0 || (n_yarn > 0 && (!indptr || !indices || !data || !y)) || (n_nodes > 0 && !x))
        return fail(VKPD_EINVAL, "bad arguments");
    int count = 0;
    if (vkpd_device_count(&count) != VKPD_OK || count == 0)
        return fail(VKPD_ECUDA, "no CUDA device available (the vkpd library has no CPU path)");
    if (n_yarn == 0) return VKPD_OK;
    const int64_t nnz = indptr[n_yarn];
    for (int64_t j = 0; j < nnz; ++j)
        if (indices[j] < 0 || indices[j] >= n_nodes) return fail(VKPD_EINVAL, "interpolation column out of range");
    DBuf<long long> dp, dc;
    DBuf<double> dw, dx, dy;
    CK(dp.alloc(n_yarn + 1)); CK(dc.alloc(std::max<int64_t>(1, nnz))); CK(dw.alloc(std::max<int64_t>(1, nnz)));
    CK(dx.alloc((size_t)3 * std::max<int64_t>(1, n_nodes))); CK(dy.alloc((size_t)3 * n_yarn));
    CK(cudaMemcpy(dp.p, indptr, sizeof(long long) * (n_yarn + 1), cudaMemcpyHostToDevice));
    if (nnz > 0) {
        CK(cudaMemcpy(dc.p, indices, sizeof(long long) * nnz, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dw.p, data, sizeof(double) * nnz, cudaMemcpyHostToDevice));
    }
    if (n_nodes > 0) CK(cudaMemcpy(dx.p, x, sizeof(double) * 3 * n_nodes, cudaMemcpyHostToDevice));
    vk::k_v2y_host_order<<<cdiv((int)n_yarn, 256), 256>>>((int)n_yarn, dp.p, dc.p, dw.p, dx.p, dy.p);
    CK(cudaGetLastError());
    CK(cudaMemcpy(y, dy.p, sizeof(double) * 3 * n_yarn, cudaMemcpyDeviceToHost));
    return VKPD_OK;
}
int vkpd_equilibrium(vkpd_ctx* ctx, const double* inertia_target, const double* x0, const double* pin_vals,
                     int iterations, double* x_out, int* failed_iter) {
    if (!inertia_target || !x0 || !x_out) return fail(VKPD_EINVAL, "null array");
    CTX_CALL(equilibrium(inertia_target, x0, pin_vals, iterations, x_out, failed_iter));
}
int vkpd_set_gammas(vkpd_ctx* ctx, const double* gamma_s, const double* gamma_v) {
    if (!gamma_s || !gamma_v) return fail(VKPD_EINVAL, "null gamma arrays");
    CTX_CALL(set_gammas(gamma_s, gamma_v));
}
int vkpd_set_colliders(vkpd_ctx* ctx, int n, const int* kinds, const double* params, double contact_stiffness) {
    if (n > 0 && (!kinds || !params)) return fail(VKPD_EINVAL, "null collider arrays");
    CTX_CALL(set_colliders(n, kinds, params, contact_stiffness));
}
int vkpd_step_async(vkpd_ctx* ctx, int iterations, double damping) { CTX_CALL(step_async(iterations, damping)); }
int vkpd_simulate(vkpd_ctx* ctx, int steps, int iterations, double damping, const double* forces, int forces_per_step,
                  const double* pin_path, double* frames, int* failed_frame, int* failed_iter) {
    CTX_CALL(simulate(steps, iterations, damping, forces, forces_per_step, pin_path, frames, failed_frame,
                      failed_iter));
}
int vkpd_sync(vkpd_ctx* ctx, int* failed_iter) { CTX_CALL(sync(failed_iter)); }
int vkpd_step(vkpd_ctx* ctx, int iterations, double damping, int* failed_iter) {
    if (!ctx) return fail(VKPD_EINVAL, "null context");
    int rc = vkpd_step_async(ctx, iterations, damping);
    if (rc) return rc;
    return vkpd_sync(ctx, failed_iter);
}
int vkpd_profile_step(vkpd_ctx* ctx, int iterations, double damping, double* lms, double* gms, double* fms) {
    CTX_CALL(profile(iterations, damping, lms, gms, fms));
}
int vkpd_elastic_rhs(vkpd_ctx* ctx, const double* x, double* rhs, double* F, double* R, double* V) {
    if (!x || !rhs) return fail(VKPD_EINVAL, "null buffer");
    CTX_CALL(elastic_rhs(x, rhs, F, R, V));
}
int vkpd_global_solve(vkpd_ctx* ctx, const double* B, const double* P, double* X, int k) {
    if (!B || !X) return fail(VKPD_EINVAL, "null buffer");
    CTX_CALL(global_solve(B, P, X, k));
}
int vkpd_apply_K(vkpd_ctx* ctx, const double* X, double* Y) {
    if (!X || !Y) return fail(VKPD_EINVAL, "null buffer");
    CTX_CALL(apply_K(X, Y));
}
#ifdef VK_PCG_TRACE
int vkpd_debug_pcg_trace(unsigned long long* out, int max) {
    int n = 0;
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(&n, vk::g_pcg_trace_n, sizeof(int));
    n = std::min(n, max);
    if (n) cudaMemcpyFromSymbol(out, vk::g_pcg_trace, sizeof(unsigned long long) * n);
    int zero = 0;
    cudaMemcpyToSymbol(vk::g_pcg_trace_n, &zero, sizeof(int));
    return n;
}
#endif
int vkpd_dev_residual(vkpd_ctx* ctx, const void* x_int, const void* xhat_int, void* r_free) {
    if (!x_int || !xhat_int || !r_free) return fail(VKPD_EINVAL, "null device buffer");
    CTX_CALL(dev_residual(x_int, xhat_int, r_free));
}
int vkpd_dev_apply_K(vkpd_ctx* ctx, const void* X_int, void* Y_free) {
    if (!X_int || !Y_free) return fail(VKPD_EINVAL, "null device buffer");
    CTX_CALL(dev_apply_K(X_int, Y_free));
}
int vkpd_dev_inv_diag(vkpd_ctx* ctx, void* out_free) {
    if (!out_free) return fail(VKPD_EINVAL, "null device buffer");
    CTX_CALL(dev_inv_diag(out_free));
}
int vkpd_dev_cheb_step(vkpd_ctx* ctx, const void* d_int, void* res_free, void* y_free, void* dnext_int, double c1,
                       double c2) {
    CTX_CALL(dev_cheb_step(d_int, res_free, y_free, dnext_int, c1, c2));
}
int vkpd_get_gershgorin(vkpd_ctx* ctx, int with_pinned_cols, double* g) {
    if (!g) return fail(VKPD_EINVAL, "null argument");
    CTX_CALL(gershgorin(with_pinned_cols, g));
}
int vkpd_get_node_order(vkpd_ctx* ctx, int64_t* int_of_orig) {
    if (!int_of_orig) return fail(VKPD_EINVAL, "null buffer");
    CTX_CALL(node_order(int_of_orig));
}
int vkpd_get_sizes(vkpd_ctx* ctx, int64_t* n, int64_t* n_free, int64_t* n_pinned, int* precision) {
    if (!ctx) return fail(VKPD_EINVAL, "null context");
    ctx->impl->sizes(n, n_free, n_pinned, precision);
    return VKPD_OK;
}
int vkpd_a_jacobi_refine(vkpd_ctx* ctx, const double* Bf, const double* X0f, int k, int sweeps, int aggregation,
                         double omega, int chebyshev, double rho, double* Xf, double* hist, int* n_hist,
                         int* diverged) {
    if (!Bf || !X0f || !Xf) return fail(VKPD_EINVAL, "null buffer");
    CTX_CALL(aj_refine(Bf, X0f, k, sweeps, aggregation, omega, chebyshev, rho, Xf, hist, n_hist, diverged));
}
int vkpd_power_rho(vkpd_ctx* ctx, double omega, int iters, const double* v0, double* rho) {
    if (!rho) return fail(VKPD_EINVAL, "null buffer");
    CTX_CALL(power_rho(omega, iters, v0, rho));
}
int vkpd_cms_set_basis(vkpd_ctx* ctx, int m, const double* T, const double* Kred_inv) {
    if (m > 0 && (!T || !Kred_inv)) return fail(VKPD_EINVAL, "null buffer");
    CTX_CALL(cms_set_basis(m, T, Kred_inv));
}
int vkpd_cms_set_blocks(vkpd_ctx* ctx, int n_dom, const int64_t* row_ptr, const int64_t* rows, const int64_t* col_ptr,
                        const int64_t* colmap, const double* A, int n_modes, int64_t nb, const int64_t* boundary,
                        const double* Kred_inv) {
    if (n_dom < 0 || (n_dom > 0 && (!row_ptr || !col_ptr)) || (nb > 0 && !boundary) || !Kred_inv)
        return fail(VKPD_EINVAL, "null buffer");
    CTX_CALL(cms_set_blocks(n_dom, row_ptr, rows, col_ptr, colmap, A, n_modes, nb, boundary, Kred_inv));
}
int vkpd_cms_timing(vkpd_ctx* ctx, double* apply_ms, double* sweeps_ms) { CTX_CALL(cms_timing(apply_ms, sweeps_ms)); }
int vkpd_step_cms(vkpd_ctx* ctx, int iterations, double damping, int sweeps, int aggregation, double omega,
                  int chebyshev, double rho, int* failed_iter) {
    CTX_CALL(step_cms(iterations, damping, sweeps, aggregation, omega, chebyshev, rho, failed_iter));
}
int vkpd_time_local(vkpd_ctx* ctx, int reps, double* local_ms, double* pass_ms) {
    CTX_CALL(time_local(reps, local_ms, pass_ms));
}
int vkpd_cms_solve(vkpd_ctx* ctx, const double* B, const double* P, int k, int sweeps, int aggregation, double omega,
                   int chebyshev, double rho, double* X) {
    if (!B || !X) return fail(VKPD_EINVAL, "null buffer");
    CTX_CALL(cms_solve(B, P, k, sweeps, aggregation, omega, chebyshev, rho, X));
}
int vkpd_get_stats(vkpd_ctx* ctx, vkpd_stats* st) {
    if (!st) return fail(VKPD_EINVAL, "null stats");
    CTX_CALL(stats(st));
}

int vkpd_projection_jacobians(int64_t n, const double* F, double* JR, double* JV) {
    if (n < 0 || (n > 0 && (!F || !JR || !JV))) return fail(VKPD_EINVAL, "bad arguments");
    int count = 0;
    if (vkpd_device_count(&count) != VKPD_OK || count == 0)
        return fail(VKPD_ECUDA, "no CUDA device available (the vkpd library has no CPU path)");
    for (int64_t i = 0; i < 9 * n; ++i)
        if (!std::isfinite(F[i])) return fail(VKPD_EINVAL, "non-finite deformation gradient in batch");
    if (n == 0) return VKPD_OK;
    DBuf<double> dF, dR, dV;
    CK(dF.alloc((size_t)9 * n)); CK(dR.alloc((size_t)81 * n)); CK(dV.alloc((size_t)81 * n));
    CK(cudaMemcpy(dF.p, F, sizeof(double) * 9 * n, cudaMemcpyHostToDevice));
    vk::k_proj_jacobians<<<cdiv(n, 128), 128>>>((int)n, dF.p, dR.p, dV.p);
    CK(cudaGetLastError());
    CK(cudaMemcpy(JR, dR.p, sizeof(double) * 81 * n, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(JV, dV.p, sizeof(double) * 81 * n, cudaMemcpyDeviceToHost));
    return VKPD_OK;
}

int vkpd_batch_projections(int precision, int64_t n, const double* F, double* R, double* V,
                           unsigned int* n_robust, unsigned int* n_fallback) {
    if (n < 0 || (n > 0 && (!F || !R || !V))) return fail(VKPD_EINVAL, "bad arguments");
    if (precision != VKPD_FP32 && precision != VKPD_FP64) return fail(VKPD_EINVAL, "precision must be 32 or 64");
    int count = 0;
    if (vkpd_device_count(&count) != VKPD_OK || count == 0)
        return fail(VKPD_ECUDA, "no CUDA device available (the vkpd library has no CPU path)");
    for (int64_t i = 0; i < 9 * n; ++i)
        if (!std::isfinite(F[i])) return fail(VKPD_EINVAL, "non-finite deformation gradient in batch");
    if (n == 0) return VKPD_OK;
    DBuf<double> dF, dR, dV;
    DBuf<vk::ProjStats> st;
    CK(dF.alloc((size_t)9 * n)); CK(dR.alloc((size_t)9 * n)); CK(dV.alloc((size_t)9 * n));
    CK(st.alloc(1));
    CK(cudaMemset(st.p, 0, sizeof(vk::ProjStats)));
    CK(cudaMemcpy(dF.p, F, sizeof(double) * 9 * n, cudaMemcpyHostToDevice));
    if (precision == VKPD_FP32) vk::k_project<float><<<cdiv(n, 128), 128>>>((int)n, dF.p, dR.p, dV.p, st.p);
    else vk::k_project<double><<<cdiv(n, 128), 128>>>((int)n, dF.p, dR.p, dV.p, st.p);
    CK(cudaGetLastError());
    CK(cudaMemcpy(R, dR.p, sizeof(double) * 9 * n, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(V, dV.p, sizeof(double) * 9 * n, cudaMemcpyDeviceToHost));
    vk::ProjStats hs;
    CK(cudaMemcpy(&hs, st.p, sizeof(hs), cudaMemcpyDeviceToHost));
    if (n_robust) *n_robust = hs.robust;
    if (n_fallback) *n_fallback = hs.fallback;
    return VKPD_OK;
}

int vkpd_hess_create(const vkpd_mesh_desc* mesh, int device, vkpd_hess** out) {
    if (!mesh || !out) return fail(VKPD_EINVAL, "null argument");
    if (!mesh->tets || !mesh->shape_grad || !mesh->volume || !mesh->gamma_s || !mesh->gamma_v)
        return fail(VKPD_EINVAL, "missing mesh array");
    if (mesh->n_pins > 0 && !mesh->pins) return fail(VKPD_EINVAL, "missing pin array");
    int count = 0;
    if (vkpd_device_count(&count) != VKPD_OK || count == 0)
        return fail(VKPD_ECUDA, "no CUDA device available (the vkpd library has no CPU path)");
    if (device < 0 || device >= count) return fail(VKPD_EINVAL, "bad device ordinal");
    DeviceGuard guard_(device);
    std::unique_ptr<vkpd_hess> h(new vkpd_hess);
    int rc = h->impl.init(mesh, device);
    if (rc != VKPD_OK) return rc;
    *out = h.release();
    return VKPD_OK;
}
void vkpd_hess_destroy(vkpd_hess* h) {
    if (h) {
        DeviceGuard guard_(h->impl.device);
        delete h;
    }
}
#define HESS_CALL(expr)                                  \
    do {                                                 \
        if (!h) return fail(VKPD_EINVAL, "null context"); \
        DeviceGuard guard_(h->impl.device);              \
        return h->impl.expr;                             \
    } while (0)
int vkpd_hess_set_gammas(vkpd_hess* h, const double* gs, const double* gv) { HESS_CALL(set_gammas(gs, gv)); }
int vkpd_hess_energy_grad(vkpd_hess* h, const double* x, double* energy, double* grad) {
    HESS_CALL(energy_grad(x, energy, grad));
}
int vkpd_hess_gamma_jt(vkpd_hess* h, const double* x, const double* lam, double* out) {
    HESS_CALL(gamma_jt(x, lam, out));
}
int vkpd_hess_linearize(vkpd_hess* h, const double* x) { HESS_CALL(linearize(x)); }
int vkpd_hess_csr(vkpd_hess* h, int64_t* indptr, int64_t* indices, double* data, int64_t* nnz) {
    if (!nnz) return fail(VKPD_EINVAL, "null nnz");
    HESS_CALL(csr(indptr, indices, data, nnz));
}
int vkpd_hess_apply(vkpd_hess* h, double mass_scale, const double* p, double* y) {
    HESS_CALL(apply(mass_scale, p, y));
}
int vkpd_hess_solve(vkpd_hess* h, double mass_scale, double ridge, const double* b, double* x, double tol,
                    int max_iters, int* iters, double* relres) {
    HESS_CALL(solve(mass_scale, ridge, b, x, tol, max_iters, iters, relres));
}

}  // extern "C"

// Host context of the fitting-side second-order machinery (hessian.cuh), float64,
// caller node order.  Included by vkpd.cu inside its anonymous namespace (uses DBuf,
// CK, fail, cdiv).
//
//   energy_grad   elastic_energy + elastic_gradient          (pdsolver.py:72-97)
//   gamma_jt      gamma_jacobian(mesh, x)^T lam              (fitting.py:172-190)
//   linearize     the per-tet 9x9 blocks of exact_elastic_hessian at x (pdsolver.py:100-118)
//   csr           exact_elastic_hessian as a CSR matrix (3nV x 3nV)
//   apply         (H + s M/dt^2) p on all dofs
//   solve         (H + s M/dt^2 + ridge I)_ff d = b_f by preconditioned MINRES: the exact
//                 Newton step of newton_polish (pdsolver.py:402-414) and the adjoint solve of
//                 adjoint_gradient (fitting.py:227-235)

struct HessCtx {
    int n = 0, nE = 0, nP = 0, device = 0;
    double dt = 0.0;
    cudaStream_t stream = nullptr;
    DBuf<int4> tets, slot4;
    DBuf<double> G, w, vol, corner, mdt2, M, hdiag, He;
    DBuf<int> inc_ptr, inc_code, nb_ptr, nb_col;
    DBuf<unsigned char> pinned;
    std::vector<int> nbptr_h, nbcol_h;
    std::vector<unsigned char> pinned_h;
    std::vector<double> mdt2_h;
    DBuf<long long> row_ptr;
    bool linearized = false;
    // work vectors (3n)
    DBuf<double> xv, pv, yv, shift, energy, partials, scal;
    DBuf<double> r1, r2, my, mv, mw, mw2, mx, mav, mb, dinv;
    DBuf<vk::hs::MinresState> st;

    ~HessCtx() {
        if (stream) cudaStreamDestroy(stream);
    }

    vk::hs::Args args() const {
        vk::hs::Args a;
        a.n = n; a.nE = nE; a.tets = tets.p; a.G = G.p; a.w = w.p; a.vol = vol.p; a.slot4 = slot4.p;
        a.corner = corner.p;
        return a;
    }

    int init(const vkpd_mesh_desc* d, int dev) {
        device = dev;
        n = (int)d->n_nodes;
        nE = (int)d->n_tets;
        nP = (int)d->n_pins;
        dt = d->dt;
        if (n <= 0 || nE <= 0) return fail(VKPD_EINVAL, "empty mesh");
        if (d->n_nodes > (1ll << 29) || 4ll * d->n_tets > (1ll << 31) - 1)
            return fail(VKPD_EINVAL, "mesh too large for 32-bit indexing");
        if (!(dt > 0.0)) return fail(VKPD_EINVAL, "dt must be positive");
        if (d->node_mass == nullptr) return fail(VKPD_EINVAL, "mesh node masses not lumped yet");
        pinned_h.assign(n, 0);
        for (int k = 0; k < nP; ++k) {
            const int64_t id = d->pins[k];
            if (id < 0 || id >= n) return fail(VKPD_EINVAL, "pin index out of range");
            pinned_h[id] = 1;
        }
        std::vector<int4> tets_h(nE);
        for (int e = 0; e < nE; ++e) {
            if (d->gamma_s[e] < 0.0 || d->gamma_v[e] < 0.0) return fail(VKPD_EINVAL, "negative material coefficient");
            if (!(d->volume[e] > 0.0)) return fail(VKPD_EINVAL, "non-positive element volume");
            int id[4];
            for (int k = 0; k < 4; ++k) {
                const int64_t v = d->tets[4 * (size_t)e + k];
                if (v < 0 || v >= n) return fail(VKPD_EINVAL, "tet node index out of range");
                id[k] = (int)v;
            }
            tets_h[e] = make_int4(id[0], id[1], id[2], id[3]);
        }
        // incidence runs in tet order (np.add.at order) and each corner's slot
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
        // node neighbourhoods (sorted, self included): the CSR block pattern
        nbptr_h.assign(n + 1, 0);
        nbcol_h.clear();
        std::vector<int> s;
        for (int i = 0; i < n; ++i) {
            s.clear();
            s.push_back(i);
            for (int k = iptr[i]; k < iptr[i + 1]; ++k) {
                const int* t = &tets_h[icode[k] % nE].x;
                for (int a = 0; a < 4; ++a) s.push_back(t[a]);
            }
            std::sort(s.begin(), s.end());
            s.erase(std::unique(s.begin(), s.end()), s.end());
            nbcol_h.insert(nbcol_h.end(), s.begin(), s.end());
            nbptr_h[i + 1] = (int)nbcol_h.size();
        }
        std::vector<double> Gp((size_t)12 * nE);
        for (int e = 0; e < nE; ++e)
            for (int k = 0; k < 12; ++k) Gp[(size_t)k * nE + e] = d->shape_grad[(size_t)12 * e + k];
        mdt2_h.resize(n);
        for (int j = 0; j < n; ++j) mdt2_h[j] = d->node_mass[j] / (dt * dt);

        CK(cudaSetDevice(device));
        CK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
        cudaStream_t st_ = stream;
        CK(tets.alloc(nE)); CK(tets.upload(tets_h.data(), nE, st_));
        CK(slot4.alloc(nE)); CK(slot4.upload(slot_h.data(), nE, st_));
        CK(G.alloc(Gp.size())); CK(G.upload(Gp.data(), Gp.size(), st_));
        CK(vol.alloc(nE)); CK(vol.upload(d->volume, nE, st_));
        CK(w.alloc((size_t)2 * nE));
        CK(inc_ptr.alloc(n + 1)); CK(inc_ptr.upload(iptr.data(), n + 1, st_));
        CK(inc_code.alloc(icode.size())); CK(inc_code.upload(icode.data(), icode.size(), st_));
        CK(nb_ptr.alloc(n + 1)); CK(nb_ptr.upload(nbptr_h.data(), n + 1, st_));
        CK(nb_col.alloc(nbcol_h.size())); CK(nb_col.upload(nbcol_h.data(), nbcol_h.size(), st_));
        CK(pinned.alloc(n)); CK(pinned.upload(pinned_h.data(), n, st_));
        CK(mdt2.alloc(n)); CK(mdt2.upload(mdt2_h.data(), n, st_));
        CK(corner.alloc((size_t)3 * 4 * nE));
        const size_t m = (size_t)3 * n;
        for (DBuf<double>* b : {&xv, &pv, &yv, &r1, &r2, &my, &mv, &mw, &mw2, &mx, &mav, &mb, &dinv, &hdiag})
            CK(b->alloc(m));
        CK(shift.alloc(n));
        CK(energy.alloc(nE));
        CK(partials.alloc(vk::hs::kMrBlocks));
        CK(scal.alloc(4));
        CK(st.alloc(1));
        return set_gammas(d->gamma_s, d->gamma_v);
    }

    int set_gammas(const double* gs, const double* gv) {
        if (!gs || !gv) return fail(VKPD_EINVAL, "null material array");
        for (int e = 0; e < nE; ++e)
            if (gs[e] < 0.0 || gv[e] < 0.0) return fail(VKPD_EINVAL, "negative material coefficient");
        CK(cudaMemcpyAsync(w.p, gs, sizeof(double) * nE, cudaMemcpyHostToDevice, stream));
        CK(cudaMemcpyAsync(w.p + nE, gv, sizeof(double) * nE, cudaMemcpyHostToDevice, stream));
        CK(cudaStreamSynchronize(stream));
        linearized = false;
        return VKPD_OK;
    }

    int upload3(const double* h, double* dptr) {
        for (size_t i = 0; i < (size_t)3 * n; ++i)
            if (!std::isfinite(h[i])) return fail(VKPD_EINVAL, "non-finite node positions");
        CK(cudaMemcpyAsync(dptr, h, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, stream));
        return VKPD_OK;
    }

    int energy_grad(const double* x, double* E, double* grad) {
        if (!x) return fail(VKPD_EINVAL, "null positions");
        if (int rc = upload3(x, xv.p)) return rc;
        vk::hs::k_hs_eval<<<cdiv(nE, 128), 128, 0, stream>>>(args(), xv.p, grad != nullptr, energy.p, nullptr,
                                                             nullptr);
        CK(cudaGetLastError());
        if (E) {
            vk::hs::k_hs_sum_partials<<<vk::hs::kMrBlocks, 256, 0, stream>>>(nE, energy.p, partials.p);
            vk::hs::k_hs_sum_final<<<1, 1, 0, stream>>>(vk::hs::kMrBlocks, partials.p, scal.p);
            CK(cudaGetLastError());
            CK(cudaMemcpyAsync(E, scal.p, sizeof(double), cudaMemcpyDeviceToHost, stream));
        }
        if (grad) {
            vk::hs::k_hs_gather<<<cdiv(n, 256), 256, 0, stream>>>(n, inc_ptr.p, corner.p, nullptr, nullptr, nullptr,
                                                                  yv.p, nullptr);
            CK(cudaGetLastError());
            CK(cudaMemcpyAsync(grad, yv.p, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, stream));
        }
        CK(cudaStreamSynchronize(stream));
        return VKPD_OK;
    }

    int gamma_jt(const double* x, const double* lam, double* out) {
        if (!x || !lam || !out) return fail(VKPD_EINVAL, "null argument");
        if (int rc = upload3(x, xv.p)) return rc;
        if (int rc = upload3(lam, pv.p)) return rc;
        DBuf<double> jt;
        CK(jt.alloc((size_t)2 * nE));
        vk::hs::k_hs_eval<<<cdiv(nE, 128), 128, 0, stream>>>(args(), xv.p, 0, nullptr, pv.p, jt.p);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(out, jt.p, sizeof(double) * 2 * nE, cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        return VKPD_OK;
    }

    int linearize(const double* x) {
        if (!x) return fail(VKPD_EINVAL, "null positions");
        if (int rc = upload3(x, xv.p)) return rc;
        if (!M.p) CK(M.alloc((size_t)81 * nE));
        vk::hs::k_hs_linearize<<<cdiv(nE, 64), 64, 0, stream>>>(args(), xv.p, M.p);
        CK(cudaGetLastError());
        vk::hs::k_hs_diag<<<cdiv(nE, 128), 128, 0, stream>>>(args(), M.p);
        vk::hs::k_hs_gather<<<cdiv(n, 256), 256, 0, stream>>>(n, inc_ptr.p, corner.p, nullptr, nullptr, nullptr,
                                                              hdiag.p, nullptr);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(stream));
        linearized = true;
        return VKPD_OK;
    }

    int csr(int64_t* indptr, int64_t* indices, double* data, int64_t* nnz) {
        if (!linearized) return fail(VKPD_EINVAL, "Hessian not linearized (call vkpd_hess_linearize)");
        const int64_t total = (int64_t)9 * nbptr_h[n];
        if (!indptr) { *nnz = total; return VKPD_OK; }
        if (*nnz < total) return fail(VKPD_EINVAL, "CSR buffers too small");
        std::vector<long long> rp((size_t)3 * n + 1);
        rp[0] = 0;
        for (int i = 0; i < n; ++i) {
            const int deg = nbptr_h[i + 1] - nbptr_h[i];
            for (int c = 0; c < 3; ++c) {
                const long long r0 = rp[(size_t)3 * i + c];
                rp[(size_t)3 * i + c + 1] = r0 + 3 * deg;
                int64_t k = r0;
                for (int q = nbptr_h[i]; q < nbptr_h[i + 1]; ++q)
                    for (int dd = 0; dd < 3; ++dd) indices[k++] = 3 * (int64_t)nbcol_h[q] + dd;
            }
        }
        for (size_t r = 0; r < rp.size(); ++r) indptr[r] = rp[r];
        CK(row_ptr.alloc(rp.size()));
        CK(row_ptr.upload(rp.data(), rp.size(), stream));
        if (!He.p) CK(He.alloc((size_t)144 * nE));
        DBuf<double> dd;
        CK(dd.alloc(total));
        vk::hs::k_hs_block<<<cdiv(nE, 64), 64, 0, stream>>>(args(), M.p, He.p);
        vk::hs::k_hs_csr_fill<<<cdiv(3 * n, 128), 128, 0, stream>>>(n, nE, inc_ptr.p, inc_code.p, tets.p, nb_ptr.p,
                                                                    nb_col.p, He.p, row_ptr.p, dd.p);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(data, dd.p, sizeof(double) * total, cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        *nnz = total;
        return VKPD_OK;
    }

    int set_shift(double mass_scale, double ridge) {
        std::vector<double> sh(n);
        for (int j = 0; j < n; ++j) sh[j] = mass_scale * mdt2_h[j] + ridge;
        CK(cudaMemcpyAsync(shift.p, sh.data(), sizeof(double) * n, cudaMemcpyHostToDevice, stream));
        CK(cudaStreamSynchronize(stream));
        return VKPD_OK;
    }

    int apply(double mass_scale, const double* p, double* y) {
        if (!linearized) return fail(VKPD_EINVAL, "Hessian not linearized (call vkpd_hess_linearize)");
        if (!p || !y) return fail(VKPD_EINVAL, "null argument");
        if (int rc = set_shift(mass_scale, 0.0)) return rc;
        CK(cudaMemcpyAsync(pv.p, p, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, stream));
        vk::hs::k_hs_apply<<<cdiv(nE, 128), 128, 0, stream>>>(args(), M.p, pv.p, nullptr);
        vk::hs::k_hs_gather<<<cdiv(n, 256), 256, 0, stream>>>(n, inc_ptr.p, corner.p, nullptr, shift.p, pv.p, yv.p,
                                                              nullptr);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(y, yv.p, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        return VKPD_OK;
    }

    // (H + s M/dt^2 + ridge I)_ff x_f = b_f; pinned dofs of b ignored, x = 0 there
    int solve(double mass_scale, double ridge, const double* b, double* x, double tol, int max_iters, int* iters,
              double* relres) {
        if (!linearized) return fail(VKPD_EINVAL, "Hessian not linearized (call vkpd_hess_linearize)");
        if (!b || !x) return fail(VKPD_EINVAL, "null argument");
        if (!(tol > 0.0)) tol = 1e-12;
        if (max_iters <= 0) max_iters = 10 * 3 * n + 100;
        for (size_t i = 0; i < (size_t)3 * n; ++i)
            if (!std::isfinite(b[i])) return fail(VKPD_EINVAL, "non-finite right-hand side");
        if (int rc = set_shift(mass_scale, ridge)) return rc;
        // masked b and the |diag| Jacobi preconditioner on the free dofs
        std::vector<double> bm((size_t)3 * n), hd((size_t)3 * n), di((size_t)3 * n);
        CK(cudaMemcpyAsync(hd.data(), hdiag.p, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        for (int i = 0; i < n; ++i)
            for (int c = 0; c < 3; ++c) {
                const size_t k = (size_t)3 * i + c;
                if (pinned_h[i]) { bm[k] = 0.0; di[k] = 0.0; continue; }
                bm[k] = b[k];
                const double dg = std::fabs(hd[k] + mass_scale * mdt2_h[i] + ridge);
                di[k] = dg > 0.0 ? 1.0 / dg : 1.0;
            }
        CK(cudaMemcpyAsync(mb.p, bm.data(), sizeof(double) * 3 * n, cudaMemcpyHostToDevice, stream));
        CK(cudaMemcpyAsync(dinv.p, di.data(), sizeof(double) * 3 * n, cudaMemcpyHostToDevice, stream));
        namespace H = vk::hs;
        const long long m = 3ll * n;
        const int B = H::kMrBlocks;
        H::k_mr_init<<<B, 256, 0, stream>>>(m, mb.p, dinv.p, r1.p, r2.p, my.p, mx.p, mw.p, mw2.p, partials.p);
        H::k_mr_init_scalar<<<1, 1, 0, stream>>>(st.p, partials.p, tol);
        H::k_mr_v<<<B, 256, 0, stream>>>(m, st.p, my.p, mv.p);
        CK(cudaGetLastError());
        const int* done = &st.p->done;
        H::MinresState hst{};
        int it = 0;
        while (it < max_iters) {
            const int chunk = std::min(16, max_iters - it);
            for (int k = 0; k < chunk; ++k, ++it) {
                H::k_hs_apply<<<cdiv(nE, 128), 128, 0, stream>>>(args(), M.p, mv.p, done);
                H::k_hs_gather<<<cdiv(n, 256), 256, 0, stream>>>(n, inc_ptr.p, corner.p, pinned.p, shift.p, mv.p,
                                                                 mav.p, done);
                H::k_mr_a<<<B, 256, 0, stream>>>(m, st.p, mav.p, mv.p, r1.p, my.p, partials.p);
                H::k_mr_s1<<<1, 1, 0, stream>>>(st.p, partials.p);
                H::k_mr_b<<<B, 256, 0, stream>>>(m, st.p, my.p, r1.p, r2.p, dinv.p, partials.p);
                H::k_mr_s2<<<1, 1, 0, stream>>>(st.p, partials.p, it);
                H::k_mr_c<<<B, 256, 0, stream>>>(m, st.p, it, mv.p, my.p, mw.p, mw2.p, mx.p);
            }
            CK(cudaGetLastError());
            CK(cudaMemcpyAsync(&hst, st.p, sizeof(hst), cudaMemcpyDeviceToHost, stream));
            CK(cudaStreamSynchronize(stream));
            if (hst.done) break;
        }
        // true relative residual |b_f - A_ff x_f| / |b_f|
        H::k_hs_apply<<<cdiv(nE, 128), 128, 0, stream>>>(args(), M.p, mx.p, nullptr);
        H::k_hs_gather<<<cdiv(n, 256), 256, 0, stream>>>(n, inc_ptr.p, corner.p, pinned.p, shift.p, mx.p, mav.p,
                                                         nullptr);
        CK(cudaGetLastError());
        std::vector<double> ax((size_t)3 * n);
        CK(cudaMemcpyAsync(ax.data(), mav.p, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, stream));
        CK(cudaMemcpyAsync(x, mx.p, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        double rn = 0.0, bn = 0.0;
        for (size_t k = 0; k < bm.size(); ++k) {
            const double r = bm[k] - ax[k];
            rn += r * r;
            bn += bm[k] * bm[k];
        }
        if (iters) *iters = hst.itn;
        if (relres) *relres = bn > 0.0 ? std::sqrt(rn / bn) : std::sqrt(rn);
        for (size_t k = 0; k < bm.size(); ++k)
            if (!std::isfinite(x[k])) return fail(VKPD_ENONFINITE, "exact Hessian solve produced non-finite values");
        return VKPD_OK;
    }
};

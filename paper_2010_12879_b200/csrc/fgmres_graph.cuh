// FGMRES(m) with the whole restart cycle on the device (included by solve.cu
// inside its anonymous namespace, after the block-Arnoldi kernels).
//
// Same algorithm and per-rhs semantics as fgmres_batch (right-preconditioned
// FGMRES(m), linsolve.py:200-298: true residual at every restart and at exit,
// inner stop on |g_j|/|b| <= tol or hnorm = 0, max_iters flagged not raised,
// non-finite values -> SolverError), with the Givens rotations, the
// convergence decisions and the least-squares back substitution moved to
// single-thread device kernels, so a restart cycle needs no host round trip:
//
//   cycle graph = r = b - A x, |r|              (true residual)
//                 k_fg_restart                  (per-rhs beta, active, g, H = 0)
//                 v_0 = r / beta
//                 IF(step 0) { V-cycle z_0 = M^-1 v_0, w = A z_0, Gram-corrected
//                              CGS2 against v_0..v_j, |w|, k_fg_givens, v_1 = w/h }
//                 k_fg_gate                     (condition of the next step)
//                 IF(step 1) { ... }  ...  IF(step m-1) { ... }
//                 k_fg_lsq                      (y = H^-1 g per rhs)
//                 x += Z y
//
// Each step j is its own conditional body with the basis pointers V_j, Z_j
// fixed at capture, so the per-step kernels are exactly the host loop's.  The
// host launches one cycle graph per restart and reads three integers back.

struct FgDev {
    double H[2][32 * 31];   // [c][i * m + j] (upper Hessenberg after rotations)
    double cs[2][32], sn[2][32], g[2][33];
    double bnorm[2];
    double tol;
    int active[2], done[2], jc[2], its_c[2];
    int its, max_iters, status, cont, any_active, m;
};

inline void fg_small_alloc(Amg &h) {
    if (h.fg_state.n == 0) {
        h.fg_state.alloc((sizeof(FgDev) + 7) / 8);
        h.fg_y.alloc(2 * 32);
        h.fg_jc.alloc(2);
        h.fg_gram.alloc((size_t)2 * 32 * 32);
    }
}

template <int R>
__global__ void k_fg_init(FgDev *st, const double *bb, double tol, int max_iters, int m) {
    if (threadIdx.x != 0) return;
    st->its = 0;
    st->status = 0;
    st->cont = 0;
    st->any_active = 0;
    st->tol = tol;
    st->max_iters = max_iters;
    st->m = m;
    for (int c = 0; c < 2; ++c) {
        const double bn = c < R ? sqrt(bb[c]) : 0.0;
        st->bnorm[c] = bn;
        st->done[c] = c < R ? (bn == 0.0) : 1;
        st->active[c] = 0;
        st->jc[c] = 0;
        st->its_c[c] = 0;
    }
}

// restart (linsolve.py:244-248): beta = |r|, converged on the true residual,
// g = beta e_1, H = 0, scale factors 1 / beta; condition of step 0
template <int R>
__global__ void k_fg_restart(FgDev *st, const double *rr, double *mult, cudaGraphConditionalHandle h0) {
    const int m = st->m;
    for (int t = threadIdx.x; t < R * (m + 1) * m; t += blockDim.x) st->H[t / ((m + 1) * m)][t % ((m + 1) * m)] = 0.0;
    if (threadIdx.x == 0) {
        int any = 0;
        for (int c = 0; c < R; ++c) {
            const double beta = sqrt(rr[c]);
            const double rel = st->bnorm[c] > 0 ? beta / st->bnorm[c] : 0.0;
            if (rel <= st->tol) st->done[c] = 1;
            st->active[c] = !st->done[c];
            any = any || st->active[c];
            for (int i = 0; i <= m; ++i) st->g[c][i] = 0.0;
            st->g[c][0] = beta;
            st->jc[c] = 0;
            mult[c] = st->active[c] ? 1.0 / beta : 0.0;
        }
        st->any_active = any;
        st->cont = any && st->its < st->max_iters && st->status == 0;
        cudaGraphSetConditional(h0, st->cont);
    }
}

// one Arnoldi step's bookkeeping per rhs (the host loop of fgmres_batch):
// H column from the orthogonalisation coefficients, previous rotations,
// the new rotation, g, the residual estimate and the stop decision
template <int R>
__global__ void k_fg_givens(FgDev *st, const double *hcol, const double *nn, int j, double *mult, double *trace) {
    if (threadIdx.x != 0) return;
    const int m = st->m;
    const int its = ++st->its;
    bool more = false;
    for (int c = 0; c < R; ++c) {
        if (!st->active[c]) { mult[c] = 0.0; continue; }
        ++st->its_c[c];
        const double hn = sqrt(nn[c]);
        if (!isfinite(hn)) { st->status = 1; mult[c] = 0.0; continue; }
        double *Hc = st->H[c];
        double *cs = st->cs[c], *sn = st->sn[c], *g = st->g[c];
        for (int i = 0; i <= j; ++i) Hc[i * m + j] = hcol[i * R + c];
        for (int i = 0; i < j; ++i) {
            const double u = Hc[i * m + j], v = Hc[(i + 1) * m + j];
            Hc[i * m + j] = __dadd_rn(__dmul_rn(cs[i], u), __dmul_rn(sn[i], v));
            Hc[(i + 1) * m + j] = __dadd_rn(__dmul_rn(-sn[i], u), __dmul_rn(cs[i], v));
        }
        const double hjj = Hc[j * m + j];
        const double den = hypot(hjj, hn);
        if (den == 0.0) { cs[j] = 1.0; sn[j] = 0.0; }
        else { cs[j] = hjj / den; sn[j] = hn / den; }
        Hc[j * m + j] = __dadd_rn(__dmul_rn(cs[j], hjj), __dmul_rn(sn[j], hn));
        g[j + 1] = __dmul_rn(-sn[j], g[j]);
        g[j] = __dmul_rn(cs[j], g[j]);
        st->jc[c] = j + 1;
        const double est = fabs(g[j + 1]) / st->bnorm[c];
        if (trace && its <= st->max_iters) trace[(int64_t)(its - 1) * R + c] = est;
        if (hn == 0.0 || est <= st->tol) {
            st->active[c] = 0;
            mult[c] = 0.0;
        } else {
            mult[c] = 1.0 / hn;
            more = true;
        }
    }
    st->cont = more && st->status == 0 && its < st->max_iters && j + 1 < m;
}

__global__ void k_fg_gate(const FgDev *st, cudaGraphConditionalHandle hnd) {
    cudaGraphSetConditional(hnd, st->cont);
}

// least squares per rhs (back substitution, linsolve.py:288-291)
template <int R>
__global__ void k_fg_lsq(FgDev *st, double *y, int *jc) {
    const int c = threadIdx.x;
    if (c >= R) return;
    const int m = st->m, jj = st->jc[c];
    const double *Hc = st->H[c];
    for (int i = jj - 1; i >= 0; --i) {
        double acc = st->g[c][i];
        for (int k = i + 1; k < jj; ++k) acc = __dsub_rn(acc, __dmul_rn(Hc[i * m + k], y[c * m + k]));
        y[c * m + i] = acc / Hc[i * m + i];
    }
    bool ok = true;
    for (int i = 0; i < jj; ++i) ok = ok && isfinite(y[c * m + i]);
    if (!ok) st->status = 1;
    jc[c] = jj;
}

// the step-j body: exactly the per-step kernels of fgmres_batch
template <int R>
void fg_step(Amg &h, int j, int m, FgDev *st, double *trace, cudaStream_t s) {
    constexpr int NI2 = 4;
    const int64_t n = h.lv[0].nvec;
    double *Vb = h.fg_basis.get(), *Zb = h.fg_prec.get();
    double *w = h.kq.get(), *sc = h.scal.get();
    const int SH1 = S_H, SH2 = S_H + 128, SMUL = S_TMP + 2;
    const int G = grid_for(n, 256, 148 * 16);
    const int nparts = kDotGrid;
    double *vj = Vb + (int64_t)j * n * R, *zj = Zb + (int64_t)j * n * R;
    amg_vcycle(h, vj, zj, R, s);
    level0_apply<R>(h, 0, false, zj, nullptr, w, s);
    for (int i0 = 0; i0 <= j; i0 += NI2) {
        const int ni = std::min(NI2, j + 1 - i0);
        k_mdot2<R, NI2><<<nparts, 256, 0, s>>>(n, n, Vb, i0, ni, w, vj, h.partials.get());
        k_mfinal<<<2 * NI2 * R, 256, 0, s>>>(h.partials.get(), nparts, 2 * NI2 * R, sc + SH1 + 2 * i0 * R);
        SPFD_LAUNCH_CHECK();
    }
    k_gram_step<R, NI2><<<1, 256, 0, s>>>(sc + SH1, j, m, h.fg_gram.get(), sc + SH2);
    k_maxpy<R><<<G, 256, 0, s>>>(n, n, Vb, j + 1, sc + SH2, w);
    SPFD_LAUNCH_CHECK();
    dot<R>(h, n, w, w, S_TMP, F_STORE, s);
    k_fg_givens<R><<<1, 32, 0, s>>>(st, sc + SH2, sc + S_TMP, j, sc + SMUL, trace);
    SPFD_LAUNCH_CHECK();
    if (j + 1 < m) {
        k_scale_r<R><<<G, 256, 0, s>>>(n, sc + SMUL, w, Vb + (int64_t)(j + 1) * n * R);
        SPFD_LAUNCH_CHECK();
    }
}

// Capture the restart-cycle graph for (R, m).  Returns false when capture
// is unavailable (the caller falls back to fgmres_batch).
template <int R>
bool fg_graph_build(Amg &h, int m) {
    const double *b = h.kb.get();   // the graph solves kb -> kx (fixed buffers)
    double *x = h.kx.get();
    if (h.fg_exec[R] && h.fg_exec_m[R] == m) return true;
    if (h.fg_exec[R]) { cudaGraphExecDestroy(h.fg_exec[R]); h.fg_exec[R] = nullptr; }
    if (h.fg_failed[R]) return false;
    if (!h.cap) SPFD_CUDA(cudaStreamCreateWithFlags(&h.cap, cudaStreamNonBlocking));
    if (!h.cap2) SPFD_CUDA(cudaStreamCreateWithFlags(&h.cap2, cudaStreamNonBlocking));
    const int64_t n = h.lv[0].nvec;
    double *sc = h.scal.get(), *r = h.kr.get();
    FgDev *st = reinterpret_cast<FgDev *>(h.fg_state.get());
    double *trace = h.fg_trace.get();
    const int SMUL = S_TMP + 2;
    const int G = grid_for(n, 256, 148 * 16);
    cudaGraph_t g = nullptr;
    SPFD_CUDA(cudaGraphCreate(&g, 0));
    std::vector<cudaGraphConditionalHandle> hnd(m);
    for (int j = 0; j < m; ++j) SPFD_CUDA(cudaGraphConditionalHandleCreate(&hnd[j], g, 0, cudaGraphCondAssignDefault));
    std::string why;
    SPFD_CUDA(cudaStreamBeginCaptureToGraph(h.cap, g, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    try {
        cudaStream_t s = h.cap;
        level0_apply<R>(h, 1, false, x, b, r, s);        // true residual
        dot<R>(h, n, r, r, S_TMP, F_STORE, s);
        SPFD_CUDA(cudaMemsetAsync(h.fg_gram.get(), 0, h.fg_gram.bytes(), s));
        k_fg_restart<R><<<1, 256, 0, s>>>(st, sc + S_TMP, sc + SMUL, hnd[0]);
        k_scale_r<R><<<G, 256, 0, s>>>(n, sc + SMUL, r, h.fg_basis.get());
        SPFD_LAUNCH_CHECK();
        for (int j = 0; j < m; ++j) {
            cudaStreamCaptureStatus cst;
            cudaGraph_t cg;
            const cudaGraphNode_t *deps = nullptr;
            size_t ndeps = 0;
            SPFD_CUDA(cudaStreamGetCaptureInfo(s, &cst, nullptr, &cg, &deps, &ndeps));
            cudaGraphNodeParams np{};
            np.type = cudaGraphNodeTypeConditional;
            np.conditional.handle = hnd[j];
            np.conditional.type = cudaGraphCondTypeIf;
            np.conditional.size = 1;
            cudaGraphNode_t node;
            SPFD_CUDA(cudaGraphAddNode(&node, cg, deps, ndeps, &np));
            cudaGraph_t body = np.conditional.phGraph_out[0];
            SPFD_CUDA(cudaStreamBeginCaptureToGraph(h.cap2, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
            std::string inner;
            try {
                fg_step<R>(h, j, m, st, trace, h.cap2);
            } catch (const std::exception &e) {
                inner = e.what();
            }
            cudaGraph_t bout = nullptr;
            cudaError_t ec = cudaStreamEndCapture(h.cap2, &bout);
            if (!inner.empty()) throw std::runtime_error(inner);
            if (ec != cudaSuccess) throw std::runtime_error(std::string("step capture: ") + cudaGetErrorString(ec));
            SPFD_CUDA(cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies));
            if (j + 1 < m) {
                k_fg_gate<<<1, 1, 0, s>>>(st, hnd[j + 1]);
                SPFD_LAUNCH_CHECK();
            }
        }
        k_fg_lsq<R><<<1, 32, 0, s>>>(st, h.fg_y.get(), h.fg_jc.get());
        k_combine_r<R><<<G, 256, 0, s>>>(n, n, m, h.fg_jc.get(), h.fg_y.get(), h.fg_prec.get(), x);
        SPFD_LAUNCH_CHECK();
    } catch (const std::exception &e) {
        why = e.what();
    }
    cudaGraph_t out = nullptr;
    cudaError_t ec = cudaStreamEndCapture(h.cap, &out);
    cudaGraphExec_t exec = nullptr;
    if (why.empty() && ec == cudaSuccess) {
        ec = cudaGraphInstantiate(&exec, g, 0);
        if (ec != cudaSuccess) why = std::string("instantiate: ") + cudaGetErrorString(ec);
    } else if (why.empty()) {
        why = std::string("end capture: ") + cudaGetErrorString(ec);
    }
    cudaGetLastError();
    if (!why.empty()) {
        if (getenv("SPFD_DEBUG")) fprintf(stderr, "[spfd] FGMRES graph capture failed (%s): host loop\n", why.c_str());
        h.fg_failed[R] = true;
        return false;
    }
    cudaGraphDestroy(g);
    h.fg_exec[R] = exec;
    h.fg_exec_m[R] = m;
    return true;
}

template <int R>
spfd_report fgmres_batch(Amg &h, const double *b, double *x, const spfd_config &cfg, double *h_trace,
                         cudaStream_t s);

// SPFD_FGMRES_GRAPH=0 selects the host-driven loop (fgmres_batch); read per
// solve so tests can A/B the two
bool fgmres_graph_enabled() {
    const char *e = getenv("SPFD_FGMRES_GRAPH");
    return !(e && std::string(e) == "0");
}

template <int R>
spfd_report fgmres_graph(Amg &h, const double *b_in, double *x_out, const spfd_config &cfg, double *h_trace,
                         cudaStream_t s) {
    spfd_report rep{};
    double *b = h.kb.get(), *x = h.kx.get();
    const int64_t n = h.lv[0].nvec;
    const int m = cfg.restart;
    SPFD_CHECK(m >= 1 && m <= 31, SPFD_EINVAL, "restart must be in [1, 31] for the device FGMRES");
    if (h.fg_m < m || h.fg_R < R) {
        amg_drop_graphs(h);
        h.fg_basis.alloc((int64_t)(m + 1) * n * R);
        h.fg_prec.alloc((int64_t)m * n * R);
        h.fg_m = m;
        h.fg_R = R;
    }
    fg_small_alloc(h);
    if (h.fg_trace_cap < (int64_t)cfg.max_iters) {
        amg_drop_graphs(h);
        h.fg_trace_cap = std::max<int64_t>(cfg.max_iters, 1024);
        h.fg_trace.alloc(h.fg_trace_cap * 2);
    }
    double *sc = h.scal.get();
    if (b_in != b) SPFD_CUDA(cudaMemcpyAsync(b, b_in, n * R * sizeof(double), cudaMemcpyDeviceToDevice, s));
    SPFD_CUDA(cudaMemsetAsync(x, 0, n * R * sizeof(double), s));
    SPFD_CUDA(cudaMemsetAsync(x_out, 0, n * R * sizeof(double), s));
    SPFD_CUDA(cudaMemsetAsync(sc, 0, S_END * sizeof(double), s));
    dot<R>(h, n, b, b, S_BB, F_STORE, s);
    double hb[R];
    SPFD_CUDA(cudaMemcpyAsync(hb, sc + S_BB, R * sizeof(double), cudaMemcpyDeviceToHost, s));
    SPFD_CUDA(cudaStreamSynchronize(s));
    double bnorm[R];
    bool all = true;
    for (int c = 0; c < R; ++c) {
        bnorm[c] = std::sqrt(hb[c]);
        if (!std::isfinite(bnorm[c])) { rep.status = SPFD_ENONFINITE; return rep; }
        all = all && bnorm[c] == 0.0;
        rep.rel_residual[c] = 0.0;
    }
    if (all) { rep.converged = 1; return rep; }
    if (cfg.max_iters > 0 && !fg_graph_build<R>(h, m)) return fgmres_batch<R>(h, b_in, x_out, cfg, h_trace, s);
    FgDev *st = reinterpret_cast<FgDev *>(h.fg_state.get());
    k_fg_init<R><<<1, 32, 0, s>>>(st, sc + S_BB, cfg.rel_tol, cfg.max_iters, m);
    SPFD_LAUNCH_CHECK();
    int hs[3];  // its, status, any_active
    int its = 0;
    while (its < cfg.max_iters) {
        SPFD_CUDA(cudaEventRecord(h.ev_alpha, s));
        SPFD_CUDA(cudaStreamWaitEvent(h.cap, h.ev_alpha, 0));
        SPFD_CUDA(cudaGraphLaunch(h.fg_exec[R], h.cap));
        SPFD_CUDA(cudaEventRecord(h.ev_x, h.cap));
        SPFD_CUDA(cudaStreamWaitEvent(s, h.ev_x, 0));
        SPFD_CUDA(cudaMemcpyAsync(&hs[0], &st->its, sizeof(int), cudaMemcpyDeviceToHost, s));
        SPFD_CUDA(cudaMemcpyAsync(&hs[1], &st->status, sizeof(int), cudaMemcpyDeviceToHost, s));
        SPFD_CUDA(cudaMemcpyAsync(&hs[2], &st->any_active, sizeof(int), cudaMemcpyDeviceToHost, s));
        SPFD_CUDA(cudaStreamSynchronize(s));
        its = hs[0];
        if (hs[1]) { rep.status = SPFD_ENONFINITE; rep.iterations = its; return rep; }  // (x_out = 0)
        if (!hs[2]) break;  // every rhs converged on the true residual at the restart
    }
    // true residual at exit (linsolve.py:296-298)
    level0_apply<R>(h, 1, false, x, b, h.kr.get(), s);
    dot<R>(h, n, h.kr.get(), h.kr.get(), S_TMP, F_STORE, s);
    double rr[R];
    int itc[2];
    SPFD_CUDA(cudaMemcpyAsync(rr, sc + S_TMP, R * sizeof(double), cudaMemcpyDeviceToHost, s));
    SPFD_CUDA(cudaMemcpyAsync(itc, st->its_c, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
    SPFD_CUDA(cudaStreamSynchronize(s));
    if (h_trace && its > 0)
        SPFD_CUDA(cudaMemcpy(h_trace, h.fg_trace.get(), (size_t)std::min(its, cfg.max_iters) * R * sizeof(double),
                             cudaMemcpyDeviceToHost));
    rep.converged = 1;
    int itmax = 0;
    for (int c = 0; c < R; ++c) {
        const double rel = bnorm[c] > 0 ? std::sqrt(rr[c]) / bnorm[c] : 0.0;
        rep.rel_residual[c] = rel;
        if (!(rel <= cfg.rel_tol)) rep.converged = 0;
        itmax = std::max(itmax, itc[c]);
    }
    rep.iterations = itmax;
    SPFD_CUDA(cudaMemcpyAsync(x_out, x, n * R * sizeof(double), cudaMemcpyDeviceToDevice, s));
    return rep;
}

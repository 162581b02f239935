// extern "C" boundary of libspfd_b200.so (include/spfd_b200.h).
#include <atomic>
#include <chrono>
#include <cstring>
#include <string>

#include "amg.cuh"
#include "comm.cuh"
#include "field.cuh"

struct spfd_op_s {
    spfd::Operator *op;
};
struct spfd_amg_s {
    spfd::Amg *amg;
    spfd::Operator *op;  // not owned
};
struct spfd_comm_s {
    spfd::Comm *comm;
};
struct spfd_field_s {
    spfd::Field *f;
    int64_t n_faces, n_cells, n_edges;
};

namespace spfd {

extern int g_fine_kind_override;
extern int g_pcg_graph_override;
static thread_local std::string g_last_error;
static std::atomic<int64_t> g_launches{0};
int64_t launch_count() { return g_launches.load(); }
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
void set_last_error(const std::string &msg) { g_last_error = msg; }

template <class F>
static int guarded(F &&f) {
    try {
        f();
        return SPFD_OK;
    } catch (const Error &e) {
        set_last_error(e.what());
        return e.code;
    } catch (const std::bad_alloc &) {
        set_last_error("host allocation failed");
        return SPFD_ENOMEM;
    } catch (const std::exception &e) {
        set_last_error(e.what());
        return SPFD_ECUDA;
    }
}

static inline cudaStream_t S(void *p) { return (cudaStream_t)p; }

}  // namespace spfd

using namespace spfd;

extern "C" {

const char *spfd_last_error(void) { return g_last_error.c_str(); }

const char *spfd_version(void) { return "spfd_b200 0.1 (sm_100a, fp64)"; }

int spfd_op_create(const int64_t *h_dims, const double *h_spacing, const uint16_t *ids, const double *lut,
                   int64_t lut_len, int pin, void *stream, spfd_op_t *out) {
    NvtxRange range_("spfd_op_create");
    return guarded([&] {
        SPFD_CHECK(out != nullptr && h_dims != nullptr && h_spacing != nullptr, SPFD_EINVAL, "null argument");
        Operator *op = op_create(h_dims, h_spacing, ids, lut, lut_len, pin, S(stream));
        *out = new spfd_op_s{op};
        pool_trim();
    });
}

int spfd_op_destroy(spfd_op_t op) {
    return guarded([&] {
        if (!op) return;
        delete op->op;
        delete op;
    });
}

int spfd_op_info_get(spfd_op_t h, spfd_op_info *info) {
    return guarded([&] {
        SPFD_CHECK(h && info, SPFD_EINVAL, "null argument");
        const Operator &op = *h->op;
        info->dims[0] = op.nx; info->dims[1] = op.ny; info->dims[2] = op.nz;
        info->n_nodes = op.n_nodes;
        info->n_edges = op.n_edges;
        info->n_dofs = op.n_dofs;
        info->n_conductive = op.n_cond;
        info->n_components = op.n_comp;
        info->n_cond_voxels = op.n_cond_vox;
        info->nnz = op.nnz;
        info->span_len = op.L;
        info->n_rows = op.n_rows;
        info->device_bytes = op.device_bytes();
    });
}

int spfd_op_export(spfd_op_t h, int what, void *dst, void *stream) {
    return guarded([&] {
        SPFD_CHECK(h && dst, SPFD_EINVAL, "null argument");
        op_export(*h->op, what, dst, S(stream));
    });
}

int spfd_op_csr(spfd_op_t h, int64_t *indptr, int32_t *indices, double *data, void *stream) {
    return guarded([&] {
        SPFD_CHECK(h && indptr && indices && data, SPFD_EINVAL, "null argument");
        op_csr(*h->op, indptr, indices, data, S(stream));
    });
}

int spfd_stencil_apply(spfd_op_t h, const double *x, double *y, int nrhs, void *stream) {
    return guarded([&] {
        SPFD_CHECK(h && x && y && (nrhs == 1 || nrhs == 2), SPFD_EINVAL, "bad argument");
        Operator &op = *h->op;
        op_dofs_to_span(op, x, op.ws_a.get(), nrhs, S(stream));
        op_stencil_span(op, op.ws_a.get(), op.ws_b.get(), nrhs, S(stream));
        op_span_to_dofs(op, op.ws_b.get(), y, nrhs, S(stream));
    });
}

int spfd_rhs_assemble(spfd_op_t h, const double *a, double *rhs, int nrhs, void *stream) {
    NvtxRange range_("spfd_rhs_assemble");
    return guarded([&] {
        SPFD_CHECK(h && a && rhs && (nrhs == 1 || nrhs == 2), SPFD_EINVAL, "bad argument");
        Operator &op = *h->op;
        op_rhs_span(op, a, op.ws_a.get(), nrhs, S(stream));
        op_span_to_dofs(op, op.ws_a.get(), rhs, nrhs, S(stream));
    });
}

int spfd_edge_voltages(spfd_op_t h, const double *a, const double *psi, double omega, double *v, int nrhs,
                       void *stream) {
    return guarded([&] {
        SPFD_CHECK(h && a && psi && v && (nrhs == 1 || nrhs == 2), SPFD_EINVAL, "bad argument");
        Operator &op = *h->op;
        op_dofs_to_span(op, psi, op.ws_a.get(), nrhs, S(stream));
        op_edge_voltages(op, a, op.ws_a.get(), omega, v, nrhs, S(stream));
    });
}

int spfd_node_field(spfd_op_t h, const double *v, double *node, int nrhs, void *stream) {
    return guarded([&] {
        SPFD_CHECK(h && v && node && (nrhs == 1 || nrhs == 2), SPFD_EINVAL, "bad argument");
        op_node_field(*h->op, v, node, nrhs, S(stream));
    });
}

int spfd_voxel_average(spfd_op_t h, const double *node, double *vox, int nrhs, void *stream) {
    return guarded([&] {
        SPFD_CHECK(h && node && vox && (nrhs == 1 || nrhs == 2), SPFD_EINVAL, "bad argument");
        op_voxel_average(*h->op, node, vox, nrhs, S(stream));
    });
}

int spfd_efield_voxavg(spfd_op_t h, const double *a, const double *psi, double omega, double *vox, int nrhs,
                       void *stream) {
    NvtxRange range_("spfd_efield_voxavg");
    return guarded([&] {
        SPFD_CHECK(h && a && psi && vox && (nrhs == 1 || nrhs == 2), SPFD_EINVAL, "bad argument");
        Operator &op = *h->op;
        op_dofs_to_span(op, psi, op.ws_a.get(), nrhs, S(stream));
        op_efield_voxavg_span(op, a, op.ws_a.get(), omega, vox, op.ws_b.get(), nrhs, S(stream));
    });
}

static void check_cfg(const spfd_config *c) {
    SPFD_CHECK(c != nullptr, SPFD_EINVAL, "null config");
    SPFD_CHECK(c->rel_tol > 0.0, SPFD_EINVAL, "rel_tol must be positive");
    SPFD_CHECK(c->restart >= 1, SPFD_EINVAL, "restart must be >= 1");
    SPFD_CHECK(c->jacobi_damping > 0.0 && c->jacobi_damping <= 1.0, SPFD_EINVAL, "jacobi_damping must be in (0, 1]");
    SPFD_CHECK(c->max_iters >= 1, SPFD_EINVAL, "max_iters must be >= 1");
    SPFD_CHECK(c->coarse_cap >= 1 && c->max_levels >= 1, SPFD_EINVAL, "coarse_cap and max_levels must be >= 1");
}

// Setup peak of library pool memory per fine DOF (temporaries + the
// hierarchy), measured with SPFD_SETUP_TRACE=1: C3 793 B/DOF.
constexpr double kSetupPeakBytesPerDof = 800.0;

int spfd_amg_setup_op(spfd_op_t h, const spfd_config *cfg, void *stream, spfd_amg_t *out) {
    NvtxRange range_("spfd_amg_setup_op");
    return guarded([&] {
        SPFD_CHECK(h && out, SPFD_EINVAL, "null argument");
        check_cfg(cfg);
        SPFD_CHECK(h->op->n_dofs >= 1, SPFD_EEMPTY, "empty Poisson system");
        // reserve the pool for the setup's peak in one step (pool_reserve):
        // the peak per DOF of the last setup in this process, else a C3/C4
        // measured figure
        static double peak_per_dof = kSetupPeakBytesPerDof;
        const auto t0 = std::chrono::steady_clock::now();
        const size_t base = pool_used();
        pool_reserve((size_t)(peak_per_dof * (double)h->op->n_dofs));
        pool_used_high_reset();
        Amg *a = amg_setup_op(h->op, *cfg, S(stream));
        const size_t peak = pool_used_high_reset();
        if (peak > base) peak_per_dof = std::max(peak_per_dof, (double)(peak - base) / (double)h->op->n_dofs);
        if (getenv("SPFD_SETUP_TRACE"))
            fprintf(stderr, "[setup] pool peak %.1f MB over %.1f MB in use (%.0f B/DOF)\n", (peak - base) / 1e6,
                    base / 1e6, (double)(peak - base) / (double)h->op->n_dofs);
        // setup time = the whole call (pool reservation and the fine-level
        // CSR export included), on the host clock after the stream drained
        SPFD_CUDA(cudaStreamSynchronize(S(stream)));
        a->setup_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        *out = new spfd_amg_s{a, h->op};
        pool_trim();
    });
}

int spfd_amg_setup_csr(int64_t n, int64_t nnz, const int64_t *indptr, const int32_t *indices, const double *data,
                       const spfd_config *cfg, void *stream, spfd_amg_t *out) {
    NvtxRange range_("spfd_amg_setup_csr");
    return guarded([&] {
        SPFD_CHECK(out && indptr && (nnz == 0 || (indices && data)), SPFD_EINVAL, "null argument");
        check_cfg(cfg);
        Amg *a = amg_setup_csr(n, nnz, indptr, indices, data, *cfg, S(stream));
        *out = new spfd_amg_s{a, nullptr};
        pool_trim();
    });
}

int spfd_amg_destroy(spfd_amg_t h) {
    return guarded([&] {
        if (!h) return;
        delete h->amg;
        delete h;
    });
}

int spfd_amg_info_get(spfd_amg_t h, spfd_amg_info *info) {
    return guarded([&] {
        SPFD_CHECK(h && info, SPFD_EINVAL, "null argument");
        Amg &a = *h->amg;
        std::memset(info, 0, sizeof(*info));
        info->n_levels = (int32_t)a.lv.size();
        SPFD_CHECK(a.lv.size() <= 32, SPFD_EINVAL, "too many levels for the info struct");
        for (size_t l = 0; l < a.lv.size(); ++l) {
            info->level_rows[l] = a.lv[l].n;
            info->level_nnz[l] = a.lv[l].a_nnz;
            const Csr &P = (l == 0 && a.structured) ? a.lv[l].P_dof : a.lv[l].P;
            info->prolong_nnz[l] = P.nnz;
        }
        info->setup_seconds = a.setup_seconds;
        info->device_bytes = a.device_bytes();
        info->structured = a.structured ? 1 : 0;
        info->smoother = a.smoother;
        info->cheb_degree = a.cheb_deg;
        for (size_t l = 0; l < a.cheb_lmax.size() && l < 32; ++l) info->cheb_lmax[l] = a.cheb_lmax[l];
        info->restriction_csr = (a.structured && a.lv.size() > 1 && a.lv[0].Rspan.rows > 0) ? 1 : 0;
        if (a.structured && a.lv.size() > 1 && a.lv[0].Pspan.rows > 0) info->restriction_csr |= 2;
    });
}

int spfd_amg_level_csr(spfd_amg_t h, int level, int which, int64_t *indptr, int32_t *indices, double *data,
                       void *stream) {
    return guarded([&] {
        SPFD_CHECK(h && indptr, SPFD_EINVAL, "null argument");
        amg_level_csr(*h->amg, level, which, indptr, indices, data, S(stream));
    });
}

int spfd_amg_level_agg(spfd_amg_t h, int level, int32_t *agg, void *stream) {
    return guarded([&] {
        SPFD_CHECK(h && agg, SPFD_EINVAL, "null argument");
        amg_level_agg(*h->amg, level, agg, S(stream));
    });
}

int spfd_vcycle(spfd_amg_t h, const double *r, double *z, int nrhs, void *stream) {
    NvtxRange range_("spfd_vcycle");
    return guarded([&] {
        SPFD_CHECK(h && r && z && nrhs >= 1 && nrhs <= h->amg->max_nrhs, SPFD_EINVAL, "bad argument");
        Amg &a = *h->amg;
        amg_to_level0(a, r, a.kb.get(), nrhs, S(stream));
        amg_vcycle(a, a.kb.get(), a.kz.get(), nrhs, S(stream));
        amg_from_level0(a, a.kz.get(), z, nrhs, S(stream));
    });
}

int spfd_solve(spfd_amg_t h, const double *b, double *x, int nrhs, const spfd_config *cfg, spfd_report *rep,
               double *h_trace, void *stream) {
    NvtxRange range_("spfd_solve");
    return guarded([&] {
        SPFD_CHECK(h && b && x && rep && nrhs >= 1 && nrhs <= h->amg->max_nrhs, SPFD_EINVAL, "bad argument");
        check_cfg(cfg);
        Amg &a = *h->amg;
        amg_to_level0(a, b, a.kb.get(), nrhs, S(stream));
        *rep = krylov_solve(a, a.kb.get(), a.kx.get(), nrhs, *cfg, h_trace, S(stream));
        amg_from_level0(a, a.kx.get(), x, nrhs, S(stream));
        SPFD_CUDA(cudaStreamSynchronize(S(stream)));
        if (rep->status == SPFD_ENONFINITE) throw Error(SPFD_ENONFINITE, "non-finite value in the Krylov iteration");
    });
}

int spfd_snapshot(spfd_op_t hop, spfd_amg_t h, const double *a, double omega, double *psi, double *vox, int nrhs,
                  const spfd_config *cfg, spfd_report *rep, void *stream) {
    NvtxRange range_("spfd_snapshot");
    return guarded([&] {
        SPFD_CHECK(hop && h && a && vox && rep && h->op == hop->op, SPFD_EINVAL, "bad argument");
        SPFD_CHECK(nrhs >= 1 && nrhs <= h->amg->max_nrhs, SPFD_EINVAL, "nrhs exceeds the hierarchy workspace");
        check_cfg(cfg);
        Amg &m = *h->amg;
        Operator &op = *hop->op;
        // rhs straight into the span layout, solve, fused E-field from the span iterate
        if (m.dist) {
            int64_t rg[4];
            dist_info(m, rg);
            op_rhs_span(op, a, m.kb.get(), nrhs, S(stream), rg[0], rg[1]);
            *rep = krylov_solve(m, m.kb.get(), m.kx.get(), nrhs, *cfg, nullptr, S(stream));
            if (rep->status == SPFD_ENONFINITE) throw Error(SPFD_ENONFINITE, "non-finite value in the Krylov iteration");
            op_node_field_span(op, a, m.kx.get(), omega, op.ws_b.get(), nrhs, S(stream), rg[0], rg[1]);
            dist_range_exchange(m, op.ws_b.get(), nrhs, S(stream));   // node plane k_{r+1} from the next rank
            op_voxavg_span(op, op.ws_b.get(), vox, nrhs, S(stream), rg[2], rg[3]);
        } else {
            op_rhs_span(op, a, m.kb.get(), nrhs, S(stream));
            *rep = krylov_solve(m, m.kb.get(), m.kx.get(), nrhs, *cfg, nullptr, S(stream));
            if (rep->status == SPFD_ENONFINITE) throw Error(SPFD_ENONFINITE, "non-finite value in the Krylov iteration");
            op_efield_voxavg_span(op, a, m.kx.get(), omega, vox, op.ws_b.get(), nrhs, S(stream));
        }
        if (psi) op_span_to_dofs(op, m.kx.get(), psi, nrhs, S(stream));
        SPFD_CUDA(cudaStreamSynchronize(S(stream)));
    });
}

int spfd_nccl_unique_id(void *h_id) {
    return guarded([&] {
        SPFD_CHECK(h_id, SPFD_EINVAL, "null argument");
        nccl_unique_id(h_id);
    });
}

int spfd_comm_init_nccl(const void *h_id, int rank, int nranks, spfd_comm_t *out) {
    return guarded([&] {
        SPFD_CHECK(h_id && out && nranks >= 1 && rank >= 0 && rank < nranks, SPFD_EINVAL, "bad argument");
        *out = new spfd_comm_s{comm_nccl(h_id, rank, nranks)};
    });
}

int spfd_comm_init_callbacks(const spfd_comm_callbacks *cb, int rank, int nranks, spfd_comm_t *out) {
    return guarded([&] {
        SPFD_CHECK(cb && out && nranks >= 1 && rank >= 0 && rank < nranks, SPFD_EINVAL, "bad argument");
        *out = new spfd_comm_s{comm_host(*cb, rank, nranks)};
    });
}

int spfd_comm_destroy(spfd_comm_t c) {
    return guarded([&] {
        if (!c) return;
        delete c->comm;
        delete c;
    });
}

int spfd_amg_distribute(spfd_amg_t h, spfd_comm_t c, int64_t replicate_below, int64_t *h_range, void *stream) {
    NvtxRange range_("spfd_amg_distribute");
    return guarded([&] {
        SPFD_CHECK(h && c && h_range, SPFD_EINVAL, "null argument");
        SPFD_CHECK(h->amg->dist == nullptr, SPFD_EINVAL, "hierarchy already distributed");
        amg_distribute(*h->amg, c->comm, replicate_below, h_range, S(stream));
        pool_trim();
    });
}

int spfd_bench_kernel(spfd_amg_t h, int which, int reps, int nrhs, double *h_ms, double *h_bytes, void *stream) {
    return guarded([&] {
        SPFD_CHECK(h && h_ms && h_bytes && which >= 0 && which <= 11, SPFD_EINVAL, "bad argument");
        *h_ms = amg_bench_kernel(*h->amg, which, reps, nrhs, h_bytes, S(stream));
    });
}

int spfd_iteration_bytes(spfd_amg_t h, int nrhs, double *h_bytes) {
    return guarded([&] {
        SPFD_CHECK(h && h_bytes && nrhs >= 1 && nrhs <= 2, SPFD_EINVAL, "bad argument");
        *h_bytes = amg_iteration_bytes(*h->amg, nrhs);
    });
}

int spfd_set_fine_kernel(int kind) {
    return guarded([&] {
        SPFD_CHECK(kind == -1 || kind == 2 || kind == 3, SPFD_EINVAL, "fine kernel kind must be -1, 2 or 3");
        g_fine_kind_override = kind;
    });
}

int spfd_set_pcg_graph(int mode) {
    return guarded([&] {
        SPFD_CHECK(mode >= -1 && mode <= 1, SPFD_EINVAL, "pcg graph mode must be -1, 0 or 1");
        g_pcg_graph_override = mode;
    });
}

static void check_box(const spfd_box *b, bool lattice) {
    SPFD_CHECK(b, SPFD_EINVAL, "null box");
    for (int a = 0; a < 3; ++a) {
        SPFD_CHECK(lattice ? b->dims[a] >= 1 : b->dims[a] >= 0, SPFD_EINVAL,
                   lattice ? "lattice dims must be >= 1" : "dims must be three integers >= 0");
        SPFD_CHECK(b->spacing[a] > 0.0, SPFD_EINVAL, "spacing must be positive");
    }
}

int spfd_field_create(const spfd_box *grid, const spfd_config *cfg, spfd_field_t *out) {
    return guarded([&] {
        SPFD_CHECK(out, SPFD_EINVAL, "null argument");
        check_box(grid, false);
        check_cfg(cfg);
        const int64_t nx = grid->dims[0], ny = grid->dims[1], nz = grid->dims[2];
        auto *h = new spfd_field_s{nullptr, (nx + 1) * ny * nz + nx * (ny + 1) * nz + nx * ny * (nz + 1), nx * ny * nz,
                                   nx * (ny + 1) * (nz + 1) + (nx + 1) * ny * (nz + 1) + (nx + 1) * (ny + 1) * nz};
        try {
            h->f = field_create(*grid, *cfg);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

int spfd_field_destroy(spfd_field_t f) {
    return guarded([&] {
        if (!f) return;
        field_destroy(f->f);
        delete f;
    });
}

int spfd_coil_field(int64_t n, const double *pts, int nseg, const double *verts, double scale, double *out,
                    void *stream) {
    NvtxRange range_("spfd_coil_field");
    return guarded([&] {
        SPFD_CHECK(n >= 0 && nseg >= 1 && (n == 0 || (pts && verts && out)), SPFD_EINVAL, "bad argument");
        coil_field(n, pts, nseg, verts, scale, out, S(stream));
    });
}

int spfd_field_interpolate(spfd_field_t f, const spfd_box *lattice, const double *b, double *flux, void *stream) {
    NvtxRange range_("spfd_field_interpolate");
    return guarded([&] {
        SPFD_CHECK(f && b && flux, SPFD_EINVAL, "null argument");
        check_box(lattice, true);
        field_interpolate(*f->f, *lattice, b, flux, S(stream));
    });
}

int spfd_field_divergence(spfd_field_t f, const double *flux, double *div, void *stream) {
    return guarded([&] {
        SPFD_CHECK(f && flux && div, SPFD_EINVAL, "null argument");
        field_divergence(*f->f, flux, div, S(stream));
    });
}

int spfd_field_clean(spfd_field_t f, const double *in, double *out, double tol, spfd_clean_info *info, void *stream) {
    NvtxRange range_("spfd_field_clean");
    return guarded([&] {
        SPFD_CHECK(f && in && out && info, SPFD_EINVAL, "null argument");
        field_clean(*f->f, 1, in, out, tol, info, S(stream));
    });
}

int spfd_field_clean_batch(spfd_field_t f, int nrhs, const double *in, double *out, double tol,
                           spfd_clean_info *info, void *stream) {
    NvtxRange range_("spfd_field_clean_batch");
    return guarded([&] {
        SPFD_CHECK(f && in && out && info, SPFD_EINVAL, "null argument");
        SPFD_CHECK(nrhs == 1 || nrhs == 2, SPFD_EINVAL, "nrhs must be 1 or 2");
        field_clean(*f->f, nrhs, in, out, tol, info, S(stream));
    });
}

int spfd_field_gauge(spfd_field_t f, const double *flux, double *a, double tol, spfd_gauge_info *info, void *stream) {
    NvtxRange range_("spfd_field_gauge");
    return guarded([&] {
        SPFD_CHECK(f && flux && a && info, SPFD_EINVAL, "null argument");
        field_gauge(*f->f, 0, flux, a, tol, info, S(stream));
    });
}

int spfd_field_gauge_tree(spfd_field_t f, int tree, const double *flux, double *a, double tol, spfd_gauge_info *info,
                          void *stream) {
    NvtxRange range_("spfd_field_gauge_tree");
    return guarded([&] {
        SPFD_CHECK(f && flux && a && info, SPFD_EINVAL, "null argument");
        SPFD_CHECK(tree == 0 || tree == 1, SPFD_EINVAL, "tree must be 0 (comb) or 1 (bfs)");
        field_gauge(*f->f, tree, flux, a, tol, info, S(stream));
    });
}

int spfd_field_circulation(spfd_field_t f, const double *a, const double *flux, double *defect, void *stream) {
    return guarded([&] {
        SPFD_CHECK(f && a && flux && defect, SPFD_EINVAL, "null argument");
        field_circulation(*f->f, a, flux, defect, S(stream));
    });
}

int spfd_exposure_stats(const double *values, int64_t n, double scale, const int64_t *vox_index,
                        const uint16_t *ids_box, int32_t n_ids, double *scaled, int64_t *h_count, double *h_mean,
                        double *h_max, double *h_p99, double *h_global, void *stream) {
    NvtxRange range_("spfd_exposure_stats");
    return guarded([&] {
        SPFD_CHECK(values && vox_index && ids_box && scaled && h_count && h_mean && h_max && h_p99 && h_global,
                   SPFD_EINVAL, "null argument");
        exposure_stats(values, n, scale, vox_index, ids_box, n_ids, scaled, h_count, h_mean, h_max, h_p99, h_global,
                       S(stream));
    });
}

int64_t spfd_launch_count(void) { return spfd::launch_count(); }

int spfd_copy(void *dst, const void *src, int64_t bytes) {
    return guarded([&] {
        if (bytes > 0) SPFD_CUDA(cudaMemcpy(dst, src, (size_t)bytes, cudaMemcpyDefault));
    });
}

}  // extern "C"

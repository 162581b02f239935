// Smoothed-aggregation AMG hierarchy and Krylov solvers (device).
#pragma once
#include <vector>

#include "op.cuh"

namespace spfd {

struct Csr {
    int64_t rows = 0, cols = 0, nnz = 0;
    DevBuf<int64_t> ptr;   // rows + 1
    DevBuf<int32_t> col;   // nnz (sorted per row)
    DevBuf<double> val;    // nnz
    void alloc(int64_t r, int64_t c, int64_t z) {
        rows = r; cols = c; nnz = z;
        ptr.alloc(r + 1); col.alloc(z); val.alloc(z);
    }
    int64_t bytes() const { return ptr.bytes() + col.bytes() + val.bytes(); }
};

struct CsrView {
    const int64_t *ptr;
    const int32_t *col;
    const double *val;
    int64_t rows;
};
inline CsrView view(const Csr &m) { return CsrView{m.ptr.get(), m.col.get(), m.val.get(), m.rows}; }

struct Level {
    int64_t n = 0;            // unknowns on this level
    int64_t nvec = 0;         // vector length (span L on a structured level 0)
    int64_t a_nnz = 0;        // nnz(A_l) (reference CSR count)
    Csr A;                    // CSR (absent on a structured level 0 after setup)
    Csr P, R;                 // solve-layout prolongation / restriction
    Csr P_dof, R_dof;         // DOF-numbered copies (structured level 0 only; exports)
    DevBuf<int32_t> agg;      // aggregate per row (DOF numbering)
    DevBuf<int32_t> agg_pos;  // structured level 0: aggregate id + 1 per span position (0 = none)
    DevBuf<int64_t> mem_ptr;  // structured level 0: aggregate -> member positions (CSR of T^T)
    DevBuf<int32_t> mem_pos;
    DevBuf<double> dinv;      // [nvec]
    DevBuf<double> odinv;     // [nvec] omega * dinv
    DevBuf<double> vr, vx, vd, vt;  // workspaces [nvec * max_nrhs]
    int p_group = 4, r_group = 32, a_group = 32;  // lanes per row in CSR kernels
    Csr AP;                   // coarse levels, V(1,1): A_l P_l for the fused prolongation + post-smooth
    int ap_group = 4;
    Csr Rspan;                // structured level 0: R = P^T with span-position columns and rows in the
    int rspan_group = 4;      //   level-1 solve order (build_rspan; the V-cycle's restriction)
    Csr Q;                    // coarse levels, V(1,1): Q = P - diag(omega D^-1) A P (pattern of A P), so the
    int q_group = 4;          //   prolongation + post-smooth is z = omega D^-1 (r + d) + Q e (build_q)
    Csr Pspan;                // structured level 0: P with span-position rows and level-1 solve columns
    int pspan_group = 4;      //   (build_rspan; the V-cycle's prolongation)
};

struct Dist;   // z-slab decomposition (dist.cuh)
struct Comm;   // transport (comm.cuh)

struct Amg {
    std::vector<Level> lv;
    Operator *op = nullptr;   // structured level 0 (not owned)
    bool structured = false;
    int64_t nc = 0;           // coarsest size
    DevBuf<double> cinv;      // dense inverse of the coarsest matrix (nc x nc)
    double omega = 2.0 / 3.0;
    int pre = 1, post = 1;
    int64_t box[3] = {0, 0, 0};  // > 0: level 0 is the cell Laplacian div div^T of this voxel box
    double box_od = 0.0;         // omega / 6, its (constant) omega D^-1
    int smoother = 0;         // SPFD_SMOOTHER_JACOBI | SPFD_SMOOTHER_CHEBYSHEV
    int cheb_deg = 2;         // Chebyshev polynomial degree per sweep
    std::vector<double> cheb_lmax;  // lambda_max(D^-1 A_l) estimates (Chebyshev)
    int max_nrhs = 2;
    double setup_seconds = 0.0;
    // Krylov workspace (level-0 layout, interleaved nrhs)
    DevBuf<double> kx, kr, kz, kp, kq, kb;
    DevBuf<double> partials;  // per-CTA dot partials
    DevBuf<double> scal;      // device scalars
    DevBuf<double> fg_basis, fg_prec;  // FGMRES basis (allocated on demand)
    int64_t fg_m = 0;
    int fg_R = 1;             // rhs count the FGMRES basis was sized for
    std::vector<int32_t> l1_perm;  // solve-layout level-1 index -> reference index (empty = identity)
    int vc_partials = 0;      // r.z partials written by the last V-cycle (0 = none)
    Dist *dist = nullptr;     // set by amg_distribute (owned)
    cudaStream_t side = nullptr;            // PCG x-update overlap stream
    cudaEvent_t ev_alpha = nullptr, ev_x = nullptr;
    // PCG as one CUDA graph per rhs count: a device-side WHILE node over the
    // iteration body (convergence tested on the device, no host round trip)
    cudaStream_t cap = nullptr;             // private capture stream
    cudaGraphExec_t pcg_exec[3] = {nullptr, nullptr, nullptr};
    int64_t pcg_body_launches[3] = {0, 0, 0};
    int pcg_kind[3] = {-1, -1, -1};         // fine-kernel kind captured in each graph
    DevBuf<double> pcg_trace;               // [cap_iters * 2] per-iteration residual estimates
    int64_t pcg_trace_cap = 0;
    // FGMRES restart cycle as one graph per rhs count (fgmres_graph.cuh)
    cudaStream_t cap2 = nullptr;            // second capture stream (conditional step bodies)
    cudaGraphExec_t fg_exec[3] = {nullptr, nullptr, nullptr};
    int fg_exec_m[3] = {0, 0, 0};
    bool fg_failed[3] = {false, false, false};
    DevBuf<double> fg_state, fg_y, fg_gram, fg_trace;
    DevBuf<int> fg_jc;
    int64_t fg_trace_cap = 0;
    Amg() = default;
    Amg(const Amg &) = delete;
    Amg &operator=(const Amg &) = delete;
    ~Amg();
    int64_t device_bytes() const;
};

Amg *amg_setup_op(Operator *op, const spfd_config &cfg, cudaStream_t s);
Amg *amg_setup_csr(int64_t n, int64_t nnz, const int64_t *ptr, const int32_t *col, const double *val,
                   const spfd_config &cfg, cudaStream_t s);
void amg_vcycle(Amg &h, const double *r, double *z, int nrhs, cudaStream_t s);  // level-0 layout, interleaved
void amg_level_csr(Amg &h, int level, int which, int64_t *ptr, int32_t *col, double *val, cudaStream_t s);
void amg_level_agg(Amg &h, int level, int32_t *agg, cudaStream_t s);

// level-0 layout helpers (span for structured, identity for CSR)
void amg_to_level0(Amg &h, const double *planar, double *inter, int nrhs, cudaStream_t s);
void amg_from_level0(Amg &h, const double *inter, double *planar, int nrhs, cudaStream_t s);

int csr_group(int64_t nnz, int64_t rows);  // lanes per row of the CSR kernels
void level1_unpermute(Amg &h, cudaStream_t s);  // reference level-1 numbering (amg_setup.cu)
void build_rspan(Amg &h, cudaStream_t s);  // CSR restriction + prolongation over span positions (amg_setup.cu)
void build_pspan(Amg &h, const int32_t *solve_to_ref, cudaStream_t s);
void build_q(Amg &h, cudaStream_t s);  // combined coarse prolongation + post-smooth operators (amg_setup.cu)
void amg_drop_graphs(Amg &h);  // destroy captured solve graphs (buffers changed; solve.cu)
void amg_distribute(Amg &h, Comm *comm, int64_t replicate_below, int64_t *range, cudaStream_t s);
void dist_range_exchange(Amg &h, double *v, int nrhs, cudaStream_t s);
void dist_info(const Amg &h, int64_t *out);  // pb, pe, voxel-row begin, end
double amg_bench_kernel(Amg &h, int which, int reps, int nrhs, double *bytes, cudaStream_t s);
// algorithmic bytes of one PCG iteration (SpMV, V-cycle, vector updates)
double amg_iteration_bytes(const Amg &h, int nrhs);
// Chebyshev smoother: power-iteration estimates of lambda_max(D^-1 A_l)
void amg_estimate_lmax(Amg &h, cudaStream_t s);
// Level 0 of a CSR hierarchy built on the cell Laplacian div div^T of an
// nx x ny x nz voxel box (diagonal 6, -1 per shared face): apply it as a
// matrix-free constant-coefficient stencil instead of reading the CSR.
void amg_set_box_level0(Amg &h, const int64_t dims[3], cudaStream_t s);
spfd_report krylov_solve(Amg &h, const double *b_inter, double *x_inter, int nrhs, const spfd_config &cfg,
                         double *h_trace, cudaStream_t s);

}  // namespace spfd

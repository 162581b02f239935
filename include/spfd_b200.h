/*
 * spfd_b200 — C-ABI of the B200-native SPFD Poisson hot path.
 *
 * The reference (`/root/reference/pkg/src/spfd`) is pure Python and has no
 * FFI; its "operator API" is the Python functions each entry point below
 * replaces (cited per function).  The Python package
 * `paper_2010_12879_b200` binds this header with ctypes; INTEGRATION.md shows
 * the binding a maintainer of the reference would add.
 *
 * Conventions
 *   - every data pointer is a DEVICE pointer (CUDA global memory) unless the
 *     parameter name starts with `h_`; sizes are int64_t; every call that
 *     launches work takes a `cudaStream_t` passed as `void *` (NULL = legacy
 *     default stream) and is asynchronous unless stated otherwise;
 *   - multi-RHS vectors ("nrhs" = 1 or 2, e.g. the real/imag parts of a
 *     phasor) are PLANAR at the boundary: rhs k occupies
 *     [k*len, (k+1)*len);
 *   - node / edge / voxel orderings are exactly the reference's:
 *     x-fastest linear indices, edges in three blocks x, y, z
 *     (fit_operators.py:1-16); DOF vectors are in ascending node order
 *     (fit_operators.py:406-407);
 *   - all arithmetic is IEEE binary64;
 *   - status codes map onto the reference exceptions in Python
 *     (see SPFD_E* below); spfd_last_error() returns a thread-local message.
 */
#ifndef SPFD_B200_H
#define SPFD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
#define SPFD_OK         0
#define SPFD_EINVAL     1 /* ValueError   (bad shape / argument)                     */
#define SPFD_ENONFINITE 2 /* SolverError  (linsolve.py:218-219, 267-268, 293-294)    */
#define SPFD_ENOTPOS    3 /* SolverError  (linsolve.py:172-176 non-positive diagonal) */
#define SPFD_EEMPTY     4 /* EmptySystemError (fit_operators.py:396-397, 443-444)     */
#define SPFD_ENOCONV    5 /* never returned as an error: report flag only            */
#define SPFD_ECUDA      6 /* RuntimeError (CUDA failure)                             */
#define SPFD_ENCCL      7 /* RuntimeError (NCCL failure)                             */
#define SPFD_ENOMEM     8 /* MemoryError                                             */
#define SPFD_EINCOMPAT  9 /* IncompatibleFluxError (gauging.py:167-171)             */
#define SPFD_EPROJECTION 10 /* ProjectionError (field_source.py:319-329)            */
#define SPFD_ELATTICE  11 /* LatticeError (field_source.py:228-232)                 */
#define SPFD_ESINGULAR 12 /* SingularPointError (field_source.py:187-188)           */

const char *spfd_last_error(void);
/* Library version string and the SM architecture the kernels were built for. */
const char *spfd_version(void);

/* ---- opaque handles ---------------------------------------------------- */
typedef struct spfd_op_s  *spfd_op_t;   /* assembled voxel operator            */
typedef struct spfd_amg_s *spfd_amg_t;  /* AMG hierarchy (+ solve workspace)   */

/* ---- operator (fit_operators.py:311-457, voxel_model.py:153-159,470-511) */

typedef struct {
    int64_t dims[3];          /* voxels nx, ny, nz                              */
    int64_t n_nodes;          /* (nx+1)(ny+1)(nz+1)                             */
    int64_t n_edges;          /* three edge blocks                              */
    int64_t n_dofs;           /* free conductive nodes                          */
    int64_t n_conductive;     /* conductive nodes                               */
    int64_t n_components;     /* conductive components (= pinned nodes if pin)  */
    int64_t n_cond_voxels;    /* voxels with kappa > 0                          */
    int64_t nnz;              /* nonzeros of the reduced 7-point matrix         */
    int64_t span_len;         /* internal row-span layout length (>= n_dofs)    */
    int64_t n_rows;           /* (ny+1)(nz+1) x-rows of the node box           */
    int64_t device_bytes;     /* device memory owned by the handle             */
} spfd_op_info;

/* Build the operator from tissue ids and a conductivity LUT.
 * Replaces assemble_poisson()'s operator half (fit_operators.py:367-436):
 * kappa = lut[ids] (voxel_model.py:153-159), edge conductances
 * (fit_operators.py:289-324), conductive components and pinning of the
 * lowest-index node per component (voxel_model.py:470-511,
 * fit_operators.py:394-408), DOF numbering, and the matrix-free stencil.
 *   ids   : uint16[nx*ny*nz], x-fastest                (device)
 *   lut   : double[lut_len], kappa per tissue id      (device)
 *   pin   : 1 = pin one node per component (reference default)
 * Errors: SPFD_EINVAL (id >= lut_len, bad dims), SPFD_EEMPTY (no conductive
 * voxel).  Synchronises `stream` before returning. */
int spfd_op_create(const int64_t *h_dims, const double *h_spacing,
                   const uint16_t *ids, const double *lut, int64_t lut_len,
                   int pin, void *stream, spfd_op_t *out);
int spfd_op_destroy(spfd_op_t op);
int spfd_op_info_get(spfd_op_t op, spfd_op_info *h_info);

/* Exports (device destinations, sizes from spfd_op_info):
 *   SPFD_EXPORT_EDGE_CONDUCTANCE  double[n_edges]   (fit_operators.py:311)
 *   SPFD_EXPORT_DOF_TO_NODE       int64[n_dofs]     (PoissonSystem.dof_to_node)
 *   SPFD_EXPORT_NODE_TO_DOF       int64[n_nodes]    (-1 = not a DOF)
 *   SPFD_EXPORT_PINNED            int64[n_components]
 *   SPFD_EXPORT_VOXEL_INDICES     int64[n_cond_voxels] (dosimetry.py:101-104)
 *   SPFD_EXPORT_DIAGONAL          double[n_dofs]    (matrix diagonal)          */
#define SPFD_EXPORT_EDGE_CONDUCTANCE 0
#define SPFD_EXPORT_DOF_TO_NODE      1
#define SPFD_EXPORT_NODE_TO_DOF      2
#define SPFD_EXPORT_PINNED           3
#define SPFD_EXPORT_VOXEL_INDICES    4
#define SPFD_EXPORT_DIAGONAL         5
int spfd_op_export(spfd_op_t op, int what, void *dst, void *stream);

/* Materialise the reduced matrix as CSR (sorted columns) — the reference's
 * PoissonSystem.matrix, bit-identical values (fit_operators.py:421-436).
 *   indptr int64[n_dofs+1], indices int32[nnz], data double[nnz]          */
int spfd_op_csr(spfd_op_t op, int64_t *indptr, int32_t *indices, double *data,
                void *stream);

/* y = A x with the matrix-free 7-point stencil (DOF-ordered, planar nrhs).
 * Same products, same order as the reference csr_matvec. */
int spfd_stencil_apply(spfd_op_t op, const double *x, double *y, int nrhs,
                       void *stream);

/* rhs = -G^T M_kappa a restricted to DOFs (fit_operators.py:438-441).
 *   a   : double[nrhs][n_edges]  edge vector potential(s)
 *   rhs : double[nrhs][n_dofs]                                            */
int spfd_rhs_assemble(spfd_op_t op, const double *a, double *rhs, int nrhs,
                      void *stream);

/* ---- E-field chain (dosimetry.py:27-116) ------------------------------- */

/* v = omega*(a + psi[head] - psi[tail]) on every edge (dosimetry.py:27-47).
 *   a double[nrhs][n_edges], psi double[nrhs][n_dofs], v double[nrhs][n_edges] */
int spfd_edge_voltages(spfd_op_t op, const double *a, const double *psi,
                       double omega, double *v, int nrhs, void *stream);
/* per-node |E| from edge voltages (dosimetry.py:50-85); node double[nrhs][n_nodes] */
int spfd_node_field(spfd_op_t op, const double *v, double *node, int nrhs,
                    void *stream);
/* 8-corner mean on conductive voxels (dosimetry.py:88-116); vox double[nrhs][n_cond_voxels] */
int spfd_voxel_average(spfd_op_t op, const double *node, double *vox, int nrhs,
                       void *stream);
/* Fused chain a, psi -> voxel |E| without materialising edge voltages or the
 * node box: bit-identical to the three calls above. */
int spfd_efield_voxavg(spfd_op_t op, const double *a, const double *psi,
                       double omega, double *vox, int nrhs, void *stream);

/* ---- AMG + Krylov (linsolve.py:26-298) ---------------------------------- */

typedef struct {
    double  rel_tol;             /* 1e-12 reference default                  */
    int32_t max_iters;           /* 1000                                     */
    int32_t restart;             /* 30 (FGMRES)                              */
    int32_t pre_sweeps;          /* 1                                        */
    int32_t post_sweeps;         /* 1                                        */
    double  jacobi_damping;      /* 2/3                                      */
    double  strength_threshold;  /* 0.08, halved per level                   */
    int32_t coarse_cap;          /* 500                                      */
    int32_t max_levels;          /* 20                                       */
    int32_t method;              /* SPFD_METHOD_PCG | SPFD_METHOD_FGMRES     */
    int32_t max_nrhs;            /* workspace sizing: 1 or 2                 */
    int32_t smoother;            /* SPFD_SMOOTHER_JACOBI (0, the reference's
                                    damped Jacobi) | SPFD_SMOOTHER_CHEBYSHEV */
    int32_t cheb_degree;         /* Chebyshev polynomial degree per sweep
                                    (0 -> 2); pre/post_sweeps repeat it      */
} spfd_config;
#define SPFD_METHOD_PCG    0
#define SPFD_METHOD_FGMRES 1
#define SPFD_SMOOTHER_JACOBI    0
#define SPFD_SMOOTHER_CHEBYSHEV 1

typedef struct {
    int32_t n_levels;
    int64_t level_rows[32];
    int64_t level_nnz[32];       /* nnz of A_l (level 0: stencil matrix nnz) */
    int64_t prolong_nnz[32];     /* nnz of P_l (0 on the coarsest level)     */
    double  setup_seconds;       /* device-timed                             */
    int64_t device_bytes;
    int32_t structured;          /* 1 = level 0 is the matrix-free stencil   */
    int32_t smoother;            /* SPFD_SMOOTHER_*                          */
    int32_t cheb_degree;
    double  cheb_lmax[32];       /* Chebyshev: power-iteration estimate of
                                    lambda_max(D^-1 A_l) per level           */
    int32_t restriction_csr;     /* bit 0: the fine restriction runs as R = P^T
                                    in CSR (else matrix-free through T);
                                    bit 1: the fine prolongation as P in CSR */
} spfd_amg_info;

/* Hierarchy on the operator (level 0 = matrix-free stencil) or on a
 * generic CSR (device arrays, sorted or unsorted columns).
 * Replaces amg_setup() (linsolve.py:120-169) including plain_aggregation
 * (_kernels.py:79-120) with identical aggregates.
 * Errors: SPFD_ENOTPOS (non-positive diagonal), SPFD_EINVAL.
 * Synchronises `stream`. */
int spfd_amg_setup_op(spfd_op_t op, const spfd_config *h_cfg, void *stream,
                      spfd_amg_t *out);
int spfd_amg_setup_csr(int64_t n, int64_t nnz, const int64_t *indptr,
                       const int32_t *indices, const double *data,
                       const spfd_config *h_cfg, void *stream, spfd_amg_t *out);
int spfd_amg_destroy(spfd_amg_t amg);
int spfd_amg_info_get(spfd_amg_t amg, spfd_amg_info *h_info);

/* Level export (device destinations; sizes from spfd_amg_info):
 *   which = 0: A_l, 1: P_l, 2: R_l as CSR (indptr int64[rows+1], indices
 *   int32[nnz], data double[nnz]); level 0 A is the operator CSR.
 *   spfd_amg_level_agg: int32[rows_l] aggregate id per row of level l.    */
int spfd_amg_level_csr(spfd_amg_t amg, int level, int which, int64_t *indptr,
                       int32_t *indices, double *data, void *stream);
int spfd_amg_level_agg(spfd_amg_t amg, int level, int32_t *agg, void *stream);

/* z = V-cycle(r) (linsolve.py:179-197), planar nrhs, level-0 ordering
 * (DOF order for an operator hierarchy, row order for a CSR one). */
int spfd_vcycle(spfd_amg_t amg, const double *r, double *z, int nrhs,
                void *stream);

typedef struct {
    int32_t iterations;          /* Krylov iterations (max over rhs)         */
    int32_t converged;           /* all rhs at rel_residual <= rel_tol       */
    double  rel_residual[2];     /* true ||b - A x|| / ||b|| per rhs          */
    double  solve_seconds;       /* device-timed                             */
    int32_t status;              /* SPFD_OK or the error code                */
} spfd_report;

/* Solve A x = b (x starts at 0).  method from cfg (PCG default; FGMRES(m)
 * with the reference semantics, linsolve.py:200-298).  Non-convergence is
 * a report flag, not an error.  h_trace (may be NULL) receives
 * max_iters*nrhs residual estimates (iteration-major).
 * Synchronises `stream` (the report is host data). */
int spfd_solve(spfd_amg_t amg, const double *b, double *x, int nrhs,
               const spfd_config *h_cfg, spfd_report *h_rep, double *h_trace,
               void *stream);

/* ---- device-resident snapshot pipeline (pipeline.py:158-175, C5) ------- */

/* One snapshot on a resident operator + hierarchy: rhs assembly, solve and
 * fused E-field/voxel average, all on `stream`.  vox double[nrhs][n_cond_voxels];
 * psi (may be NULL) double[nrhs][n_dofs]. */
int spfd_snapshot(spfd_op_t op, spfd_amg_t amg, const double *a, double omega,
                  double *psi, double *vox, int nrhs, const spfd_config *h_cfg,
                  spfd_report *h_rep, void *stream);

/* ---- multi-GPU z-slabs --------------------------------------- */

typedef struct spfd_comm_s *spfd_comm_t;

/* Host transport (testing several processes on one GPU, or any custom
 * transport): the library synchronises its stream, then calls
 *   exchange(user, n, peer[], kind[], buf[], bytes[])  kind 0 = send, 1 = recv
 *   allgather(user, send, recv, bytes)                 rank-ordered
 * with DEVICE buffers; both must complete before returning 0. */
typedef struct {
    void *user;
    int (*exchange)(void *user, int n, const int *peer, const int *kind, void *const *buf, const int64_t *bytes);
    int (*allgather)(void *user, const void *send, void *recv, int64_t bytes);
} spfd_comm_callbacks;

/* NCCL transport over NVLink / NVSwitch (NCCL loaded with dlopen).
 * h_unique_id: 128-byte ncclUniqueId produced by spfd_nccl_unique_id on
 * one rank and broadcast (e.g. with torch.distributed). */
int spfd_nccl_unique_id(void *h_unique_id);
int spfd_comm_init_nccl(const void *h_unique_id, int rank, int nranks, spfd_comm_t *out);
int spfd_comm_init_callbacks(const spfd_comm_callbacks *h_cb, int rank, int nranks, spfd_comm_t *out);
int spfd_comm_destroy(spfd_comm_t comm);

/* Attach a z-slab decomposition to an operator hierarchy (collective; every
 * rank holds the identical operator and hierarchy, so aggregates and
 * iteration counts do not depend on the number of GPUs).  Rank r owns the
 * node planes [k_r, k_{r+1}) balanced by span positions; coarse rows belong
 * to the rank owning their aggregate's lowest member; levels below
 * `replicate_below` rows are solved redundantly on every rank.  Afterwards
 * spfd_solve / spfd_snapshot run distributed: halo planes and coarse halos
 * travel over the transport, dot products are allgathered and summed in rank
 * order (bitwise reproducible for a fixed rank count).  Vectors stay
 * full-length; only the owned range is computed.
 *   h_range[0..5] (out): first/last+1 DOF, first/last+1 conductive voxel
 *   owned by this rank (psi / vox outputs are valid there), and the owned
 *   node planes [k_r, k_{r+1}). */
int spfd_amg_distribute(spfd_amg_t amg, spfd_comm_t comm, int64_t replicate_below, int64_t *h_range,
                        void *stream);

/* ---- field sources, cleaning, gauging, statistics ------ */

/* A voxel grid (dims = voxels per axis, StaggeredGrid) or a sampling
 * lattice (dims = points per axis, field_source.Lattice). */
typedef struct {
    int64_t dims[3];
    double  spacing[3];
    double  origin[3];
} spfd_box;

typedef struct spfd_field_s *spfd_field_t;  /* per-grid workspace + cleaning AMG */

/* cfg: AMG / Krylov settings of the divergence-cleaning solve (the
 * reference passes its SolveConfig, field_source.py:313-316). */
int spfd_field_create(const spfd_box *h_grid, const spfd_config *h_cfg, spfd_field_t *out);
int spfd_field_destroy(spfd_field_t f);

/* f3: Biot-Savart field of a closed polyline (coil_field,
 * field_source.py:163-197).  pts double[n][3], verts double[nseg+1][3],
 * out double[n][3]; scale = mu0 I / (4 pi).  SPFD_ESINGULAR when a point is
 * within 1e-12 m of a segment.  Synchronises `stream`. */
int spfd_coil_field(int64_t n, const double *pts, int nseg, const double *verts, double scale,
                    double *out, void *stream);

/* f3: face fluxes from lattice samples (interpolate_to_faces,
 * field_source.py:254-272): trilinear interpolation / linear extrapolation
 * of the normal component at each face centre times the face area.
 *   b double[n_points][3] (FieldSampleSet.b, lattice x-fastest),
 *   flux double[n_faces].  Bit-identical to the reference.
 * SPFD_ELATTICE for a single-point lattice axis off the query plane. */
int spfd_field_interpolate(spfd_field_t f, const spfd_box *h_lattice, const double *b, double *flux,
                           void *stream);

/* f2: cell net outflux div = build_divergence(grid) @ flux
 * (fit_operators.py:276-286), bit-identical.  div double[n_cells]. */
int spfd_field_divergence(spfd_field_t f, const double *flux, double *div, void *stream);

typedef struct {
    double  rel_before;          /* ||div flux|| / ||flux||                  */
    double  rel_after;           /* after the projection (= before if none)  */
    int32_t solved;              /* 1 if the projection solve ran            */
    int32_t iterations;
    double  solve_rel_residual;
    double  setup_seconds;       /* AMG setup on div divT (first call only)  */
} spfd_clean_info;

/* f2: divergence_clean (field_source.py:292-329): out = in if the relative
 * cell-outflux norm is <= tol, else in - divT phi with
 * (div divT) phi = div in.  Default: a direct spectral solve (div divT is the
 * 7-point cell Laplacian with zero exterior: sine transforms in x and y, one
 * tridiagonal solve per mode along z), residual at rounding level, i.e.
 * within the reference's rel_tol = min(1e-12, tol/(4 rel)); h_info
 * iterations = 0.  SPFD_CLEAN_SOLVER=amg: the reference's method, AMG +
 * Krylov at that rel_tol, the hierarchy on div divT built on the first call
 * and kept by the handle.  SPFD_EPROJECTION on non-convergence or a
 * violated postcondition.  out may alias in. */
int spfd_field_clean(spfd_field_t f, const double *in, double *out, double tol,
                     spfd_clean_info *h_info, void *stream);
/* The same for nrhs = 1 or 2 flux vectors (planar [nrhs][n_faces], e.g.
 * the real and imaginary sample sets of a snapshot) with one batched
 * Krylov solve at the stricter of the two tolerances; per-vector decisions
 * and post-checks as above; h_info[nrhs]. */
int spfd_field_clean_batch(spfd_field_t f, int nrhs, const double *in, double *out, double tol,
                           spfd_clean_info *h_info, void *stream);

typedef struct {
    double  rel_residual;        /* ||C a - flux|| / ||flux||                */
    int64_t worst_face;          /* argmax |defect| if above tol, else -1    */
    double  worst_defect;
} spfd_gauge_info;

/* f1: comb-tree gauging (build_comb_tree + gauge_vector_potential,
 * gauging.py:34-71,137-172): edge potential a double[n_edges] with zero
 * tree edges reproducing the face fluxes, by three column prefix scans;
 * then the circulation residual over all faces is checked against tol
 * (SPFD_EINCOMPAT, info filled).  Zero fluxes give a = 0. */
int spfd_field_gauge(spfd_field_t f, const double *flux, double *a, double tol,
                     spfd_gauge_info *h_info, void *stream);
/* The same with the spanning tree selected (build_tree(grid, kind),
 * gauging.py:122-127): tree 0 = comb, 1 = BFS from node 0
 * (build_bfs_tree, gauging.py:74-119: all x-edges, the y-edges of the plane
 * i = 0 and the z-edges of the line i = j = 0), whose FIFO elimination
 * (_kernels.py:12-76) unrolls into running sums along x. */
int spfd_field_gauge_tree(spfd_field_t f, int tree, const double *flux, double *a, double tol,
                          spfd_gauge_info *h_info, void *stream);

/* circulation_residual (gauging.py:127-134): defect double[n_faces] */
int spfd_field_circulation(spfd_field_t f, const double *a, const double *flux, double *defect,
                           void *stream);

/* f4: exposure statistics (build_exposure_report + percentile99,
 * dosimetry.py:119-127,195-234) over n voxel values:
 *   scaled[v] = values[v] * scale (RMS_FACTOR or 1), tissue of v =
 *   ids_box[vox_index[v]]; per tissue id < n_ids: count, mean, max and the
 *   nearest-rank 99th percentile (sorted index ceil(0.99 c) - 1); h_global =
 *   {p99, max} over all values.  p99 and max are exact selections.
 * Host outputs have n_ids entries.  Synchronises `stream`. */
int spfd_exposure_stats(const double *values, int64_t n, double scale, const int64_t *vox_index,
                        const uint16_t *ids_box, int32_t n_ids, double *scaled, int64_t *h_count,
                        double *h_mean, double *h_max, double *h_p99, double *h_global, void *stream);

/* ---- measurement ---------------------------------------------------------- */

/* Time `reps` back-to-back launches of one solve kernel between CUDA
 * events on `stream` (after 3 warm-up launches):
 *   which = 0 fine SpMV q = A p (+ p.q partials), 1 fused pre-smooth +
 *   defect (also the restriction input), 2 post-smooth sweep (+ r.z),
 *   3 one full V-cycle, 4 fine matrix-free prolongation, 5 restriction
 *   sums over the aggregates, 6 level-1 pre-smooth residual, 7 level-1
 *   fused prolongation + post-smooth, 8 PCG r update (+ r.r), 9 PCG p update,
 *   10 fused pre-smooth + restriction input, 11 fused prolongation +
 *   post-smooth (10, 11: only while the fused fine kernel is selected).
 * h_ms: ms per launch; h_bytes: algorithmic bytes per launch (3: the whole
 * V-cycle).  Kernels 4-7 need the corresponding levels (else EINVAL). */
int spfd_bench_kernel(spfd_amg_t amg, int which, int reps, int nrhs, double *h_ms, double *h_bytes,
                      void *stream);
/* Algorithmic HBM bytes of one PCG iteration with `nrhs` batched rhs: the
 * SpMV, the V-cycle (every level) and the three vector updates. */
int spfd_iteration_bytes(spfd_amg_t amg, int nrhs, double *h_bytes);
/* Tuning knob (not part of the reference API): select the fine-level
 * stencil kernel used by every later solve / V-cycle in this process.
 * kind = -1 default (environment SPFD_SPAN_KERNEL=flat|pf, else pf), 2 flat
 * per-position kernel, 3 the same with the tile's streamed arrays
 * bulk-prefetched into L2.  Both give bit-identical stencil outputs; this
 * exists for A/B tests. */
int spfd_set_fine_kernel(int kind);
/* Tuning knob: run PCG as one CUDA graph with a device-side WHILE node
 * (mode 1, the default) or as the host-driven loop (mode 0); -1 restores the
 * default / environment (SPFD_PCG_GRAPH).  Same arithmetic, same bits. */
int spfd_set_pcg_graph(int mode);
/* Number of kernels this library has launched so far (process-wide). */
int64_t spfd_launch_count(void);
/* Synchronous copy between any host/device pointers (host transports). */
int spfd_copy(void *dst, const void *src, int64_t bytes);

#ifdef __cplusplus
}
#endif
#endif /* SPFD_B200_H */

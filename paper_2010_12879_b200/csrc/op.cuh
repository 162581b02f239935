// Voxel operator: grid, conductances, DOF map and the row-span layout.
//
// Row-span layout ("spans"): every x-row (j, k) of the node box stores the
// contiguous index range [lo, hi) that covers all conductive nodes of the row
// (DOFs and pinned nodes).  Vectors, conductances and masks live in a flat
// array of length L = sum(hi - lo), rows in (k, j) order, so positions are in
// ascending node order exactly like the reference's DOF numbering with the
// (rare) non-DOF positions kept as zeros.  The +x/+y/+z neighbours of a node
// are found through the 16-byte row table; no per-node index is stored.
#pragma once
#include "common.cuh"

namespace spfd {

constexpr int kTile = 1024;          // positions per CTA in span kernels
constexpr int kSpanThreads = 256;    // threads per CTA in span kernels

struct Operator {
    int64_t nx, ny, nz;              // voxels
    int64_t NX, NY, NZ;              // nodes per axis
    double sx, sy, sz;               // spacing
    double gx, gy, gz;               // dual-area / length per edge axis
    int64_t n_nodes, n_edges, n_vox;
    int64_t eoff[3];                 // edge block offsets
    int64_t n_dofs = 0, n_cond = 0, n_comp = 0, n_cond_vox = 0, nnz = 0;
    int64_t L = 0, n_rows = 0, n_tiles = 0;
    int pin = 1;

    DevBuf<int4> rows;               // [n_rows+1] {off, lo, hi, j|k<<?>}  (sentinel at end)
    DevBuf<int32_t> tile_row;        // [n_tiles+1] first row of each tile
    DevBuf<double> wx, wy, wz;       // [L] edge conductance of the +axis edge at each position
    DevBuf<double> diag;             // [L] reference-order diagonal (0 for non-DOF)
    DevBuf<double> dinv;             // [L] 1/diag (0 for non-DOF)
    DevBuf<uint32_t> dofmask;        // [(L+31)/32]
    DevBuf<int32_t> pos_to_dof;      // [L]  -1 = not a DOF
    DevBuf<int32_t> dof_to_pos;      // [N]
    DevBuf<int64_t> pinned;          // [n_comp]
    DevBuf<uint8_t> vox_cond;        // [n_vox] kappa > 0
    DevBuf<int32_t> vrow_off;        // [ny*nz+1] conductive-voxel offsets per voxel row
    DevBuf<int32_t> nnz_row;         // [N+1] CSR row pointer cache (int32 counts, built lazily)
    DevBuf<double> ws_a, ws_b;       // span workspaces [L*2]
    int64_t device_bytes() const {
        return rows.bytes() + tile_row.bytes() + wx.bytes() + wy.bytes() + wz.bytes() +
               diag.bytes() + dinv.bytes() + dofmask.bytes() + pos_to_dof.bytes() +
               dof_to_pos.bytes() + pinned.bytes() + vox_cond.bytes() + vrow_off.bytes() +
               nnz_row.bytes() + ws_a.bytes() + ws_b.bytes();
    }
};

// Views passed by value into kernels.
struct SpanView {
    const int4 *rows;
    const int32_t *tile_row;
    const double *wx, *wy, *wz;
    const uint32_t *mask;
    int64_t L;
    int NY;        // rows per k-plane (= ny+1)
    int n_rows;
};

inline SpanView span_view(const Operator &op) {
    return SpanView{op.rows.get(), op.tile_row.get(), op.wx.get(), op.wy.get(), op.wz.get(),
                    op.dofmask.get(), op.L, (int)op.NY, (int)op.n_rows};
}

// Owned position range [pb, pe) of a span kernel launch (z-slab).
struct PosRange {
    int64_t pb, pe;
    int tile0, tiles;
};
PosRange pos_range(const Operator &op, int64_t pb, int64_t pe);  // pe < 0: up to L

// Host entry points implemented in op.cu
Operator *op_create(const int64_t *dims, const double *spacing, const uint16_t *ids,
                    const double *lut, int64_t lut_len, int pin, cudaStream_t s);
void op_export(Operator &op, int what, void *dst, cudaStream_t s);
void op_csr(Operator &op, int64_t *indptr, int32_t *indices, double *data, cudaStream_t s);
void op_dofs_to_span(const Operator &op, const double *planar, double *span, int nrhs,
                     cudaStream_t s);
void op_span_to_dofs(const Operator &op, const double *span, double *planar, int nrhs,
                     cudaStream_t s);
void op_stencil_span(const Operator &op, const double *x, double *y, int nrhs, cudaStream_t s);
void op_rhs_span(const Operator &op, const double *a, double *rhs_span, int nrhs,
                 cudaStream_t s, int64_t pb = 0, int64_t pe = -1);
void op_node_field_span(const Operator &op, const double *a, const double *psi_span, double omega,
                        double *node_span, int nrhs, cudaStream_t s, int64_t pb, int64_t pe);
void op_voxavg_span(const Operator &op, const double *node_span, double *vox, int nrhs, cudaStream_t s,
                    int64_t vr_b, int64_t vr_e);
void op_edge_voltages(const Operator &op, const double *a, const double *psi_span,
                      double omega, double *v, int nrhs, cudaStream_t s);
void op_node_field(const Operator &op, const double *v, double *node, int nrhs, cudaStream_t s);
void op_voxel_average(const Operator &op, const double *node, double *vox, int nrhs,
                      cudaStream_t s);
void op_efield_voxavg_span(const Operator &op, const double *a, const double *psi_span,
                           double omega, double *vox, double *node_span_ws, int nrhs,
                           cudaStream_t s);

}  // namespace spfd

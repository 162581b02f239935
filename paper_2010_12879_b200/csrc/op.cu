// Voxel operator construction, matrix-free 7-point stencil, RHS assembly,
// CSR materialisation and the E-field / voxel-average chain (sm_100a).
//
// Reference parity: every floating-point expression below reproduces the
// reference's numpy/scipy evaluation order with explicitly rounded ops
// (no FMA contraction), so conductances, the matrix, the RHS, the stencil
// product and the E-field chain are bit-identical to
//   fit_operators.py:289-324 (edge_conductance / _mean4),
//   fit_operators.py:421-441 (COO->CSR assembly, bincount RHS),
//   scipy csr_matvec (sorted-column accumulation),
//   dosimetry.py:27-116 (edge voltages, node |E|, corner mean).
#include <cub/cub.cuh>

#include "op.cuh"

namespace spfd {

// ------------------------------------------------------------------------
// small helpers
// ------------------------------------------------------------------------

template <class T>
static void exclusive_scan(const T *in, T *out, int64_t n, cudaStream_t s) {
    size_t bytes = 0;
    SPFD_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, s));
    DevBuf<uint8_t> tmp;
    tmp.alloc(bytes);
    SPFD_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), bytes, in, out, n, s));
    SPFD_CUDA(cudaStreamSynchronize(s));
}

template <class T>
static T read_scalar(const T *dev, cudaStream_t s) {
    T h;
    SPFD_CUDA(cudaMemcpyAsync(&h, dev, sizeof(T), cudaMemcpyDeviceToHost, s));
    SPFD_CUDA(cudaStreamSynchronize(s));
    return h;
}

__device__ __forceinline__ bool mask_bit(const uint32_t *m, int64_t p) {
    return (m[p >> 5] >> (p & 31)) & 1u;
}

// Position of node (i, row r) or -1 when outside the row's span.
__device__ __forceinline__ int span_pos(const int4 *rows, int r, int i) {
    int4 q = rows[r];
    return (i >= q.y && i < q.z) ? q.x + (i - q.y) : -1;
}

// Row containing position p, searching rows [r0, r1] (r0 contains the
// CTA's first position).  Empty rows share the offset of the next row, so
// the last row with off <= p is the non-empty one.
__device__ __forceinline__ int find_row(const int4 *rows, int r0, int r1, int p) {
    int lo = r0, hi = r1;  // invariant: rows[lo].x <= p
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (rows[mid].x <= p) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// ------------------------------------------------------------------------
// operator construction
// ------------------------------------------------------------------------

struct Geo {
    int nx, ny, nz, NX, NY, NZ;
};

__global__ void k_vox_cond(const uint16_t *ids, const double *lut, int64_t lut_len,
                           int64_t n_vox, uint8_t *cond, int *bad) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n_vox;
         v += (int64_t)gridDim.x * blockDim.x) {
        uint16_t id = ids[v];
        if (id >= lut_len) { *bad = 1; cond[v] = 0; continue; }
        cond[v] = lut[id] > 0.0 ? 1 : 0;
    }
}

__device__ __forceinline__ bool vox_ok(const uint8_t *c, Geo g, int i, int j, int k) {
    if (i < 0 || j < 0 || k < 0 || i >= g.nx || j >= g.ny || k >= g.nz) return false;
    return c[i + (int64_t)g.nx * (j + (int64_t)g.ny * k)] != 0;
}

// Conductive edge = a conductive voxel among its <= 4 neighbours
// (voxel_model.py:448-456).
__device__ __forceinline__ bool edge_cond(const uint8_t *c, Geo g, int axis, int i, int j, int k) {
    if (axis == 0)
        return vox_ok(c, g, i, j - 1, k - 1) || vox_ok(c, g, i, j - 1, k) ||
               vox_ok(c, g, i, j, k - 1) || vox_ok(c, g, i, j, k);
    if (axis == 1)
        return vox_ok(c, g, i - 1, j, k - 1) || vox_ok(c, g, i - 1, j, k) ||
               vox_ok(c, g, i, j, k - 1) || vox_ok(c, g, i, j, k);
    return vox_ok(c, g, i - 1, j - 1, k) || vox_ok(c, g, i - 1, j, k) ||
           vox_ok(c, g, i, j - 1, k) || vox_ok(c, g, i, j, k);
}

// Node conductive = touches a conductive voxel (voxel_model.py:459-467);
// initialise union-find parents.
__global__ void k_node_init(const uint8_t *vc, Geo g, int64_t n_nodes, int32_t *parent) {
    for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < n_nodes;
         n += (int64_t)gridDim.x * blockDim.x) {
        int i = (int)(n % g.NX);
        int64_t t = n / g.NX;
        int j = (int)(t % g.NY);
        int k = (int)(t / g.NY);
        bool c = false;
        for (int dk = -1; dk <= 0 && !c; ++dk)
            for (int dj = -1; dj <= 0 && !c; ++dj)
                for (int di = -1; di <= 0 && !c; ++di) c = vox_ok(vc, g, i + di, j + dj, k + dk);
        parent[n] = c ? (int32_t)n : -1;
    }
}

__device__ __forceinline__ int32_t uf_find(int32_t *parent, int32_t x) {
    int32_t p = parent[x];
    while (p != x) {
        int32_t gp = parent[p];
        if (gp != p) parent[x] = gp;  // path halving; benign race
        x = p;
        p = parent[x];
    }
    return x;
}

// Lock-free union: always hang the larger root under the smaller one, so
// every component's final root is its lowest node index (the node the
// reference pins, fit_operators.py:398-399).
__device__ void uf_union(int32_t *parent, int32_t a, int32_t b) {
    while (true) {
        a = uf_find(parent, a);
        b = uf_find(parent, b);
        if (a == b) return;
        int32_t hi = a > b ? a : b, lo = a > b ? b : a;
        if (atomicCAS(&parent[hi], hi, lo) == hi) return;
    }
}

__global__ void k_union_edges(const uint8_t *vc, Geo g, int64_t n_nodes, int32_t *parent) {
    for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < n_nodes;
         n += (int64_t)gridDim.x * blockDim.x) {
        if (parent[n] < 0) continue;
        int i = (int)(n % g.NX);
        int64_t t = n / g.NX;
        int j = (int)(t % g.NY);
        int k = (int)(t / g.NY);
        if (i < g.nx && edge_cond(vc, g, 0, i, j, k)) uf_union(parent, (int32_t)n, (int32_t)(n + 1));
        if (j < g.ny && edge_cond(vc, g, 1, i, j, k)) uf_union(parent, (int32_t)n, (int32_t)(n + g.NX));
        if (k < g.nz && edge_cond(vc, g, 2, i, j, k))
            uf_union(parent, (int32_t)n, (int32_t)(n + (int64_t)g.NX * g.NY));
    }
}

// Final compression; flags: 1 = conductive, 2 = component root (pinned).
__global__ void k_uf_flags(int32_t *parent, int64_t n_nodes, uint8_t *flags) {
    for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < n_nodes;
         n += (int64_t)gridDim.x * blockDim.x) {
        int32_t p = parent[n];
        if (p < 0) { flags[n] = 0; continue; }
        int32_t r = uf_find(parent, (int32_t)n);
        flags[n] = (uint8_t)(1 | (r == (int32_t)n ? 2 : 0));
    }
}

// One warp per node row: span [lo, hi) over conductive nodes.
__global__ void k_row_span(const uint8_t *flags, Geo g, int64_t n_rows, int *lo_out,
                           int *hi_out, int *len_out) {
    int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    for (int64_t r = warp; r < n_rows; r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const uint8_t *f = flags + r * g.NX;
        int lo = INT_MAX, hi = -1;
        for (int i = lane; i < g.NX; i += 32)
            if (f[i]) { lo = min(lo, i); hi = max(hi, i); }
        for (int o = 16; o > 0; o >>= 1) {
            lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        if (lane == 0) {
            if (hi < 0) { lo_out[r] = 0; hi_out[r] = 0; len_out[r] = 0; }
            else { lo_out[r] = lo; hi_out[r] = hi + 1; len_out[r] = hi + 1 - lo; }
        }
    }
}

// row table entry {offset, lo, hi, j}
__global__ void k_rows_pack(const int *lo, const int *hi, const int *off, int64_t n_rows,
                            int64_t L, int NY, int4 *rows) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r <= n_rows;
         r += (int64_t)gridDim.x * blockDim.x) {
        if (r == n_rows) rows[r] = make_int4((int)L, 0, 0, 0);
        else rows[r] = make_int4(off[r], lo[r], hi[r], (int)(r % NY));
    }
}

__global__ void k_tile_rows(const int4 *rows, int64_t n_rows, int64_t n_tiles, int32_t *tile_row) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t <= n_tiles;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t p = t * kTile;
        int lo = 0, hi = (int)n_rows - 1;
        while (lo < hi) {
            int mid = (lo + hi + 1) >> 1;
            if (rows[mid].x <= p) lo = mid; else hi = mid - 1;
        }
        tile_row[t] = lo;
    }
}

// Sum of the <= 4 voxel conductivities around an edge in the reference's
// (da, db) order, then *0.25, then *geom (fit_operators.py:289-324).
__device__ __forceinline__ double kap(const uint16_t *ids, const double *lut, Geo g, int i, int j,
                                      int k) {
    if (i < 0 || j < 0 || k < 0 || i >= g.nx || j >= g.ny || k >= g.nz) return 0.0;
    return lut[ids[i + (int64_t)g.nx * (j + (int64_t)g.ny * k)]];
}

__device__ double edge_w(const uint16_t *ids, const double *lut, Geo g, int axis, int i, int j,
                         int k, double geom) {
    double a0, a1, a2, a3;
    if (axis == 0) {
        if (i >= g.nx) return 0.0;
        a0 = kap(ids, lut, g, i, j - 1, k - 1); a1 = kap(ids, lut, g, i, j - 1, k);
        a2 = kap(ids, lut, g, i, j, k - 1);     a3 = kap(ids, lut, g, i, j, k);
    } else if (axis == 1) {
        if (j >= g.ny) return 0.0;
        a0 = kap(ids, lut, g, i - 1, j, k - 1); a1 = kap(ids, lut, g, i - 1, j, k);
        a2 = kap(ids, lut, g, i, j, k - 1);     a3 = kap(ids, lut, g, i, j, k);
    } else {
        if (k >= g.nz) return 0.0;
        a0 = kap(ids, lut, g, i - 1, j - 1, k); a1 = kap(ids, lut, g, i - 1, j, k);
        a2 = kap(ids, lut, g, i, j - 1, k);     a3 = kap(ids, lut, g, i, j, k);
    }
    double acc = add_rn(add_rn(add_rn(a0, a1), a2), a3);
    return mul_rn(mul_rn(acc, 0.25), geom);
}

// One warp per row: conductances and DOF flags at every span position.
__global__ void k_fill_span(const uint16_t *ids, const double *lut, const uint8_t *flags, Geo g,
                            const int4 *rows, int64_t n_rows, double gx, double gy, double gz,
                            int pin, double *wx, double *wy, double *wz, int32_t *isdof) {
    int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    for (int64_t r = warp; r < n_rows; r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        int4 q = rows[r];
        int j = (int)(r % g.NY), k = (int)(r / g.NY);
        for (int i = q.y + lane; i < q.z; i += 32) {
            int p = q.x + (i - q.y);
            wx[p] = edge_w(ids, lut, g, 0, i, j, k, gx);
            wy[p] = edge_w(ids, lut, g, 1, i, j, k, gy);
            wz[p] = edge_w(ids, lut, g, 2, i, j, k, gz);
            uint8_t f = flags[r * g.NX + i];
            bool dof = (f & 1) && !(pin && (f & 2));
            isdof[p] = dof ? 1 : 0;
        }
    }
}

// Pack DOF flags into a bitmap, build pos_to_dof / dof_to_pos.
__global__ void k_dof_maps(const int32_t *isdof, const int32_t *dofidx, int64_t L,
                           int32_t *pos_to_dof, int32_t *dof_to_pos, uint32_t *mask) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < L;
         p += (int64_t)gridDim.x * blockDim.x) {
        bool d = isdof[p] != 0;
        unsigned b = __ballot_sync(__activemask(), d);
        if (d) { pos_to_dof[p] = dofidx[p]; dof_to_pos[dofidx[p]] = (int32_t)p; }
        else pos_to_dof[p] = -1;
        if ((threadIdx.x & 31) == 0) mask[p >> 5] = b;
    }
}

// Neighbour weights of the -x/-y/-z edges of position p (row r, column i).
struct MinusW {
    double wxm, wym, wzm;
    int pxm, pym, pzm;  // positions (or -1)
};

__device__ __forceinline__ MinusW minus_edges(const SpanView &v, int p, int r, int i, int4 q) {
    MinusW m;
    m.pxm = (i > q.y) ? p - 1 : -1;
    int j = r % v.NY;
    m.pym = (j > 0) ? span_pos(v.rows, r - 1, i) : -1;
    m.pzm = (r >= v.NY) ? span_pos(v.rows, r - v.NY, i) : -1;
    m.wxm = m.pxm >= 0 ? v.wx[m.pxm] : 0.0;
    m.wym = m.pym >= 0 ? v.wy[m.pym] : 0.0;
    m.wzm = m.pzm >= 0 ? v.wz[m.pzm] : 0.0;
    return m;
}

// Reference-order diagonal: tail edges x,y,z then head edges x,y,z
// (COO order of fit_operators.py:425-428 summed by csr_sum_duplicates).
__global__ void k_diag(SpanView v, double *diag, double *dinv, int *bad) {
    int t = blockIdx.x;
    int r0 = v.tile_row[t], r1 = v.tile_row[t + 1];
    for (int u = 0; u < kTile / kSpanThreads; ++u) {
        int p = t * kTile + u * kSpanThreads + threadIdx.x;
        if (p >= v.L) break;
        int r = find_row(v.rows, r0, r1, p);
        int4 q = v.rows[r];
        int i = q.y + (p - q.x);
        MinusW m = minus_edges(v, p, r, i, q);
        double d = add_rn(add_rn(add_rn(add_rn(add_rn(v.wx[p], v.wy[p]), v.wz[p]), m.wxm), m.wym),
                          m.wzm);
        bool dof = mask_bit(v.mask, p);
        if (dof && !(d > 0.0)) *bad = 1;
        diag[p] = dof ? d : 0.0;
        dinv[p] = dof ? 1.0 / d : 0.0;
    }
}

// Conductive voxels per voxel row.
__global__ void k_vrow_count(const uint8_t *vc, Geo g, int64_t n_vrows, int *cnt) {
    int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    for (int64_t r = warp; r < n_vrows; r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const uint8_t *c = vc + r * g.nx;
        int s = 0;
        for (int i = lane; i < g.nx; i += 32) s += c[i];
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) cnt[r] = s;
    }
}

// Per DOF: number of CSR entries (self + DOF neighbours).
__global__ void k_csr_count(SpanView v, const int32_t *pos_to_dof, int32_t *cnt) {
    int t = blockIdx.x;
    int r0 = v.tile_row[t], r1 = v.tile_row[t + 1];
    for (int u = 0; u < kTile / kSpanThreads; ++u) {
        int p = t * kTile + u * kSpanThreads + threadIdx.x;
        if (p >= v.L) break;
        int d = pos_to_dof[p];
        if (d < 0) continue;
        int r = find_row(v.rows, r0, r1, p);
        int4 q = v.rows[r];
        int i = q.y + (p - q.x);
        int j = r % v.NY;
        int c = 1;
        int nb[6];
        nb[0] = (r >= v.NY) ? span_pos(v.rows, r - v.NY, i) : -1;
        nb[1] = (j > 0) ? span_pos(v.rows, r - 1, i) : -1;
        nb[2] = (i > q.y) ? p - 1 : -1;
        nb[3] = (i + 1 < q.z) ? p + 1 : -1;
        nb[4] = (r + 1 < v.n_rows && j + 1 < v.NY) ? span_pos(v.rows, r + 1, i) : -1;
        nb[5] = (r + v.NY < v.n_rows) ? span_pos(v.rows, r + v.NY, i) : -1;
        // off-diagonals exist only for active edges between two DOFs
        double w[6];
        MinusW m = minus_edges(v, p, r, i, q);
        w[0] = m.wzm; w[1] = m.wym; w[2] = m.wxm; w[3] = v.wx[p]; w[4] = v.wy[p]; w[5] = v.wz[p];
        for (int s = 0; s < 6; ++s) c += (nb[s] >= 0 && w[s] > 0.0 && pos_to_dof[nb[s]] >= 0);
        cnt[d] = c;
    }
}

__global__ void k_csr_fill(SpanView v, const int32_t *pos_to_dof, const double *diag,
                           const int64_t *indptr, int32_t *indices, double *data) {
    int t = blockIdx.x;
    int r0 = v.tile_row[t], r1 = v.tile_row[t + 1];
    for (int u = 0; u < kTile / kSpanThreads; ++u) {
        int p = t * kTile + u * kSpanThreads + threadIdx.x;
        if (p >= v.L) break;
        int d = pos_to_dof[p];
        if (d < 0) continue;
        int r = find_row(v.rows, r0, r1, p);
        int4 q = v.rows[r];
        int i = q.y + (p - q.x);
        int j = r % v.NY;
        int nb[6];
        nb[0] = (r >= v.NY) ? span_pos(v.rows, r - v.NY, i) : -1;
        nb[1] = (j > 0) ? span_pos(v.rows, r - 1, i) : -1;
        nb[2] = (i > q.y) ? p - 1 : -1;
        nb[3] = (i + 1 < q.z) ? p + 1 : -1;
        nb[4] = (r + 1 < v.n_rows && j + 1 < v.NY) ? span_pos(v.rows, r + 1, i) : -1;
        nb[5] = (r + v.NY < v.n_rows) ? span_pos(v.rows, r + v.NY, i) : -1;
        MinusW m = minus_edges(v, p, r, i, q);
        double w[6] = {m.wzm, m.wym, m.wxm, v.wx[p], v.wy[p], v.wz[p]};
        int64_t o = indptr[d];
        for (int s = 0; s < 6; ++s) {
            if (s == 3) { indices[o] = d; data[o] = diag[p]; ++o; }
            if (nb[s] >= 0 && w[s] > 0.0) {
                int dn = pos_to_dof[nb[s]];
                if (dn >= 0) { indices[o] = dn; data[o] = -w[s]; ++o; }
            }
        }
    }
}

Operator *op_create(const int64_t *dims, const double *spacing, const uint16_t *ids,
                    const double *lut, int64_t lut_len, int pin, cudaStream_t s) {
    SPFD_CHECK(dims[0] >= 1 && dims[1] >= 1 && dims[2] >= 1, SPFD_EINVAL, "dims must be >= 1");
    SPFD_CHECK(spacing[0] > 0 && spacing[1] > 0 && spacing[2] > 0, SPFD_EINVAL,
               "spacing must be positive");
    SPFD_CHECK(lut_len >= 1, SPFD_EINVAL, "empty conductivity LUT");
    auto *op = new Operator();
    try {
        op->nx = dims[0]; op->ny = dims[1]; op->nz = dims[2];
        op->NX = op->nx + 1; op->NY = op->ny + 1; op->NZ = op->nz + 1;
        op->sx = spacing[0]; op->sy = spacing[1]; op->sz = spacing[2];
        // geom = face_area(axis) / spacing[axis] with face_area = s[t0]*s[t1]
        op->gx = (op->sy * op->sz) / op->sx;
        op->gy = (op->sx * op->sz) / op->sy;
        op->gz = (op->sx * op->sy) / op->sz;
        op->n_nodes = op->NX * op->NY * op->NZ;
        op->n_vox = op->nx * op->ny * op->nz;
        int64_t ex = op->nx * op->NY * op->NZ, ey = op->NX * op->ny * op->NZ,
                ez = op->NX * op->NY * op->nz;
        op->eoff[0] = 0; op->eoff[1] = ex; op->eoff[2] = ex + ey;
        op->n_edges = ex + ey + ez;
        op->pin = pin;
        SPFD_CHECK(op->n_nodes < (int64_t)INT32_MAX, SPFD_EINVAL, "grid too large for int32 node ids");
        Geo g{(int)op->nx, (int)op->ny, (int)op->nz, (int)op->NX, (int)op->NY, (int)op->NZ};
        const int T = 256;

        DevBuf<int> bad;
        bad.alloc(1);
        SPFD_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(int), s));
        op->vox_cond.alloc(op->n_vox);
        k_vox_cond<<<grid_for(op->n_vox, T, 148 * 32), T, 0, s>>>(ids, lut, lut_len, op->n_vox,
                                                                   op->vox_cond.get(), bad.get());
        SPFD_LAUNCH_CHECK();
        SPFD_CHECK(read_scalar(bad.get(), s) == 0, SPFD_EINVAL, "tissue id outside the LUT");

        // components (union-find over conductive edges)
        DevBuf<int32_t> parent;
        parent.alloc(op->n_nodes);
        DevBuf<uint8_t> flags;
        flags.alloc(op->n_nodes);
        int gn = grid_for(op->n_nodes, T, 148 * 32);
        k_node_init<<<gn, T, 0, s>>>(op->vox_cond.get(), g, op->n_nodes, parent.get());
        k_union_edges<<<gn, T, 0, s>>>(op->vox_cond.get(), g, op->n_nodes, parent.get());
        k_uf_flags<<<gn, T, 0, s>>>(parent.get(), op->n_nodes, flags.get());
        SPFD_LAUNCH_CHECK();

        // pinned nodes = component roots in ascending node order
        {
            DevBuf<int64_t> pin_tmp, cnt;
            pin_tmp.alloc(op->n_nodes);
            cnt.alloc(1);
            // flagged select of node indices with flags & 2
            cub::TransformInputIterator<uint8_t, RootFlag, const uint8_t *> rf(flags.get(), RootFlag());
            cub::CountingInputIterator<int64_t> ci(0);
            size_t bytes = 0;
            SPFD_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, ci, rf, pin_tmp.get(), cnt.get(),
                                                 op->n_nodes, s));
            DevBuf<uint8_t> tmp;
            tmp.alloc(bytes);
            SPFD_CUDA(cub::DeviceSelect::Flagged(tmp.get(), bytes, ci, rf, pin_tmp.get(), cnt.get(),
                                                 op->n_nodes, s));
            op->n_comp = read_scalar(cnt.get(), s);
            if (op->n_comp == 0) throw Error(SPFD_EEMPTY, "model has no conductive voxels: empty Poisson system");
            op->pinned.alloc(op->n_comp);
            SPFD_CUDA(cudaMemcpyAsync(op->pinned.get(), pin_tmp.get(), op->n_comp * sizeof(int64_t),
                                      cudaMemcpyDeviceToDevice, s));
        }

        // row spans
        op->n_rows = op->NY * op->NZ;
        DevBuf<int> lo, hi, len, off;
        lo.alloc(op->n_rows); hi.alloc(op->n_rows); len.alloc(op->n_rows + 1); off.alloc(op->n_rows + 1);
        SPFD_CUDA(cudaMemsetAsync(len.get() + op->n_rows, 0, sizeof(int), s));
        k_row_span<<<grid_for(op->n_rows * 32, T, 148 * 32), T, 0, s>>>(flags.get(), g, op->n_rows,
                                                                         lo.get(), hi.get(), len.get());
        SPFD_LAUNCH_CHECK();
        {
            DevBuf<int64_t> len64, off64;
            len64.alloc(op->n_rows + 1); off64.alloc(op->n_rows + 1);
            // widen to int64 for the total, then check it fits int32
            cub::TransformInputIterator<int64_t, WidenI32, const int *> wl(len.get(), WidenI32());
            size_t bytes = 0;
            SPFD_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, wl, off64.get(), op->n_rows + 1, s));
            DevBuf<uint8_t> tmp;
            tmp.alloc(bytes);
            SPFD_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), bytes, wl, off64.get(), op->n_rows + 1, s));
            op->L = read_scalar(off64.get() + op->n_rows, s);
            SPFD_CHECK(op->L < (int64_t)INT32_MAX - kTile, SPFD_EINVAL, "span layout exceeds int32");
            exclusive_scan(len.get(), off.get(), op->n_rows + 1, s);
        }
        op->rows.alloc(op->n_rows + 1);
        k_rows_pack<<<grid_for(op->n_rows + 1, T), T, 0, s>>>(lo.get(), hi.get(), off.get(), op->n_rows,
                                                             op->L, (int)op->NY, op->rows.get());
        op->n_tiles = (op->L + kTile - 1) / kTile;
        op->tile_row.alloc(op->n_tiles + 1);
        k_tile_rows<<<grid_for(op->n_tiles + 1, T), T, 0, s>>>(op->rows.get(), op->n_rows, op->n_tiles,
                                                              op->tile_row.get());
        SPFD_LAUNCH_CHECK();

        // span arrays
        int64_t L = op->L;
        op->wx.alloc(L + 4); op->wy.alloc(L + 4); op->wz.alloc(L + 4);  // +4: aligned bulk-copy supersets
        op->diag.alloc(L); op->dinv.alloc(L);
        op->pos_to_dof.alloc(L);
        op->dofmask.alloc((L + 31) / 32 + 1);
        SPFD_CUDA(cudaMemsetAsync(op->dofmask.get(), 0, op->dofmask.bytes(), s));
        DevBuf<int32_t> isdof, dofidx;
        isdof.alloc(L + 1); dofidx.alloc(L + 1);
        SPFD_CUDA(cudaMemsetAsync(isdof.get() + L, 0, sizeof(int32_t), s));
        k_fill_span<<<grid_for(op->n_rows * 32, T, 148 * 32), T, 0, s>>>(
            ids, lut, flags.get(), g, op->rows.get(), op->n_rows, op->gx, op->gy, op->gz, pin,
            op->wx.get(), op->wy.get(), op->wz.get(), isdof.get());
        SPFD_LAUNCH_CHECK();
        exclusive_scan(isdof.get(), dofidx.get(), L + 1, s);
        op->n_dofs = read_scalar(dofidx.get() + L, s);
        op->dof_to_pos.alloc(op->n_dofs);
        // grid must be a multiple of warps covering L exactly per warp for ballot packing
        {
            int64_t nthreads = ((L + 31) / 32) * 32;
            k_dof_maps<<<(int)((nthreads + T - 1) / T), T, 0, s>>>(isdof.get(), dofidx.get(), L,
                                                                   op->pos_to_dof.get(),
                                                                   op->dof_to_pos.get(),
                                                                   op->dofmask.get());
            SPFD_LAUNCH_CHECK();
        }
        {
            SpanView v = span_view(*op);
            SPFD_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(int), s));
            if (op->n_tiles > 0)
                k_diag<<<(int)op->n_tiles, kSpanThreads, 0, s>>>(v, op->diag.get(), op->dinv.get(), bad.get());
            SPFD_LAUNCH_CHECK();
            if (pin && op->n_dofs > 0)
                SPFD_CHECK(read_scalar(bad.get(), s) == 0, SPFD_EEMPTY,
                           "reduced system has a non-positive diagonal entry");
        }
        // conductive count = DOFs + pinned (pin) or DOFs (no pin)
        op->n_cond = op->n_dofs + (pin ? op->n_comp : 0);

        // voxel rows
        int64_t nvr = op->ny * op->nz;
        DevBuf<int> vcnt;
        vcnt.alloc(nvr + 1);
        SPFD_CUDA(cudaMemsetAsync(vcnt.get() + nvr, 0, sizeof(int), s));
        k_vrow_count<<<grid_for(nvr * 32, T, 148 * 32), T, 0, s>>>(op->vox_cond.get(), g, nvr, vcnt.get());
        SPFD_LAUNCH_CHECK();
        op->vrow_off.alloc(nvr + 1);
        exclusive_scan(vcnt.get(), op->vrow_off.get(), nvr + 1, s);
        op->n_cond_vox = read_scalar(op->vrow_off.get() + nvr, s);

        // CSR nnz
        {
            op->nnz_row.alloc(op->n_dofs + 1);
            SPFD_CUDA(cudaMemsetAsync(op->nnz_row.get(), 0, op->nnz_row.bytes(), s));
            SpanView v = span_view(*op);
            if (op->n_tiles > 0)
                k_csr_count<<<(int)op->n_tiles, kSpanThreads, 0, s>>>(v, op->pos_to_dof.get(),
                                                                        op->nnz_row.get());
            SPFD_LAUNCH_CHECK();
            DevBuf<int64_t> sum;
            sum.alloc(1);
            size_t bytes = 0;
            SPFD_CUDA(cub::DeviceReduce::Sum(nullptr, bytes, op->nnz_row.get(), sum.get(), op->n_dofs, s));
            DevBuf<uint8_t> tmp;
            tmp.alloc(bytes);
            SPFD_CUDA(cub::DeviceReduce::Sum(tmp.get(), bytes, op->nnz_row.get(), sum.get(), op->n_dofs, s));
            op->nnz = read_scalar(sum.get(), s);
        }
        op->ws_a.alloc(2 * L + 2);
        op->ws_b.alloc(2 * L + 2);
        SPFD_CUDA(cudaStreamSynchronize(s));
        if (op->n_dofs == 0 && pin) {
            // every component is a single pinned node: the reference also
            // returns an empty (0x0) system in this case
        }
        return op;
    } catch (...) {
        delete op;
        throw;
    }
}

// ------------------------------------------------------------------------
// DOF <-> span conversions (planar [nrhs][N] <-> interleaved [L][nrhs])
// ------------------------------------------------------------------------

__global__ void k_dofs_to_span(const int32_t *pos_to_dof, int64_t L, int64_t N, const double *in,
                               double *out, int nrhs) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < L;
         p += (int64_t)gridDim.x * blockDim.x) {
        int d = pos_to_dof[p];
        for (int k = 0; k < nrhs; ++k) out[p * nrhs + k] = d >= 0 ? in[k * N + d] : 0.0;
    }
}

__global__ void k_span_to_dofs(const int32_t *dof_to_pos, int64_t N, const double *in, double *out,
                               int nrhs) {
    for (int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; d < N;
         d += (int64_t)gridDim.x * blockDim.x) {
        int64_t p = dof_to_pos[d];
        for (int k = 0; k < nrhs; ++k) out[k * N + d] = in[p * nrhs + k];
    }
}

void op_dofs_to_span(const Operator &op, const double *planar, double *span, int nrhs,
                     cudaStream_t s) {
    k_dofs_to_span<<<grid_for(op.L, 256, 148 * 32), 256, 0, s>>>(op.pos_to_dof.get(), op.L, op.n_dofs,
                                                                 planar, span, nrhs);
    SPFD_LAUNCH_CHECK();
}

void op_span_to_dofs(const Operator &op, const double *span, double *planar, int nrhs,
                     cudaStream_t s) {
    if (op.n_dofs == 0) return;
    k_span_to_dofs<<<grid_for(op.n_dofs, 256, 148 * 32), 256, 0, s>>>(op.dof_to_pos.get(), op.n_dofs,
                                                                      span, planar, nrhs);
    SPFD_LAUNCH_CHECK();
}

// ------------------------------------------------------------------------
// matrix-free 7-point stencil  y = A x   (span layout, R interleaved rhs)
// ------------------------------------------------------------------------

template <int R>
struct Vec;
template <>
struct Vec<1> {
    using T = double;
    __device__ static T zero() { return 0.0; }
};
template <>
struct Vec<2> {
    using T = double2;
    __device__ static T zero() { return make_double2(0.0, 0.0); }
};

__device__ __forceinline__ double acc_prod(double s, double a, double x) { return add_rn(s, mul_rn(a, x)); }
__device__ __forceinline__ double2 acc_prod(double2 s, double a, double2 x) {
    return make_double2(add_rn(s.x, mul_rn(a, x.x)), add_rn(s.y, mul_rn(a, x.y)));
}

template <int R>
__global__ void __launch_bounds__(kSpanThreads) k_stencil(SpanView v, const typename Vec<R>::T *__restrict__ x,
                                                          typename Vec<R>::T *__restrict__ y) {
    using T = typename Vec<R>::T;
    int t = blockIdx.x;
    int r0 = v.tile_row[t], r1 = v.tile_row[t + 1];
#pragma unroll
    for (int u = 0; u < kTile / kSpanThreads; ++u) {
        int p = t * kTile + u * kSpanThreads + threadIdx.x;
        if (p >= v.L) break;
        int r = find_row(v.rows, r0, r1, p);
        int4 q = v.rows[r];
        int i = q.y + (p - q.x);
        int j = r % v.NY;
        T zero = Vec<R>::zero();
        T xc = x[p];
        double wxp = v.wx[p], wyp = v.wy[p], wzp = v.wz[p];
        double wxm = 0.0, wym = 0.0, wzm = 0.0;
        T xxm = zero, xym = zero, xzm = zero, xxp = zero, xyp = zero, xzp = zero;
        if (i > q.y) { wxm = v.wx[p - 1]; xxm = x[p - 1]; }
        if (i + 1 < q.z) xxp = x[p + 1];
        if (j > 0) {
            int pn = span_pos(v.rows, r - 1, i);
            if (pn >= 0) { wym = v.wy[pn]; xym = x[pn]; }
        }
        if (j + 1 < v.NY) {
            int pn = span_pos(v.rows, r + 1, i);
            if (pn >= 0) xyp = x[pn];
        }
        if (r >= v.NY) {
            int pn = span_pos(v.rows, r - v.NY, i);
            if (pn >= 0) { wzm = v.wz[pn]; xzm = x[pn]; }
        }
        if (r + v.NY < v.n_rows) {
            int pn = span_pos(v.rows, r + v.NY, i);
            if (pn >= 0) xzp = x[pn];
        }
        double d = add_rn(add_rn(add_rn(add_rn(add_rn(wxp, wyp), wzp), wxm), wym), wzm);
        // sorted-column order: z-, y-, x-, diag, x+, y+, z+
        T s = zero;
        s = acc_prod(s, -wzm, xzm);
        s = acc_prod(s, -wym, xym);
        s = acc_prod(s, -wxm, xxm);
        s = acc_prod(s, d, xc);
        s = acc_prod(s, -wxp, xxp);
        s = acc_prod(s, -wyp, xyp);
        s = acc_prod(s, -wzp, xzp);
        y[p] = mask_bit(v.mask, p) ? s : zero;
    }
}

void op_stencil_span(const Operator &op, const double *x, double *y, int nrhs, cudaStream_t s) {
    if (op.n_tiles == 0) return;
    SpanView v = span_view(op);
    if (nrhs == 1)
        k_stencil<1><<<(int)op.n_tiles, kSpanThreads, 0, s>>>(v, x, y);
    else
        k_stencil<2><<<(int)op.n_tiles, kSpanThreads, 0, s>>>(v, (const double2 *)x, (double2 *)y);
    SPFD_LAUNCH_CHECK();
}

// ------------------------------------------------------------------------
// RHS assembly  rhs = (sum_tail w a - sum_head w a)[dofs]  (fit_operators.py:438-441)
// ------------------------------------------------------------------------

struct EdgeIdx {
    int64_t eoff1, eoff2;
    int nx, ny, nz, NX, NY;
    __device__ int64_t ex(int i, int j, int k) const { return i + (int64_t)nx * (j + (int64_t)NY * k); }
    __device__ int64_t ey(int i, int j, int k) const {
        return eoff1 + i + (int64_t)NX * (j + (int64_t)ny * k);
    }
    __device__ int64_t ez(int i, int j, int k) const {
        return eoff2 + i + (int64_t)NX * (j + (int64_t)NY * k);
    }
};

inline EdgeIdx edge_idx(const Operator &op) {
    return EdgeIdx{op.eoff[1], op.eoff[2], (int)op.nx, (int)op.ny, (int)op.nz, (int)op.NX, (int)op.NY};
}

template <int R>
__global__ void __launch_bounds__(kSpanThreads) k_rhs(SpanView v, EdgeIdx e, const double *__restrict__ a,
                                                      int64_t E, typename Vec<R>::T *__restrict__ rhs, PosRange pr) {
    using T = typename Vec<R>::T;
    int t = pr.tile0 + blockIdx.x;
    int r0 = v.tile_row[t], r1 = v.tile_row[t + 1];
    for (int u = 0; u < kTile / kSpanThreads; ++u) {
        int p = t * kTile + u * kSpanThreads + threadIdx.x;
        if (p >= pr.pe) break;
        if (p < pr.pb) continue;
        int r = find_row(v.rows, r0, r1, p);
        int4 q = v.rows[r];
        int i = q.y + (p - q.x);
        int j = r % v.NY, k = r / v.NY;
        MinusW m = minus_edges(v, p, r, i, q);
        double wxp = v.wx[p], wyp = v.wy[p], wzp = v.wz[p];
        double out[R];
#pragma unroll
        for (int c = 0; c < R; ++c) {
            const double *ac = a + c * E;
            double tsum = 0.0, hsum = 0.0;
            if (wxp > 0.0) tsum = add_rn(tsum, mul_rn(wxp, ac[e.ex(i, j, k)]));
            if (wyp > 0.0) tsum = add_rn(tsum, mul_rn(wyp, ac[e.ey(i, j, k)]));
            if (wzp > 0.0) tsum = add_rn(tsum, mul_rn(wzp, ac[e.ez(i, j, k)]));
            if (m.wxm > 0.0) hsum = add_rn(hsum, mul_rn(m.wxm, ac[e.ex(i - 1, j, k)]));
            if (m.wym > 0.0) hsum = add_rn(hsum, mul_rn(m.wym, ac[e.ey(i, j - 1, k)]));
            if (m.wzm > 0.0) hsum = add_rn(hsum, mul_rn(m.wzm, ac[e.ez(i, j, k - 1)]));
            out[c] = mask_bit(v.mask, p) ? sub_rn(tsum, hsum) : 0.0;
        }
        if constexpr (R == 1) rhs[p] = out[0];
        else rhs[p] = make_double2(out[0], out[1]);
    }
}

PosRange pos_range(const Operator &op, int64_t pb, int64_t pe) {
    if (pe > op.L || pe < 0) pe = op.L;
    if (pb < 0) pb = 0;
    PosRange r{pb, pe, (int)(pb / kTile), 0};
    r.tiles = (int)((pe + kTile - 1) / kTile) - r.tile0;
    return r;
}

void op_rhs_span(const Operator &op, const double *a, double *rhs_span, int nrhs, cudaStream_t s, int64_t pb,
                 int64_t pe) {
    PosRange pr = pos_range(op, pb, pe);
    if (pr.tiles <= 0) return;
    SpanView v = span_view(op);
    EdgeIdx e = edge_idx(op);
    if (nrhs == 1)
        k_rhs<1><<<pr.tiles, kSpanThreads, 0, s>>>(v, e, a, op.n_edges, rhs_span, pr);
    else
        k_rhs<2><<<pr.tiles, kSpanThreads, 0, s>>>(v, e, a, op.n_edges, (double2 *)rhs_span, pr);
    SPFD_LAUNCH_CHECK();
}

// ------------------------------------------------------------------------
// E-field chain
// ------------------------------------------------------------------------

// Edge voltages over all edges (box layout); psi in span layout (planar per
// rhs handled by the caller through interleaved span input).
__global__ void k_edge_volt(const int4 *rows, EdgeIdx e, int64_t E, const double *a,
                            const double *psi_span, int nrhs, double omega, double *vout) {
    for (int64_t ed = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; ed < E;
         ed += (int64_t)gridDim.x * blockDim.x) {
        int axis;
        int64_t loc;
        int dx;
        if (ed < e.eoff1) { axis = 0; loc = ed; dx = e.nx; }
        else if (ed < e.eoff2) { axis = 1; loc = ed - e.eoff1; dx = e.NX; }
        else { axis = 2; loc = ed - e.eoff2; dx = e.NX; }
        int i = (int)(loc % dx);
        int64_t t = loc / dx;
        int dy = axis == 1 ? e.ny : e.NY;
        int j = (int)(t % dy);
        int k = (int)(t / dy);
        int rt = j + e.NY * k;
        int rh = rt, ih = i;
        if (axis == 0) ih = i + 1;
        else if (axis == 1) rh = rt + 1;
        else rh = rt + e.NY;
        int pt = span_pos(rows, rt, i), ph = span_pos(rows, rh, ih);
        for (int c = 0; c < nrhs; ++c) {
            double ps_t = pt >= 0 ? psi_span[(int64_t)pt * nrhs + c] : 0.0;
            double ps_h = ph >= 0 ? psi_span[(int64_t)ph * nrhs + c] : 0.0;
            vout[c * E + ed] = mul_rn(omega, sub_rn(add_rn(a[c * E + ed], ps_h), ps_t));
        }
    }
}

void op_edge_voltages(const Operator &op, const double *a, const double *psi_span, double omega,
                      double *v, int nrhs, cudaStream_t s) {
    k_edge_volt<<<grid_for(op.n_edges, 256, 148 * 32), 256, 0, s>>>(op.rows.get(), edge_idx(op),
                                                                    op.n_edges, a, psi_span, nrhs,
                                                                    omega, v);
    SPFD_LAUNCH_CHECK();
}

struct EfGeo {
    Geo g;
    EdgeIdx e;
    double sx, sy, sz;
};

// per-axis component: mean of the (<= 2) conductive incident edge fields
__device__ __forceinline__ double axis_comp(double vt, bool mt, double vh, bool mh, double sa) {
    double evt = mt ? __ddiv_rn(mul_rn(vt, 1.0), sa) : 0.0;
    double evh = mh ? __ddiv_rn(mul_rn(vh, 1.0), sa) : 0.0;
    double num = add_rn(add_rn(0.0, evt), evh);
    // num / max(cnt, 1) with cnt in {0, 1, 2}: dividing by 1 or 2 is exact
    // as the identity / a multiply by 0.5 (same IEEE result, no divide)
    if (!mt && !mh) return 0.0;
    return (mt && mh) ? mul_rn(num, 0.5) : num;
}

__device__ __forceinline__ double field_mag(double cx, double cy, double cz) {
    double tot = add_rn(add_rn(add_rn(0.0, mul_rn(cx, cx)), mul_rn(cy, cy)), mul_rn(cz, cz));
    return __dsqrt_rn(tot);
}

// Node |E| over the node box from edge voltages (dosimetry.py:50-85).
__global__ void k_node_field_box(const uint8_t *vc, EfGeo f, int64_t E, int64_t n_nodes,
                                 const double *v, int nrhs, double *node) {
    Geo g = f.g;
    for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < n_nodes;
         n += (int64_t)gridDim.x * blockDim.x) {
        int i = (int)(n % g.NX);
        int64_t t = n / g.NX;
        int j = (int)(t % g.NY);
        int k = (int)(t / g.NY);
        bool mxt = i < g.nx && edge_cond(vc, g, 0, i, j, k);
        bool mxh = i > 0 && edge_cond(vc, g, 0, i - 1, j, k);
        bool myt = j < g.ny && edge_cond(vc, g, 1, i, j, k);
        bool myh = j > 0 && edge_cond(vc, g, 1, i, j - 1, k);
        bool mzt = k < g.nz && edge_cond(vc, g, 2, i, j, k);
        bool mzh = k > 0 && edge_cond(vc, g, 2, i, j, k - 1);
        for (int c = 0; c < nrhs; ++c) {
            const double *vv = v + c * E;
            double cx = axis_comp(mxt ? vv[f.e.ex(i, j, k)] : 0.0, mxt,
                                  mxh ? vv[f.e.ex(i - 1, j, k)] : 0.0, mxh, f.sx);
            double cy = axis_comp(myt ? vv[f.e.ey(i, j, k)] : 0.0, myt,
                                  myh ? vv[f.e.ey(i, j - 1, k)] : 0.0, myh, f.sy);
            double cz = axis_comp(mzt ? vv[f.e.ez(i, j, k)] : 0.0, mzt,
                                  mzh ? vv[f.e.ez(i, j, k - 1)] : 0.0, mzh, f.sz);
            node[c * n_nodes + n] = field_mag(cx, cy, cz);
        }
    }
}

void op_node_field(const Operator &op, const double *v, double *node, int nrhs, cudaStream_t s) {
    Geo g{(int)op.nx, (int)op.ny, (int)op.nz, (int)op.NX, (int)op.NY, (int)op.NZ};
    EfGeo f{g, edge_idx(op), op.sx, op.sy, op.sz};
    k_node_field_box<<<grid_for(op.n_nodes, 256, 148 * 32), 256, 0, s>>>(
        op.vox_cond.get(), f, op.n_edges, op.n_nodes, v, nrhs, node);
    SPFD_LAUNCH_CHECK();
}

// Voxel average with a node accessor; one warp per voxel row, conductive
// voxels compacted in x-fastest order (dosimetry.py:88-116).
template <class NodeAt>
__device__ void voxel_row_avg(const uint8_t *vc, Geo g, const int32_t *vrow_off, int64_t vr,
                              int64_t n_cv, NodeAt at, int nrhs, double *vox) {
    int lane = threadIdx.x & 31;
    int j = (int)(vr % g.ny), k = (int)(vr / g.ny);
    const uint8_t *c = vc + vr * g.nx;
    int base = vrow_off[vr];
    for (int i0 = 0; i0 < g.nx; i0 += 32) {
        int i = i0 + lane;
        bool on = i < g.nx && c[i];
        unsigned b = __ballot_sync(0xffffffffu, on);
        if (on) {
            int slot = base + __popc(b & ((1u << lane) - 1u));
            for (int cc = 0; cc < nrhs; ++cc) {
                double acc = 0.0;
                for (int di = 0; di < 2; ++di)
                    for (int dj = 0; dj < 2; ++dj)
                        for (int dk = 0; dk < 2; ++dk) acc = add_rn(acc, at(cc, i + di, j + dj, k + dk));
                vox[cc * n_cv + slot] = mul_rn(acc, 0.125);
            }
        }
        base += __popc(b);
    }
}

struct BoxNodeAt {
    const double *node;
    int64_t n_nodes;
    int NX, NY;
    __device__ double operator()(int c, int i, int j, int k) const {
        return node[c * n_nodes + i + (int64_t)NX * (j + (int64_t)NY * k)];
    }
};

__global__ void k_voxavg_box(const uint8_t *vc, Geo g, const int32_t *vrow_off, int64_t n_vrows,
                             int64_t n_cv, BoxNodeAt at, int nrhs, double *vox) {
    int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    for (int64_t vr = warp; vr < n_vrows; vr += ((int64_t)gridDim.x * blockDim.x) >> 5)
        voxel_row_avg(vc, g, vrow_off, vr, n_cv, at, nrhs, vox);
}

void op_voxel_average(const Operator &op, const double *node, double *vox, int nrhs, cudaStream_t s) {
    Geo g{(int)op.nx, (int)op.ny, (int)op.nz, (int)op.NX, (int)op.NY, (int)op.NZ};
    int64_t nvr = op.ny * op.nz;
    BoxNodeAt at{node, op.n_nodes, (int)op.NX, (int)op.NY};
    k_voxavg_box<<<grid_for(nvr * 32, 256, 148 * 32), 256, 0, s>>>(op.vox_cond.get(), g, op.vrow_off.get(),
                                                                   nvr, op.n_cond_vox, at, nrhs, vox);
    SPFD_LAUNCH_CHECK();
}

// Fused: node |E| on span positions straight from (a, psi_span, w), then the
// voxel average reading the span node field.  Bit-identical to the three
// separate stages (inactive edges contribute exact zeros).
template <int R>
__global__ void __launch_bounds__(kSpanThreads, 4) k_node_field_span(SpanView v, EdgeIdx e, const double *__restrict__ a,
                                                                  int64_t E, const double *__restrict__ psi,
                                                                  double omega, double sx, double sy, double sz,
                                                                  double *__restrict__ node, PosRange pr) {
    int t = pr.tile0 + blockIdx.x;
    int r0 = v.tile_row[t], r1 = v.tile_row[t + 1];
    int r = r0;
    for (int u = 0; u < kTile / kSpanThreads; ++u) {
        int p = t * kTile + u * kSpanThreads + threadIdx.x;
        if (p >= pr.pe) break;
        if (p < pr.pb) continue;
        r = find_row(v.rows, r, r1, p);  // positions grow with u: search from the last row
        int4 q = v.rows[r];
        int i = q.y + (p - q.x);
        int j = q.w, k = (r - j) / v.NY;
        MinusW m = minus_edges(v, p, r, i, q);
        double wxp = v.wx[p], wyp = v.wy[p], wzp = v.wz[p];
        int pxp = (wxp > 0.0) ? p + 1 : -1;
        int pyp = (wyp > 0.0) ? span_pos(v.rows, r + 1, i) : -1;
        int pzp = (wzp > 0.0) ? span_pos(v.rows, r + v.NY, i) : -1;
#pragma unroll
        for (int c = 0; c < R; ++c) {
            const double *ac = a + c * E;
            double pc = psi[(int64_t)p * R + c];
            auto ps = [&](int pp) { return pp >= 0 ? psi[(int64_t)pp * R + c] : 0.0; };
            double vxt = wxp > 0.0 ? mul_rn(omega, sub_rn(add_rn(ac[e.ex(i, j, k)], ps(pxp)), pc)) : 0.0;
            double vxh = m.wxm > 0.0 ? mul_rn(omega, sub_rn(add_rn(ac[e.ex(i - 1, j, k)], pc), ps(m.pxm))) : 0.0;
            double vyt = wyp > 0.0 ? mul_rn(omega, sub_rn(add_rn(ac[e.ey(i, j, k)], ps(pyp)), pc)) : 0.0;
            double vyh = m.wym > 0.0 ? mul_rn(omega, sub_rn(add_rn(ac[e.ey(i, j - 1, k)], pc), ps(m.pym))) : 0.0;
            double vzt = wzp > 0.0 ? mul_rn(omega, sub_rn(add_rn(ac[e.ez(i, j, k)], ps(pzp)), pc)) : 0.0;
            double vzh = m.wzm > 0.0 ? mul_rn(omega, sub_rn(add_rn(ac[e.ez(i, j, k - 1)], pc), ps(m.pzm))) : 0.0;
            double cx = axis_comp(vxt, wxp > 0.0, vxh, m.wxm > 0.0, sx);
            double cy = axis_comp(vyt, wyp > 0.0, vyh, m.wym > 0.0, sy);
            double cz = axis_comp(vzt, wzp > 0.0, vzh, m.wzm > 0.0, sz);
            node[(int64_t)p * R + c] = field_mag(cx, cy, cz);
        }
    }
}

template <int R>
struct SpanNodeAt {
    const int4 *rows;
    const double *node;
    int NY;
    __device__ double operator()(int c, int i, int j, int k) const {
        int4 q = rows[j + NY * k];
        return node[(int64_t)(q.x + (i - q.y)) * R + c];
    }
};

template <int R>
__global__ void k_voxavg_span(const uint8_t *vc, Geo g, const int32_t *vrow_off, int64_t vr_b, int64_t n_vrows,
                              int64_t n_cv, SpanNodeAt<R> at, double *vox) {
    int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    for (int64_t vr = vr_b + warp; vr < n_vrows; vr += ((int64_t)gridDim.x * blockDim.x) >> 5)
        voxel_row_avg(vc, g, vrow_off, vr, n_cv, at, R, vox);
}

void op_node_field_span(const Operator &op, const double *a, const double *psi_span, double omega,
                        double *node_span, int nrhs, cudaStream_t s, int64_t pb, int64_t pe) {
    PosRange pr = pos_range(op, pb, pe);
    if (pr.tiles <= 0) return;
    SpanView v = span_view(op);
    EdgeIdx e = edge_idx(op);
    if (nrhs == 1)
        k_node_field_span<1><<<pr.tiles, kSpanThreads, 0, s>>>(v, e, a, op.n_edges, psi_span, omega, op.sx, op.sy,
                                                               op.sz, node_span, pr);
    else
        k_node_field_span<2><<<pr.tiles, kSpanThreads, 0, s>>>(v, e, a, op.n_edges, psi_span, omega, op.sx, op.sy,
                                                               op.sz, node_span, pr);
    SPFD_LAUNCH_CHECK();
}

void op_voxavg_span(const Operator &op, const double *node_span, double *vox, int nrhs, cudaStream_t s,
                    int64_t vr_b, int64_t vr_e) {
    Geo g{(int)op.nx, (int)op.ny, (int)op.nz, (int)op.NX, (int)op.NY, (int)op.NZ};
    int64_t nvr = op.ny * op.nz;
    if (vr_e < 0 || vr_e > nvr) vr_e = nvr;
    if (vr_e <= vr_b) return;
    int gv = grid_for((vr_e - vr_b) * 32, 256, 148 * 32);
    if (nrhs == 1)
        k_voxavg_span<1><<<gv, 256, 0, s>>>(op.vox_cond.get(), g, op.vrow_off.get(), vr_b, vr_e, op.n_cond_vox,
                                            SpanNodeAt<1>{op.rows.get(), node_span, (int)op.NY}, vox);
    else
        k_voxavg_span<2><<<gv, 256, 0, s>>>(op.vox_cond.get(), g, op.vrow_off.get(), vr_b, vr_e, op.n_cond_vox,
                                            SpanNodeAt<2>{op.rows.get(), node_span, (int)op.NY}, vox);
    SPFD_LAUNCH_CHECK();
}

void op_efield_voxavg_span(const Operator &op, const double *a, const double *psi_span, double omega,
                           double *vox, double *node_span_ws, int nrhs, cudaStream_t s) {
    op_node_field_span(op, a, psi_span, omega, node_span_ws, nrhs, s, 0, -1);
    op_voxavg_span(op, node_span_ws, vox, nrhs, s, 0, -1);
}

// ------------------------------------------------------------------------
// exports
// ------------------------------------------------------------------------

__global__ void k_export_w(const int4 *rows, EdgeIdx e, int64_t E, const double *wx, const double *wy,
                           const double *wz, double *out) {
    for (int64_t ed = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; ed < E;
         ed += (int64_t)gridDim.x * blockDim.x) {
        int axis;
        int64_t loc;
        int dx, dy;
        if (ed < e.eoff1) { axis = 0; loc = ed; dx = e.nx; dy = e.NY; }
        else if (ed < e.eoff2) { axis = 1; loc = ed - e.eoff1; dx = e.NX; dy = e.ny; }
        else { axis = 2; loc = ed - e.eoff2; dx = e.NX; dy = e.NY; }
        int i = (int)(loc % dx);
        int64_t t = loc / dx;
        int j = (int)(t % dy), k = (int)(t / dy);
        int p = span_pos(rows, j + e.NY * k, i);
        const double *w = axis == 0 ? wx : (axis == 1 ? wy : wz);
        out[ed] = p >= 0 ? w[p] : 0.0;
    }
}

__global__ void k_export_nodes(SpanView v, const int32_t *pos_to_dof, int NX, int64_t *d2n,
                               int64_t *n2d, const double *diag, double *diag_out) {
    int t = blockIdx.x;
    int r0 = v.tile_row[t], r1 = v.tile_row[t + 1];
    for (int u = 0; u < kTile / kSpanThreads; ++u) {
        int p = t * kTile + u * kSpanThreads + threadIdx.x;
        if (p >= v.L) break;
        int d = pos_to_dof[p];
        if (d < 0) continue;
        int r = find_row(v.rows, r0, r1, p);
        int4 q = v.rows[r];
        int64_t node = (int64_t)(q.y + (p - q.x)) + (int64_t)NX * r;
        if (d2n) d2n[d] = node;
        if (n2d) n2d[node] = d;
        if (diag_out) diag_out[d] = diag[p];
    }
}

__global__ void k_fill_i64(int64_t *p, int64_t n, int64_t val) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n;
         x += (int64_t)gridDim.x * blockDim.x)
        p[x] = val;
}

__global__ void k_export_voxidx(const uint8_t *vc, Geo g, const int32_t *vrow_off, int64_t n_vrows,
                                int64_t *out) {
    int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    for (int64_t vr = warp; vr < n_vrows; vr += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const uint8_t *c = vc + vr * g.nx;
        int base = vrow_off[vr];
        for (int i0 = 0; i0 < g.nx; i0 += 32) {
            int i = i0 + lane;
            bool on = i < g.nx && c[i];
            unsigned b = __ballot_sync(0xffffffffu, on);
            if (on) out[base + __popc(b & ((1u << lane) - 1u))] = i + (int64_t)g.nx * vr;
            base += __popc(b);
        }
    }
}

void op_export(Operator &op, int what, void *dst, cudaStream_t s) {
    SpanView v = span_view(op);
    Geo g{(int)op.nx, (int)op.ny, (int)op.nz, (int)op.NX, (int)op.NY, (int)op.NZ};
    switch (what) {
        case SPFD_EXPORT_EDGE_CONDUCTANCE:
            k_export_w<<<grid_for(op.n_edges, 256, 148 * 32), 256, 0, s>>>(
                op.rows.get(), edge_idx(op), op.n_edges, op.wx.get(), op.wy.get(), op.wz.get(), (double *)dst);
            break;
        case SPFD_EXPORT_DOF_TO_NODE:
            if (op.n_tiles)
                k_export_nodes<<<(int)op.n_tiles, kSpanThreads, 0, s>>>(v, op.pos_to_dof.get(), (int)op.NX,
                                                                         (int64_t *)dst, nullptr, nullptr, nullptr);
            break;
        case SPFD_EXPORT_NODE_TO_DOF:
            k_fill_i64<<<grid_for(op.n_nodes, 256, 148 * 32), 256, 0, s>>>((int64_t *)dst, op.n_nodes, -1);
            if (op.n_tiles)
                k_export_nodes<<<(int)op.n_tiles, kSpanThreads, 0, s>>>(v, op.pos_to_dof.get(), (int)op.NX,
                                                                         nullptr, (int64_t *)dst, nullptr, nullptr);
            break;
        case SPFD_EXPORT_PINNED:
            SPFD_CUDA(cudaMemcpyAsync(dst, op.pinned.get(), op.n_comp * sizeof(int64_t),
                                      cudaMemcpyDeviceToDevice, s));
            break;
        case SPFD_EXPORT_VOXEL_INDICES: {
            int64_t nvr = op.ny * op.nz;
            k_export_voxidx<<<grid_for(nvr * 32, 256, 148 * 32), 256, 0, s>>>(op.vox_cond.get(), g,
                                                                              op.vrow_off.get(), nvr,
                                                                              (int64_t *)dst);
            break;
        }
        case SPFD_EXPORT_DIAGONAL:
            if (op.n_tiles)
                k_export_nodes<<<(int)op.n_tiles, kSpanThreads, 0, s>>>(v, op.pos_to_dof.get(), (int)op.NX,
                                                                         nullptr, nullptr, op.diag.get(),
                                                                         (double *)dst);
            break;
        default:
            throw Error(SPFD_EINVAL, "unknown export selector");
    }
    SPFD_LAUNCH_CHECK();
}

void op_csr(Operator &op, int64_t *indptr, int32_t *indices, double *data, cudaStream_t s) {
    // indptr = exclusive scan of per-row counts (int32 counts -> int64)
    cub::TransformInputIterator<int64_t, WidenI32, const int32_t *> wl(op.nnz_row.get(), WidenI32());
    size_t bytes = 0;
    SPFD_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, wl, indptr, op.n_dofs + 1, s));
    DevBuf<uint8_t> tmp;
    tmp.alloc(bytes);
    SPFD_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), bytes, wl, indptr, op.n_dofs + 1, s));
    SpanView v = span_view(op);
    if (op.n_tiles)
        k_csr_fill<<<(int)op.n_tiles, kSpanThreads, 0, s>>>(v, op.pos_to_dof.get(), op.diag.get(), indptr,
                                                             indices, data);
    SPFD_LAUNCH_CHECK();
    SPFD_CUDA(cudaStreamSynchronize(s));
}

}  // namespace spfd

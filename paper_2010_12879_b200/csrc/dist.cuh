// z-slab decomposition of the solve (included at the end of solve.cu).
//
// Every rank holds the identical operator and AMG hierarchy (built by the
// same deterministic setup), so the aggregates -- and therefore the
// preconditioner and the iteration count -- do not depend on the number of
// GPUs.  The solve is distributed:
//   * fine level: rank r owns the node planes [k_r, k_{r+1}) (contiguous span
//     positions, balanced by count); every stencil pass exchanges one plane
//     with each neighbour (contiguous ranges, no packing);
//   * level l >= 1 with at least `replicate_below` rows: a row (aggregate)
//     belongs to the rank owning its lowest member; smoothers / transfers run
//     on the owned rows of owned-row CSRs; the off-rank columns they read are
//     exchanged with per-neighbour index lists computed at setup (every rank
//     can compute every other rank's needs because the hierarchy is shared);
//   * smaller levels are replicated: their input is the rank-ordered sum of
//     per-rank partial restrictions (allgather), then every rank runs the
//     rest of the V-cycle redundantly;
//   * dot products: per-rank partials allgathered and summed in rank order,
//     so results are bitwise reproducible for a fixed number of ranks.
// Vectors stay full length (global indexing); only owned entries and the
// halos are valid.
#pragma once

#include "comm.cuh"

struct ListHalo {
    struct Peer {
        int rank = 0;
        int64_t nsend = 0, nrecv = 0;
        DevBuf<int32_t> sidx, ridx;
        DevBuf<double> sbuf, rbuf;
    };
    std::vector<Peer> peers;
};

struct DistLevel {
    bool dist = false;        // rows distributed (else replicated from here on)
    bool r_partial = false;   // next level replicated: R_loc = all next rows x owned columns
    DevBuf<int32_t> own;      // owned rows (sorted)
    int64_t n_own = 0;
    DevBuf<int32_t> next_own; // owned next-level rows (rowmap of R_loc when !r_partial)
    int64_t n_next_own = 0;
    Csr A_loc, P_loc, R_loc;  // owned-row CSRs with global columns
    ListHalo hA, hR, hP;
    DevBuf<int32_t> owner;    // owner rank of every row of this level
    int gA = 8, gP = 4, gR = 8;
};

struct Dist {
    Comm *comm = nullptr;
    int rank = 0, size = 1;
    int kb = 0, ke = 0;                    // owned node planes
    int64_t pb = 0, pe = 0;                // owned span positions
    int64_t lo_recv[2] = {0, 0}, lo_send[2] = {0, 0}, hi_recv[2] = {0, 0}, hi_send[2] = {0, 0};
    std::vector<int64_t> plane_pos;        // first position of every plane (+ L)
    std::vector<int> kbounds;              // plane boundaries per rank (size + 1)
    DevBuf<int64_t> pbounds;               // position boundaries per rank (size + 1)
    bool l1_dist = false;
    DevBuf<int32_t> agg_own;               // owned level-1 rows
    int64_t n_agg_own = 0;
    ListHalo hu, he;
    std::vector<DistLevel> lv;             // index = level (entry 0 unused)
    DevBuf<double> gsend, grecv;           // allgather scratch
    DevBuf<double> hgather;                // distributed FGMRES: gathered Hessenberg partials
    int64_t dof_b = 0, dof_e = 0, vox_b = 0, vox_e = 0;
    int64_t vrow_b = 0, vrow_e = 0;
    // interior positions [ib, ie): stencil neighbours all owned -> computed on
    // a side stream while the halo planes travel
    int64_t ib = 0, ie = 0;
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    // distributed PCG: one batch of iterations captured as a CUDA graph per
    // rhs count (stream-ordered transports only; pcg_dist)
    cudaGraphExec_t batch_exec[3] = {nullptr, nullptr, nullptr};
    int batch_nb[3] = {0, 0, 0};
    const double *batch_trace[3] = {nullptr, nullptr, nullptr};
    int64_t batch_launches[3] = {0, 0, 0};
    bool batch_failed[3] = {false, false, false};
    ~Dist() {
        for (auto &e : batch_exec)
            if (e) cudaGraphExecDestroy(e);
        if (ev_fork) cudaEventDestroy(ev_fork);
        if (ev_join) cudaEventDestroy(ev_join);
        if (side) cudaStreamDestroy(side);
    }
};

// ------------------------------------------------------------- kernels --

__global__ void k_pack(const int32_t *idx, int64_t n, int R, const double *v, double *buf) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        for (int c = 0; c < R; ++c) buf[i * R + c] = v[(int64_t)idx[i] * R + c];
}
__global__ void k_unpack(const int32_t *idx, int64_t n, int R, const double *buf, double *v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        for (int c = 0; c < R; ++c) v[(int64_t)idx[i] * R + c] = buf[i * R + c];
}

// out[i] = sum over ranks (in rank order) of parts[p][i]; optional x0 = od * out
__global__ void k_rank_sum(const double *parts, int size, int64_t m, int R, double *out, const double *od,
                           double *x0) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m * R;
         i += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int p = 0; p < size; ++p) s += parts[(int64_t)p * m * R + i];
        out[i] = s;
        if (x0) x0[i] = od[i / R] * s;
    }
}

// gathered per-rank scalars [size][R] -> rank-ordered sum into slot, then `what`
template <int R>
__global__ void k_rank_finalize(const double *g, int size, double *scal, int slot, int what) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    for (int c = 0; c < R; ++c) {
        double s = 0.0;
        for (int p = 0; p < size; ++p) s += g[p * R + c];
        scal[slot + c] = s;
        bool active = scal[S_ACTIVE + c] != 0.0;
        if (what == F_ALPHA) {
            scal[S_ALPHA + c] = (active && s != 0.0) ? scal[S_RHO + c] / s : 0.0;
        } else if (what == F_BETA_INIT) {
            scal[S_RHO + c] = s;
            scal[S_BETA + c] = 0.0;
        } else if (what == F_BETA) {
            double old = scal[S_RHO + c];
            scal[S_BETA + c] = (active && old != 0.0) ? s / old : 0.0;
            scal[S_RHO + c] = s;
        }
    }
}

// owner rank of a span position (boundaries per rank)
__device__ __forceinline__ int owner_of(const int64_t *pb, int size, int64_t p) {
    int lo = 0, hi = size - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (pb[mid] <= p) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// level-1 owner: rank owning the aggregate's lowest member position
__global__ void k_owner_l1(const int64_t *mptr, const int32_t *mpos, int64_t n_agg, const int64_t *pb, int size,
                           int32_t *owner) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n_agg; c += (int64_t)gridDim.x * blockDim.x)
        owner[c] = owner_of(pb, size, mpos[mptr[c]]);
}

__global__ void k_fill_i32(int32_t *p, int64_t n, int32_t v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

// anchor (lowest member row) of every aggregate of a CSR level
__global__ void k_anchor(const int32_t *agg, int64_t n, int32_t *anchor) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        atomicMin(&anchor[agg[i]], (int32_t)i);
}
__global__ void k_owner_from_anchor(const int32_t *anchor, int64_t n_next, const int32_t *owner_l, int32_t *owner_n) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n_next; c += (int64_t)gridDim.x * blockDim.x)
        owner_n[c] = owner_l[anchor[c]];
}

// flag[i] = (owner[i] == who)
__global__ void k_flag_owner(const int32_t *owner, int64_t n, int who, int32_t *flag) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        flag[i] = owner[i] == who ? 1 : 0;
}

// mark columns of the rows owned by `rows_of` whose owner is `col_owner`
__global__ void k_mark_cols(CsrView m, const int32_t *row_owner, int rows_of, const int32_t *col_owner, int col_of,
                            int32_t *flag) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < m.rows; r += (int64_t)gridDim.x * blockDim.x) {
        if (row_owner[r] != rows_of) continue;
        for (int64_t q = m.ptr[r]; q < m.ptr[r + 1]; ++q) {
            int c = m.col[q];
            if (col_owner[c] == col_of) flag[c] = 1;
        }
    }
}

// fine level: members (positions) of aggregates owned by `agg_of` whose position owner is `pos_of`
__global__ void k_mark_members(const int64_t *mptr, const int32_t *mpos, int64_t n_agg, const int32_t *owner1,
                               int agg_of, const int64_t *pb, int size, int pos_of, int32_t *flag) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n_agg; c += (int64_t)gridDim.x * blockDim.x) {
        if (owner1[c] != agg_of) continue;
        for (int64_t q = mptr[c]; q < mptr[c + 1]; ++q) {
            int p = mpos[q];
            if (owner_of(pb, size, p) == pos_of) flag[p] = 1;
        }
    }
}

// fine level: aggregates of positions in [w0, w1) whose owner is `agg_of`
__global__ void k_mark_aggs(const int32_t *aggp, int64_t w0, int64_t w1, const int32_t *owner1, int agg_of,
                            int32_t *flag) {
    for (int64_t p = w0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < w1; p += (int64_t)gridDim.x * blockDim.x) {
        int g1 = aggp[p];
        if (g1 > 0 && owner1[g1 - 1] == agg_of) flag[g1 - 1] = 1;
    }
}

// owned-row CSR extraction (rows = list, columns kept global)
__global__ void k_rowlen(CsrView m, const int32_t *rows, int64_t n, int64_t *len) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int r = rows[i];
        len[i] = m.ptr[r + 1] - m.ptr[r];
    }
}
__global__ void k_rowcopy(CsrView m, const int32_t *rows, int64_t n, const int64_t *optr, int32_t *ocol,
                          double *oval) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int r = rows[i];
        int64_t o = optr[i];
        for (int64_t q = m.ptr[r]; q < m.ptr[r + 1]; ++q, ++o) { ocol[o] = m.col[q]; oval[o] = m.val[q]; }
    }
}
// all rows, only columns owned by `me`
__global__ void k_colcount(CsrView m, const int32_t *col_owner, int me, int64_t *len) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < m.rows; r += (int64_t)gridDim.x * blockDim.x) {
        int64_t c = 0;
        for (int64_t q = m.ptr[r]; q < m.ptr[r + 1]; ++q) c += col_owner[m.col[q]] == me;
        len[r] = c;
    }
}
__global__ void k_colcopy(CsrView m, const int32_t *col_owner, int me, const int64_t *optr, int32_t *ocol,
                          double *oval) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < m.rows; r += (int64_t)gridDim.x * blockDim.x) {
        int64_t o = optr[r];
        for (int64_t q = m.ptr[r]; q < m.ptr[r + 1]; ++q)
            if (col_owner[m.col[q]] == me) { ocol[o] = m.col[q]; oval[o] = m.val[q]; ++o; }
    }
}

// restriction for a distributed level 1: owned aggregates only
template <int R>
__global__ void k_agg_sum_list(const int64_t *mptr, const int32_t *mpos, const int32_t *list, int64_t n,
                               const double *u, double *rc, const double *od_c, double *x0_c) {
    using W = V<R>;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t g = list[i];
        typename W::T s = W::zero();
        for (int64_t q = mptr[g]; q < mptr[g + 1]; ++q) s = W::add(s, W::ld(u, mpos[q]));
        W::st(rc, g, s);
        if (x0_c) W::st(x0_c, g, W::scale(od_c[g], s));
    }
}
// replicated level 1: partial sums over the members inside [pb, pe)
template <int R>
__global__ void k_agg_sum_partial(const int64_t *mptr, const int32_t *mpos, int64_t n_agg, int64_t pb, int64_t pe,
                                  const double *u, double *part) {
    using W = V<R>;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < n_agg; g += (int64_t)gridDim.x * blockDim.x) {
        typename W::T s = W::zero();
        for (int64_t q = mptr[g]; q < mptr[g + 1]; ++q) {
            const int p = mpos[q];
            if (p >= pb && p < pe) s = W::add(s, W::ld(u, p));
        }
        W::st(part, g, s);
    }
}

__global__ void k_count_dofs(const uint32_t *mask, int64_t pb, int64_t *out) {
    __shared__ unsigned long long sh;
    if (threadIdx.x == 0) sh = 0;
    __syncthreads();
    unsigned long long local = 0;
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w * 32 < pb; w += (int64_t)gridDim.x * blockDim.x) {
        uint32_t bits = mask[w];
        int64_t lim = pb - w * 32;
        if (lim < 32) bits &= (1u << lim) - 1u;
        local += __popc(bits);
    }
    atomicAdd(&sh, local);
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd((unsigned long long *)out, sh);
}

// ---------------------------------------------------------------- setup --

template <class T>
static T d2h(const T *p, cudaStream_t s) {
    T v;
    SPFD_CUDA(cudaMemcpyAsync(&v, p, sizeof(T), cudaMemcpyDeviceToHost, s));
    SPFD_CUDA(cudaStreamSynchronize(s));
    return v;
}

// compact indices with flag != 0 (ascending) into out; returns count
static int64_t compact_flags(const int32_t *flag, int64_t n, DevBuf<int32_t> &out, cudaStream_t s) {
    DevBuf<int32_t> tmp;
    tmp.alloc(n + 1);
    DevBuf<int64_t> cnt;
    cnt.alloc(1);
    cub::CountingInputIterator<int32_t> it(0);
    size_t bytes = 0;
    SPFD_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, it, flag, tmp.get(), cnt.get(), n, s));
    DevBuf<uint8_t> ws;
    ws.alloc(bytes);
    SPFD_CUDA(cub::DeviceSelect::Flagged(ws.get(), bytes, it, flag, tmp.get(), cnt.get(), n, s));
    int64_t k = d2h(cnt.get(), s);
    out.alloc(k > 0 ? k : 1);
    if (k > 0) SPFD_CUDA(cudaMemcpyAsync(out.get(), tmp.get(), k * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    SPFD_CUDA(cudaStreamSynchronize(s));
    return k;
}

static void extract_rows(const Csr &m, const DevBuf<int32_t> &rows, int64_t n, Csr &out, cudaStream_t s) {
    const int T = 256;
    DevBuf<int64_t> len;
    len.alloc(n + 1);
    SPFD_CUDA(cudaMemsetAsync(len.get(), 0, len.bytes(), s));
    if (n) k_rowlen<<<grid_for(n, T), T, 0, s>>>(view(m), rows.get(), n, len.get());
    DevBuf<int64_t> ptr;
    ptr.alloc(n + 1);
    {
        size_t bytes = 0;
        SPFD_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, len.get(), ptr.get(), n + 1, s));
        DevBuf<uint8_t> ws;
        ws.alloc(bytes);
        SPFD_CUDA(cub::DeviceScan::ExclusiveSum(ws.get(), bytes, len.get(), ptr.get(), n + 1, s));
    }
    int64_t nnz = d2h(ptr.get() + n, s);
    out.alloc(n, m.cols, nnz);
    SPFD_CUDA(cudaMemcpyAsync(out.ptr.get(), ptr.get(), (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
    if (n) k_rowcopy<<<grid_for(n, T), T, 0, s>>>(view(m), rows.get(), n, ptr.get(), out.col.get(), out.val.get());
    SPFD_LAUNCH_CHECK();
    SPFD_CUDA(cudaStreamSynchronize(s));
}

static void extract_cols(const Csr &m, const int32_t *col_owner, int me, Csr &out, cudaStream_t s) {
    const int T = 256;
    int64_t n = m.rows;
    DevBuf<int64_t> len, ptr;
    len.alloc(n + 1);
    ptr.alloc(n + 1);
    SPFD_CUDA(cudaMemsetAsync(len.get(), 0, len.bytes(), s));
    k_colcount<<<grid_for(n, T), T, 0, s>>>(view(m), col_owner, me, len.get());
    {
        size_t bytes = 0;
        SPFD_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, len.get(), ptr.get(), n + 1, s));
        DevBuf<uint8_t> ws;
        ws.alloc(bytes);
        SPFD_CUDA(cub::DeviceScan::ExclusiveSum(ws.get(), bytes, len.get(), ptr.get(), n + 1, s));
    }
    int64_t nnz = d2h(ptr.get() + n, s);
    out.alloc(n, m.cols, nnz);
    SPFD_CUDA(cudaMemcpyAsync(out.ptr.get(), ptr.get(), (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
    k_colcopy<<<grid_for(n, T), T, 0, s>>>(view(m), col_owner, me, ptr.get(), out.col.get(), out.val.get());
    SPFD_LAUNCH_CHECK();
    SPFD_CUDA(cudaStreamSynchronize(s));
}

// build a list halo for vector entries indexed 0..nv-1:
//   mark(q, who, flag): flag[i] = 1 for entries rank `q` needs from rank `who`
template <class Mark>
static void build_list_halo(ListHalo &hl, int me, int size, int64_t nv, int maxr, Mark mark, cudaStream_t s) {
    DevBuf<int32_t> flag;
    flag.alloc(nv + 1);
    for (int q = 0; q < size; ++q) {
        if (q == me) continue;
        ListHalo::Peer pr;
        pr.rank = q;
        SPFD_CUDA(cudaMemsetAsync(flag.get(), 0, flag.bytes(), s));
        mark(q, me, flag.get());  // what q needs from me
        pr.nsend = compact_flags(flag.get(), nv, pr.sidx, s);
        SPFD_CUDA(cudaMemsetAsync(flag.get(), 0, flag.bytes(), s));
        mark(me, q, flag.get());  // what I need from q
        pr.nrecv = compact_flags(flag.get(), nv, pr.ridx, s);
        if (pr.nsend == 0 && pr.nrecv == 0) continue;
        pr.sbuf.alloc(pr.nsend * maxr + 1);
        pr.rbuf.alloc(pr.nrecv * maxr + 1);
        hl.peers.push_back(std::move(pr));
    }
}

static void list_exchange(Comm &c, ListHalo &hl, double *v, int R, cudaStream_t s) {
    if (hl.peers.empty()) return;
    for (auto &p : hl.peers)
        if (p.nsend) k_pack<<<grid_for(p.nsend, 256), 256, 0, s>>>(p.sidx.get(), p.nsend, R, v, p.sbuf.get());
    SPFD_LAUNCH_CHECK();
    c.begin();
    for (auto &p : hl.peers) {
        c.send(p.rank, p.sbuf.get(), p.nsend * R * sizeof(double));
        c.recv(p.rank, p.rbuf.get(), p.nrecv * R * sizeof(double));
    }
    c.end(s);
    for (auto &p : hl.peers)
        if (p.nrecv) k_unpack<<<grid_for(p.nrecv, 256), 256, 0, s>>>(p.ridx.get(), p.nrecv, R, p.rbuf.get(), v);
    SPFD_LAUNCH_CHECK();
}

// fine level: one node plane with each neighbour (contiguous ranges)
static void range_exchange(Dist &D, double *v, int R, cudaStream_t s) {
    Comm &c = *D.comm;
    c.begin();
    if (D.rank > 0) {
        c.send(D.rank - 1, v + D.lo_send[0] * R, (D.lo_send[1] - D.lo_send[0]) * R * sizeof(double));
        c.recv(D.rank - 1, v + D.lo_recv[0] * R, (D.lo_recv[1] - D.lo_recv[0]) * R * sizeof(double));
    }
    if (D.rank < D.size - 1) {
        c.send(D.rank + 1, v + D.hi_send[0] * R, (D.hi_send[1] - D.hi_send[0]) * R * sizeof(double));
        c.recv(D.rank + 1, v + D.hi_recv[0] * R, (D.hi_recv[1] - D.hi_recv[0]) * R * sizeof(double));
    }
    c.end(s);
}

// One fine-level stencil pass over the owned planes with its input's halo
// exchange overlapped: the interior planes (all neighbours owned) run on the
// side stream while `xin`'s boundary planes travel, then the two boundary
// planes.  Partials (DOT) are written contiguously: interior, low, high.
template <int R, int MODE, bool DOT>
int launch_fine_ov(Dist &D, const Operator &op, const SpanArgs &sa, double *xin, cudaStream_t s) {
    static const bool ov = !(getenv("SPFD_HALO_OVERLAP") && std::string(getenv("SPFD_HALO_OVERLAP")) == "0");
    if (!ov || D.size == 1 || D.ie <= D.ib) {
        range_exchange(D, xin, R, s);
        return launch_fine<R, MODE, DOT>(op, sa, s);
    }
    SPFD_CUDA(cudaEventRecord(D.ev_fork, s));
    SPFD_CUDA(cudaStreamWaitEvent(D.side, D.ev_fork, 0));
    SpanArgs si = sa;
    si.pb = D.ib;
    si.pe = D.ie;
    const int g1 = launch_fine<R, MODE, DOT>(op, si, D.side);
    range_exchange(D, xin, R, s);
    SpanArgs sl = sa;
    sl.pb = D.pb;
    sl.pe = D.ib;
    if (sl.partials) sl.partials += (int64_t)g1 * R;
    const int g2 = D.ib > D.pb ? launch_fine<R, MODE, DOT>(op, sl, s) : 0;
    SpanArgs sh = sa;
    sh.pb = D.ie;
    sh.pe = D.pe;
    if (sh.partials) sh.partials += (int64_t)(g1 + g2) * R;
    const int g3 = D.pe > D.ie ? launch_fine<R, MODE, DOT>(op, sh, s) : 0;
    SPFD_CUDA(cudaEventRecord(D.ev_join, D.side));
    SPFD_CUDA(cudaStreamWaitEvent(s, D.ev_join, 0));
    return g1 + g2 + g3;
}

void amg_distribute_impl(Amg &h, Comm *comm, int64_t replicate_below, int64_t *range, cudaStream_t s) {
    // validate everything before touching the hierarchy
    SPFD_CHECK(h.structured, SPFD_EINVAL, "distribution needs an operator (structured) hierarchy");
    SPFD_CHECK(h.pre <= 1 && h.post == 1, SPFD_EINVAL, "distributed V-cycle supports pre_sweeps <= 1, post_sweeps == 1");
    SPFD_CHECK(h.smoother == SPFD_SMOOTHER_JACOBI, SPFD_EINVAL, "distributed V-cycle supports the Jacobi smoother");
    SPFD_CHECK(comm != nullptr && comm->size >= 1 && comm->rank >= 0 && comm->rank < comm->size, SPFD_EINVAL,
               "invalid communicator");
    SPFD_CHECK(h.op->NZ >= 2 * comm->size, SPFD_EINVAL, "fewer than two node planes per rank");
    level1_unpermute(h, s);  // the slab decomposition works in the reference numbering
    const int T = 256;
    const Operator &op = *h.op;
    auto *D = new Dist();
    try {
        D->comm = comm;
        D->rank = comm->rank;
        D->size = comm->size;
        const int size = D->size, me = D->rank, R = h.max_nrhs;
        // --- fine partition: planes balanced by span positions
        std::vector<int4> rows(op.n_rows + 1);
        SPFD_CUDA(cudaMemcpyAsync(rows.data(), op.rows.get(), rows.size() * sizeof(int4), cudaMemcpyDeviceToHost, s));
        SPFD_CUDA(cudaStreamSynchronize(s));
        const int NZ = (int)op.NZ, NY = (int)op.NY;
        D->plane_pos.resize(NZ + 1);
        for (int k = 0; k < NZ; ++k) D->plane_pos[k] = rows[(size_t)k * NY].x;
        D->plane_pos[NZ] = op.L;
        SPFD_CHECK(NZ >= 2 * size, SPFD_EINVAL, "fewer than two node planes per rank");
        D->kbounds.assign(size + 1, 0);
        D->kbounds[size] = NZ;
        for (int p = 1; p < size; ++p) {
            int64_t target = op.L * p / size;
            int k = D->kbounds[p - 1] + 1;
            while (k < NZ - (size - p) && D->plane_pos[k] < target) ++k;
            D->kbounds[p] = k;
        }
        std::vector<int64_t> pbh(size + 1);
        for (int p = 0; p <= size; ++p) pbh[p] = D->plane_pos[D->kbounds[p]];
        D->pbounds.alloc(size + 1);
        SPFD_CUDA(cudaMemcpyAsync(D->pbounds.get(), pbh.data(), (size + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s));
        D->kb = D->kbounds[me];
        D->ke = D->kbounds[me + 1];
        D->pb = pbh[me];
        D->pe = pbh[me + 1];
        auto plane = [&](int k, int64_t *r2) { r2[0] = D->plane_pos[k]; r2[1] = D->plane_pos[k + 1]; };
        if (me > 0) { plane(D->kb, D->lo_send); plane(D->kb - 1, D->lo_recv); }
        if (me < size - 1) { plane(D->ke - 1, D->hi_send); plane(D->ke, D->hi_recv); }
        D->ib = D->plane_pos[D->kb + (me > 0 ? 1 : 0)];
        D->ie = D->plane_pos[D->ke - (me < size - 1 ? 1 : 0)];
        SPFD_CUDA(cudaStreamCreateWithFlags(&D->side, cudaStreamNonBlocking));
        SPFD_CUDA(cudaEventCreateWithFlags(&D->ev_fork, cudaEventDisableTiming));
        SPFD_CUDA(cudaEventCreateWithFlags(&D->ev_join, cudaEventDisableTiming));
        // DOF and voxel ranges owned (outputs)
        {
            DevBuf<int64_t> cnt;
            cnt.alloc(2);
            SPFD_CUDA(cudaMemsetAsync(cnt.get(), 0, 2 * sizeof(int64_t), s));
            k_count_dofs<<<148 * 4, 256, 0, s>>>(op.dofmask.get(), D->pb, cnt.get());
            k_count_dofs<<<148 * 4, 256, 0, s>>>(op.dofmask.get(), D->pe, cnt.get() + 1);
            SPFD_LAUNCH_CHECK();
            D->dof_b = d2h(cnt.get(), s);
            D->dof_e = d2h(cnt.get() + 1, s);
            int64_t nz = op.nz, ny = op.ny;
            D->vrow_b = std::min<int64_t>(D->kb, nz) * ny;
            D->vrow_e = std::min<int64_t>(D->ke, nz) * ny;
            D->vox_b = d2h(op.vrow_off.get() + D->vrow_b, s);
            D->vox_e = d2h(op.vrow_off.get() + D->vrow_e, s);
        }
        const int nl = (int)h.lv.size();
        D->lv.resize(nl);
        int64_t gmax = 2 * R;
        if (nl > 1) {
            Level &F = h.lv[0];
            Level &L1 = h.lv[1];
            const int64_t n1 = L1.n;
            DistLevel &d1 = D->lv[1];
            d1.owner.alloc(n1);
            k_owner_l1<<<grid_for(n1, T), T, 0, s>>>(F.mem_ptr.get(), F.mem_pos.get(), n1, D->pbounds.get(), size,
                                                     d1.owner.get());
            SPFD_LAUNCH_CHECK();
            D->l1_dist = size > 1 && n1 >= replicate_below && nl > 2;
            if (D->l1_dist) {
                DevBuf<int32_t> flag;
                flag.alloc(n1 + 1);
                k_flag_owner<<<grid_for(n1, T), T, 0, s>>>(d1.owner.get(), n1, me, flag.get());
                D->n_agg_own = compact_flags(flag.get(), n1, D->agg_own, s);
                const int64_t *pbd = D->pbounds.get();
                const int32_t *own1 = d1.owner.get();
                // u halo: members of aggregates owned by q located in my range (what q needs from me)
                build_list_halo(D->hu, me, size, op.L, R,
                                [&](int q, int who, int32_t *fl) {
                                    k_mark_members<<<grid_for(n1, T), T, 0, s>>>(F.mem_ptr.get(), F.mem_pos.get(), n1,
                                                                                 own1, q, pbd, size, who, fl);
                                },
                                s);
                // e halo: aggregates (owned by `who`) of the positions q's stencil touches
                build_list_halo(D->he, me, size, n1, R,
                                [&](int q, int who, int32_t *fl) {
                                    int k0 = std::max(0, D->kbounds[q] - 1), k1 = std::min(NZ, D->kbounds[q + 1] + 1);
                                    int64_t w0 = D->plane_pos[k0], w1 = D->plane_pos[k1];
                                    k_mark_aggs<<<grid_for(w1 - w0, T), T, 0, s>>>(F.agg_pos.get(), w0, w1, own1, who,
                                                                                  fl);
                                },
                                s);
                d1.dist = true;
            } else {
                gmax = std::max<int64_t>(gmax, n1 * R);
            }
            // coarse levels
            for (int l = 1; l < nl - 1 && D->lv[l].dist; ++l) {
                Level &L = h.lv[l];
                Level &C = h.lv[l + 1];
                DistLevel &dl = D->lv[l];
                DistLevel &dn = D->lv[l + 1];
                const int64_t n = L.n, nn = C.n;
                {
                    DevBuf<int32_t> flag;
                    flag.alloc(n + 1);
                    k_flag_owner<<<grid_for(n, T), T, 0, s>>>(dl.owner.get(), n, me, flag.get());
                    dl.n_own = compact_flags(flag.get(), n, dl.own, s);
                }
                extract_rows(L.A, dl.own, dl.n_own, dl.A_loc, s);
                extract_rows(L.P, dl.own, dl.n_own, dl.P_loc, s);
                dl.gA = csr_group(dl.A_loc.nnz, dl.A_loc.rows);
                dl.gP = csr_group(dl.P_loc.nnz, dl.P_loc.rows);
                const int32_t *own_l = dl.owner.get();
                build_list_halo(dl.hA, me, size, n, R,
                                [&](int q, int who, int32_t *fl) {
                                    k_mark_cols<<<grid_for(n, T), T, 0, s>>>(view(L.A), own_l, q, own_l, who, fl);
                                },
                                s);
                // next level ownership: owner of the aggregate's lowest member
                dn.owner.alloc(nn);
                {
                    DevBuf<int32_t> anchor;
                    anchor.alloc(nn);
                    k_fill_i32<<<grid_for(nn, T), T, 0, s>>>(anchor.get(), nn, INT32_MAX);
                    k_anchor<<<grid_for(n, T), T, 0, s>>>(L.agg.get(), n, anchor.get());
                    k_owner_from_anchor<<<grid_for(nn, T), T, 0, s>>>(anchor.get(), nn, own_l, dn.owner.get());
                    SPFD_LAUNCH_CHECK();
                }
                const bool next_dist = nn >= replicate_below && l + 1 < nl - 1;
                if (next_dist) {
                    const int32_t *own_n = dn.owner.get();
                    DevBuf<int32_t> flag;
                    flag.alloc(nn + 1);
                    k_flag_owner<<<grid_for(nn, T), T, 0, s>>>(own_n, nn, me, flag.get());
                    dl.n_next_own = compact_flags(flag.get(), nn, dl.next_own, s);
                    extract_rows(L.R, dl.next_own, dl.n_next_own, dl.R_loc, s);
                    build_list_halo(dl.hR, me, size, n, R,
                                    [&](int q, int who, int32_t *fl) {
                                        k_mark_cols<<<grid_for(nn, T), T, 0, s>>>(view(L.R), own_n, q, own_l, who, fl);
                                    },
                                    s);
                    build_list_halo(dl.hP, me, size, nn, R,
                                    [&](int q, int who, int32_t *fl) {
                                        k_mark_cols<<<grid_for(n, T), T, 0, s>>>(view(L.P), own_l, q, own_n, who, fl);
                                    },
                                    s);
                    dn.dist = true;
                } else {
                    dl.r_partial = true;
                    extract_cols(L.R, own_l, me, dl.R_loc, s);
                    gmax = std::max<int64_t>(gmax, nn * R);
                }
                dl.gR = csr_group(dl.R_loc.nnz, dl.R_loc.rows);
            }
        }
        D->gsend.alloc(gmax);
        D->grecv.alloc(gmax * size);
        range[0] = D->dof_b; range[1] = D->dof_e; range[2] = D->vox_b; range[3] = D->vox_e;
        range[4] = D->kb; range[5] = D->ke;
        h.dist = D;
    } catch (...) {
        delete D;
        throw;
    }
}

// ---------------------------------------------------------- V-cycle --

template <int R>
void allgather_sum(Dist &D, const double *part, int64_t m, double *out, const double *od, double *x0, cudaStream_t s) {
    D.comm->allgather(part, D.grecv.get(), m * R * sizeof(double), s);
    k_rank_sum<<<grid_for(m * R, 256, 148 * 8), 256, 0, s>>>(D.grecv.get(), D.size, m, R, out, od, x0);
    SPFD_LAUNCH_CHECK();
}

template <int R>
void vcycle_dist_level(Amg &h, int l, const double *r, double *z, cudaStream_t s) {
    Dist &D = *h.dist;
    DistLevel &dl = D.lv[l];
    if (!dl.dist) {
        vcycle_level<R>(h, l, r, z, s);
        return;
    }
    Level &L = h.lv[l];
    Level &C = h.lv[l + 1];
    const int nl = (int)h.lv.size();
    const double *od = L.odinv.get();
    double *d = L.vd.get();
    // d = r - A x0 (x0 = od r written for the owned rows by the restriction)
    list_exchange(*D.comm, dl.hA, L.vt.get(), R, s);
    launch_csr<R, 1, false>(dl.A_loc, dl.gA, L.vt.get(), r, od, nullptr, d, nullptr, s, nullptr, nullptr, dl.own.get());
    const bool x0n = l + 1 < nl - 1;
    if (!dl.r_partial) {
        list_exchange(*D.comm, dl.hR, d, R, s);
        launch_csr<R, 0, false>(dl.R_loc, dl.gR, d, nullptr, nullptr, nullptr, C.vr.get(), nullptr, s, C.odinv.get(),
                                x0n ? C.vt.get() : nullptr, dl.next_own.get());
        vcycle_dist_level<R>(h, l + 1, C.vr.get(), C.vx.get(), s);
        list_exchange(*D.comm, dl.hP, C.vx.get(), R, s);
    } else {
        launch_csr<R, 0, false>(dl.R_loc, dl.gR, d, nullptr, nullptr, nullptr, D.gsend.get(), nullptr, s);
        allgather_sum<R>(D, D.gsend.get(), C.n, C.vr.get(), C.odinv.get(), x0n ? C.vt.get() : nullptr, s);
        vcycle_level<R>(h, l + 1, C.vr.get(), C.vx.get(), s);
    }
    // x1 = od r + P e on owned rows, then one Jacobi sweep
    launch_csr<R, 4, false>(dl.P_loc, dl.gP, C.vx.get(), r, od, nullptr, d, nullptr, s, nullptr, nullptr, dl.own.get());
    list_exchange(*D.comm, dl.hA, d, R, s);
    launch_csr<R, 3, false>(dl.A_loc, dl.gA, d, r, od, nullptr, z, nullptr, s, nullptr, nullptr, dl.own.get());
}

// fine level (structured) of a distributed hierarchy; returns the number of
// r.z partial blocks written by the post-smooth (own range)
template <int R>
int vcycle_dist_fine(Amg &h, double *r, double *z, cudaStream_t s) {
    Dist &D = *h.dist;
    Level &L = h.lv[0];
    const Operator &op = *h.op;
    const double *od = L.odinv.get();
    double *d = L.vd.get(), *u = L.vr.get();
    if (h.lv.size() == 1) {  // single-level: replicate the dense solve
        vcycle_level<R>(h, 0, r, z, s);
        return 0;
    }
    Level &C = h.lv[1];
    const int nl = (int)h.lv.size();
    SpanArgs sa{nullptr, r, od, nullptr, nullptr, nullptr, d, nullptr};
    sa.pb = D.pb;
    sa.pe = D.pe;
    launch_fine_ov<R, 2, false>(D, op, sa, r, s);        // d = r - A(od r)
    SpanArgs sb = sa;
    sb.r = d;
    sb.y = u;
    launch_fine_ov<R, 2, false>(D, op, sb, d, s);        // u = d - A(od d)
    const bool x0 = nl > 2;
    if (D.l1_dist) {
        list_exchange(*D.comm, D.hu, u, R, s);
        k_agg_sum_list<R><<<grid_for(D.n_agg_own, 256, 148 * 16), 256, 0, s>>>(
            L.mem_ptr.get(), L.mem_pos.get(), D.agg_own.get(), D.n_agg_own, u, C.vr.get(), C.odinv.get(),
            x0 ? C.vt.get() : nullptr);
        SPFD_LAUNCH_CHECK();
        vcycle_dist_level<R>(h, 1, C.vr.get(), C.vx.get(), s);
        list_exchange(*D.comm, D.he, C.vx.get(), R, s);
    } else {
        k_agg_sum_partial<R><<<grid_for(C.n, 256, 148 * 16), 256, 0, s>>>(L.mem_ptr.get(), L.mem_pos.get(), C.n, D.pb,
                                                                         D.pe, u, D.gsend.get());
        SPFD_LAUNCH_CHECK();
        allgather_sum<R>(D, D.gsend.get(), C.n, C.vr.get(), C.odinv.get(), x0 ? C.vt.get() : nullptr, s);
        vcycle_level<R>(h, 1, C.vr.get(), C.vx.get(), s);
    }
    SpanArgs sc{nullptr, r, od, nullptr, C.vx.get(), L.agg_pos.get(), d, nullptr};
    sc.pb = D.pb;
    sc.pe = D.pe;
    launch_fine<R, 4, false>(op, sc, s);                 // x1 = od r + e - od A e
    SpanArgs sd{d, r, od, nullptr, nullptr, nullptr, z, h.partials.get()};
    sd.pb = D.pb;
    sd.pe = D.pe;
    return launch_fine_ov<R, 3, true>(D, op, sd, d, s);  // z = x1 + od (r - A x1), r.z partials
}

// ------------------------------------------------------------- PCG --

template <int R>
void finalize_dist(Amg &h, int nblocks, int slot, int what, cudaStream_t s) {
    Dist &D = *h.dist;
    k_finalize<R><<<1, kFinThreads, 0, s>>>(h.partials.get(), nblocks, h.scal.get(), S_LOC, F_STORE, 0.0);
    SPFD_LAUNCH_CHECK();
    D.comm->allgather(h.scal.get() + S_LOC, D.grecv.get(), R * sizeof(double), s);
    k_rank_finalize<R><<<1, 32, 0, s>>>(D.grecv.get(), D.size, h.scal.get(), slot, what);
    SPFD_LAUNCH_CHECK();
}

template <int R>
void dot_dist(Amg &h, const double *a, const double *b, int slot, int what, cudaStream_t s) {
    Dist &D = *h.dist;
    const int64_t n = D.pe - D.pb;
    k_dot<R><<<kDotGrid, kDotThreads, 0, s>>>(n, a + D.pb * R, b + D.pb * R, h.partials.get());
    SPFD_LAUNCH_CHECK();
    finalize_dist<R>(h, kDotGrid, slot, what, s);
}

template <int R>
int apply_dist(Amg &h, int mode, bool dot, double *x, const double *r, double *y, cudaStream_t s) {
    Dist &D = *h.dist;
    const Operator &op = *h.op;
    SpanArgs sa{x, r, h.lv[0].odinv.get(), nullptr, nullptr, nullptr, y, h.partials.get()};
    sa.pb = D.pb;
    sa.pe = D.pe;
    if (mode == 0)
        return dot ? launch_fine_ov<R, 0, true>(D, op, sa, x, s) : launch_fine_ov<R, 0, false>(D, op, sa, x, s);
    return dot ? launch_fine_ov<R, 1, true>(D, op, sa, x, s) : launch_fine_ov<R, 1, false>(D, op, sa, x, s);
}

// Convergence test of one distributed PCG iteration on the device (the
// host loop's test): counts the iteration, records the estimates, and once
// the loop would stop (all rhs converged, a non-finite estimate or the
// iteration cap) freezes the solve -- every rhs inactive, so the alpha of
// the iterations still queued behind it is 0 and x, r stay as they are.
// The host reads the scalars once per batch of iterations instead of once
// per iteration.
__global__ void k_dist_check(double *scal, int R, double *trace) {
    if (scal[S_G_DONE] != 0.0) return;
    const int it = (int)scal[S_G_IT] + 1;
    scal[S_G_IT] = it;
    const double tol = scal[S_G_TOL];
    const int maxit = (int)scal[S_G_MAXIT];
    bool done = true, bad = false;
    for (int c = 0; c < R; ++c) {
        const double bb = scal[S_BB + c], rr = scal[S_RR + c];
        const double bn = sqrt(bb);
        const double est = bn > 0 ? sqrt(rr) / bn : 0.0;
        if (!isfinite(est)) bad = true;
        trace[(int64_t)(it - 1) * R + c] = est;
        if (est > tol) done = false;
        const bool conv = bb == 0.0 || sqrt(rr) <= tol * bn;
        scal[S_ACTIVE + c] = conv ? 0.0 : 1.0;
    }
    if (bad) scal[S_G_STATUS] = 1.0;
    if (done || bad || it >= maxit) {
        scal[S_G_DONE] = 1.0;
        for (int c = 0; c < R; ++c) scal[S_ACTIVE + c] = 0.0;
    }
}

// iterations queued per host read (SPFD_DIST_BATCH, default 4; 1 = the
// per-iteration loop)
inline int dist_batch() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("SPFD_DIST_BATCH");
        v = e ? atoi(e) : 4;
        if (v < 1) v = 1;
    }
    return v;
}

// SPFD_DIST_GRAPH=0: queue the distributed iteration batches as individual
// launches even on a stream-ordered transport
inline bool dist_graph_enabled() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("SPFD_DIST_GRAPH");
        v = (e && std::string(e) == "0") ? 0 : 1;
    }
    return v == 1;
}

// One batch of nb iterations (the kernels and transport calls `body` issues
// on the stream it is given) replayed as a CUDA graph: captured on the
// hierarchy's private capture stream the first time, ordered after and
// before the work on s by events.  Returns false (the caller launches the
// batch itself) when the batch cannot be captured.
template <int R, class Body>
bool dist_batch_graph(Amg &h, int nb, Body &&body, cudaStream_t s) {
    Dist &D = *h.dist;
    if (D.batch_exec[R] && (D.batch_nb[R] != nb || D.batch_trace[R] != h.pcg_trace.get())) {
        cudaGraphExecDestroy(D.batch_exec[R]);
        D.batch_exec[R] = nullptr;
    }
    if (!D.batch_exec[R]) {
        if (D.batch_failed[R]) return false;
        if (!h.cap) SPFD_CUDA(cudaStreamCreateWithFlags(&h.cap, cudaStreamNonBlocking));
        const int64_t l0 = launch_count();
        SPFD_CUDA(cudaStreamBeginCapture(h.cap, cudaStreamCaptureModeRelaxed));
        std::string why;
        try {
            body(nb, h.cap);
        } catch (const std::exception &e) {
            why = e.what();
        }
        cudaGraph_t g = nullptr;
        cudaError_t ec = cudaStreamEndCapture(h.cap, &g);
        cudaGraphExec_t exec = nullptr;
        if (why.empty() && ec == cudaSuccess) {
            ec = cudaGraphInstantiate(&exec, g, 0);
            if (ec != cudaSuccess) why = std::string("instantiate: ") + cudaGetErrorString(ec);
        } else if (why.empty()) {
            why = std::string("end capture: ") + cudaGetErrorString(ec);
        }
        if (g) cudaGraphDestroy(g);
        cudaGetLastError();  // clear a sticky capture error
        if (!why.empty()) {
            if (getenv("SPFD_DEBUG")) fprintf(stderr, "[spfd] distributed batch capture failed (%s)\n", why.c_str());
            D.batch_failed[R] = true;
            return false;
        }
        D.batch_exec[R] = exec;
        D.batch_nb[R] = nb;
        D.batch_trace[R] = h.pcg_trace.get();
        D.batch_launches[R] = launch_count() - l0;
        if (getenv("SPFD_DEBUG"))
            fprintf(stderr, "[spfd] distributed batch graph captured: %d iterations, %lld launches\n", nb,
                    (long long)D.batch_launches[R]);
    } else {
        for (int64_t k = 0; k < D.batch_launches[R]; ++k) count_launch();
    }
    SPFD_CUDA(cudaEventRecord(h.ev_alpha, s));
    SPFD_CUDA(cudaStreamWaitEvent(h.cap, h.ev_alpha, 0));
    SPFD_CUDA(cudaGraphLaunch(D.batch_exec[R], h.cap));
    SPFD_CUDA(cudaEventRecord(h.ev_x, h.cap));
    SPFD_CUDA(cudaStreamWaitEvent(s, h.ev_x, 0));
    return true;
}

template <int R>
spfd_report pcg_dist(Amg &h, const double *b, double *x, const spfd_config &cfg, double *h_trace, cudaStream_t s) {
    Dist &D = *h.dist;
    spfd_report rep{};
    const int64_t n = h.lv[0].nvec;
    const int64_t no = D.pe - D.pb, off = D.pb * R;
    double *r = h.kr.get(), *z = h.kz.get(), *p = h.kp.get(), *q = h.kq.get();
    double *sc = h.scal.get();
    SPFD_CUDA(cudaMemsetAsync(x, 0, n * R * sizeof(double), s));
    SPFD_CUDA(cudaMemsetAsync(p, 0, n * R * sizeof(double), s));
    SPFD_CUDA(cudaMemsetAsync(sc, 0, S_H * sizeof(double), s));
    double ones[2] = {1.0, 1.0};
    SPFD_CUDA(cudaMemcpyAsync(sc + S_ACTIVE, ones, R * sizeof(double), cudaMemcpyHostToDevice, s));
    dot_dist<R>(h, b, b, S_BB, F_STORE, s);
    double hs[S_H];
    SPFD_CUDA(cudaMemcpyAsync(hs, sc, S_H * sizeof(double), cudaMemcpyDeviceToHost, s));
    SPFD_CUDA(cudaStreamSynchronize(s));
    double bnorm[2] = {std::sqrt(hs[S_BB]), R > 1 ? std::sqrt(hs[S_BB + 1]) : 0.0};
    for (int c = 0; c < R; ++c)
        if (!std::isfinite(bnorm[c])) { rep.status = SPFD_ENONFINITE; return rep; }
    bool all_zero = true;
    for (int c = 0; c < R; ++c) all_zero = all_zero && bnorm[c] == 0.0;
    if (all_zero) { rep.converged = 1; return rep; }
    const double tol = cfg.rel_tol;
    if (h.pcg_trace_cap < cfg.max_iters) {
        h.pcg_trace_cap = std::max<int64_t>(cfg.max_iters, 1024);
        h.pcg_trace.alloc(h.pcg_trace_cap * 2);
    }
    {
        // S_G_TOL, S_G_MAXIT, S_G_IT, S_G_INIT, S_G_STATUS, S_G_DONE, (2 spare)
        const double g[8] = {tol, (double)cfg.max_iters, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        static_assert(S_G_DONE - S_G < 8 && S_END - S_G == 8, "graph scalar slots");
        SPFD_CUDA(cudaMemcpyAsync(sc + S_G, g, sizeof g, cudaMemcpyHostToDevice, s));
    }
    int it = 0;
    bool restart = true;
    while (true) {
        if (restart) {
            apply_dist<R>(h, 1, false, x, b, r, s);                 // r = b - A x (own range)
            SPFD_CUDA(cudaMemcpyAsync(sc + S_ACTIVE, ones, R * sizeof(double), cudaMemcpyHostToDevice, s));
            const double zero = 0.0;
            SPFD_CUDA(cudaMemcpyAsync(sc + S_G_DONE, &zero, sizeof(double), cudaMemcpyHostToDevice, s));
            int g = vcycle_dist_fine<R>(h, r, z, s);
            if (g > 0) finalize_dist<R>(h, g, S_RZ, F_BETA_INIT, s);
            else dot_dist<R>(h, r, z, S_RZ, F_BETA_INIT, s);
            SPFD_CUDA(cudaMemcpyAsync(p + off, z + off, no * R * sizeof(double), cudaMemcpyDeviceToDevice, s));
            restart = false;
        }
        if (it >= cfg.max_iters) break;
        // a batch of iterations, the convergence test on the device; the
        // ones queued behind a stop are no-ops (k_dist_check)
        const int nb = std::min(dist_batch(), cfg.max_iters - it);
        auto batch = [&](int nbat, cudaStream_t st) {
            for (int k = 0; k < nbat; ++k) {
                int g = apply_dist<R>(h, 0, true, p, nullptr, q, st);    // q = A p, p.q
                finalize_dist<R>(h, g, S_PQ, F_ALPHA, st);
                k_update_xr<R><<<kDotGrid, kDotThreads, 0, st>>>(no, sc, x + off, r + off, p + off, q + off,
                                                                h.partials.get());
                SPFD_LAUNCH_CHECK();
                finalize_dist<R>(h, kDotGrid, S_RR, F_STORE, st);
                k_dist_check<<<1, 1, 0, st>>>(sc, R, h.pcg_trace.get());
                SPFD_LAUNCH_CHECK();
                if (k + 1 == nbat) break;  // the host decides what follows the batch's last test
                int gz = vcycle_dist_fine<R>(h, r, z, st);
                if (gz > 0) finalize_dist<R>(h, gz, S_RZ, F_BETA, st);
                else dot_dist<R>(h, r, z, S_RZ, F_BETA, st);
                k_xpby<R><<<grid_for(no, 256, 148 * 16), 256, 0, st>>>(no, sc, z + off, p + off);
                SPFD_LAUNCH_CHECK();
            }
        };
        // full batches on a stream-ordered transport (NCCL) replay one
        // captured graph: no per-kernel launch cost between host reads
        const bool graphed = nb == dist_batch() && nb > 1 && D.comm->stream_ordered() && dist_graph_enabled() &&
                             dist_batch_graph<R>(h, nb, batch, s);
        if (!graphed) batch(nb, s);
        double gs[8];
        SPFD_CUDA(cudaMemcpyAsync(gs, sc + S_G, sizeof gs, cudaMemcpyDeviceToHost, s));
        SPFD_CUDA(cudaStreamSynchronize(s));
        const int nit = (int)gs[S_G_IT - S_G];
        if (h_trace && nit > it)
            SPFD_CUDA(cudaMemcpy(h_trace + (int64_t)it * R, h.pcg_trace.get() + (int64_t)it * R,
                                 (size_t)(nit - it) * R * sizeof(double), cudaMemcpyDeviceToHost));
        it = nit;
        if (gs[S_G_STATUS - S_G] != 0.0) { rep.status = SPFD_ENONFINITE; rep.iterations = it; return rep; }
        if (gs[S_G_DONE - S_G] != 0.0 || it >= cfg.max_iters) {
            int gt = apply_dist<R>(h, 1, true, x, b, q, s);
            finalize_dist<R>(h, gt, S_TMP, F_STORE, s);
            SPFD_CUDA(cudaMemcpyAsync(hs, sc, S_H * sizeof(double), cudaMemcpyDeviceToHost, s));
            SPFD_CUDA(cudaStreamSynchronize(s));
            bool ok = true;
            for (int c = 0; c < R; ++c) {
                double rel = bnorm[c] > 0 ? std::sqrt(hs[S_TMP + c]) / bnorm[c] : 0.0;
                rep.rel_residual[c] = rel;
                if (!(rel <= tol)) ok = false;
            }
            if (ok || it >= cfg.max_iters) {
                rep.converged = ok ? 1 : 0;
                break;
            }
            restart = true;
            continue;
        }
        int gz = vcycle_dist_fine<R>(h, r, z, s);
        if (gz > 0) finalize_dist<R>(h, gz, S_RZ, F_BETA, s);
        else dot_dist<R>(h, r, z, S_RZ, F_BETA, s);
        k_xpby<R><<<grid_for(no, 256, 148 * 16), 256, 0, s>>>(no, sc, z + off, p + off);
        SPFD_LAUNCH_CHECK();
    }
    // leave x valid on the halo planes too (the E-field reads one plane beyond)
    range_exchange(D, x, R, s);
    rep.iterations = it;
    return rep;
}

// Device AMG setup: strength graph, exact greedy aggregation, smoothed
// prolongation and Galerkin products (linsolve.py:106-176, _kernels.py:79-120).
//
// Parity contract: given the reference's fine matrix, the aggregates are
// identical and P, R = P^T and every coarse operator are bit-identical to the
// scipy results (products are formed without FMA and each output entry is
// summed sequentially in the order scipy's csr_matmat accumulates it).
#include <cub/cub.cuh>

#include <chrono>
#include <algorithm>
#include <cstdlib>

#include "amg.cuh"

namespace spfd {

// SPFD_SETUP_TRACE=1: per-phase wall times of the setup on stderr (each mark
// synchronises the stream; for diagnosing setup-time spread only)
static void setup_mark(const char *what, cudaStream_t s) {
    static const bool on = getenv("SPFD_SETUP_TRACE") != nullptr;
    if (!on) return;
    static auto last = std::chrono::steady_clock::now();
    static cudaEvent_t ev_last = nullptr;
    cudaEvent_t ev;
    cudaEventCreate(&ev);
    cudaEventRecord(ev, s);
    cudaStreamSynchronize(s);
    float gpu_ms = 0.f;
    if (ev_last) cudaEventElapsedTime(&gpu_ms, ev_last, ev);
    if (ev_last) cudaEventDestroy(ev_last);
    ev_last = ev;
    const auto now = std::chrono::steady_clock::now();
    // wall time since the previous mark, and the stream's time between the two marks
    fprintf(stderr, "[setup] %-28s %8.1f ms (stream %8.1f ms)\n", what,
            std::chrono::duration<double, std::milli>(now - last).count(), gpu_ms);
    last = now;
}


namespace {

template <class T>
T read1(const T *dev, cudaStream_t s) {
    T h;
    SPFD_CUDA(cudaMemcpyAsync(&h, dev, sizeof(T), cudaMemcpyDeviceToHost, s));
    SPFD_CUDA(cudaStreamSynchronize(s));
    return h;
}

template <class In, class Out>
void scan_excl(In in, Out *out, int64_t n, cudaStream_t s) {
    size_t bytes = 0;
    SPFD_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, s));
    DevBuf<uint8_t> tmp;
    tmp.alloc(bytes);
    SPFD_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), bytes, in, out, n, s));
    SPFD_CUDA(cudaStreamSynchronize(s));
}

inline int bits_for(uint64_t v) {
    int b = 1;
    while (b < 64 && (v >> b) != 0) ++b;
    return b;
}

// ---------------------------------------------------------------- diag --
__global__ void k_diag_dinv(CsrView a, double omega, double *dinv, double *odinv, double *diag_out,
                            int *bad) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < a.rows;
         r += (int64_t)gridDim.x * blockDim.x) {
        double d = 0.0;
        for (int64_t q = a.ptr[r]; q < a.ptr[r + 1]; ++q)
            if (a.col[q] == r) d = add_rn(d, a.val[q]);
        if (!(d > 0.0)) *bad = 1;
        double di = 1.0 / d;
        dinv[r] = di;
        odinv[r] = mul_rn(omega, di);
        if (diag_out) diag_out[r] = d;
    }
}

// ------------------------------------------------------------ strength --
// strong(i,j): i != j and |a_ij| >= (theta*sd_i)*sd_j, sd = sqrt|a_ii|
// (linsolve.py:106-117)
__global__ void k_strength_count(CsrView a, const double *diag, double theta, int64_t *cnt) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < a.rows;
         r += (int64_t)gridDim.x * blockDim.x) {
        double sr = __dsqrt_rn(fabs(diag[r]));
        double tr = mul_rn(theta, sr);
        int64_t c = 0;
        for (int64_t q = a.ptr[r]; q < a.ptr[r + 1]; ++q) {
            int j = a.col[q];
            if (j == r) continue;
            c += fabs(a.val[q]) >= mul_rn(tr, __dsqrt_rn(fabs(diag[j])));
        }
        cnt[r] = c;
    }
}

__global__ void k_strength_fill(CsrView a, const double *diag, double theta, const int64_t *sptr,
                                int32_t *scol, double *sval) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < a.rows;
         r += (int64_t)gridDim.x * blockDim.x) {
        double tr = mul_rn(theta, __dsqrt_rn(fabs(diag[r])));
        int64_t o = sptr[r];
        for (int64_t q = a.ptr[r]; q < a.ptr[r + 1]; ++q) {
            int j = a.col[q];
            if (j == r) continue;
            double m = fabs(a.val[q]);
            if (m >= mul_rn(tr, __dsqrt_rn(fabs(diag[j])))) { scol[o] = j; sval[o] = m; ++o; }
        }
    }
}

// pattern transpose (order within a row irrelevant for its users)
__global__ void k_count_cols(const int32_t *col, int64_t nnz, int64_t *cnt) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nnz;
         q += (int64_t)gridDim.x * blockDim.x)
        atomicAdd((unsigned long long *)&cnt[col[q]], 1ull);
}

__global__ void k_scatter_t(const int64_t *ptr, const int32_t *col, int64_t rows, int64_t *cursor,
                            int32_t *tcol) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows;
         r += (int64_t)gridDim.x * blockDim.x)
        for (int64_t q = ptr[r]; q < ptr[r + 1]; ++q) {
            unsigned long long o = atomicAdd((unsigned long long *)&cursor[col[q]], 1ull);
            tcol[o] = (int32_t)r;
        }
}

// --------------------------------------------------------- aggregation --
// Pass 1 of _kernels.py:79-120 is the greedy (index-order) selection of
// roots such that no two roots "claim" (root + strong neighbours) a common
// node.  i becomes a root iff every lower-index node r that could claim a
// node of {i} U S(i) is decided non-root; i is non-root as soon as a root
// claims a node of {i} U S(i).  Both rules are monotone, so they can be
// applied asynchronously in rounds; the fixed point is exactly the serial
// result.  Work is event driven: a decided node re-queues its dependants.
struct Graph {
    const int64_t *sp;  // strong graph S
    const int32_t *sc;
    const int64_t *tp;  // transpose S^T (claimers)
    const int32_t *tc;
};

__device__ __forceinline__ void notify_dependants(Graph g, int i, int8_t *state, int *queued, int round,
                                                  int *next, int *n_next) {
    // dependants: j > i with j in {x} U ST(x) for x in {i} U S(i)
    for (int64_t a = g.sp[i] - 1; a < g.sp[i + 1]; ++a) {
        int x = a < g.sp[i] ? i : g.sc[a];
        for (int64_t b = g.tp[x] - 1; b < g.tp[x + 1]; ++b) {
            int j = b < g.tp[x] ? x : g.tc[b];
            if (j <= i) continue;
            if (*(volatile int8_t *)&state[j] != 0) continue;
            if (atomicExch(&queued[j], round) != round) {
                int slot = atomicAdd(n_next, 1);
                next[slot] = j;
            }
        }
    }
}

__global__ void k_agg_round(Graph g, int8_t *state, int32_t *claimed, int *queued, int round,
                            const int *cur, const int *n_cur_p, int *next, int *n_next, int full_n) {
    int n_cur = full_n > 0 ? full_n : *n_cur_p;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n_cur; idx += gridDim.x * blockDim.x) {
        int i = full_n > 0 ? idx : cur[idx];
        if (*(volatile int8_t *)&state[i] != 0) continue;
        bool blocked = false, waiting = false;
        for (int64_t a = g.sp[i] - 1; a < g.sp[i + 1] && !blocked; ++a) {
            int x = a < g.sp[i] ? i : g.sc[a];
            for (int64_t b = g.tp[x] - 1; b < g.tp[x + 1]; ++b) {
                int r = b < g.tp[x] ? x : g.tc[b];
                int8_t st = *(volatile int8_t *)&state[r];
                if (st == 1) { blocked = true; break; }
                if (st == 0 && r < i) waiting = true;
            }
        }
        if (blocked) {
            state[i] = 2;
        } else if (!waiting) {
            claimed[i] = i;
            for (int64_t a = g.sp[i]; a < g.sp[i + 1]; ++a) claimed[g.sc[a]] = i;
            __threadfence();
            state[i] = 1;
        } else {
            continue;
        }
        notify_dependants(g, i, state, queued, round + 1, next, n_next);
    }
}

// The same round with one warp per worklist node: the lanes split each
// node's 2-hop scan (claimers of {i} U S(i)) and its dependant
// notifications; warp votes give the node's decision.  On the coarser
// levels, whose strong graphs are dense (hundreds to thousands of 2-hop
// pairs per node), a thread-per-node round is one long serial loop per
// node; on level 0 the warp form also wins (shorter rounds).  Same
// per-node rule, same fixed point.
__global__ void k_agg_round_warp(Graph g, int8_t *state, int32_t *claimed, int *queued, int round, const int *cur,
                                 const int *n_cur_p, int *next, int *n_next, int full_n) {
    const int lane = threadIdx.x & 31;
    const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int n_cur = full_n > 0 ? full_n : *n_cur_p;
    for (int64_t idx = wid; idx < n_cur; idx += nw) {
        const int i = full_n > 0 ? (int)idx : cur[idx];
        if (*(volatile int8_t *)&state[i] != 0) continue;
        bool blocked = false, waiting = false;
        for (int64_t a = g.sp[i] - 1; a < g.sp[i + 1]; ++a) {
            const int x = a < g.sp[i] ? i : g.sc[a];
            bool bl = false;
            for (int64_t b = g.tp[x] - 1 + lane; b < g.tp[x + 1]; b += 32) {
                const int r = b < g.tp[x] ? x : g.tc[b];
                const int8_t st = *(volatile int8_t *)&state[r];
                if (st == 1) bl = true;
                if (st == 0 && r < i) waiting = true;
            }
            if (__any_sync(0xffffffffu, bl)) { blocked = true; break; }
        }
        waiting = __any_sync(0xffffffffu, waiting);
        if (blocked) {
            if (lane == 0) state[i] = 2;
        } else if (!waiting) {
            if (lane == 0) claimed[i] = i;
            for (int64_t a = g.sp[i] + lane; a < g.sp[i + 1]; a += 32) claimed[g.sc[a]] = i;
            __threadfence();
            __syncwarp();
            if (lane == 0) state[i] = 1;
        } else {
            continue;
        }
        __syncwarp();
        // dependants: j > i with j in {x} U ST(x) for x in {i} U S(i)
        for (int64_t a = g.sp[i] - 1; a < g.sp[i + 1]; ++a) {
            const int x = a < g.sp[i] ? i : g.sc[a];
            for (int64_t b = g.tp[x] - 1 + lane; b < g.tp[x + 1]; b += 32) {
                const int j = b < g.tp[x] ? x : g.tc[b];
                if (j <= i) continue;
                if (*(volatile int8_t *)&state[j] != 0) continue;
                if (atomicExch(&queued[j], round + 1) != round + 1) {
                    const int slot = atomicAdd(n_next, 1);
                    next[slot] = j;
                }
            }
        }
    }
}

__global__ void k_swap_counts(int *n_cur, int *n_next) {
    *n_cur = *n_next;
    *n_next = 0;
}

// Pass 2: strongest already-assigned strong neighbour (strict '>', first
// maximum in CSR order); j < i always counts as assigned in the serial scan.
__global__ void k_agg_best(const int64_t *sp, const int32_t *sc, const double *sv, const int32_t *claimed,
                           int64_t n, int32_t *best, int32_t *single) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (claimed[i] >= 0) { best[i] = -2; single[i] = 0; continue; }
        int b = -1;
        double top = 0.0;
        for (int64_t q = sp[i]; q < sp[i + 1]; ++q) {
            int j = sc[q];
            if ((j < i || claimed[j] >= 0) && sv[q] > top) { top = sv[q]; b = j; }
        }
        best[i] = b;
        single[i] = b < 0 ? 1 : 0;
    }
}

__global__ void k_root_flags(const int8_t *state, int64_t n, int32_t *flag) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        flag[i] = state[i] == 1 ? 1 : 0;
}

__global__ void k_agg_final(const int32_t *claimed, const int32_t *best, const int32_t *root_rank,
                            const int32_t *single_rank, int32_t n_roots, int64_t n, int32_t *agg) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t j = i;
        while (true) {
            if (claimed[j] >= 0) { agg[i] = root_rank[claimed[j]]; break; }
            int b = best[j];
            if (b < 0) { agg[i] = n_roots + single_rank[j]; break; }
            j = b;
        }
    }
}

// ------------------------------------------------------------ ESC SpGEMM --
__global__ void k_prod_count(CsrView a, CsrView b, int64_t *cnt) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < a.rows;
         r += (int64_t)gridDim.x * blockDim.x) {
        int64_t c = 0;
        for (int64_t q = a.ptr[r]; q < a.ptr[r + 1]; ++q) {
            int k = a.col[q];
            c += b.ptr[k + 1] - b.ptr[k];
        }
        cnt[r] = c;
    }
}

// expansion in scipy csr_matmat order: A's row order, then B's row order
__global__ void k_prod_expand(CsrView a, CsrView b, int64_t row0, int64_t row1, const int64_t *off,
                              int64_t base, uint64_t ncols, uint64_t *keys, double *vals) {
    for (int64_t r = row0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < row1;
         r += (int64_t)gridDim.x * blockDim.x) {
        int64_t o = off[r] - base;
        for (int64_t q = a.ptr[r]; q < a.ptr[r + 1]; ++q) {
            int k = a.col[q];
            double av = a.val[q];
            for (int64_t t = b.ptr[k]; t < b.ptr[k + 1]; ++t) {
                keys[o] = (uint64_t)r * ncols + (uint64_t)b.col[t];
                vals[o] = mul_rn(av, b.val[t]);
                ++o;
            }
        }
    }
}

__global__ void k_heads(const uint64_t *keys, int64_t m, int32_t *head) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < m;
         q += (int64_t)gridDim.x * blockDim.x)
        head[q] = (q == 0 || keys[q] != keys[q - 1]) ? 1 : 0;
}

__global__ void k_seg_starts(const int32_t *head, const int64_t *segid, int64_t m, int64_t *start) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < m;
         q += (int64_t)gridDim.x * blockDim.x)
        if (head[q]) start[segid[q]] = q;
}

// sequential per-segment sum (the order scipy accumulates sums[k])
__global__ void k_seg_sum(const uint64_t *keys, const double *vals, const int64_t *start, int64_t nseg,
                          int64_t m, bool drop_zero, uint64_t *okey, double *oval, int32_t *keep) {
    for (int64_t sg = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; sg < nseg;
         sg += (int64_t)gridDim.x * blockDim.x) {
        int64_t b = start[sg], e = sg + 1 < nseg ? start[sg + 1] : m;
        double v = 0.0;
        for (int64_t q = b; q < e; ++q) v = add_rn(v, vals[q]);
        okey[sg] = keys[b];
        oval[sg] = v;
        keep[sg] = (!drop_zero || v != 0.0) ? 1 : 0;
    }
}

__global__ void k_compact(const uint64_t *key, const double *val, const int32_t *keep, const int64_t *pos,
                          int64_t nseg, uint64_t ncols, int64_t out_base, int32_t *col, double *oval,
                          int64_t *rowcnt) {
    for (int64_t sg = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; sg < nseg;
         sg += (int64_t)gridDim.x * blockDim.x) {
        if (!keep[sg]) continue;
        int64_t o = out_base + pos[sg];
        uint64_t k = key[sg];
        col[o] = (int32_t)(k % ncols);
        oval[o] = val[sg];
        atomicAdd((unsigned long long *)&rowcnt[k / ncols], 1ull);
    }
}

__global__ void k_find_chunk(const int64_t *off, int64_t rows, int64_t r0, int64_t budget, int64_t *out) {
    // largest r1 in (r0, rows] with off[r1] - off[r0] <= budget (at least r0+1)
    int64_t lo = r0 + 1, hi = rows;
    int64_t base = off[r0];
    while (lo < hi) {
        int64_t mid = (lo + hi + 1) / 2;
        if (off[mid] - base <= budget) lo = mid; else hi = mid - 1;
    }
    *out = lo;
}

struct Pieces {
    std::vector<DevBuf<int32_t>> cols;
    std::vector<DevBuf<double>> vals;
    std::vector<int64_t> counts;
};

constexpr int64_t kChunkProducts = 48ll << 20;  // products per ESC chunk (~1.5 GB of keys/values + sort
                                                // scratch: stays inside the pool's kept floor, see pool_trim)

// C = A * B (sorted columns, optional zero dropping).
void spgemm(const CsrView &a, const CsrView &b, int64_t bcols, Csr &c, bool drop_zero, cudaStream_t s) {
    const int T = 256;
    int64_t rows = a.rows;
    DevBuf<int64_t> cnt, off, rowcnt;
    cnt.alloc(rows + 1);
    off.alloc(rows + 1);
    rowcnt.alloc(rows + 1);
    SPFD_CUDA(cudaMemsetAsync(cnt.get() + rows, 0, sizeof(int64_t), s));
    SPFD_CUDA(cudaMemsetAsync(rowcnt.get(), 0, rowcnt.bytes(), s));
    if (rows > 0) k_prod_count<<<grid_for(rows, T), T, 0, s>>>(a, b, cnt.get());
    SPFD_LAUNCH_CHECK();
    scan_excl(cnt.get(), off.get(), rows + 1, s);
    int64_t total = read1(off.get() + rows, s);
    uint64_t ncols = (uint64_t)(bcols > 0 ? bcols : 1);
    int end_bit = bits_for((uint64_t)rows * ncols);

    Pieces pc;
    DevBuf<int64_t> chunk_end;
    chunk_end.alloc(1);
    int64_t r0 = 0, out_total = 0;
    while (r0 < rows) {
        k_find_chunk<<<1, 1, 0, s>>>(off.get(), rows, r0, kChunkProducts, chunk_end.get());
        int64_t r1 = read1(chunk_end.get(), s);
        int64_t base = read1(off.get() + r0, s);
        int64_t m = read1(off.get() + r1, s) - base;
        if (m > 0) {
            DevBuf<uint64_t> k0, k1, okey;
            DevBuf<double> v0, v1, oval;
            k0.alloc(m); k1.alloc(m); v0.alloc(m); v1.alloc(m);
            k_prod_expand<<<grid_for(r1 - r0, T), T, 0, s>>>(a, b, r0, r1, off.get(), base, ncols, k0.get(),
                                                             v0.get());
            SPFD_LAUNCH_CHECK();
            size_t bytes = 0;
            SPFD_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, k0.get(), k1.get(), v0.get(), v1.get(),
                                                      m, 0, end_bit, s));
            {
                DevBuf<uint8_t> tmp;
                tmp.alloc(bytes);
                SPFD_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), bytes, k0.get(), k1.get(), v0.get(),
                                                          v1.get(), m, 0, end_bit, s));
                SPFD_CUDA(cudaStreamSynchronize(s));
            }
            k0.release(); v0.release();
            DevBuf<int32_t> head;
            DevBuf<int64_t> segid;
            head.alloc(m);
            segid.alloc(m + 1);
            k_heads<<<grid_for(m, T), T, 0, s>>>(k1.get(), m, head.get());
            {
                cub::TransformInputIterator<int64_t, WidenI32, const int32_t *> wi(head.get(), WidenI32());
                // inclusive ids minus one -> exclusive scan then use directly
                scan_excl(wi, segid.get(), m, s);
            }
            int64_t nseg = read1(segid.get() + (m - 1), s) + read1(head.get() + (m - 1), s);
            DevBuf<int64_t> start;
            start.alloc(nseg);
            k_seg_starts<<<grid_for(m, T), T, 0, s>>>(head.get(), segid.get(), m, start.get());
            head.release(); segid.release();
            okey.alloc(nseg); oval.alloc(nseg);
            DevBuf<int32_t> keep;
            keep.alloc(nseg + 1);
            SPFD_CUDA(cudaMemsetAsync(keep.get() + nseg, 0, sizeof(int32_t), s));
            k_seg_sum<<<grid_for(nseg, T), T, 0, s>>>(k1.get(), v1.get(), start.get(), nseg, m, drop_zero,
                                                      okey.get(), oval.get(), keep.get());
            SPFD_LAUNCH_CHECK();
            k1.release(); v1.release(); start.release();
            DevBuf<int64_t> pos;
            pos.alloc(nseg + 1);
            {
                cub::TransformInputIterator<int64_t, WidenI32, const int32_t *> wi(keep.get(), WidenI32());
                scan_excl(wi, pos.get(), nseg + 1, s);
            }
            int64_t kept = read1(pos.get() + nseg, s);
            DevBuf<int32_t> pcol;
            DevBuf<double> pval;
            pcol.alloc(kept); pval.alloc(kept);
            k_compact<<<grid_for(nseg, T), T, 0, s>>>(okey.get(), oval.get(), keep.get(), pos.get(), nseg, ncols,
                                                      0, pcol.get(), pval.get(), rowcnt.get());
            SPFD_LAUNCH_CHECK();
            SPFD_CUDA(cudaStreamSynchronize(s));
            pc.cols.push_back(std::move(pcol));
            pc.vals.push_back(std::move(pval));
            pc.counts.push_back(kept);
            out_total += kept;
        }
        r0 = r1;
    }
    c.alloc(rows, bcols, out_total);
    int64_t o = 0;
    for (size_t q = 0; q < pc.counts.size(); ++q) {
        if (pc.counts[q] == 0) continue;
        SPFD_CUDA(cudaMemcpyAsync(c.col.get() + o, pc.cols[q].get(), pc.counts[q] * sizeof(int32_t),
                                  cudaMemcpyDeviceToDevice, s));
        SPFD_CUDA(cudaMemcpyAsync(c.val.get() + o, pc.vals[q].get(), pc.counts[q] * sizeof(double),
                                  cudaMemcpyDeviceToDevice, s));
        o += pc.counts[q];
    }
    scan_excl(rowcnt.get(), c.ptr.get(), rows + 1, s);
}

// transpose with (col, row)-sorted output: stable radix sort on col*rows+row
__global__ void k_t_keys(CsrView a, uint64_t nrows, uint64_t *keys, double *vals) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < a.rows;
         r += (int64_t)gridDim.x * blockDim.x)
        for (int64_t q = a.ptr[r]; q < a.ptr[r + 1]; ++q) {
            keys[q] = (uint64_t)a.col[q] * nrows + (uint64_t)r;
            vals[q] = a.val[q];
        }
}

__global__ void k_t_out(const uint64_t *keys, const double *vals, int64_t nnz, uint64_t nrows, int32_t *col,
                        double *val, int64_t *rowcnt) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nnz;
         q += (int64_t)gridDim.x * blockDim.x) {
        col[q] = (int32_t)(keys[q] % nrows);
        val[q] = vals[q];
        atomicAdd((unsigned long long *)&rowcnt[keys[q] / nrows], 1ull);
    }
}

void transpose(const CsrView &a, int64_t acols, Csr &t, cudaStream_t s) {
    const int T = 256;
    int64_t nnz = read1(a.ptr + a.rows, s);
    t.alloc(acols, a.rows, nnz);
    DevBuf<int64_t> rowcnt;
    rowcnt.alloc(acols + 1);
    SPFD_CUDA(cudaMemsetAsync(rowcnt.get(), 0, rowcnt.bytes(), s));
    if (nnz > 0) {
        DevBuf<uint64_t> k0, k1;
        DevBuf<double> v0, v1;
        k0.alloc(nnz); k1.alloc(nnz); v0.alloc(nnz); v1.alloc(nnz);
        uint64_t nrows = (uint64_t)(a.rows > 0 ? a.rows : 1);
        k_t_keys<<<grid_for(a.rows, T), T, 0, s>>>(a, nrows, k0.get(), v0.get());
        int end_bit = bits_for((uint64_t)acols * nrows);
        size_t bytes = 0;
        SPFD_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, k0.get(), k1.get(), v0.get(), v1.get(), nnz, 0,
                                                  end_bit, s));
        DevBuf<uint8_t> tmp;
        tmp.alloc(bytes);
        SPFD_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), bytes, k0.get(), k1.get(), v0.get(), v1.get(), nnz,
                                                  0, end_bit, s));
        k_t_out<<<grid_for(nnz, T), T, 0, s>>>(k1.get(), v1.get(), nnz, nrows, t.col.get(), t.val.get(),
                                               rowcnt.get());
        SPFD_LAUNCH_CHECK();
        SPFD_CUDA(cudaStreamSynchronize(s));
    }
    scan_excl(rowcnt.get(), t.ptr.get(), acols + 1, s);
}

// P = T - (omega*dinv_i) * AT (entries of AT with zero results dropped;
// scipy binop semantics of `tentative - smoothed`, linsolve.py:146-150)
__global__ void k_make_p(CsrView at, const int32_t *agg, const double *dinv, double omega, int64_t *cnt,
                         double *val_out, int32_t *keep) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < at.rows;
         r += (int64_t)gridDim.x * blockDim.x) {
        double scale = mul_rn(omega, dinv[r]);
        int64_t c = 0;
        for (int64_t q = at.ptr[r]; q < at.ptr[r + 1]; ++q) {
            double sm = mul_rn(at.val[q], scale);
            double v = at.col[q] == agg[r] ? sub_rn(1.0, sm) : sub_rn(0.0, sm);
            val_out[q] = v;
            keep[q] = v != 0.0;
            c += v != 0.0;
        }
        cnt[r] = c;
    }
}

__global__ void k_compact_rows(CsrView src, const double *vals, const int32_t *keep, const int64_t *optr,
                               int32_t *ocol, double *oval) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < src.rows;
         r += (int64_t)gridDim.x * blockDim.x) {
        int64_t o = optr[r];
        for (int64_t q = src.ptr[r]; q < src.ptr[r + 1]; ++q)
            if (keep[q]) { ocol[o] = src.col[q]; oval[o] = vals[q]; ++o; }
    }
}

// ------------------------------------------------------ dense inverse ----
__global__ void k_dense_from_csr(CsrView a, int64_t n, double *m) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x)
        for (int64_t q = a.ptr[r]; q < a.ptr[r + 1]; ++q) m[r * n + a.col[q]] = add_rn(m[r * n + a.col[q]], a.val[q]);
}

__global__ void k_eye(int64_t n, double *m) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n * n;
         q += (int64_t)gridDim.x * blockDim.x)
        m[q] = (q / n == q % n) ? 1.0 : 0.0;
}

// Gauss-Jordan step k on [M | Inv] (SPD: no pivoting needed)
__global__ void k_gj_save(const double *m, int64_t n, int64_t k, double *f, int *bad) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        f[i] = m[i * n + k];
        if (i == k && !(f[i] > 0.0 && isfinite(f[i]))) *bad = 1;
    }
}

__global__ void k_gj_norm(double *m, double *inv, int64_t n, int64_t k, const double *f) {
    double piv = f[k];
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n;
         c += (int64_t)gridDim.x * blockDim.x) {
        m[k * n + c] /= piv;
        inv[k * n + c] /= piv;
    }
}

__global__ void k_gj_elim(double *m, double *inv, int64_t n, int64_t k, const double *f) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n * n;
         q += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = q / n, c = q % n;
        if (i == k) continue;
        double fi = f[i];
        if (fi == 0.0) continue;
        m[i * n + c] -= fi * m[k * n + c];
        inv[i * n + c] -= fi * inv[k * n + c];
    }
}

void dense_inverse(const Csr &a, DevBuf<double> &inv, cudaStream_t s) {
    int64_t n = a.rows;
    SPFD_CHECK(n <= 16384, SPFD_EINVAL, "coarsest level too large for a dense factorisation");
    DevBuf<double> m, f;
    DevBuf<int> bad;
    m.alloc(n * n); f.alloc(n); bad.alloc(1);
    inv.alloc(n * n);
    SPFD_CUDA(cudaMemsetAsync(m.get(), 0, m.bytes(), s));
    SPFD_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(int), s));
    const int T = 256;
    k_dense_from_csr<<<grid_for(n, T), T, 0, s>>>(view(a), n, m.get());
    k_eye<<<grid_for(n * n, T), T, 0, s>>>(n, inv.get());
    for (int64_t k = 0; k < n; ++k) {
        k_gj_save<<<grid_for(n, T), T, 0, s>>>(m.get(), n, k, f.get(), bad.get());
        k_gj_norm<<<grid_for(n, T), T, 0, s>>>(m.get(), inv.get(), n, k, f.get());
        k_gj_elim<<<grid_for(n * n, T), T, 0, s>>>(m.get(), inv.get(), n, k, f.get());
    }
    SPFD_LAUNCH_CHECK();
    SPFD_CHECK(read1(bad.get(), s) == 0, SPFD_ENOTPOS, "coarsest matrix is not positive definite");
}

// ------------------------------------------------- structured level 0 ----
__global__ void k_dofs_to_span_1(const int32_t *pos_to_dof, int64_t L, const double *in, double *out) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < L;
         p += (int64_t)gridDim.x * blockDim.x) {
        int d = pos_to_dof[p];
        out[p] = d >= 0 ? in[d] : 0.0;
    }
}

__global__ void k_agg_pos(const int32_t *pos_to_dof, int64_t L, const int32_t *agg, int32_t *out) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < L;
         p += (int64_t)gridDim.x * blockDim.x) {
        int d = pos_to_dof[p];
        out[p] = d >= 0 ? agg[d] + 1 : 0;  // aggregate id + 1, 0 = none
    }
}

__global__ void k_member_init(const int32_t *dof_to_pos, int64_t n, int32_t *pos) {
    for (int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; d < n; d += (int64_t)gridDim.x * blockDim.x)
        pos[d] = dof_to_pos[d];
}

__global__ void k_count_agg(const int32_t *agg, int64_t n, int64_t *cnt) {
    for (int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; d < n; d += (int64_t)gridDim.x * blockDim.x)
        atomicAdd((unsigned long long *)&cnt[agg[d]], 1ull);
}

// members of every aggregate in ascending position order: stable radix sort
// of (aggregate id, position) pairs in DOF order (positions ascend with DOFs)
void build_members(const int32_t *agg, int64_t n, int64_t n_agg, const int32_t *dof_to_pos, DevBuf<int64_t> &mptr,
                   DevBuf<int32_t> &mpos, cudaStream_t s) {
    const int T = 256;
    DevBuf<int32_t> k1, v0;
    k1.alloc(n); v0.alloc(n);
    mpos.alloc(n);
    k_member_init<<<grid_for(n, T), T, 0, s>>>(dof_to_pos, n, v0.get());
    size_t bytes = 0;
    int end_bit = bits_for((uint64_t)n_agg);
    SPFD_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, agg, k1.get(), v0.get(), mpos.get(), n, 0, end_bit, s));
    DevBuf<uint8_t> tmp;
    tmp.alloc(bytes);
    SPFD_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), bytes, agg, k1.get(), v0.get(), mpos.get(), n, 0, end_bit, s));
    DevBuf<int64_t> cnt;
    cnt.alloc(n_agg + 1);
    SPFD_CUDA(cudaMemsetAsync(cnt.get(), 0, cnt.bytes(), s));
    k_count_agg<<<grid_for(n, T), T, 0, s>>>(agg, n, cnt.get());
    SPFD_LAUNCH_CHECK();
    mptr.alloc(n_agg + 1);
    scan_excl(cnt.get(), mptr.get(), n_agg + 1, s);
}

// lanes per row of the CSR kernels: small groups keep the per-row
// reduction/epilogue overhead low (the coarse rows hold ~10-40 entries)
int pick_group(int64_t nnz, int64_t rows) {
    static int forced = -1;
    if (forced < 0) {
        const char *e = getenv("SPFD_CSR_GROUP");
        forced = e ? atoi(e) : 0;
    }
    if (forced == 4 || forced == 8 || forced == 16 || forced == 32) return forced;
    double avg = rows > 0 ? (double)nnz / (double)rows : 1.0;
    // (measured on C3: the level-1 operator, ~30 nnz/row, runs fastest with
    // 4 lanes -- fewer shuffle levels, more rows in flight per warp)
    int g = avg <= 40.0 ? 4 : (avg <= 48.0 ? 8 : 16);
    // small coarse matrices: widen the groups until the launch fills the
    // machine (latency, not bandwidth, bounds those levels); rows of several
    // hundred entries get up to a whole CTA (k_csr_wide)
    const int gmax = avg >= 128.0 ? 256 : 32;
    while (g < gmax && rows * (int64_t)g < (int64_t)148 * 32 * 64 && g * 2 <= 2 * avg) g *= 2;
    return g;
}

// One coarsening step on level l (CSR A in level numbering).  Returns false
// on stagnation.
// tentative prolongator T: one unit entry per row (column = aggregate)
__global__ void k_tent_fill(int64_t n, int64_t *ptr, double *val) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x) {
        ptr[i] = i;
        if (i < n) val[i] = 1.0;
    }
}

bool coarsen(Level &L, const Csr &A, double theta, double omega, Csr &Ac, Csr &P, Csr &R, DevBuf<int32_t> &agg,
             cudaStream_t s) {
    const int T = 256;
    int64_t n = A.rows;
    CsrView av = view(A);
    DevBuf<double> diag;
    diag.alloc(n);
    {
        DevBuf<double> d1, d2;
        d1.alloc(n); d2.alloc(n);
        DevBuf<int> bad;
        bad.alloc(1);
        SPFD_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(int), s));
        k_diag_dinv<<<grid_for(n, T), T, 0, s>>>(av, omega, d1.get(), d2.get(), diag.get(), bad.get());
        SPFD_CHECK(read1(bad.get(), s) == 0, SPFD_ENOTPOS, "matrix has a non-positive diagonal entry");
    }
    // strength graph
    DevBuf<int64_t> scnt, sptr;
    scnt.alloc(n + 1); sptr.alloc(n + 1);
    SPFD_CUDA(cudaMemsetAsync(scnt.get() + n, 0, sizeof(int64_t), s));
    k_strength_count<<<grid_for(n, T), T, 0, s>>>(av, diag.get(), theta, scnt.get());
    scan_excl(scnt.get(), sptr.get(), n + 1, s);
    int64_t snnz = read1(sptr.get() + n, s);
    DevBuf<int32_t> scol;
    DevBuf<double> sval;
    scol.alloc(snnz); sval.alloc(snnz);
    k_strength_fill<<<grid_for(n, T), T, 0, s>>>(av, diag.get(), theta, sptr.get(), scol.get(), sval.get());
    // transpose pattern
    DevBuf<int64_t> tcnt, tptr, cursor;
    tcnt.alloc(n + 1); tptr.alloc(n + 1); cursor.alloc(n + 1);
    SPFD_CUDA(cudaMemsetAsync(tcnt.get(), 0, tcnt.bytes(), s));
    if (snnz) k_count_cols<<<grid_for(snnz, T), T, 0, s>>>(scol.get(), snnz, tcnt.get());
    scan_excl(tcnt.get(), tptr.get(), n + 1, s);
    SPFD_CUDA(cudaMemcpyAsync(cursor.get(), tptr.get(), (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
    DevBuf<int32_t> tcol;
    tcol.alloc(snnz);
    k_scatter_t<<<grid_for(n, T), T, 0, s>>>(sptr.get(), scol.get(), n, cursor.get(), tcol.get());
    SPFD_LAUNCH_CHECK();

    setup_mark("strength + transpose", s);
    // pass 1
    DevBuf<int8_t> state;
    DevBuf<int32_t> claimed;
    DevBuf<int> queued, wl0, wl1, counts;
    state.alloc(n); claimed.alloc(n); queued.alloc(n); wl0.alloc(n); wl1.alloc(n); counts.alloc(2);
    SPFD_CUDA(cudaMemsetAsync(state.get(), 0, n, s));
    SPFD_CUDA(cudaMemsetAsync(claimed.get(), 0xff, n * sizeof(int32_t), s));
    SPFD_CUDA(cudaMemsetAsync(queued.get(), 0xff, n * sizeof(int), s));
    SPFD_CUDA(cudaMemsetAsync(counts.get(), 0, 2 * sizeof(int), s));
    Graph g{sptr.get(), scol.get(), tptr.get(), tcol.get()};
    int *cur = wl0.get(), *nxt = wl1.get();
    int *n_cur = counts.get(), *n_next = counts.get() + 1;
    const int G = 148 * 8;
    // warp per node where the strong graph is dense (see k_agg_round_warp;
    // SPFD_AGG_WARP=0: thread per node everywhere)
    // one warp per node on every level (C3 pass 1: level 0 259 -> 111 ms,
    // level 1 430 -> 47 ms, level 2 270 -> 19 ms); SPFD_AGG_WARP=0: one thread
    const char *aw = getenv("SPFD_AGG_WARP");
    const bool warp_round = !(aw && std::string(aw) == "0");
    if (warp_round)
        k_agg_round_warp<<<G, T, 0, s>>>(g, state.get(), claimed.get(), queued.get(), 0, cur, n_cur, nxt, n_next,
                                         (int)n);
    else
        k_agg_round<<<grid_for(n, T, G), T, 0, s>>>(g, state.get(), claimed.get(), queued.get(), 0, cur, n_cur, nxt,
                                                   n_next, (int)n);
    k_swap_counts<<<1, 1, 0, s>>>(n_cur, n_next);
    std::swap(cur, nxt);
    int round = 1;
    while (true) {
        for (int b = 0; b < 64; ++b, ++round) {
            if (warp_round)
                k_agg_round_warp<<<G, T, 0, s>>>(g, state.get(), claimed.get(), queued.get(), round, cur, n_cur, nxt,
                                                 n_next, 0);
            else
                k_agg_round<<<G, T, 0, s>>>(g, state.get(), claimed.get(), queued.get(), round, cur, n_cur, nxt,
                                            n_next, 0);
            k_swap_counts<<<1, 1, 0, s>>>(n_cur, n_next);
            std::swap(cur, nxt);
        }
        SPFD_LAUNCH_CHECK();
        if (read1(n_cur, s) == 0) break;
        SPFD_CHECK(round < 4 * (int)n + 1000, SPFD_ECUDA, "aggregation did not terminate");
    }
    setup_mark("aggregation pass 1", s);
    // pass 2 + numbering
    DevBuf<int32_t> best, single, rootflag, root_rank, single_rank;
    best.alloc(n); single.alloc(n + 1); rootflag.alloc(n + 1); root_rank.alloc(n + 1); single_rank.alloc(n + 1);
    SPFD_CUDA(cudaMemsetAsync(single.get() + n, 0, sizeof(int32_t), s));
    SPFD_CUDA(cudaMemsetAsync(rootflag.get() + n, 0, sizeof(int32_t), s));
    k_agg_best<<<grid_for(n, T), T, 0, s>>>(sptr.get(), scol.get(), sval.get(), claimed.get(), n, best.get(),
                                             single.get());
    k_root_flags<<<grid_for(n, T), T, 0, s>>>(state.get(), n, rootflag.get());
    scan_excl(rootflag.get(), root_rank.get(), n + 1, s);
    scan_excl(single.get(), single_rank.get(), n + 1, s);
    int32_t n_roots = read1(root_rank.get() + n, s);
    int32_t n_single = read1(single_rank.get() + n, s);
    int64_t n_agg = (int64_t)n_roots + n_single;
    agg.alloc(n);
    k_agg_final<<<grid_for(n, T), T, 0, s>>>(claimed.get(), best.get(), root_rank.get(), single_rank.get(),
                                              n_roots, n, agg.get());
    SPFD_LAUNCH_CHECK();
    if (n_agg >= n) return false;

    // tentative T (n x n_agg, ones) and AT = A * T (zeros kept)
    Csr Tm;
    Tm.alloc(n, n_agg, n);
    k_tent_fill<<<grid_for(n + 1, T), T, 0, s>>>(n, Tm.ptr.get(), Tm.val.get());  // ptr = 0..n, values 1
    SPFD_LAUNCH_CHECK();
    SPFD_CUDA(cudaMemcpyAsync(Tm.col.get(), agg.get(), n * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    Csr AT;
    setup_mark("aggregation pass 2", s);
    spgemm(av, view(Tm), n_agg, AT, false, s);
    Tm = Csr();
    // P
    {
        DevBuf<double> dinv;
        dinv.alloc(n);
        DevBuf<double> od;
        od.alloc(n);
        DevBuf<int> bad;
        bad.alloc(1);
        SPFD_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(int), s));
        k_diag_dinv<<<grid_for(n, T), T, 0, s>>>(av, omega, dinv.get(), od.get(), nullptr, bad.get());
        DevBuf<int64_t> pcnt;
        pcnt.alloc(n + 1);
        SPFD_CUDA(cudaMemsetAsync(pcnt.get() + n, 0, sizeof(int64_t), s));
        DevBuf<double> pv;
        DevBuf<int32_t> keep;
        pv.alloc(AT.nnz); keep.alloc(AT.nnz);
        k_make_p<<<grid_for(n, T), T, 0, s>>>(view(AT), agg.get(), dinv.get(), omega, pcnt.get(), pv.get(),
                                              keep.get());
        DevBuf<int64_t> pptr;
        pptr.alloc(n + 1);
        scan_excl(pcnt.get(), pptr.get(), n + 1, s);
        int64_t pnnz = read1(pptr.get() + n, s);
        P.alloc(n, n_agg, pnnz);
        SPFD_CUDA(cudaMemcpyAsync(P.ptr.get(), pptr.get(), (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
        k_compact_rows<<<grid_for(n, T), T, 0, s>>>(view(AT), pv.get(), keep.get(), pptr.get(), P.col.get(),
                                                    P.val.get());
        SPFD_LAUNCH_CHECK();
        SPFD_CUDA(cudaStreamSynchronize(s));
    }
    AT = Csr();
    transpose(view(P), n_agg, R, s);
    Csr AP;
    setup_mark("prolongator P, R", s);
    spgemm(av, view(P), n_agg, AP, true, s);
    spgemm(view(R), view(AP), n_agg, Ac, true, s);
    setup_mark("Galerkin R A P", s);
    (void)L;
    return true;
}

}  // namespace

int csr_group(int64_t nnz, int64_t rows) { return pick_group(nnz, rows); }

int64_t Amg::device_bytes() const {
    int64_t b = cinv.bytes() + kx.bytes() + kr.bytes() + kz.bytes() + kp.bytes() + kq.bytes() + kb.bytes() +
                partials.bytes() + scal.bytes() + fg_basis.bytes() + fg_prec.bytes();
    for (auto &l : lv)
        b += l.A.bytes() + l.P.bytes() + l.R.bytes() + l.P_dof.bytes() + l.R_dof.bytes() + l.Rspan.bytes() + l.Pspan.bytes() + l.Q.bytes() + l.agg.bytes() +
             l.dinv.bytes() + l.odinv.bytes() + l.agg_pos.bytes() + l.mem_ptr.bytes() + l.mem_pos.bytes() + l.vr.bytes() + l.vx.bytes() + l.vd.bytes() + l.vt.bytes() + l.AP.bytes();
    return b;
}

void alloc_krylov(Amg &h, int64_t nvec0, int max_nrhs);

// ---- level-1 renumbering (solve layout) ------------------------------------
// Level-1 unknowns (aggregates) renumbered along a Morton curve of their
// root nodes; every level-1 structure the single-GPU V-cycle uses is
// permuted consistently on the device, keeping each row's entry order, so
// the V-cycle computes the same sums in the same order (same bits).
template <class T>
static std::vector<T> d2h(const DevBuf<T> &b, size_t n) {
    std::vector<T> v(n);
    if (n) SPFD_CUDA(cudaMemcpy(v.data(), b.get(), n * sizeof(T), cudaMemcpyDeviceToHost));
    return v;
}
__host__ __device__ inline uint64_t morton3(uint32_t x, uint32_t y, uint32_t z) {
    auto spread = [](uint64_t v) {
        v &= 0x1fffff;
        v = (v | v << 32) & 0x1f00000000ffffull;
        v = (v | v << 16) & 0x1f0000ff0000ffull;
        v = (v | v << 8) & 0x100f00f00f00f00full;
        v = (v | v << 4) & 0x10c30c30c30c30c3ull;
        v = (v | v << 2) & 0x1249249249249249ull;
        return v;
    };
    return spread(x) | spread(y) << 1 | spread(z) << 2;
}
__global__ void k_perm_len(const int64_t *ptr, const int32_t *P, int64_t n, int64_t *len) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t o = P ? P[r] : r;
        len[r] = ptr[o + 1] - ptr[o];
    }
}
// new row r = old row P[r] (entry order kept), columns relabelled by cmap
__global__ void k_perm_rows(const int64_t *ptr, const int32_t *col, const double *val, const int32_t *P,
                            const int32_t *cmap, const int64_t *nptr, int64_t n, int32_t *ncol, double *nval) {
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    for (int64_t r = warp; r < n; r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t o = P ? P[r] : r;
        const int64_t b = ptr[o], e = ptr[o + 1], t0 = nptr[r];
        for (int64_t q = b + lane; q < e; q += 32) {
            const int32_t c = col[q];
            ncol[t0 + (q - b)] = cmap ? cmap[c] : c;
            if (val) nval[t0 + (q - b)] = val[q];
        }
    }
}
__global__ void k_gather_d(const double *x, const int32_t *P, int64_t n, double *y) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
        y[r] = x[P[r]];
}
__global__ void k_inv_perm(const int32_t *P, int64_t n, int32_t *inv) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
        inv[P[r]] = (int32_t)r;
}
__global__ void k_relabel_aggpos(int32_t *ap, int64_t n, const int32_t *inv) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x)
        if (ap[p] > 0) ap[p] = inv[ap[p] - 1] + 1;
}
__global__ void k_root_keys(const int64_t *mptr, const int32_t *mpos, int64_t n1, const int4 *rows, int64_t n_rows,
                            int NY, uint64_t *key, int32_t *idx) {
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < n1; g += (int64_t)gridDim.x * blockDim.x) {
        const int p = mpos[mptr[g]];  // root: the aggregate's first member
        int lo = 0, hi = (int)n_rows - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (rows[mid].x <= p) lo = mid; else hi = mid - 1;
        }
        const int4 q = rows[lo];
        key[g] = morton3((uint32_t)(q.y + (p - q.x)), (uint32_t)(lo % NY), (uint32_t)(lo / NY));
        idx[g] = (int32_t)g;
    }
}

// permute rows (P: new -> old, device) and relabel columns (cmap, device) of a CSR in place
static void perm_csr(Csr &m, const int32_t *P, const int32_t *cmap, cudaStream_t s) {
    const int T = 256;
    DevBuf<int64_t> len, nptr;
    len.alloc(m.rows + 1);
    nptr.alloc(m.rows + 1);
    SPFD_CUDA(cudaMemsetAsync(len.get() + m.rows, 0, sizeof(int64_t), s));
    k_perm_len<<<grid_for(m.rows, T), T, 0, s>>>(m.ptr.get(), P, m.rows, len.get());
    SPFD_LAUNCH_CHECK();
    scan_excl(len.get(), nptr.get(), m.rows + 1, s);
    DevBuf<int32_t> ncol;
    DevBuf<double> nval;
    ncol.alloc(m.nnz);
    nval.alloc(m.nnz);
    k_perm_rows<<<grid_for(m.rows * 32, T), T, 0, s>>>(m.ptr.get(), m.col.get(), m.val.get(), P, cmap, nptr.get(),
                                                       m.rows, ncol.get(), nval.get());
    SPFD_LAUNCH_CHECK();
    m.ptr = std::move(nptr);
    m.col = std::move(ncol);
    m.val = std::move(nval);
}

// Apply a renumbering of the level-1 unknowns (P: new index -> current
// index, device array) to every structure the single-GPU V-cycle reads;
// h.l1_perm keeps new -> reference index (empty = reference numbering).
void level1_permute(Amg &h, const int32_t *P, cudaStream_t s) {
    const int T = 256;
    Level &L0 = h.lv[0], &L1 = h.lv[1];
    // the captured PCG graphs hold the buffers replaced below: recapture
    amg_drop_graphs(h);
    const int64_t n1 = L1.n;
    DevBuf<int32_t> inv;
    inv.alloc(n1);
    k_inv_perm<<<grid_for(n1, T), T, 0, s>>>(P, n1, inv.get());
    SPFD_LAUNCH_CHECK();
    perm_csr(L1.A, P, inv.get(), s);
    if (L1.AP.rows) perm_csr(L1.AP, P, nullptr, s);
    perm_csr(L1.P, P, nullptr, s);
    perm_csr(L1.R, nullptr, inv.get(), s);
    for (DevBuf<double> *b : {&L1.odinv, &L1.dinv}) {
        DevBuf<double> nb;
        nb.alloc(b->n);
        if (b->n > (size_t)n1)  // alignment padding beyond the rows
            SPFD_CUDA(cudaMemsetAsync(nb.get() + n1, 0, (b->n - n1) * sizeof(double), s));
        k_gather_d<<<grid_for(n1, T), T, 0, s>>>(b->get(), P, n1, nb.get());
        SPFD_LAUNCH_CHECK();
        *b = std::move(nb);
    }
    k_relabel_aggpos<<<grid_for(L0.nvec, T), T, 0, s>>>(L0.agg_pos.get(), L0.nvec, inv.get());
    SPFD_LAUNCH_CHECK();
    {   // member lists: a CSR without values
        DevBuf<int64_t> len, nptr;
        len.alloc(n1 + 1);
        nptr.alloc(n1 + 1);
        SPFD_CUDA(cudaMemsetAsync(len.get() + n1, 0, sizeof(int64_t), s));
        k_perm_len<<<grid_for(n1, T), T, 0, s>>>(L0.mem_ptr.get(), P, n1, len.get());
        SPFD_LAUNCH_CHECK();
        scan_excl(len.get(), nptr.get(), n1 + 1, s);
        DevBuf<int32_t> npos;
        npos.alloc(L0.mem_pos.n);
        k_perm_rows<<<grid_for(n1 * 32, T), T, 0, s>>>(L0.mem_ptr.get(), L0.mem_pos.get(), nullptr, P, nullptr,
                                                       nptr.get(), n1, npos.get(), nullptr);
        SPFD_LAUNCH_CHECK();
        L0.mem_ptr = std::move(nptr);
        L0.mem_pos = std::move(npos);
    }
    // compose the bookkeeping on the host (n1 ints)
    std::vector<int32_t> hp(n1);
    SPFD_CUDA(cudaMemcpyAsync(hp.data(), P, n1 * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    SPFD_CUDA(cudaStreamSynchronize(s));
    std::vector<int32_t> comp(n1);
    bool ident = true;
    for (int64_t g = 0; g < n1; ++g) {
        comp[g] = h.l1_perm.empty() ? hp[g] : h.l1_perm[hp[g]];
        ident = ident && comp[g] == g;
    }
    if (ident) h.l1_perm.clear();
    else h.l1_perm = std::move(comp);
    build_rspan(h, s);  // rows follow the new level-1 numbering
    build_q(h, s);
}

// back to the reference numbering (before distributing the hierarchy)
void level1_unpermute(Amg &h, cudaStream_t s) {
    if (h.l1_perm.empty()) return;
    const int64_t n1 = h.lv[1].n;
    std::vector<int32_t> Q(n1);
    for (int64_t g = 0; g < n1; ++g) Q[h.l1_perm[g]] = (int32_t)g;  // reference index -> current index
    DevBuf<int32_t> dq;
    dq.alloc(n1);
    SPFD_CUDA(cudaMemcpyAsync(dq.get(), Q.data(), n1 * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    level1_permute(h, dq.get(), s);
}

// Morton order of the level-1 aggregates' root nodes (device keys + CUB sort)
// The fine-level restriction r_c = R d as the reference computes it
// (linsolve.py:190-195, R = P^T), on a CSR whose columns are span positions
// and whose rows follow the level-1 solve numbering: one gather-SpMV over
// nnz(P) entries instead of the matrix-free form's stencil pass over d plus
// the aggregate sums.  The entries of each row keep R's order, so the result
// does not depend on the level-1 numbering.  SPFD_RSPAN=0: matrix-free.
__global__ void k_rspan_len(const int64_t *__restrict__ rptr, const int32_t *__restrict__ perm, int64_t n1,
                            int64_t *__restrict__ len) {
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < n1; g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = perm ? perm[g] : g;
        len[g] = rptr[r + 1] - rptr[r];
    }
}

__global__ void k_rspan_fill(CsrView R, const int32_t *__restrict__ perm, const int32_t *__restrict__ dof_to_pos,
                             const int64_t *__restrict__ optr, int64_t n1, int32_t *__restrict__ col,
                             double *__restrict__ val) {
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < n1; g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = perm ? perm[g] : g;
        const int64_t a = R.ptr[r], b = R.ptr[r + 1], o = optr[g];
        for (int64_t q = a; q < b; ++q) {
            col[o + (q - a)] = dof_to_pos[R.col[q]];
            val[o + (q - a)] = R.val[q];
        }
    }
}

// The fine-level prolongation x1 = x0 + P e on the reference's P (rows: span
// positions, empty for non-DOF positions; columns: level-1 solve indices),
// each row's entries in P's stored order.  About 3.6 entries per row: a
// short-row gather-SpMV from the L2-resident coarse vector instead of the
// matrix-free (I - omega D^-1 A) T e, whose 7-point stencil re-reads the
// aggregate map and the conductances at every neighbour.  SPFD_PSPAN=0:
// matrix-free.
__global__ void k_inv_perm_i(const int32_t *__restrict__ solve_to_ref, int64_t n, int32_t *__restrict__ ref_to_solve) {
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < n; g += (int64_t)gridDim.x * blockDim.x)
        ref_to_solve[solve_to_ref[g]] = (int32_t)g;
}

__global__ void k_pspan_len(const int64_t *__restrict__ pptr, const int32_t *__restrict__ pos_to_dof, int64_t L,
                            int64_t *__restrict__ len) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < L; p += (int64_t)gridDim.x * blockDim.x) {
        const int32_t d = pos_to_dof[p];
        len[p] = d >= 0 ? pptr[d + 1] - pptr[d] : 0;
    }
}

__global__ void k_pspan_fill(CsrView P, const int32_t *__restrict__ pos_to_dof, const int32_t *__restrict__ ref_to_solve,
                             const int64_t *__restrict__ optr, int64_t L, int32_t *__restrict__ col,
                             double *__restrict__ val) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < L; p += (int64_t)gridDim.x * blockDim.x) {
        const int32_t d = pos_to_dof[p];
        if (d < 0) continue;
        const int64_t a = P.ptr[d], b = P.ptr[d + 1], o = optr[p];
        for (int64_t q = a; q < b; ++q) {
            const int32_t c = P.col[q];
            col[o + (q - a)] = ref_to_solve ? ref_to_solve[c] : c;
            val[o + (q - a)] = P.val[q];
        }
    }
}

void build_pspan(Amg &h, const int32_t *solve_to_ref, cudaStream_t s) {
    const bool on = !(getenv("SPFD_PSPAN") && std::string(getenv("SPFD_PSPAN")) == "0");
    Level &L0 = h.lv[0];
    L0.Pspan = Csr{};
    if (!on || !h.structured || h.lv.size() < 2 || L0.P_dof.rows == 0) return;
    const int T = 256;
    const int64_t n1 = h.lv[1].n, L = L0.nvec;
    DevBuf<int32_t> r2s;
    if (solve_to_ref) {
        r2s.alloc(n1);
        k_inv_perm_i<<<grid_for(n1, T), T, 0, s>>>(solve_to_ref, n1, r2s.get());
        SPFD_LAUNCH_CHECK();
    }
    DevBuf<int64_t> len;
    len.alloc(L + 1);
    SPFD_CUDA(cudaMemsetAsync(len.get() + L, 0, sizeof(int64_t), s));
    k_pspan_len<<<grid_for(L, T), T, 0, s>>>(L0.P_dof.ptr.get(), h.op->pos_to_dof.get(), L, len.get());
    SPFD_LAUNCH_CHECK();
    Csr &M = L0.Pspan;
    M.rows = L;
    M.cols = n1;
    M.ptr.alloc(L + 1);
    scan_excl(len.get(), M.ptr.get(), L + 1, s);
    M.nnz = read1(M.ptr.get() + L, s);
    M.col.alloc(M.nnz);
    M.val.alloc(M.nnz);
    k_pspan_fill<<<grid_for(L, T), T, 0, s>>>(view(L0.P_dof), h.op->pos_to_dof.get(), r2s.n ? r2s.get() : nullptr,
                                              M.ptr.get(), L, M.col.get(), M.val.get());
    SPFD_LAUNCH_CHECK();
    // ~3.6 entries per row: one thread per row (coalesced epilogue; measured
    // 161 us vs 195 us with 2 lanes and 316 us with 4 on C3)
    L0.pspan_group = 1;
    if (const char *e = getenv("SPFD_GROUP_PSPAN")) L0.pspan_group = atoi(e);
}

// Coarse-level V(1,1) prolongation + post-smooth as one operator:
//   z = od r + P e + od (d - (A P) e) = od (r + d) + Q e,  Q = P - diag(od) A P
// with the pattern of A P (which contains P's: A has a full diagonal and the
// product keeps zeros).  One gather-SpMV over nnz(A P) entries instead of
// P and A P (k_csr_pp).  A row of P outside A P's pattern drops Q for the
// level.  SPFD_Q=0 keeps k_csr_pp.
__global__ void k_q_fill(CsrView P, CsrView AP, const double *__restrict__ od, double *__restrict__ qv,
                         int *__restrict__ bad) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < AP.rows; r += (int64_t)gridDim.x * blockDim.x) {
        const double o = od[r];
        int64_t p = P.ptr[r];
        const int64_t p1 = P.ptr[r + 1];
        for (int64_t q = AP.ptr[r]; q < AP.ptr[r + 1]; ++q) {
            double v = -(o * AP.val[q]);
            if (p < p1 && P.col[p] == AP.col[q]) v += P.val[p++];
            qv[q] = v;
        }
        if (p != p1) *bad = 1;
    }
}

void build_q(Amg &h, cudaStream_t s) {
    const bool on = !(getenv("SPFD_Q") && std::string(getenv("SPFD_Q")) == "0");
    const int T = 256;
    for (size_t l = 0; l < h.lv.size(); ++l) {
        Level &L = h.lv[l];
        L.Q = Csr{};
        if (!on || L.AP.rows == 0 || L.P.rows != L.AP.rows) continue;
        Csr &Q = L.Q;
        Q.rows = L.AP.rows;
        Q.cols = L.AP.cols;
        Q.nnz = L.AP.nnz;
        Q.ptr.alloc(Q.rows + 1);
        Q.col.alloc(Q.nnz);
        Q.val.alloc(Q.nnz);
        SPFD_CUDA(cudaMemcpyAsync(Q.ptr.get(), L.AP.ptr.get(), (Q.rows + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
        SPFD_CUDA(cudaMemcpyAsync(Q.col.get(), L.AP.col.get(), Q.nnz * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
        DevBuf<int> bad;
        bad.alloc(1);
        SPFD_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(int), s));
        k_q_fill<<<grid_for(Q.rows, T), T, 0, s>>>(view(L.P), view(L.AP), L.odinv.get(), Q.val.get(), bad.get());
        SPFD_LAUNCH_CHECK();
        if (read1(bad.get(), s) != 0) { L.Q = Csr{}; continue; }
        L.q_group = L.ap_group;
        const std::string key = std::string("SPFD_GROUP_Q") + std::to_string(l);
        if (const char *e = getenv(key.c_str())) L.q_group = atoi(e);
    }
}

void build_rspan(Amg &h, cudaStream_t s) {
    const bool on = !(getenv("SPFD_RSPAN") && std::string(getenv("SPFD_RSPAN")) == "0");
    if (h.lv.empty()) return;
    Level &L0 = h.lv[0];
    L0.Rspan = Csr{};
    L0.Pspan = Csr{};
    if (!h.structured || h.lv.size() < 2 || L0.R_dof.rows == 0) return;
    const int T = 256;
    const int64_t n1 = h.lv[1].n;
    DevBuf<int32_t> perm;
    if (!h.l1_perm.empty()) {
        perm.alloc(n1);
        SPFD_CUDA(cudaMemcpyAsync(perm.get(), h.l1_perm.data(), n1 * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    }
    build_pspan(h, perm.n ? perm.get() : nullptr, s);
    if (!on) return;
    DevBuf<int64_t> len;
    len.alloc(n1 + 1);
    SPFD_CUDA(cudaMemsetAsync(len.get() + n1, 0, sizeof(int64_t), s));
    k_rspan_len<<<grid_for(n1, T), T, 0, s>>>(L0.R_dof.ptr.get(), perm.n ? perm.get() : nullptr, n1, len.get());
    SPFD_LAUNCH_CHECK();
    Csr &M = L0.Rspan;
    M.rows = n1;
    M.cols = L0.nvec;
    M.ptr.alloc(n1 + 1);
    scan_excl(len.get(), M.ptr.get(), n1 + 1, s);
    M.nnz = read1(M.ptr.get() + n1, s);
    M.col.alloc(M.nnz);
    M.val.alloc(M.nnz);
    k_rspan_fill<<<grid_for(n1, T), T, 0, s>>>(view(L0.R_dof), perm.n ? perm.get() : nullptr,
                                               h.op->dof_to_pos.get(), M.ptr.get(), n1, M.col.get(), M.val.get());
    SPFD_LAUNCH_CHECK();
    L0.rspan_group = pick_group(M.nnz, M.rows);
    if (const char *e = getenv("SPFD_GROUP_RSPAN")) L0.rspan_group = atoi(e);
}

static void morton_level1(Amg &h, cudaStream_t s) {
    const int T = 256;
    Level &L0 = h.lv[0], &L1 = h.lv[1];
    const Operator &op = *h.op;
    const int64_t n1 = L1.n;
    DevBuf<uint64_t> key, key2;
    DevBuf<int32_t> idx, P;
    key.alloc(n1); key2.alloc(n1); idx.alloc(n1); P.alloc(n1);
    k_root_keys<<<grid_for(n1, T), T, 0, s>>>(L0.mem_ptr.get(), L0.mem_pos.get(), n1, op.rows.get(), op.n_rows,
                                              (int)op.NY, key.get(), idx.get());
    SPFD_LAUNCH_CHECK();
    SPFD_CUDA(cudaMemsetAsync(P.get(), 0, n1 * sizeof(int32_t), s));  // (initcheck: CUB's stores are not tracked)
    size_t bytes = 0;
    SPFD_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, key.get(), key2.get(), idx.get(), P.get(), (int)n1, 0,
                                              64, s));
    DevBuf<uint8_t> tmp;
    tmp.alloc(bytes);
    SPFD_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), bytes, key.get(), key2.get(), idx.get(), P.get(), (int)n1, 0,
                                              64, s));
    level1_permute(h, P.get(), s);
}

// level-1 CSR in the reference numbering into caller buffers (exports)
static void export_level1(const Amg &h, const Csr &m, bool rows_perm, bool cols_perm, int64_t *ptr, int32_t *col,
                          double *val) {
    const auto &perm = h.l1_perm;  // current -> reference
    std::vector<int32_t> inv(perm.size());
    for (size_t g = 0; g < perm.size(); ++g) inv[perm[g]] = (int32_t)g;
    auto hp = d2h(m.ptr, m.rows + 1);
    auto hc = d2h(m.col, m.nnz);
    auto hv = d2h(m.val, m.nnz);
    std::vector<int64_t> np(m.rows + 1, 0);
    std::vector<int32_t> nc(m.nnz);
    std::vector<double> nv(m.nnz);
    for (int64_t o = 0; o < m.rows; ++o) {
        const int64_t r = rows_perm ? inv[o] : o;
        np[o + 1] = np[o] + (hp[r + 1] - hp[r]);
        for (int64_t q = hp[r], t = np[o]; q < hp[r + 1]; ++q, ++t) {
            nc[t] = cols_perm ? perm[hc[q]] : hc[q];
            nv[t] = hv[q];
        }
    }
    SPFD_CUDA(cudaMemcpy(ptr, np.data(), np.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
    if (m.nnz) {
        SPFD_CUDA(cudaMemcpy(col, nc.data(), nc.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
        SPFD_CUDA(cudaMemcpy(val, nv.data(), nv.size() * sizeof(double), cudaMemcpyHostToDevice));
    }
}

static void finish_level(Level &L, const Csr &A, double omega, cudaStream_t s) {
    const int T = 256;
    L.dinv.alloc(L.nvec);
    L.odinv.alloc(L.nvec + 4);
    DevBuf<int> bad;
    bad.alloc(1);
    SPFD_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(int), s));
    k_diag_dinv<<<grid_for(A.rows, T), T, 0, s>>>(view(A), omega, L.dinv.get(), L.odinv.get(), nullptr, bad.get());
    SPFD_LAUNCH_CHECK();
    SPFD_CHECK(read1(bad.get(), s) == 0, SPFD_ENOTPOS, "matrix has a non-positive diagonal entry");
}

static Amg *build(Amg *h, Csr &&A0, const spfd_config &cfg, cudaStream_t s) {
    const int T = 256;
    cudaEvent_t e0, e1;
    SPFD_CUDA(cudaEventCreate(&e0));
    SPFD_CUDA(cudaEventCreate(&e1));
    SPFD_CUDA(cudaEventRecord(e0, s));
    setup_mark("(setup start)", s);
    auto wall0 = std::chrono::steady_clock::now();
    h->omega = cfg.jacobi_damping;
    h->pre = cfg.pre_sweeps;
    h->post = cfg.post_sweeps;
    SPFD_CHECK(cfg.smoother == SPFD_SMOOTHER_JACOBI || cfg.smoother == SPFD_SMOOTHER_CHEBYSHEV, SPFD_EINVAL,
               "unknown smoother");
    SPFD_CHECK(cfg.cheb_degree >= 0 && cfg.cheb_degree <= 16, SPFD_EINVAL, "chebyshev degree must be in [1, 16]");
    h->smoother = cfg.smoother;
    h->cheb_deg = cfg.cheb_degree > 0 ? cfg.cheb_degree : 2;
    h->max_nrhs = cfg.max_nrhs < 1 ? 1 : (cfg.max_nrhs > 2 ? 2 : cfg.max_nrhs);
    int R = h->max_nrhs;

    std::vector<Csr> mats;
    mats.push_back(std::move(A0));
    h->lv.emplace_back();
    h->lv[0].n = mats[0].rows;
    h->lv[0].a_nnz = mats[0].nnz;
    int depth = 0;
    while (mats.back().rows > cfg.coarse_cap && (int)h->lv.size() < cfg.max_levels) {
        Csr Ac, P, Rm;
        DevBuf<int32_t> agg;
        double theta = cfg.strength_threshold * std::pow(0.5, depth);
        bool ok = coarsen(h->lv.back(), mats.back(), theta, h->omega, Ac, P, Rm, agg, s);
        h->lv.back().agg = std::move(agg);
        if (!ok) break;
        h->lv.back().P = std::move(P);
        h->lv.back().R = std::move(Rm);
        h->lv.emplace_back();
        h->lv.back().n = Ac.rows;
        h->lv.back().a_nnz = Ac.nnz;
        mats.push_back(std::move(Ac));
        ++depth;
    }
    int nl = (int)h->lv.size();
    setup_mark("levels built", s);
    // per-level solve data
    for (int l = 0; l < nl; ++l) {
        Level &L = h->lv[l];
        bool st0 = (l == 0 && h->structured);
        L.nvec = st0 ? h->op->L : L.n;
        if (st0) {
            // dinv / odinv in span layout from the operator's exact diagonal
            L.dinv.alloc(L.nvec);
            L.odinv.alloc(L.nvec + 4);
            SPFD_CUDA(cudaMemcpyAsync(L.dinv.get(), h->op->dinv.get(), L.nvec * sizeof(double),
                                      cudaMemcpyDeviceToDevice, s));
            // odinv = omega * dinv computed on the DOF CSR then mapped
            DevBuf<double> d1, d2;
            d1.alloc(L.n); d2.alloc(L.n);
            DevBuf<int> bad;
            bad.alloc(1);
            SPFD_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(int), s));
            k_diag_dinv<<<grid_for(L.n, T), T, 0, s>>>(view(mats[0]), h->omega, d1.get(), d2.get(), nullptr,
                                                        bad.get());
            k_dofs_to_span_1<<<grid_for(L.nvec, T), T, 0, s>>>(h->op->pos_to_dof.get(), L.nvec, d2.get(),
                                                               L.odinv.get());
            SPFD_LAUNCH_CHECK();
            if (l < nl - 1) {
                // matrix-free transfers: aggregate per span position and the
                // member lists of T^T (ascending positions); P/R kept in DOF
                // numbering only for export
                L.agg_pos.alloc(L.nvec + 4);
                k_agg_pos<<<grid_for(L.nvec, T), T, 0, s>>>(h->op->pos_to_dof.get(), L.nvec, L.agg.get(),
                                                            L.agg_pos.get());
                SPFD_LAUNCH_CHECK();
                build_members(L.agg.get(), L.n, h->lv[l + 1].n, h->op->dof_to_pos.get(), L.mem_ptr, L.mem_pos, s);
                L.P_dof = std::move(L.P);
                L.R_dof = std::move(L.R);
            }
        } else {
            finish_level(L, mats[l], h->omega, s);
            L.A = std::move(mats[l]);
        }
        if (l < nl - 1 && !(l == 0 && h->structured)) {
            L.p_group = pick_group(L.P.nnz, L.P.rows);
            L.r_group = pick_group(L.R.nnz, L.R.rows);
        }
        if (!(l == 0 && h->structured)) L.a_group = pick_group(L.A.nnz, L.A.rows);
        // tuning overrides: SPFD_GROUP_{A,P,R,AP}<level>=lanes
        auto over = [&](const char *kind, int &g) {
            const std::string key = std::string("SPFD_GROUP_") + kind + std::to_string(l);
            if (const char *e = getenv(key.c_str())) g = atoi(e);
        };
        over("A", L.a_group);
        over("P", L.p_group);
        over("R", L.r_group);
        // V(1,1) on a coarse level: z = x1 + od (d - (A P) e) with d the pre-smoothing
        // defect replaces "x1 = x0 + P e; z = x1 + od (r - A x1)" -- one pass over
        // P and A P (whose gathers hit the small coarse vector) instead of P and A
        static const bool use_ap = !(getenv("SPFD_AP") && std::string(getenv("SPFD_AP")) == "0");
        if (use_ap && l >= 1 && l < nl - 1 && h->pre == 1 && h->post == 1 && h->smoother == SPFD_SMOOTHER_JACOBI) {
            spgemm(view(L.A), view(L.P), L.P.cols, L.AP, false, s);
            // only where A P is no larger than A (C3: levels 2-3; on level 1
            // the product holds ~1.3x A's entries and measured no faster)
            if (L.AP.nnz > L.A.nnz) L.AP = Csr{};
            else L.ap_group = pick_group(L.AP.nnz, L.AP.rows);
            over("AP", L.ap_group);
        }
        L.vr.alloc(L.nvec * R);
        L.vx.alloc(L.nvec * R);
        L.vd.alloc(L.nvec * R);
        L.vt.alloc(L.nvec * R);
    }
    setup_mark("per-level solve data", s);
    // coarsest dense inverse
    {
        Level &C = h->lv[nl - 1];
        const Csr &Am = (nl - 1 == 0 && h->structured) ? mats[0] : C.A;
        h->nc = C.n;
        dense_inverse(Am, h->cinv, s);
        if (nl - 1 == 0 && h->structured) {
            // single-level structured hierarchy: keep the DOF CSR
        }
    }
    // solve layout: level 1 in Morton order of the aggregate roots (gathers of
    // neighbouring aggregates share cache lines); exports and the distributed
    // path see the reference numbering (export_level1, level1_unpermute)
    if (!(getenv("SPFD_MORTON") && std::string(getenv("SPFD_MORTON")) == "0") && h->structured && nl > 2)
        morton_level1(*h, s);
    build_rspan(*h, s);
    build_q(*h, s);
    setup_mark("dense inverse + Morton", s);
    alloc_krylov(*h, h->lv[0].nvec, R);
    setup_mark("workspace", s);
    if (h->smoother == SPFD_SMOOTHER_CHEBYSHEV) amg_estimate_lmax(*h, s);
    SPFD_CUDA(cudaEventRecord(e1, s));
    SPFD_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    SPFD_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    (void)wall0;
    h->setup_seconds = ms * 1e-3;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return h;
}

Amg *amg_setup_op(Operator *op, const spfd_config &cfg, cudaStream_t s) {
    auto *h = new Amg();
    try {
        h->op = op;
        h->structured = true;
        Csr A0;
        A0.alloc(op->n_dofs, op->n_dofs, op->nnz);
        op_csr(*op, A0.ptr.get(), A0.col.get(), A0.val.get(), s);
        return build(h, std::move(A0), cfg, s);
    } catch (...) {
        delete h;
        throw;
    }
}

__global__ void k_copy_sorted_rows(int64_t n, const int64_t *ptr, const int32_t *col, const double *val,
                                   int32_t *ocol, double *oval) {
    // insertion sort per row (input may be unsorted); rows are short
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x) {
        int64_t b = ptr[r], e = ptr[r + 1];
        for (int64_t q = b; q < e; ++q) { ocol[q] = col[q]; oval[q] = val[q]; }
        for (int64_t q = b + 1; q < e; ++q) {
            int32_t c = ocol[q];
            double v = oval[q];
            int64_t t = q - 1;
            while (t >= b && ocol[t] > c) { ocol[t + 1] = ocol[t]; oval[t + 1] = oval[t]; --t; }
            ocol[t + 1] = c;
            oval[t + 1] = v;
        }
    }
}

Amg *amg_setup_csr(int64_t n, int64_t nnz, const int64_t *ptr, const int32_t *col, const double *val,
                   const spfd_config &cfg, cudaStream_t s) {
    SPFD_CHECK(n >= 1, SPFD_EINVAL, "matrix must have at least one row");
    auto *h = new Amg();
    try {
        Csr A0;
        A0.alloc(n, n, nnz);
        SPFD_CUDA(cudaMemcpyAsync(A0.ptr.get(), ptr, (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
        k_copy_sorted_rows<<<grid_for(n, 256), 256, 0, s>>>(n, ptr, col, val, A0.col.get(), A0.val.get());
        SPFD_LAUNCH_CHECK();
        return build(h, std::move(A0), cfg, s);
    } catch (...) {
        delete h;
        throw;
    }
}

void amg_level_csr(Amg &h, int level, int which, int64_t *ptr, int32_t *col, double *val, cudaStream_t s) {
    SPFD_CHECK(level >= 0 && level < (int)h.lv.size(), SPFD_EINVAL, "level out of range");
    Level &L = h.lv[level];
    const Csr *m = nullptr;
    if (which == 0) {
        if (level == 0 && h.structured) {
            op_csr(*h.op, ptr, col, val, s);
            return;
        }
        m = &L.A;
    } else if (which == 1) {
        m = (level == 0 && h.structured) ? &L.P_dof : &L.P;
    } else if (which == 2) {
        m = (level == 0 && h.structured) ? &L.R_dof : &L.R;
    }
    SPFD_CHECK(m != nullptr && m->rows > 0, SPFD_EINVAL, "no such matrix on this level");
    if (level == 1 && !h.l1_perm.empty()) {  // solve layout is renumbered: export the reference order
        SPFD_CUDA(cudaStreamSynchronize(s));
        export_level1(h, *m, which != 2, which != 1, ptr, col, val);
        return;
    }
    SPFD_CUDA(cudaMemcpyAsync(ptr, m->ptr.get(), (m->rows + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
    if (m->nnz) {
        SPFD_CUDA(cudaMemcpyAsync(col, m->col.get(), m->nnz * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
        SPFD_CUDA(cudaMemcpyAsync(val, m->val.get(), m->nnz * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }
    SPFD_CUDA(cudaStreamSynchronize(s));
}

void amg_level_agg(Amg &h, int level, int32_t *agg, cudaStream_t s) {
    SPFD_CHECK(level >= 0 && level < (int)h.lv.size(), SPFD_EINVAL, "level out of range");
    Level &L = h.lv[level];
    SPFD_CHECK(L.agg.get() != nullptr && L.agg.n >= (size_t)L.n, SPFD_EINVAL, "no aggregates on this level");
    SPFD_CUDA(cudaMemcpyAsync(agg, L.agg.get(), L.n * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    SPFD_CUDA(cudaStreamSynchronize(s));
}

}  // namespace spfd

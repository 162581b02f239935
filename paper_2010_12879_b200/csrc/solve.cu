// V-cycle (linsolve.py:179-197), PCG and FGMRES(m) (linsolve.py:200-298)
// on device.  Level 0 is either the matrix-free stencil in the span layout
// or a CSR; coarse levels are CSR; the coarsest level applies the dense
// inverse.  All reductions are two-stage with a fixed order (per-CTA
// partials, then one CTA summing the partials in index order): repeated
// solves are bitwise identical (test_linsolve.py:157-166).
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <string>

#include <cub/cub.cuh>

#include "amg.cuh"
#include "comm.cuh"

namespace spfd {

namespace {

constexpr int kDotGrid = 148 * 4;
constexpr int kDotThreads = 256;

// device scalar slots (per rhs k)
enum {
    S_RHO = 0, S_PQ = 2, S_RR = 4, S_ALPHA = 6, S_BETA = 8, S_BB = 10, S_RZ = 12, S_ACTIVE = 14,
    S_TMP = 16, S_LOC = 20, S_H = 32,  // S_LOC: per-rank partial scalars; FGMRES Hessenberg column from S_H
    S_G = S_H + 256,                    // graph PCG: tol, max_iters, iteration, init flag, status
    S_G_TOL = S_G, S_G_MAXIT = S_G + 1, S_G_IT = S_G + 2, S_G_INIT = S_G + 3, S_G_STATUS = S_G + 4,
    S_G_DONE = S_G + 5,  // distributed PCG: iterations batched between host reads (pcg_dist)
    S_END = S_G + 8
};

__device__ __forceinline__ bool mbit(const uint32_t *m, int64_t p) { return (m[p >> 5] >> (p & 31)) & 1u; }

__device__ __forceinline__ int spos(const int4 *rows, int r, int i) {
    int4 q = rows[r];
    return (i >= q.y && i < q.z) ? q.x + (i - q.y) : -1;
}

__device__ __forceinline__ int frow(const int4 *rows, int r0, int r1, int p) {
    int lo = r0, hi = r1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (rows[mid].x <= p) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// R-wide vector element (R = 1: double, R = 2: double2 real/imag pair)
template <int R> struct V;
template <> struct V<1> {
    using T = double;
    static __device__ __forceinline__ T ld(const double *p, int64_t i) { return p[i]; }
    static __device__ __forceinline__ void st(double *p, int64_t i, T v) { p[i] = v; }
    static __device__ __forceinline__ T zero() { return 0.0; }
    static __device__ __forceinline__ T axpy(double a, T x, T y) { return add_rn(y, mul_rn(a, x)); }  // exact y + a*x
    static __device__ __forceinline__ T fma_(double a, T x, T y) { return fma(a, x, y); }
    static __device__ __forceinline__ T sub(T a, T b) { return a - b; }
    static __device__ __forceinline__ T add(T a, T b) { return a + b; }
    static __device__ __forceinline__ T scale(double a, T x) { return a * x; }
    static __device__ __forceinline__ double dot(T a, T b, int) { return a * b; }
    static __device__ __forceinline__ double comp(T a, int) { return a; }
};
template <> struct V<2> {
    using T = double2;
    static __device__ __forceinline__ T ld(const double *p, int64_t i) { return reinterpret_cast<const double2 *>(p)[i]; }
    static __device__ __forceinline__ void st(double *p, int64_t i, T v) { reinterpret_cast<double2 *>(p)[i] = v; }
    static __device__ __forceinline__ T zero() { return make_double2(0.0, 0.0); }
    static __device__ __forceinline__ T axpy(double a, T x, T y) {
        return make_double2(add_rn(y.x, mul_rn(a, x.x)), add_rn(y.y, mul_rn(a, x.y)));
    }
    static __device__ __forceinline__ T fma_(double a, T x, T y) { return make_double2(fma(a, x.x, y.x), fma(a, x.y, y.y)); }
    static __device__ __forceinline__ T sub(T a, T b) { return make_double2(a.x - b.x, a.y - b.y); }
    static __device__ __forceinline__ T add(T a, T b) { return make_double2(a.x + b.x, a.y + b.y); }
    static __device__ __forceinline__ T scale(double a, T x) { return make_double2(a * x.x, a * x.y); }
    static __device__ __forceinline__ double dot(T a, T b, int c) { return c == 0 ? a.x * b.x : a.y * b.y; }
    static __device__ __forceinline__ double comp(T a, int c) { return c == 0 ? a.x : a.y; }
};

// Neighbourhood of one span position: the 6 edge weights and the positions
// of the 6 neighbours (-1 outside the conductive spans).
struct Nbr {
    double wxp, wyp, wzp, wxm, wym, wzm, diag;
    int pxm, pym, pzm, pxp, pyp, pzp;
};

__device__ __forceinline__ Nbr neighbours(const SpanView &v, int p, int r, int4 q) {
    Nbr n;
    const int i = q.y + (p - q.x), j = q.w;
    n.wxp = v.wx[p]; n.wyp = v.wy[p]; n.wzp = v.wz[p];
    n.wxm = 0.0; n.wym = 0.0; n.wzm = 0.0;
    n.pxm = (i > q.y) ? p - 1 : -1;
    n.pxp = (i + 1 < q.z) ? p + 1 : -1;
    n.pym = (j > 0) ? spos(v.rows, r - 1, i) : -1;
    n.pyp = (j + 1 < v.NY) ? spos(v.rows, r + 1, i) : -1;
    n.pzm = (r >= v.NY) ? spos(v.rows, r - v.NY, i) : -1;
    n.pzp = (r + v.NY < v.n_rows) ? spos(v.rows, r + v.NY, i) : -1;
    if (n.pxm >= 0) n.wxm = v.wx[n.pxm];
    if (n.pym >= 0) n.wym = v.wy[n.pym];
    if (n.pzm >= 0) n.wzm = v.wz[n.pzm];
    // reference diagonal order: tail edges x, y, z then head edges x, y, z
    n.diag = add_rn(add_rn(add_rn(add_rn(add_rn(n.wxp, n.wyp), n.wzp), n.wxm), n.wym), n.wzm);
    return n;
}

// (A x)_p in the reference's sorted-column order; X(pos) -> V<R>::T gives
// the neighbour inputs, xc is the centre input (loaded once by the caller).
template <int R, class X>
__device__ __forceinline__ typename V<R>::T apply_row(const Nbr &n, typename V<R>::T xc, X xat) {
    using W = V<R>;
    typename W::T s = W::zero();
    if (n.pzm >= 0) s = W::axpy(-n.wzm, xat(n.pzm), s);
    if (n.pym >= 0) s = W::axpy(-n.wym, xat(n.pym), s);
    if (n.pxm >= 0) s = W::axpy(-n.wxm, xat(n.pxm), s);
    s = W::axpy(n.diag, xc, s);
    if (n.pxp >= 0) s = W::axpy(-n.wxp, xat(n.pxp), s);
    if (n.pyp >= 0) s = W::axpy(-n.wyp, xat(n.pyp), s);
    if (n.pzp >= 0) s = W::axpy(-n.wzp, xat(n.pzp), s);
    return s;
}

struct SpanArgs {
    const double *x;      // input vector (modes 0, 1, 3)
    const double *r;      // right-hand side / residual
    const double *od;     // omega * D^-1 (span)
    const double *base;   // mode 4: materialised smoother iterate (or null -> od*r)
    const double *ec;     // mode 4: coarse correction (level-1 vector)
    const int32_t *aggp;  // mode 4: aggregate of each position (-1 = none)
    double *y;            // output
    double *partials;     // per-CTA dot partials
    int64_t pb = 0;       // owned position range [pb, pe) (z-slab); defaults = all
    int64_t pe = INT64_MAX;
    int tile0 = 0;        // first tile of the launch (set by launch_fine)
    int pf_ahead = 0;     // PF: also prefetch the tile this many tiles ahead (0 = own tile only)
    int rev = 0;          // walk the tiles from the high end (L2 reuse of the previous pass's tail)
};

// Input of a fine-level stencil at a position, per mode (see k_span).
template <int R, int MODE>
__device__ __forceinline__ typename V<R>::T xin(const SpanArgs &a, int pp) {
    using W = V<R>;
    if (MODE == 2) return W::scale(a.od[pp], W::ld(a.r, pp));
    if (MODE == 4) {
        int g1 = a.aggp[pp];  // aggregate id + 1, 0 = none
        return g1 > 0 ? W::ld(a.ec, g1 - 1) : W::zero();
    }
    return W::ld(a.x, pp);
}

// Output of one fine-level stencil point for MODE (see k_span), in the
// reference's summation order (shared by every fine kernel: same bits).
template <int R, int MODE>
__device__ __forceinline__ typename V<R>::T point_out(const SpanArgs &a, const Nbr &n, int p,
                                                      typename V<R>::T &dotv) {
    using W = V<R>;
    using T = typename W::T;
    T out;
    if (MODE == 2) {
        const double *od = a.od, *rr = a.r;
        const T rc = W::ld(rr, p);
        T s = apply_row<R>(n, W::scale(od[p], rc), [&](int pp) { return W::scale(od[pp], W::ld(rr, pp)); });
        out = W::sub(rc, s);
    } else if (MODE == 4) {
        const double *ec = a.ec;
        const int32_t *ag = a.aggp;
        auto eat = [&](int pp) {
            int g1 = ag[pp];  // aggregate id + 1, 0 = none
            return g1 > 0 ? W::ld(ec, g1 - 1) : W::zero();
        };
        const T ecc = eat(p);
        const double odc = a.od[p];
        T s = apply_row<R>(n, ecc, eat);
        T b = a.base ? W::ld(a.base, p) : W::scale(odc, W::ld(a.r, p));
        out = W::sub(W::add(b, ecc), W::scale(odc, s));
    } else {
        const double *xx = a.x;
        const T xc = W::ld(xx, p);
        T s = apply_row<R>(n, xc, [&](int pp) { return W::ld(xx, pp); });
        if (MODE == 0) {
            out = s;
            dotv = xc;
        } else if (MODE == 1) {
            out = W::sub(W::ld(a.r, p), s);
        } else {
            const T rc = W::ld(a.r, p);
            out = W::add(xc, W::scale(a.od[p], W::sub(rc, s)));
            dotv = rc;
        }
    }
    return out;
}

// MODE 0: y = A x (+ partial x.y)
// MODE 1: y = r - A x (+ partial y.y)
// MODE 2: y = r - A (od r)            (implicit first Jacobi sweep + defect)
// MODE 3: y = x + od (r - A x) (+ partial r.y)   (Jacobi sweep)
// MODE 4: y = base + e - od (A e), e = T ec      (matrix-free prolongation
//         with P = (I - omega D^-1 A) T; base = od r when null)
// Bulk L2 prefetch (TMA engine, no registers) of the byte range
// [p0, p1) * esz of a streamed array; 16-byte granules.
__device__ __forceinline__ void l2_prefetch(const void *base, int64_t p0, int64_t p1, int esz) {
    if (!base || p1 <= p0) return;
    uintptr_t b = reinterpret_cast<uintptr_t>(base) + (uintptr_t)(p0 * esz);
    uintptr_t e = reinterpret_cast<uintptr_t>(base) + (uintptr_t)(p1 * esz);
    b = (b + 15) & ~(uintptr_t)15;
    e &= ~(uintptr_t)15;
    if (e <= b) return;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(b), "r"((unsigned)(e - b)) : "memory");
}

// One thread of the CTA queues the tile's streamed (center-position) arrays
// into L2, so the per-position dependent load chains below hit L2 instead
// of waiting on DRAM (PF = true).
template <int R, int MODE>
__device__ __forceinline__ void tile_prefetch(const SpanView &v, const SpanArgs &a, int64_t p0, int64_t p1) {
    l2_prefetch(v.wx, p0, p1, 8);
    l2_prefetch(v.wy, p0, p1, 8);
    l2_prefetch(v.wz, p0, p1, 8);
    if (MODE == 0 || MODE == 1 || MODE == 3) l2_prefetch(a.x, p0, p1, 8 * R);
    if (MODE != 0) l2_prefetch(a.r, p0, p1, 8 * R);
    if (MODE >= 2) l2_prefetch(a.od, p0, p1, 8);
    if (MODE == 4) { l2_prefetch(a.aggp, p0, p1, 4); l2_prefetch(a.base, p0, p1, 8 * R); }
}

// One tile of a fine-level stencil pass: positions [t * kTile, +kTile) that
// lie in [pb, pend); accumulates the thread's dot contribution.
template <int R, int MODE, bool DOT, bool RANGED>
__device__ __forceinline__ void span_tile(const SpanView &v, const SpanArgs &a, int t, int64_t pend,
                                          double (&dot)[R]) {
    using W = V<R>;
    using T = typename W::T;
    const int r0 = v.tile_row[t], r1 = v.tile_row[t + 1];
    int row = r0;
    for (int u = 0; u < kTile / kSpanThreads; ++u) {
        const int p = t * kTile + u * kSpanThreads + threadIdx.x;
        if (p >= pend || (RANGED && p < a.pb)) continue;  // no divergent loop exit before block_sum
        row = frow(v.rows, row, r1, p);
        const int4 q = v.rows[row];
        const Nbr n = neighbours(v, p, row, q);
        const bool dof = mbit(v.mask, p);
        T dotv = W::zero();
        T out = point_out<R, MODE>(a, n, p, dotv);
        if (!dof) out = W::zero();
        W::st(a.y, p, out);
        if (DOT) {
#pragma unroll
            for (int c = 0; c < R; ++c) {
                if (MODE == 0 || MODE == 3) dot[c] += W::dot(dotv, out, c);
                else dot[c] += W::dot(out, out, c);
            }
        }
    }
}

#ifndef SPFD_SPAN_MINB
#define SPFD_SPAN_MINB 6
#endif
// the SpMV + dot instance spills 8 bytes at 6 CTAs per SM; 5 is spill-free
// but measured 2% slower at C3 (125.4 vs 122.5 us), so both stay at 6
#ifndef SPFD_SPMV_MINB
#define SPFD_SPMV_MINB 6
#endif
template <int R, int MODE, bool DOT, bool RANGED = false, bool PF = false, int MINB = SPFD_SPAN_MINB>
__global__ void __launch_bounds__(kSpanThreads, MINB) k_span(SpanView v, SpanArgs a) {
    __shared__ double red[32 * R];
    // blk: the tile's index within the launch (CTAs run in blockIdx order;
    // rev walks the tiles from the high end).  Dot partials are stored by
    // blk, so the reduction order does not depend on the direction.
    const int blk = a.rev ? (int)gridDim.x - 1 - (int)blockIdx.x : (int)blockIdx.x;
    const int t = RANGED ? a.tile0 + blk : blk;
    const int64_t pend = RANGED ? (a.pe < v.L ? a.pe : v.L) : v.L;
    if (PF && threadIdx.x == 0) {
        if (a.pf_ahead <= 0 || blockIdx.x < a.pf_ahead) {  // first wave: its own tile
            const int64_t q0 = (int64_t)t * kTile, q1 = q0 + kTile < pend ? q0 + kTile : pend;
            tile_prefetch<R, MODE>(v, a, q0, q1);
        }
        if (a.pf_ahead > 0) {  // later CTAs find their tile queued by an earlier one
            const int ta = a.rev ? t - a.pf_ahead : t + a.pf_ahead;
            const int64_t q0 = (int64_t)ta * kTile, q1 = q0 + kTile < pend ? q0 + kTile : pend;
            if (ta >= 0) tile_prefetch<R, MODE>(v, a, q0, q1);
        }
    }
    if (PF) __syncwarp();  // warp 0 reconverges after thread 0's prefetch (synccheck)
    double dot[R];
#pragma unroll
    for (int c = 0; c < R; ++c) dot[c] = 0.0;
    span_tile<R, MODE, DOT, RANGED>(v, a, t, pend, dot);
    if (DOT) {
        block_sum<R>(dot, red);
        if (threadIdx.x == 0)
#pragma unroll
            for (int c = 0; c < R; ++c) a.partials[blk * R + c] = dot[c];
    }
}

// Restriction r_c = T^T u: sequential sum over each aggregate's member
// positions (ascending) -- deterministic, no atomics.  Optionally also
// writes x0_c = od_c * r_c, the next level's implicit first Jacobi sweep.
template <int R>
__global__ void k_agg_sum(const int64_t *mptr, const int32_t *mpos, int64_t n_agg, const double *u, double *rc,
                          const double *od_c, double *x0_c, int rev) {
    using W = V<R>;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_agg; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t g = rev ? n_agg - 1 - i : i;
        typename W::T s = W::zero();
        const int64_t q1 = mptr[g + 1];
        // 4 members in flight; the sum keeps the ascending member order
        for (int64_t q = mptr[g]; q < q1; q += 4) {
            int pp[4];
            typename W::T uv[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) pp[k] = q + k < q1 ? mpos[q + k] : -1;
#pragma unroll
            for (int k = 0; k < 4; ++k) uv[k] = pp[k] >= 0 ? W::ld(u, pp[k]) : W::zero();
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (pp[k] >= 0) s = W::add(s, uv[k]);
        }
        W::st(rc, g, s);
        if (x0_c) W::st(x0_c, g, W::scale(od_c[g], s));
    }
}

// ---- CSR kernels (G lanes per row) ------------------------------------
// MODE 0: y = M x (aux: also od_aux * y);  1: y = r - M x;  2: y = r - M(odinv r);
// MODE 3: y = x + odinv (r - M x);  4: y = odinv r + M e (prolongation, x=e)
// MODE 5: y = base + M e (prolongation on a materialised smoother iterate)
// MODE 6: y = odinv (r + base) + M e (coarse prolongation + post-smooth through Q, build_q)
// L2 bulk prefetch of the column/value ranges of rows [row, row + n) (the
// warp's next rows in the grid-stride loop).
__device__ __forceinline__ void csr_prefetch(const CsrView &m, int64_t row, int n) {
    if (row >= m.rows) return;
    const int64_t e = row + n < m.rows ? row + n : m.rows;
    const int64_t q0 = m.ptr[row], q1 = m.ptr[e];
    l2_prefetch(m.col, q0, q1, 4);
    l2_prefetch(m.val, q0, q1, 8);
}

// Row epilogue of the CSR kernels: reduce the G lanes' partial sums with a
// fixed xor tree (all lanes take part), then the row leader (`lead`) applies
// MODE to global row gr:
//   0: y = sum (+ aux = od_aux y)   1/2: y = r - sum   3: y = x + od (r - sum)
//   4: y = od r + sum   5: y = base + sum   6: y = od (r + base) + sum
template <int G, int R, int MODE, bool DOT>
__device__ __forceinline__ void csr_row_out(typename V<R>::T acc, bool lead, int64_t gr, const double *__restrict__ x,
                                            const double *__restrict__ r, const double *__restrict__ od,
                                            const double *__restrict__ base, double *__restrict__ y,
                                            const double *__restrict__ od_aux, double *__restrict__ aux,
                                            double (&dot)[R]) {
    using W = V<R>;
    using T = typename W::T;
    double ac[R];
#pragma unroll
    for (int c = 0; c < R; ++c) {
        ac[c] = W::comp(acc, c);
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) ac[c] += __shfl_xor_sync(0xffffffffu, ac[c], o, G);
    }
    if (!lead) return;
    T sum;
    if constexpr (R == 1) sum = ac[0];
    else sum = make_double2(ac[0], ac[1]);
    T out;
    if (MODE == 0) out = sum;
    else if (MODE == 1 || MODE == 2) out = W::sub(W::ld(r, gr), sum);
    else if (MODE == 3) out = W::add(W::ld(x, gr), W::scale(od[gr], W::sub(W::ld(r, gr), sum)));
    else if (MODE == 4) out = W::add(W::scale(od[gr], W::ld(r, gr)), sum);
    else if (MODE == 6) out = W::add(W::scale(od[gr], W::add(W::ld(r, gr), W::ld(base, gr))), sum);
    else out = W::add(W::ld(base, gr), sum);
    W::st(y, gr, out);
    if (MODE == 0 && aux) W::st(aux, gr, W::scale(od_aux[gr], out));
    if (DOT) {
#pragma unroll
        for (int c = 0; c < R; ++c) {
            if (MODE == 0) dot[c] += W::dot(W::ld(x, gr), out, c);
            else if (MODE == 3) dot[c] += W::dot(W::ld(r, gr), out, c);
            else dot[c] += W::dot(out, out, c);
        }
    }
}

#ifndef SPFD_CSR_UNROLL_WIDE
#define SPFD_CSR_UNROLL_WIDE 4  // entries in flight per lane for groups of >= 8 lanes (8: C3 33.1 vs 32.9 ms)
#endif

template <int G, int R, int MODE, bool DOT>
__global__ void k_csr(CsrView m, const double *__restrict__ x, const double *__restrict__ r,
                      const double *__restrict__ od, const double *__restrict__ base, double *__restrict__ y,
                      double *__restrict__ partials, const double *__restrict__ od_aux, double *__restrict__ aux,
                      const int32_t *__restrict__ rowmap, int pf) {
    using W = V<R>;
    using T = typename W::T;
    __shared__ double red[32 * R];
    const int lane = threadIdx.x % G;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
    constexpr int GPW = 32 / G;  // row groups per warp
    double dot[R];
#pragma unroll
    for (int c = 0; c < R; ++c) dot[c] = 0.0;
    // warp-uniform trip count so the full-mask shuffles below are safe
    for (int64_t rbase = warp * GPW; rbase < m.rows; rbase += nwarp * GPW) {
        if (pf && (threadIdx.x & 31) == 0) csr_prefetch(m, rbase + nwarp * GPW, GPW);
        const int64_t row = rbase + (threadIdx.x & 31) / G;
        const bool valid = row < m.rows;
        T acc = W::zero();
        if (valid) {
            // U entries per lane in flight (all loads issued before the FMAs,
            // which keep the sequential per-lane order)
            constexpr int U = G >= 8 ? SPFD_CSR_UNROLL_WIDE : 4;
            const int64_t q1 = m.ptr[row + 1];
            for (int64_t q = m.ptr[row] + lane; q < q1; q += U * G) {
                int col[U];
                double a[U];
                T xv[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const bool in = q + u * G < q1;
                    col[u] = in ? m.col[q + u * G] : -1;
                    a[u] = in ? m.val[q + u * G] : 0.0;
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (col[u] >= 0) xv[u] = MODE == 2 ? W::scale(od[col[u]], W::ld(r, col[u])) : W::ld(x, col[u]);
                    else xv[u] = W::zero();
                }
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (col[u] >= 0) acc = W::fma_(a[u], xv[u], acc);
            }
        }
        csr_row_out<G, R, MODE, DOT>(acc, valid && lane == 0, (valid && rowmap) ? (int64_t)rowmap[row] : row, x, r, od, base, y,
                                     od_aux, aux, dot);
    }
    if (DOT) {
        block_sum<R>(dot, red);
        if (threadIdx.x == 0)
#pragma unroll
            for (int c = 0; c < R; ++c) partials[blockIdx.x * R + c] = dot[c];
    }
}

constexpr int kCsrThreads = 256;

// Fused coarse-level prolongation + post-smooth (V(1,1)):
//   x1 = od r + P e,   z = x1 + od (d - (A P) e)
// with d = r - A (od r) the pre-smoothing defect.  Equal to the two-pass
// "x1 = x0 + P e; z = x1 + od (r - A x1)" up to rounding (A x1 = A x0 +
// (A P) e); the gathers of both rows hit the small coarse vector e.
template <int G, int R>
__global__ void __launch_bounds__(kCsrThreads) k_csr_pp(CsrView P, CsrView M, const double *__restrict__ e,
                                                       const double *__restrict__ r, const double *__restrict__ od,
                                                       const double *__restrict__ d, double *__restrict__ z, int pf) {
    using W = V<R>;
    using T = typename W::T;
    const int lane = threadIdx.x % G;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
    constexpr int GPW = 32 / G;
    for (int64_t rbase = warp * GPW; rbase < P.rows; rbase += nwarp * GPW) {
        if (pf && (threadIdx.x & 31) == 0) {
            csr_prefetch(P, rbase + nwarp * GPW, GPW);
            csr_prefetch(M, rbase + nwarp * GPW, GPW);
        }
        const int64_t row = rbase + (threadIdx.x & 31) / G;
        const bool valid = row < P.rows;
        T ap = W::zero(), am = W::zero();
        if (valid) {
            const int64_t p1 = P.ptr[row + 1], m1 = M.ptr[row + 1];
            for (int64_t q = P.ptr[row] + lane; q < p1; q += G) ap = W::fma_(P.val[q], W::ld(e, P.col[q]), ap);
            constexpr int U = 4;
            for (int64_t q = M.ptr[row] + lane; q < m1; q += U * G) {
                int col[U];
                double a[U];
                T xv[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const bool in = q + u * G < m1;
                    col[u] = in ? M.col[q + u * G] : -1;
                    a[u] = in ? M.val[q + u * G] : 0.0;
                }
#pragma unroll
                for (int u = 0; u < U; ++u) xv[u] = col[u] >= 0 ? W::ld(e, col[u]) : W::zero();
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (col[u] >= 0) am = W::fma_(a[u], xv[u], am);
            }
        }
        double sp[R], sm[R];
#pragma unroll
        for (int c = 0; c < R; ++c) {
            sp[c] = W::comp(ap, c);
            sm[c] = W::comp(am, c);
#pragma unroll
            for (int o = G / 2; o > 0; o >>= 1) {
                sp[c] += __shfl_xor_sync(0xffffffffu, sp[c], o, G);
                sm[c] += __shfl_xor_sync(0xffffffffu, sm[c], o, G);
            }
        }
        if (valid && lane == 0) {
            T pe, me;
            if constexpr (R == 1) { pe = sp[0]; me = sm[0]; }
            else { pe = make_double2(sp[0], sp[1]); me = make_double2(sm[0], sm[1]); }
            const double o = od[row];
            const T x1 = W::add(W::scale(o, W::ld(r, row)), pe);
            W::st(z, row, W::add(x1, W::scale(o, W::sub(W::ld(d, row), me))));
        }
    }
}

// Wide rows (small coarse levels: a few thousand rows of several hundred
// entries): G = 64 / 128 / 256 lanes of one CTA per row.  Each warp reduces
// its lanes with a fixed xor tree, the row's leader adds the warp partials
// in warp order -- deterministic.  Same MODEs as k_csr.
template <int G, int R, int MODE, bool DOT>
__global__ void __launch_bounds__(kCsrThreads) k_csr_wide(CsrView m, const double *__restrict__ x,
                                                         const double *__restrict__ r, const double *__restrict__ od,
                                                         const double *__restrict__ base, double *__restrict__ y,
                                                         double *__restrict__ partials,
                                                         const double *__restrict__ od_aux, double *__restrict__ aux,
                                                         const int32_t *__restrict__ rowmap) {
    static_assert(G >= 64 && G <= kCsrThreads, "wide rows only");
    using W = V<R>;
    using T = typename W::T;
    constexpr int RPB = kCsrThreads / G, WPR = G / 32;
    __shared__ double wp[kCsrThreads / 32][R];
    __shared__ double red[32 * R];
    const int li = threadIdx.x % G, rr = threadIdx.x / G, wid = threadIdx.x >> 5;
    double dot[R];
#pragma unroll
    for (int c = 0; c < R; ++c) dot[c] = 0.0;
    const int64_t iters = (m.rows + (int64_t)gridDim.x * RPB - 1) / ((int64_t)gridDim.x * RPB);
    for (int64_t itr = 0; itr < iters; ++itr) {
        const int64_t row = (itr * gridDim.x + blockIdx.x) * RPB + rr;
        const bool valid = row < m.rows;
        T acc = W::zero();
        if (valid) {
            constexpr int U = 4;
            const int64_t q1 = m.ptr[row + 1];
            for (int64_t q = m.ptr[row] + li; q < q1; q += U * G) {
                int col[U];
                double a[U];
                T xv[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const bool in = q + u * G < q1;
                    col[u] = in ? m.col[q + u * G] : -1;
                    a[u] = in ? m.val[q + u * G] : 0.0;
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (col[u] >= 0) xv[u] = MODE == 2 ? W::scale(od[col[u]], W::ld(r, col[u])) : W::ld(x, col[u]);
                    else xv[u] = W::zero();
                }
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (col[u] >= 0) acc = W::fma_(a[u], xv[u], acc);
            }
        }
#pragma unroll
        for (int c = 0; c < R; ++c) {
            double v = W::comp(acc, c);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if ((threadIdx.x & 31) == 0) wp[wid][c] = v;
        }
        __syncthreads();
        if (valid && li == 0) {
            double ac[R];
#pragma unroll
            for (int c = 0; c < R; ++c) {
                ac[c] = 0.0;
                for (int k = 0; k < WPR; ++k) ac[c] += wp[rr * WPR + k][c];
            }
            const int64_t gr = rowmap ? (int64_t)rowmap[row] : row;
            T sum;
            if constexpr (R == 1) sum = ac[0];
            else sum = make_double2(ac[0], ac[1]);
            T out;
            if (MODE == 0) out = sum;
            else if (MODE == 1 || MODE == 2) out = W::sub(W::ld(r, gr), sum);
            else if (MODE == 3) out = W::add(W::ld(x, gr), W::scale(od[gr], W::sub(W::ld(r, gr), sum)));
            else if (MODE == 4) out = W::add(W::scale(od[gr], W::ld(r, gr)), sum);
            else if (MODE == 6) out = W::add(W::scale(od[gr], W::add(W::ld(r, gr), W::ld(base, gr))), sum);
            else out = W::add(W::ld(base, gr), sum);
            W::st(y, gr, out);
            if (MODE == 0 && aux) W::st(aux, gr, W::scale(od_aux[gr], out));
            if (DOT) {
#pragma unroll
                for (int c = 0; c < R; ++c) {
                    if (MODE == 0) dot[c] += W::dot(W::ld(x, gr), out, c);
                    else if (MODE == 3) dot[c] += W::dot(W::ld(r, gr), out, c);
                    else dot[c] += W::dot(out, out, c);
                }
            }
        }
        __syncthreads();
    }
    if (DOT) {
        block_sum<R>(dot, red);
        if (threadIdx.x == 0)
#pragma unroll
            for (int c = 0; c < R; ++c) partials[blockIdx.x * R + c] = dot[c];
    }
}

// SPFD_CSR_PF=1: L2 bulk prefetch of the next rows in the CSR kernels (A/B)
inline int csr_prefetch_enabled() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("SPFD_CSR_PF");
        v = (e && std::string(e) == "1") ? 1 : 0;
    }
    return v;
}

// CTAs per SM the grid-stride CSR launches are capped at (SPFD_CSR_GRID_PER_SM,
// default 8 = one resident wave of 256-thread CTAs: C3 32.91 vs 33.00 ms at
// 16, 33.2 at 32, 37.6 at 4; launches writing dot partials keep 16, the
// partials buffer's size).  Rows do not depend on the grid: same bits.
inline int csr_grid_per_sm() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("SPFD_CSR_GRID_PER_SM");
        v = e ? std::max(1, std::min(64, atoi(e))) : 8;
    }
    return v;
}

inline int csr_grid(int64_t rows, int G, int per_sm = 16) {
    int64_t groups = G >= kCsrThreads ? 1 : (int64_t)kCsrThreads / G;
    int64_t g = (rows + groups - 1) / groups;
    if (g < 1) g = 1;
    if (g > 148 * per_sm) g = 148 * per_sm;
    return (int)g;
}

template <int G, int R, int MODE, bool DOT>
void launch_csr_g(const Csr &m, const double *x, const double *r, const double *od, const double *base, double *y,
                  double *partials, cudaStream_t s, int grid, const double *od_aux, double *aux,
                  const int32_t *rowmap) {
    if constexpr (G > 32)
        k_csr_wide<G, R, MODE, DOT><<<grid, kCsrThreads, 0, s>>>(view(m), x, r, od, base, y, partials, od_aux, aux,
                                                                 rowmap);
    else
        k_csr<G, R, MODE, DOT><<<grid, kCsrThreads, 0, s>>>(view(m), x, r, od, base, y, partials, od_aux, aux, rowmap,
                                                            csr_prefetch_enabled());
}

template <int R, int MODE, bool DOT>
int launch_csr(const Csr &m, int G, const double *x, const double *r, const double *od, const double *base,
               double *y, double *partials, cudaStream_t s, const double *od_aux = nullptr, double *aux = nullptr,
               const int32_t *rowmap = nullptr) {
    int grid = csr_grid(m.rows, G, DOT ? 16 : csr_grid_per_sm());
    switch (G) {
        case 1: launch_csr_g<1, R, MODE, DOT>(m, x, r, od, base, y, partials, s, grid, od_aux, aux, rowmap); break;
        case 2: launch_csr_g<2, R, MODE, DOT>(m, x, r, od, base, y, partials, s, grid, od_aux, aux, rowmap); break;
        case 4: launch_csr_g<4, R, MODE, DOT>(m, x, r, od, base, y, partials, s, grid, od_aux, aux, rowmap); break;
        case 8: launch_csr_g<8, R, MODE, DOT>(m, x, r, od, base, y, partials, s, grid, od_aux, aux, rowmap); break;
        case 16: launch_csr_g<16, R, MODE, DOT>(m, x, r, od, base, y, partials, s, grid, od_aux, aux, rowmap); break;
        case 64: launch_csr_g<64, R, MODE, DOT>(m, x, r, od, base, y, partials, s, grid, od_aux, aux, rowmap); break;
        case 128: launch_csr_g<128, R, MODE, DOT>(m, x, r, od, base, y, partials, s, grid, od_aux, aux, rowmap); break;
        case 256: launch_csr_g<256, R, MODE, DOT>(m, x, r, od, base, y, partials, s, grid, od_aux, aux, rowmap); break;
        default: launch_csr_g<32, R, MODE, DOT>(m, x, r, od, base, y, partials, s, grid, od_aux, aux, rowmap); break;
    }
    SPFD_LAUNCH_CHECK();
    return grid;
}

// dense coarsest solve z = Cinv r (one warp per row)
template <int R>
__global__ void k_dense_mv(const double *cinv, int64_t n, const double *r, double *z) {
    int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    for (int64_t row = warp; row < n; row += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        double acc[R];
#pragma unroll
        for (int c = 0; c < R; ++c) acc[c] = 0.0;
        for (int64_t j = lane; j < n; j += 32) {
            double a = cinv[row * n + j];
#pragma unroll
            for (int c = 0; c < R; ++c) acc[c] = fma(a, r[j * R + c], acc[c]);
        }
#pragma unroll
        for (int c = 0; c < R; ++c)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], o);
        if (lane == 0)
#pragma unroll
            for (int c = 0; c < R; ++c) z[row * R + c] = acc[c];
    }
}

template <int R>
__global__ void k_span_gather(const int32_t *dof_to_pos, int64_t n, const double *span, double *out) {
    for (int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; d < n; d += (int64_t)gridDim.x * blockDim.x)
#pragma unroll
        for (int c = 0; c < R; ++c) out[d * R + c] = span[(int64_t)dof_to_pos[d] * R + c];
}
template <int R>
__global__ void k_span_scatter(const int32_t *pos_to_dof, int64_t L, const double *in, double *span) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < L; p += (int64_t)gridDim.x * blockDim.x) {
        int d = pos_to_dof[p];
#pragma unroll
        for (int c = 0; c < R; ++c) span[p * R + c] = d >= 0 ? in[(int64_t)d * R + c] : 0.0;
    }
}

// ---- matrix-free cell Laplacian (divergence cleaning, level 0) ----------
// div div^T on an nx x ny x nz box of cells: 6 on the diagonal, -1 per face
// shared with a neighbour cell (field.cu k_normal_fill), applied in the CSR's
// column order (z-, y-, x-, centre, x+, y+, z+).  Same MODEs as k_csr
// (0: y = A x (+ x.y), 1: y = r - A x (+ y.y), 2: y = r - A(od r),
// 3: y = x + od (r - A x) (+ r.y)); od is the constant omega / 6.
template <int R, int MODE, bool DOT>
__global__ void __launch_bounds__(256) k_box(int nx, int ny, int nz, double od, const double *__restrict__ x,
                                             const double *__restrict__ r, double *__restrict__ y,
                                             double *__restrict__ partials) {
    using W = V<R>;
    using T = typename W::T;
    __shared__ double red[32 * R];
    const int nxy = nx * ny, nc = nxy * nz;
    double dot[R];
#pragma unroll
    for (int c = 0; c < R; ++c) dot[c] = 0.0;
    const double *in = MODE == 2 ? r : x;
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < nc; c += gridDim.x * blockDim.x) {
        const int i = c % nx, t = c / nx, j = t % ny, k = t / ny;
        auto ld = [&](int q) { return MODE == 2 ? W::scale(od, W::ld(in, q)) : W::ld(in, q); };
        T v[7];
        v[0] = k > 0 ? ld(c - nxy) : W::zero();
        v[1] = j > 0 ? ld(c - nx) : W::zero();
        v[2] = i > 0 ? ld(c - 1) : W::zero();
        v[3] = ld(c);
        v[4] = i < nx - 1 ? ld(c + 1) : W::zero();
        v[5] = j < ny - 1 ? ld(c + nx) : W::zero();
        v[6] = k < nz - 1 ? ld(c + nxy) : W::zero();
        T s = W::zero();
#pragma unroll
        for (int q = 0; q < 3; ++q) s = W::sub(s, v[q]);
        s = W::axpy(6.0, v[3], s);
#pragma unroll
        for (int q = 4; q < 7; ++q) s = W::sub(s, v[q]);
        T out;
        if (MODE == 0) out = s;
        else if (MODE == 1 || MODE == 2) out = W::sub(W::ld(r, c), s);
        else out = W::add(W::ld(x, c), W::scale(od, W::sub(W::ld(r, c), s)));
        W::st(y, c, out);
        if (DOT) {
#pragma unroll
            for (int cc = 0; cc < R; ++cc) {
                if (MODE == 0) dot[cc] += W::dot(W::ld(x, c), out, cc);
                else if (MODE == 3) dot[cc] += W::dot(W::ld(r, c), out, cc);
                else dot[cc] += W::dot(out, out, cc);
            }
        }
    }
    if (DOT) {
        block_sum<R>(dot, red);
        if (threadIdx.x == 0)
#pragma unroll
            for (int cc = 0; cc < R; ++cc) partials[blockIdx.x * R + cc] = dot[cc];
    }
}

// ---- elementwise / BLAS-1 ----------------------------------------------
template <int R>
__global__ void k_odinv_r(int64_t n, const double *od, const double *r, double *x) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
#pragma unroll
        for (int c = 0; c < R; ++c) x[i * R + c] = od[i] * r[i * R + c];
}

// partial a.b per rhs (fixed grid)
template <int R>
__global__ void k_dot(int64_t n, const double *a, const double *b, double *partials) {
    using W = V<R>;
    __shared__ double red[32 * R];
    double d[R];
#pragma unroll
    for (int c = 0; c < R; ++c) d[c] = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const typename W::T av = W::ld(a, i), bv = W::ld(b, i);
#pragma unroll
        for (int c = 0; c < R; ++c) d[c] = fma(W::comp(av, c), W::comp(bv, c), d[c]);
    }
    block_sum<R>(d, red);
    if (threadIdx.x == 0)
#pragma unroll
        for (int c = 0; c < R; ++c) partials[blockIdx.x * R + c] = d[c];
}

template <int R>
__device__ __forceinline__ typename V<R>::T vfma(const double (&a)[R], typename V<R>::T x, typename V<R>::T y) {
    if constexpr (R == 1) return fma(a[0], x, y);
    else return make_double2(fma(a[0], x.x, y.x), fma(a[1], x.y, y.y));
}

// x += alpha p ; r -= alpha q ; partial r.r
template <int R>
__global__ void k_update_xr(int64_t n, const double *scal, double *x, double *r, const double *p, const double *q,
                            double *partials) {
    using W = V<R>;
    __shared__ double red[32 * R];
    double a[R], na[R], d[R];
#pragma unroll
    for (int c = 0; c < R; ++c) { a[c] = scal[S_ALPHA + c]; na[c] = -a[c]; d[c] = 0.0; }
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        W::st(x, i, vfma<R>(a, W::ld(p, i), W::ld(x, i)));
        const typename W::T rv = vfma<R>(na, W::ld(q, i), W::ld(r, i));
        W::st(r, i, rv);
#pragma unroll
        for (int c = 0; c < R; ++c) d[c] = fma(W::comp(rv, c), W::comp(rv, c), d[c]);
    }
    block_sum<R>(d, red);
    if (threadIdx.x == 0)
#pragma unroll
        for (int c = 0; c < R; ++c) partials[blockIdx.x * R + c] = d[c];
}

// split update for overlap: r -= alpha q (+ r.r) on the solve stream while
// x += alpha p runs on a side stream during the next V-cycle
template <int R>
__global__ void k_update_r(int64_t n, const double *scal, double *r, const double *q, double *partials, int rev) {
    using W = V<R>;
    __shared__ double red[32 * R];
    double na[R], d[R];
#pragma unroll
    for (int c = 0; c < R; ++c) { na[c] = -scal[S_ALPHA + c]; d[c] = 0.0; }
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = rev ? n - 1 - j : j;
        const typename W::T rv = vfma<R>(na, W::ld(q, i), W::ld(r, i));
        W::st(r, i, rv);
#pragma unroll
        for (int c = 0; c < R; ++c) d[c] = fma(W::comp(rv, c), W::comp(rv, c), d[c]);
    }
    block_sum<R>(d, red);
    if (threadIdx.x == 0)
#pragma unroll
        for (int c = 0; c < R; ++c) partials[blockIdx.x * R + c] = d[c];
}
template <int R>
__global__ void k_update_x(int64_t n, const double *scal, double *x, const double *p, int rev = 0) {
    using W = V<R>;
    double a[R];
#pragma unroll
    for (int c = 0; c < R; ++c) a[c] = scal[S_ALPHA + c];
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = rev ? n - 1 - j : j;
        W::st(x, i, vfma<R>(a, W::ld(p, i), W::ld(x, i)));
    }
}

// p = z + beta p
template <int R>
__global__ void k_xpby(int64_t n, const double *scal, const double *z, double *p, int rev = 0) {
    using W = V<R>;
    double b[R];
#pragma unroll
    for (int c = 0; c < R; ++c) b[c] = scal[S_BETA + c];
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = rev ? n - 1 - j : j;
        W::st(p, i, vfma<R>(b, W::ld(p, i), W::ld(z, i)));
    }
}

// x += alpha p ; p = z + beta p  (alpha of the previous iteration: the graph
// body's deferred x update fused into the p update -- one read of p, and the
// same two FMAs per entry as k_update_x followed by k_xpby)
template <int R>
__global__ void k_xpby_x(int64_t n, const double *scal, const double *z, double *p, double *x) {
    using W = V<R>;
    double a[R], b[R];
#pragma unroll
    for (int c = 0; c < R; ++c) { a[c] = scal[S_ALPHA + c]; b[c] = scal[S_BETA + c]; }
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const typename W::T pv = W::ld(p, i);
        W::st(x, i, vfma<R>(a, pv, W::ld(x, i)));
        W::st(p, i, vfma<R>(b, pv, W::ld(z, i)));
    }
}

// Sum per-CTA partials in index order; then apply `what`.
enum { F_STORE = 0, F_ALPHA = 1, F_BETA_INIT = 2, F_BETA = 3, F_BETA_AUTO = 4 };
// One CTA of kFinThreads: thread t sums partials t, t + T, t + 2T, ... in
// four interleaved accumulators (coalesced, four loads in flight; a
// contiguous stripe per thread made this a chain of dependent L2 reads,
// 11 us for the 8705 fine-level tiles), then a fixed tree -- a fixed order,
// so the result is reproducible run to run.
constexpr int kFinThreads = 1024;
template <int R>
__device__ __forceinline__ void fin_sum(const double *partials, int nblocks, double (&s)[R], double *red) {
    double s4[4][R];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int c = 0; c < R; ++c) s4[u][c] = 0.0;
    const int T = blockDim.x;
    int b = threadIdx.x;
    for (; b + 3 * T < nblocks; b += 4 * T)
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int c = 0; c < R; ++c) s4[u][c] += partials[(b + u * T) * R + c];
    for (; b < nblocks; b += T)
#pragma unroll
        for (int c = 0; c < R; ++c) s4[0][c] += partials[b * R + c];
#pragma unroll
    for (int c = 0; c < R; ++c) s[c] = (s4[0][c] + s4[1][c]) + (s4[2][c] + s4[3][c]);
    block_sum<R>(s, red);
}

template <int R>
__global__ void __launch_bounds__(kFinThreads) k_finalize(const double *partials, int nblocks, double *scal, int slot,
                                                          int what, double tol) {
    __shared__ double red[32 * R];
    double s[R];
    fin_sum<R>(partials, nblocks, s, red);
    if (threadIdx.x == 0) {
        if (what == F_BETA_AUTO) {  // graph PCG: the first iteration after a (re)start initialises rho
            what = scal[S_G_INIT] != 0.0 ? F_BETA_INIT : F_BETA;
            scal[S_G_INIT] = 0.0;
        }
#pragma unroll
        for (int c = 0; c < R; ++c) {
            scal[slot + c] = s[c];
            bool active = scal[S_ACTIVE + c] != 0.0;
            if (what == F_ALPHA) {
                double pq = s[c];
                scal[S_ALPHA + c] = (active && pq != 0.0) ? scal[S_RHO + c] / pq : 0.0;
            } else if (what == F_BETA_INIT) {
                scal[S_RHO + c] = s[c];
                scal[S_BETA + c] = 0.0;
            } else if (what == F_BETA) {
                double old = scal[S_RHO + c];
                scal[S_BETA + c] = (active && old != 0.0) ? s[c] / old : 0.0;
                scal[S_RHO + c] = s[c];
            }
        }
        (void)tol;
    }
}

// Graph PCG convergence test (the host loop's test, on the device): counts
// the iteration, records the residual estimates, updates the per-rhs active
// flags and ends the WHILE node on convergence, non-finite residual or the
// iteration cap.
__device__ void check_body(double *scal, int R, double *trace, cudaGraphConditionalHandle hnd) {
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
        if (it <= maxit) trace[(int64_t)(it - 1) * R + c] = est;
        if (est > tol) done = false;
        const bool conv = bb == 0.0 || sqrt(rr) <= tol * bn;
        scal[S_ACTIVE + c] = conv ? 0.0 : 1.0;
    }
    if (bad) scal[S_G_STATUS] = 1.0;
    if (done || bad || it >= maxit) cudaGraphSetConditional(hnd, 0);
}

// r.r finalize (F_STORE into S_RR) and the convergence test in one launch:
// k_finalize's summation order, then the test (check_body) on thread 0
template <int R>
__global__ void __launch_bounds__(kFinThreads) k_finalize_check(const double *partials, int nblocks, double *scal,
                                                                double *trace, cudaGraphConditionalHandle hnd) {
    __shared__ double red[32 * R];
    double s[R];
    fin_sum<R>(partials, nblocks, s, red);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int c = 0; c < R; ++c) scal[S_RR + c] = s[c];
        check_body(scal, R, trace, hnd);
    }
}

__global__ void k_set_active(double *scal, int R, double tol) {
    for (int c = 0; c < R; ++c) {
        double bb = scal[S_BB + c], rr = scal[S_RR + c];
        bool conv = bb == 0.0 || sqrt(rr) <= tol * sqrt(bb);
        scal[S_ACTIVE + c] = conv ? 0.0 : 1.0;
    }
}

}  // namespace

// ------------------------------------------------------------------------
// level-0 layout conversions
// ------------------------------------------------------------------------

__global__ void k_interleave(int64_t n, int R, const double *planar, double *inter) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        for (int c = 0; c < R; ++c) inter[i * R + c] = planar[c * n + i];
}
__global__ void k_deinterleave(int64_t n, int R, const double *inter, double *planar) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        for (int c = 0; c < R; ++c) planar[c * n + i] = inter[i * R + c];
}

void amg_to_level0(Amg &h, const double *planar, double *inter, int nrhs, cudaStream_t s) {
    if (h.structured) op_dofs_to_span(*h.op, planar, inter, nrhs, s);
    else {
        k_interleave<<<grid_for(h.lv[0].n, 256, 148 * 16), 256, 0, s>>>(h.lv[0].n, nrhs, planar, inter);
        SPFD_LAUNCH_CHECK();
    }
}

void amg_from_level0(Amg &h, const double *inter, double *planar, int nrhs, cudaStream_t s) {
    if (h.structured) op_span_to_dofs(*h.op, inter, planar, nrhs, s);
    else {
        k_deinterleave<<<grid_for(h.lv[0].n, 256, 148 * 16), 256, 0, s>>>(h.lv[0].n, nrhs, inter, planar);
        SPFD_LAUNCH_CHECK();
    }
}

void alloc_krylov(Amg &h, int64_t nvec0, int R) {
    int64_t n = nvec0 * R;
    h.kx.alloc(n); h.kr.alloc(n); h.kz.alloc(n); h.kp.alloc(n); h.kq.alloc(n); h.kb.alloc(n);
    int64_t np = kDotGrid;
    if (h.structured) np = std::max<int64_t>(np, h.op->n_tiles);
    np = std::max<int64_t>(np, 148 * 16);
    np = std::max<int64_t>(np, (int64_t)kDotGrid * 8);  // batched FGMRES dual block dots (k_mdot2: 2 x 4 x R)
    h.partials.alloc(np * 2 + 64);
    h.scal.alloc(S_END);
    SPFD_CUDA(cudaStreamCreateWithFlags(&h.side, cudaStreamNonBlocking));
    SPFD_CUDA(cudaEventCreateWithFlags(&h.ev_alpha, cudaEventDisableTiming));
    SPFD_CUDA(cudaEventCreateWithFlags(&h.ev_x, cudaEventDisableTiming));
}

// ------------------------------------------------------------------------
// level-0 operator application and the V-cycle
// ------------------------------------------------------------------------

namespace {

}  // namespace

// fine-kernel override from the C-ABI tuning knob (-1 = environment/default)
int g_fine_kind_override = -1;

namespace {

// fine-level stencil kernel: 3 = flat per-position k_span with the tile's
// streamed arrays bulk-prefetched into L2 (default), 2 = without the
// prefetch (A/B).  The variants measured slower (z-marching, smem/TMA
// staging, fused pass pairs, lane shuffles, voxel-id conductances) are
// documented in DESIGN.md and profiles/r02_fine_kernel_experiments.md.
int fine_kernel_kind() {
    if (g_fine_kind_override >= 0) return g_fine_kind_override;
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("SPFD_SPAN_KERNEL");
        v = 3;
        if (e && std::string(e) == "flat") v = 2;
        if (e && std::string(e) == "pf") v = 3;
    }
    return v;
}

// Launch one fine-level stencil pass over the owned positions [a.pb, a.pe).
// Returns the number of CTAs (dot partials written when DOT).
inline int pf_ahead() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("SPFD_PF_AHEAD");
        v = e ? atoi(e) : 0;
        if (v < 0) v = 0;
    }
    return v;
}

// Alternate sweep directions of consecutive fine-level passes (SPFD_REV=0:
// all forward).  CTAs retire roughly in launch order, so when a pass ends
// the L2 (126 MB) holds the tail of what it touched; the next pass starting
// from that end finds its first ~100 MB of weights / vectors there.  Chain
// per PCG iteration: pre-smooth R, restriction input F, aggregate sums R |
// prolongation F, post-smooth R, p update F, SpMV R, r update F.
bool alt_dirs() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("SPFD_REV");
        v = (e && std::string(e) == "0") ? 0 : 1;
    }
    return v == 1;
}

template <int R, int MODE, bool DOT>
int launch_fine(const Operator &op, const SpanArgs &a_in, cudaStream_t s) {
    SpanView v = span_view(op);
    SpanArgs a = a_in;
    a.pf_ahead = pf_ahead();
    if (a.pb > 0 || a.pe < op.L) {  // owned z-slab range
        const int64_t pe = a.pe < op.L ? a.pe : op.L;
        const int t0 = (int)(a.pb / kTile), t1 = (int)((pe + kTile - 1) / kTile);
        SpanArgs b = a;
        b.tile0 = t0;
        int g = t1 - t0;
        if (g > 0) {
            // 4 CTAs/SM: the range checks cost registers; at 6 (and 5) the ranged
            // instantiations spilled (the single-GPU kernels keep 6, measured)
            if (fine_kernel_kind() == 3) k_span<R, MODE, DOT, true, true, 4><<<g, kSpanThreads, 0, s>>>(v, b);
            else k_span<R, MODE, DOT, true, false, 4><<<g, kSpanThreads, 0, s>>>(v, b);
        }
        SPFD_LAUNCH_CHECK();
        return g;
    }
    int g = (int)op.n_tiles;
    constexpr int MB = (MODE == 0 && DOT) ? SPFD_SPMV_MINB : SPFD_SPAN_MINB;
    if (g > 0) {
        if (fine_kernel_kind() == 3) k_span<R, MODE, DOT, false, true, MB><<<g, kSpanThreads, 0, s>>>(v, a);
        else k_span<R, MODE, DOT, false, false, MB><<<g, kSpanThreads, 0, s>>>(v, a);
    }
    SPFD_LAUNCH_CHECK();
    return g;
}

// returns number of partial blocks written when DOT
template <int R>
int level0_apply(Amg &h, int mode, bool dot, const double *x, const double *r, double *y, cudaStream_t s,
                 bool rev = false) {
    Level &L = h.lv[0];
    double *part = h.partials.get();
    if (h.structured) {
        int g = (int)h.op->n_tiles;
        if (g == 0) return 0;
        SpanArgs sa{x, r, L.odinv.get(), nullptr, nullptr, nullptr, y, part};
        sa.rev = rev && alt_dirs();
        const Operator &op = *h.op;
        if (mode == 0) g = dot ? launch_fine<R, 0, true>(op, sa, s) : launch_fine<R, 0, false>(op, sa, s);
        else if (mode == 1) g = dot ? launch_fine<R, 1, true>(op, sa, s) : launch_fine<R, 1, false>(op, sa, s);
        else if (mode == 2) g = launch_fine<R, 2, false>(op, sa, s);
        else g = dot ? launch_fine<R, 3, true>(op, sa, s) : launch_fine<R, 3, false>(op, sa, s);
        return g;
    }
    if (h.box[0] > 0) {  // matrix-free cell Laplacian
        const int nx = (int)h.box[0], ny = (int)h.box[1], nz = (int)h.box[2];
        const int g = grid_for(L.n, 256, 148 * 8);
        const double od = h.box_od;
        switch (mode) {
            case 0: if (dot) k_box<R, 0, true><<<g, 256, 0, s>>>(nx, ny, nz, od, x, r, y, part);
                    else k_box<R, 0, false><<<g, 256, 0, s>>>(nx, ny, nz, od, x, r, y, part); break;
            case 1: if (dot) k_box<R, 1, true><<<g, 256, 0, s>>>(nx, ny, nz, od, x, r, y, part);
                    else k_box<R, 1, false><<<g, 256, 0, s>>>(nx, ny, nz, od, x, r, y, part); break;
            case 2: k_box<R, 2, false><<<g, 256, 0, s>>>(nx, ny, nz, od, x, r, y, part); break;
            default: if (dot) k_box<R, 3, true><<<g, 256, 0, s>>>(nx, ny, nz, od, x, r, y, part);
                     else k_box<R, 3, false><<<g, 256, 0, s>>>(nx, ny, nz, od, x, r, y, part); break;
        }
        SPFD_LAUNCH_CHECK();
        return g;
    }
    const double *od = L.odinv.get();
    switch (mode) {
        case 0: return dot ? launch_csr<R, 0, true>(L.A, L.a_group, x, r, od, nullptr, y, part, s)
                           : launch_csr<R, 0, false>(L.A, L.a_group, x, r, od, nullptr, y, part, s);
        case 1: return dot ? launch_csr<R, 1, true>(L.A, L.a_group, x, r, od, nullptr, y, part, s)
                           : launch_csr<R, 1, false>(L.A, L.a_group, x, r, od, nullptr, y, part, s);
        case 2: return launch_csr<R, 2, false>(L.A, L.a_group, x, r, od, nullptr, y, part, s);
        default: return dot ? launch_csr<R, 3, true>(L.A, L.a_group, x, r, od, nullptr, y, part, s)
                            : launch_csr<R, 3, false>(L.A, L.a_group, x, r, od, nullptr, y, part, s);
    }
}

// smoother/residual on level l (l > 0 or CSR level 0)
template <int R>
void level_apply(Amg &h, int l, int mode, const double *x, const double *r, double *y, cudaStream_t s) {
    if (l == 0) { level0_apply<R>(h, mode, false, x, r, y, s); return; }
    Level &L = h.lv[l];
    const double *od = L.odinv.get();
    switch (mode) {
        case 1: launch_csr<R, 1, false>(L.A, L.a_group, x, r, od, nullptr, y, nullptr, s); break;
        case 2: launch_csr<R, 2, false>(L.A, L.a_group, x, r, od, nullptr, y, nullptr, s); break;
        default: launch_csr<R, 3, false>(L.A, L.a_group, x, r, od, nullptr, y, nullptr, s); break;
    }
}

template <int R>
void vcycle_level(Amg &h, int l, const double *r, double *z, cudaStream_t s);

// fused coarse-level prolongation + post-smooth z = od r + P e + od (d - (A P) e)
template <int R>
void launch_pp(const Level &L, const double *e, const double *r, const double *d, double *z, cudaStream_t s) {
    if (L.Q.rows) {  // z = od (r + d) + Q e (build_q)
        launch_csr<R, 6, false>(L.Q, L.q_group, e, r, L.odinv.get(), d, z, nullptr, s);
        return;
    }
    const int G = std::min(L.ap_group, 32);
    const int grid = csr_grid(L.P.rows, G);
    const bool pf = csr_prefetch_enabled();
    switch (G) {
        case 4: k_csr_pp<4, R><<<grid, kCsrThreads, 0, s>>>(view(L.P), view(L.AP), e, r, L.odinv.get(), d, z, pf); break;
        case 8: k_csr_pp<8, R><<<grid, kCsrThreads, 0, s>>>(view(L.P), view(L.AP), e, r, L.odinv.get(), d, z, pf); break;
        case 16: k_csr_pp<16, R><<<grid, kCsrThreads, 0, s>>>(view(L.P), view(L.AP), e, r, L.odinv.get(), d, z, pf); break;
        default: k_csr_pp<32, R><<<grid, kCsrThreads, 0, s>>>(view(L.P), view(L.AP), e, r, L.odinv.get(), d, z, pf); break;
    }
    SPFD_LAUNCH_CHECK();
}

// Fine level of a structured hierarchy, transfers matrix-free through the
// aggregates (P = (I - omega D^-1 A) T, R = P^T):
//   d  = r - A(od r)                      pre-smooth + defect
//   u  = d - A(od d),  r_c = T^T u        restriction P^T d
//   x1 = od r + e - od A e,  e = T e_c    prolongation + correction
//   z  = x1 + od (r - A x1)               post-smooth
// Returns the number of CTA partials of r.z written by the last sweep
// (0 if none), so PCG needs no separate dot pass.
template <int R>
int vcycle_fine_mf(Amg &h, const double *r, double *z, cudaStream_t s) {
    Level &L = h.lv[0];
    Level &C = h.lv[1];
    double *d = L.vd.get(), *t = L.vt.get(), *u = L.vr.get();
    const size_t bytes = (size_t)L.nvec * R * sizeof(double);
    const double *od = L.odinv.get();
    const double *xbase = nullptr;
    const int rv = alt_dirs() ? 1 : 0;
    if (h.pre <= 1) {
        SpanArgs sa{nullptr, r, od, nullptr, nullptr, nullptr, d, nullptr};
        sa.rev = rv;
        launch_fine<R, 2, false>(*h.op, sa, s);
    } else {
        k_odinv_r<R><<<grid_for(L.nvec, 256, 148 * 16), 256, 0, s>>>(L.nvec, od, r, t);
        for (int it = 1; it < h.pre; ++it) {
            launch_fine<R, 3, false>(*h.op, SpanArgs{t, r, od, nullptr, nullptr, nullptr, d, nullptr}, s);
            SPFD_CUDA(cudaMemcpyAsync(t, d, bytes, cudaMemcpyDeviceToDevice, s));
        }
        launch_fine<R, 1, false>(*h.op, SpanArgs{t, r, od, nullptr, nullptr, nullptr, d, nullptr}, s);
        xbase = t;
    }
    SPFD_LAUNCH_CHECK();
    // level 1 gets r_1 and (when it smooths) its first Jacobi iterate od_1 r_1
    const bool x0 = h.pre <= 1 && (int)h.lv.size() > 2;
    if (L.Rspan.rows) {
        // r_1 = R d, R = P^T as a CSR over span positions (build_rspan)
        launch_csr<R, 0, false>(L.Rspan, L.rspan_group, d, nullptr, nullptr, nullptr, C.vr.get(), nullptr, s,
                                C.odinv.get(), x0 ? C.vt.get() : nullptr);
    } else {
        // matrix-free: u = d - A(od d), r_1 = T^T u
        launch_fine<R, 2, false>(*h.op, SpanArgs{nullptr, d, od, nullptr, nullptr, nullptr, u, nullptr}, s);
        SPFD_LAUNCH_CHECK();
        k_agg_sum<R><<<grid_for(C.n, 256, 148 * 16), 256, 0, s>>>(L.mem_ptr.get(), L.mem_pos.get(), C.n, u,
                                                                 C.vr.get(), C.odinv.get(), x0 ? C.vt.get() : nullptr,
                                                                 rv);
    }
    SPFD_LAUNCH_CHECK();
    vcycle_level<R>(h, 1, C.vr.get(), C.vx.get(), s);
    if (L.Pspan.rows) {  // x1 = x0 + P e, P in CSR over span positions (build_pspan)
        if (xbase) launch_csr<R, 5, false>(L.Pspan, L.pspan_group, C.vx.get(), r, od, xbase, d, nullptr, s);
        else launch_csr<R, 4, false>(L.Pspan, L.pspan_group, C.vx.get(), r, od, nullptr, d, nullptr, s);
    } else {
        launch_fine<R, 4, false>(*h.op, SpanArgs{nullptr, r, od, xbase, C.vx.get(), L.agg_pos.get(), d, nullptr}, s);
    }
    SPFD_LAUNCH_CHECK();
    if (h.post == 0) {
        SPFD_CUDA(cudaMemcpyAsync(z, d, bytes, cudaMemcpyDeviceToDevice, s));
        return 0;
    }
    const double *cur = d;
    int parts = 0;
    for (int it = 0; it < h.post; ++it) {
        const bool last = it == h.post - 1;
        double *dst = last ? z : (cur == d ? t : d);
        SpanArgs sa{cur, r, od, nullptr, nullptr, nullptr, dst, h.partials.get()};
        sa.rev = (h.post - it) & 1 ? rv : 0;   // the last sweep runs reversed
        if (last) parts = launch_fine<R, 3, true>(*h.op, sa, s);
        else launch_fine<R, 3, false>(*h.op, sa, s);
        cur = dst;
    }
    return parts;
}

template <int R>
void vcycle_level(Amg &h, int l, const double *r, double *z, cudaStream_t s) {
    int nl = (int)h.lv.size();
    Level &L = h.lv[l];
    if (l == nl - 1) {
        if (l == 0 && h.structured) {
            // single-level structured hierarchy: the dense inverse acts on DOF order
            const Operator &op = *h.op;
            k_span_gather<R><<<grid_for(op.n_dofs, 256, 148 * 16), 256, 0, s>>>(op.dof_to_pos.get(), op.n_dofs, r,
                                                                                L.vd.get());
            k_dense_mv<R><<<grid_for(h.nc * 32, 256, 148 * 8), 256, 0, s>>>(h.cinv.get(), h.nc, L.vd.get(),
                                                                           L.vt.get());
            k_span_scatter<R><<<grid_for(op.L, 256, 148 * 16), 256, 0, s>>>(op.pos_to_dof.get(), op.L, L.vt.get(), z);
        } else {
            k_dense_mv<R><<<grid_for(h.nc * 32, 256, 148 * 8), 256, 0, s>>>(h.cinv.get(), h.nc, r, z);
        }
        SPFD_LAUNCH_CHECK();
        return;
    }
    if (l == 0 && h.structured) {
        h.vc_partials = vcycle_fine_mf<R>(h, r, z, s);
        return;
    }
    double *d = L.vd.get(), *t = L.vt.get();
    const size_t bytes = (size_t)L.nvec * R * sizeof(double);
    const double *xbase = nullptr;  // materialised pre-smoothed iterate (pre >= 2)
    if (h.pre <= 1) {
        // implicit first sweep x = omega D^-1 r, defect d = r - A x (linsolve.py:190-193);
        // on coarse levels the restriction already wrote x = od r into vt
        if (l > 0) level_apply<R>(h, l, 1, t, r, d, s);
        else level_apply<R>(h, l, 2, nullptr, r, d, s);
    } else {
        k_odinv_r<R><<<grid_for(L.nvec, 256, 148 * 16), 256, 0, s>>>(L.nvec, L.odinv.get(), r, t);
        for (int it = 1; it < h.pre; ++it) {
            level_apply<R>(h, l, 3, t, r, d, s);
            SPFD_CUDA(cudaMemcpyAsync(t, d, bytes, cudaMemcpyDeviceToDevice, s));
        }
        level_apply<R>(h, l, 1, t, r, d, s);
        xbase = t;
    }
    Level &C = h.lv[l + 1];
    const bool x0 = h.pre <= 1 && l + 1 < nl - 1;
    launch_csr<R, 0, false>(L.R, L.r_group, d, nullptr, nullptr, nullptr, C.vr.get(), nullptr, s, C.odinv.get(),
                            x0 ? C.vt.get() : nullptr);
    vcycle_level<R>(h, l + 1, C.vr.get(), C.vx.get(), s);
    if (L.AP.rows > 0 && h.pre == 1 && h.post == 1) {
        launch_pp<R>(L, C.vx.get(), r, d, z, s);  // fused prolongation + post-smooth from the defect d
        return;
    }
    // x1 = x + P e (linsolve.py:194) -> d
    if (xbase) launch_csr<R, 5, false>(L.P, L.p_group, C.vx.get(), r, L.odinv.get(), xbase, d, nullptr, s);
    else launch_csr<R, 4, false>(L.P, L.p_group, C.vx.get(), r, L.odinv.get(), nullptr, d, nullptr, s);
    if (h.post == 0) {
        SPFD_CUDA(cudaMemcpyAsync(z, d, bytes, cudaMemcpyDeviceToDevice, s));
        return;
    }
    // post sweeps x += omega D^-1 (r - A x) (linsolve.py:195-196), last one lands in z
    const double *cur = d;
    for (int it = 0; it < h.post; ++it) {
        double *dst = (it == h.post - 1) ? z : (cur == d ? t : d);
        level_apply<R>(h, l, 3, cur, r, dst, s);
        cur = dst;
    }
}

// ---- Chebyshev smoother (SPFD_SMOOTHER_CHEBYSHEV) -------------------------
// Polynomial smoother in D^-1 A on [beta / 5, beta], beta = 1.1 x the
// power-iteration estimate of lambda_max (lower end 0.2 beta, see
// oracle/spfd_oracle.py chebyshev_coefficients), three-term
// recurrence (Saad, Iterative Methods, alg. 12.1):
//   d_0 = (1/theta) D^-1 r_0,  x_1 = x_0 + d_0
//   rho_k = 1 / (2 sigma - rho_{k-1}),  d_k = rho_k rho_{k-1} d_{k-1} + (2 rho_k / delta) D^-1 r_k
// with theta = (beta + alpha) / 2, delta = (beta - alpha) / 2, sigma = theta / delta,
// rho_0 = 1 / sigma, r_k = b - A x_k.  The same polynomial before and after
// the coarse correction keeps the V-cycle symmetric (a valid PCG
// preconditioner).  The reference has damped Jacobi only (linsolve.py:184-197);
// this is the north_star's optional smoother, restated in oracle/.
template <int R>
__global__ void k_cheb_first(int64_t n, const double *__restrict__ dinv, double c0, const double *t, double *d,
                             const double *xin, double *xout) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double di = dinv[i];
#pragma unroll
        for (int c = 0; c < R; ++c) {
            const double dv = c0 * (di * t[i * R + c]);
            d[i * R + c] = dv;
            xout[i * R + c] = xin ? xin[i * R + c] + dv : dv;
        }
    }
}

template <int R>
__global__ void k_cheb_step(int64_t n, const double *__restrict__ dinv, double c1, double c2,
                            const double *__restrict__ t, double *__restrict__ d, double *__restrict__ x) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double di = dinv[i];
#pragma unroll
        for (int c = 0; c < R; ++c) {
            const double dv = c1 * d[i * R + c] + c2 * (di * t[i * R + c]);
            d[i * R + c] = dv;
            x[i * R + c] += dv;
        }
    }
}

struct ChebCoef {
    double c0;
    double c1[16], c2[16];  // step k = 1 .. degree-1
};

ChebCoef cheb_coef(double lmax, int degree) {
    const double beta = 1.1 * lmax, alpha = 0.2 * beta;
    const double theta = 0.5 * (beta + alpha), delta = 0.5 * (beta - alpha), sigma = theta / delta;
    ChebCoef c{};
    c.c0 = 1.0 / theta;
    double rho = 1.0 / sigma;
    for (int k = 1; k < degree && k < 16; ++k) {
        const double rn = 1.0 / (2.0 * sigma - rho);
        c.c1[k] = rn * rho;
        c.c2[k] = 2.0 * rn / delta;
        rho = rn;
    }
    return c;
}

// residual y = b - A_l x on level l (span layout on a structured level 0)
template <int R>
void level_residual(Amg &h, int l, const double *x, const double *b, double *y, cudaStream_t s) {
    if (l == 0) level0_apply<R>(h, 1, false, x, b, y, s);
    else level_apply<R>(h, l, 1, x, b, y, s);
}

// one polynomial sweep on x (x == nullptr: from x = 0 into xout); t, d scratch
template <int R>
void cheb_sweep(Amg &h, int l, const ChebCoef &c, const double *b, const double *xin, double *xout, double *t,
                double *d, cudaStream_t s) {
    Level &L = h.lv[l];
    const int64_t n = L.nvec;
    const int g = grid_for(n, 256, 148 * 16);
    if (xin) {
        level_residual<R>(h, l, xin, b, t, s);
        k_cheb_first<R><<<g, 256, 0, s>>>(n, L.dinv.get(), c.c0, t, d, xin, xout);
    } else {
        k_cheb_first<R><<<g, 256, 0, s>>>(n, L.dinv.get(), c.c0, b, d, nullptr, xout);
    }
    SPFD_LAUNCH_CHECK();
    for (int k = 1; k < h.cheb_deg; ++k) {
        level_residual<R>(h, l, xout, b, t, s);
        k_cheb_step<R><<<g, 256, 0, s>>>(n, L.dinv.get(), c.c1[k], c.c2[k], t, d, xout);
        SPFD_LAUNCH_CHECK();
    }
}

template <int R>
void vcycle_cheb(Amg &h, int l, const double *r, double *z, cudaStream_t s) {
    const int nl = (int)h.lv.size();
    if (l == nl - 1) {  // coarsest: the dense inverse
        vcycle_level<R>(h, l, r, z, s);
        return;
    }
    Level &L = h.lv[l];
    Level &C = h.lv[l + 1];
    double *d = L.vd.get(), *t = L.vt.get();
    const ChebCoef c = cheb_coef(h.cheb_lmax[l], h.cheb_deg);
    // pre-smoothing from x = 0 (z holds the iterate)
    cheb_sweep<R>(h, l, c, r, nullptr, z, t, d, s);
    for (int k = 1; k < h.pre; ++k) cheb_sweep<R>(h, l, c, r, z, z, t, d, s);
    if (h.pre == 0) SPFD_CUDA(cudaMemsetAsync(z, 0, (size_t)L.nvec * R * sizeof(double), s));
    // residual, restriction
    level_residual<R>(h, l, z, r, t, s);
    if (l == 0 && h.structured) {
        double *u = L.vr.get();  // R t = T^T (t - A (omega D^-1 t))
        launch_fine<R, 2, false>(*h.op, SpanArgs{nullptr, t, L.odinv.get(), nullptr, nullptr, nullptr, u, nullptr}, s);
        k_agg_sum<R><<<grid_for(C.n, 256, 148 * 16), 256, 0, s>>>(L.mem_ptr.get(), L.mem_pos.get(), C.n, u,
                                                                 C.vr.get(), nullptr, nullptr, 0);
        SPFD_LAUNCH_CHECK();
    } else {
        launch_csr<R, 0, false>(L.R, L.r_group, t, nullptr, nullptr, nullptr, C.vr.get(), nullptr, s);
    }
    vcycle_cheb<R>(h, l + 1, C.vr.get(), C.vx.get(), s);
    // x1 = x + P e -> t
    if (l == 0 && h.structured)
        launch_fine<R, 4, false>(*h.op, SpanArgs{nullptr, r, L.odinv.get(), z, C.vx.get(), L.agg_pos.get(), t, nullptr},
                                 s);
    else
        launch_csr<R, 5, false>(L.P, L.p_group, C.vx.get(), r, L.odinv.get(), z, t, nullptr, s);
    SPFD_LAUNCH_CHECK();
    // post-smoothing from x1 (the first sweep moves the iterate from t to z)
    if (h.post == 0) {
        SPFD_CUDA(cudaMemcpyAsync(z, t, (size_t)L.nvec * R * sizeof(double), cudaMemcpyDeviceToDevice, s));
        return;
    }
    {
        // residual into d, then d := c0 D^-1 d in place and z = t + d
        level_residual<R>(h, l, t, r, d, s);
        const int g = grid_for(L.nvec, 256, 148 * 16);
        k_cheb_first<R><<<g, 256, 0, s>>>(L.nvec, L.dinv.get(), c.c0, d, d, t, z);
        SPFD_LAUNCH_CHECK();
        for (int k = 1; k < h.cheb_deg; ++k) {
            level_residual<R>(h, l, z, r, t, s);
            k_cheb_step<R><<<g, 256, 0, s>>>(L.nvec, L.dinv.get(), c.c1[k], c.c2[k], t, d, z);
            SPFD_LAUNCH_CHECK();
        }
    }
    for (int k = 1; k < h.post; ++k) cheb_sweep<R>(h, l, c, r, z, z, t, d, s);
}

__global__ void k_pi_init(int64_t n, const double *dinv, double *x) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t hsh = (uint32_t)(i * 2654435761ull) >> 8;
        x[i] = dinv[i] != 0.0 ? 0.5 + (double)(hsh & 0xffff) / 65536.0 : 0.0;
    }
}

// y = scale * dinv * y (dinv may be null) ; x = y when x != null
__global__ void k_pi_scale(int64_t n, const double *dinv, double scale, double *y, double *x) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double v = scale * (dinv ? dinv[i] * y[i] : y[i]);
        y[i] = v;
        if (x) x[i] = v;
    }
}

}  // namespace

void amg_vcycle(Amg &h, const double *r, double *z, int nrhs, cudaStream_t s) {
    h.vc_partials = 0;
    if (h.smoother == SPFD_SMOOTHER_CHEBYSHEV && h.lv.size() > 1) {
        if (nrhs == 1) vcycle_cheb<1>(h, 0, r, z, s);
        else vcycle_cheb<2>(h, 0, r, z, s);
        return;
    }
    if (nrhs == 1) vcycle_level<1>(h, 0, r, z, s);
    else vcycle_level<2>(h, 0, r, z, s);
}

void amg_set_box_level0(Amg &h, const int64_t dims[3], cudaStream_t s) {
    SPFD_CHECK(!h.structured && !h.lv.empty(), SPFD_EINVAL, "box level 0 needs a CSR hierarchy");
    const int64_t nc = dims[0] * dims[1] * dims[2];
    SPFD_CHECK(nc == h.lv[0].n && nc < (int64_t)1 << 31 && dims[0] > 0 && dims[1] > 0 && dims[2] > 0, SPFD_EINVAL,
               "box dims do not match level 0");
    // every cell has diagonal 6 (div div^T): omega D^-1 is one number
    double od = 0.0;
    SPFD_CUDA(cudaMemcpyAsync(&od, h.lv[0].odinv.get(), sizeof(double), cudaMemcpyDeviceToHost, s));
    SPFD_CUDA(cudaStreamSynchronize(s));
    SPFD_CHECK(od == h.omega * (1.0 / 6.0), SPFD_EINVAL, "level 0 is not the cell Laplacian");
    h.box_od = od;
    for (int a = 0; a < 3; ++a) h.box[a] = dims[a];
    amg_drop_graphs(h);
}

// Power iteration on D^-1 A_l from a fixed pseudo-random start (20 steps,
// ||D^-1 A x|| with ||x|| = 1 -> lambda_max from below; the Chebyshev
// interval's 1.1 factor covers the gap).
void amg_estimate_lmax(Amg &h, cudaStream_t s) {
    const int nl = (int)h.lv.size();
    h.cheb_lmax.assign(nl, 0.0);
    double *sc = h.scal.get();
    auto norm = [&](int64_t n, const double *v) {
        k_dot<1><<<kDotGrid, kDotThreads, 0, s>>>(n, v, v, h.partials.get());
        SPFD_LAUNCH_CHECK();
        k_finalize<1><<<1, kFinThreads, 0, s>>>(h.partials.get(), kDotGrid, sc, S_TMP, F_STORE, 0.0);
        SPFD_LAUNCH_CHECK();
        double v2 = 0.0;
        SPFD_CUDA(cudaMemcpyAsync(&v2, sc + S_TMP, sizeof(double), cudaMemcpyDeviceToHost, s));
        SPFD_CUDA(cudaStreamSynchronize(s));
        return std::sqrt(v2);
    };
    for (int l = 0; l < nl - 1; ++l) {
        Level &L = h.lv[l];
        const int64_t n = L.nvec;
        const int g = grid_for(n, 256, 148 * 16);
        double *x = L.vx.get(), *y = L.vd.get();
        k_pi_init<<<g, 256, 0, s>>>(n, L.dinv.get(), x);
        SPFD_LAUNCH_CHECK();
        double nx = norm(n, x), lam = 0.0;
        SPFD_CHECK(nx > 0.0, SPFD_EINVAL, "empty level in the eigenvalue estimate");
        k_pi_scale<<<g, 256, 0, s>>>(n, nullptr, 1.0 / nx, x, nullptr);
        for (int it = 0; it < 20; ++it) {
            if (l == 0) level0_apply<1>(h, 0, false, x, nullptr, y, s);
            else launch_csr<1, 0, false>(L.A, L.a_group, x, nullptr, nullptr, nullptr, y, nullptr, s);
            k_pi_scale<<<g, 256, 0, s>>>(n, L.dinv.get(), 1.0, y, nullptr);
            SPFD_LAUNCH_CHECK();
            lam = norm(n, y);
            SPFD_CHECK(std::isfinite(lam) && lam > 0.0, SPFD_ENONFINITE, "eigenvalue estimate failed");
            k_pi_scale<<<g, 256, 0, s>>>(n, nullptr, 1.0 / lam, y, x);
            SPFD_LAUNCH_CHECK();
        }
        h.cheb_lmax[l] = lam;
    }
}

// ------------------------------------------------------------------------
// PCG
// ------------------------------------------------------------------------

namespace {

template <int R>
void finalize(Amg &h, int nblocks, int slot, int what, cudaStream_t s) {
    k_finalize<R><<<1, kFinThreads, 0, s>>>(h.partials.get(), nblocks, h.scal.get(), slot, what, 0.0);
    SPFD_LAUNCH_CHECK();
}

template <int R>
void dot(Amg &h, int64_t n, const double *a, const double *b, int slot, int what, cudaStream_t s) {
    k_dot<R><<<kDotGrid, kDotThreads, 0, s>>>(n, a, b, h.partials.get());
    SPFD_LAUNCH_CHECK();
    finalize<R>(h, kDotGrid, slot, what, s);
}

// SPFD_PCG_FUSE_X=0: the x update as a separate side-stream kernel
// overlapping the V-cycle instead of fused into the next p update
bool pcg_fuse_x() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("SPFD_PCG_FUSE_X");
        v = (e && std::string(e) == "0") ? 0 : 1;
    }
    return v == 1;
}

template <int R>
spfd_report pcg(Amg &h, const double *b, double *x, const spfd_config &cfg, double *h_trace, cudaStream_t s) {
    spfd_report rep{};
    int64_t n = h.lv[0].nvec;
    double *r = h.kr.get(), *z = h.kz.get(), *p = h.kp.get(), *q = h.kq.get();
    double *sc = h.scal.get();
    SPFD_CUDA(cudaMemsetAsync(x, 0, n * R * sizeof(double), s));
    SPFD_CUDA(cudaMemsetAsync(sc, 0, (S_H) * sizeof(double), s));
    double ones[2] = {1.0, 1.0};
    SPFD_CUDA(cudaMemcpyAsync(sc + S_ACTIVE, ones, R * sizeof(double), cudaMemcpyHostToDevice, s));
    dot<R>(h, n, b, b, S_BB, F_STORE, s);
    double hs[S_H];
    SPFD_CUDA(cudaMemcpyAsync(hs, sc, S_H * sizeof(double), cudaMemcpyDeviceToHost, s));
    SPFD_CUDA(cudaStreamSynchronize(s));
    double bnorm[2] = {std::sqrt(hs[S_BB]), R > 1 ? std::sqrt(hs[S_BB + 1]) : 0.0};
    for (int c = 0; c < R; ++c)
        if (!std::isfinite(bnorm[c])) { rep.status = SPFD_ENONFINITE; return rep; }
    bool all_zero = true;
    for (int c = 0; c < R; ++c) all_zero = all_zero && bnorm[c] == 0.0;
    if (all_zero) { rep.converged = 1; return rep; }

    int it = 0;
    bool restart = true;
    double tol = cfg.rel_tol;
    const bool fuse = pcg_fuse_x();
    while (true) {
        if (restart) {
            // r = b - A x ; z = M r ; rho = r.z ; p = z
            level0_apply<R>(h, 1, false, x, b, r, s);
            SPFD_CUDA(cudaMemcpyAsync(sc + S_ACTIVE, ones, R * sizeof(double), cudaMemcpyHostToDevice, s));
            amg_vcycle(h, r, z, R, s);
            if (h.vc_partials > 0) finalize<R>(h, h.vc_partials, S_RZ, F_BETA_INIT, s);
            else dot<R>(h, n, r, z, S_RZ, F_BETA_INIT, s);
            SPFD_CUDA(cudaMemcpyAsync(p, z, n * R * sizeof(double), cudaMemcpyDeviceToDevice, s));
            restart = false;
        }
        if (it >= cfg.max_iters) break;
        const int rv = 0;
        int g = level0_apply<R>(h, 0, true, p, nullptr, q, s, true);  // q = A p, p.q
        finalize<R>(h, g, S_PQ, F_ALPHA, s);
        if (!fuse) {
            // x += alpha p on the side stream, overlapping the V-cycle (which is
            // L1/latency-bound and leaves HBM bandwidth idle); joined before p changes
            SPFD_CUDA(cudaEventRecord(h.ev_alpha, s));
            SPFD_CUDA(cudaStreamWaitEvent(h.side, h.ev_alpha, 0));
            k_update_x<R><<<grid_for(n, 256, 148 * 8), 256, 0, h.side>>>(n, sc, x, p);
            SPFD_LAUNCH_CHECK();
            SPFD_CUDA(cudaEventRecord(h.ev_x, h.side));
        }  // else: x += alpha p rides with the next p update (k_xpby_x), or is flushed below
        k_update_r<R><<<kDotGrid, kDotThreads, 0, s>>>(n, sc, r, q, h.partials.get(), rv);
        SPFD_LAUNCH_CHECK();
        finalize<R>(h, kDotGrid, S_RR, F_STORE, s);
        k_set_active<<<1, 1, 0, s>>>(sc, R, tol);
        SPFD_CUDA(cudaMemcpyAsync(hs, sc, S_H * sizeof(double), cudaMemcpyDeviceToHost, s));
        SPFD_CUDA(cudaStreamSynchronize(s));
        ++it;
        bool done = true;
        for (int c = 0; c < R; ++c) {
            double est = bnorm[c] > 0 ? std::sqrt(hs[S_RR + c]) / bnorm[c] : 0.0;
            if (!std::isfinite(est)) { rep.status = SPFD_ENONFINITE; rep.iterations = it; return rep; }
            if (h_trace && it <= cfg.max_iters) h_trace[(int64_t)(it - 1) * R + c] = est;
            if (est > tol) done = false;
        }
        if (done || it >= cfg.max_iters) {
            // true residual check (linsolve.py:296-298 semantics)
            if (fuse) {
                k_update_x<R><<<grid_for(n, 256, 148 * 8), 256, 0, s>>>(n, sc, x, p);
                SPFD_LAUNCH_CHECK();
            }
            SPFD_CUDA(cudaStreamWaitEvent(s, h.ev_x, 0));
            int gt = level0_apply<R>(h, 1, true, x, b, q, s);
            finalize<R>(h, gt, S_TMP, F_STORE, s);
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
            restart = true;  // recursive residual drifted: restart from the true residual
            continue;
        }
        amg_vcycle(h, r, z, R, s);
        if (h.vc_partials > 0) finalize<R>(h, h.vc_partials, S_RZ, F_BETA, s);  // r.z fused into the post-smooth
        else dot<R>(h, n, r, z, S_RZ, F_BETA, s);
        if (fuse) {
            k_xpby_x<R><<<grid_for(n, 256, 148 * 16), 256, 0, s>>>(n, sc, z, p, x);
        } else {
            SPFD_CUDA(cudaStreamWaitEvent(s, h.ev_x, 0));  // x += alpha p done before p changes
            k_xpby<R><<<grid_for(n, 256, 148 * 16), 256, 0, s>>>(n, sc, z, p, 0);
        }
        SPFD_LAUNCH_CHECK();
    }
    SPFD_CUDA(cudaStreamWaitEvent(s, h.ev_x, 0));
    rep.iterations = it;
    return rep;
}

// ---- PCG as one CUDA graph ------------------------------------------------
// The iteration is rotated so the convergence test ends the body:
//   z = M r, beta (rho on the first pass after a (re)start)  ->
//   x += alpha p (previous alpha), p = z + beta p  ->  q = A p, alpha  ->
//   r -= alpha q, r.r  ->  k_finalize_check (sets the WHILE condition)
// which is the host loop's arithmetic in the same order.  The body is
// captured once per rhs count into the WHILE node of a graph; a solve is
// restart prologue + one graph launch (+ the last x update), and the host
// reads the scalars once per launch instead of once per iteration.

}  // namespace
int g_pcg_graph_override = -1;  // C-ABI tuning knob (-1 = environment/default)
namespace {

bool pcg_graph_enabled() {
    if (g_pcg_graph_override >= 0) return g_pcg_graph_override == 1;
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("SPFD_PCG_GRAPH");
        v = (e && std::string(e) == "0") ? 0 : 1;
    }
    return v == 1;
}

template <int R>
void pcg_body(Amg &h, cudaGraphConditionalHandle hnd, cudaStream_t s) {
    const int64_t n = h.lv[0].nvec;
    double *r = h.kr.get(), *z = h.kz.get(), *p = h.kp.get(), *q = h.kq.get(), *x = h.kx.get();
    double *sc = h.scal.get();
    const bool fuse = pcg_fuse_x();
    if (!fuse) {
        // x += alpha p with the previous iteration's alpha, overlapping the V-cycle
        SPFD_CUDA(cudaEventRecord(h.ev_alpha, s));
        SPFD_CUDA(cudaStreamWaitEvent(h.side, h.ev_alpha, 0));
        k_update_x<R><<<grid_for(n, 256, 148 * 8), 256, 0, h.side>>>(n, sc, x, p);
        SPFD_LAUNCH_CHECK();
        SPFD_CUDA(cudaEventRecord(h.ev_x, h.side));
    }
    amg_vcycle(h, r, z, R, s);
    if (h.vc_partials > 0) finalize<R>(h, h.vc_partials, S_RZ, F_BETA_AUTO, s);
    else dot<R>(h, n, r, z, S_RZ, F_BETA_AUTO, s);
    const int rv = 0;
    if (fuse) {
        k_xpby_x<R><<<grid_for(n, 256, 148 * 16), 256, 0, s>>>(n, sc, z, p, x);
    } else {
        SPFD_CUDA(cudaStreamWaitEvent(s, h.ev_x, 0));
        k_xpby<R><<<grid_for(n, 256, 148 * 16), 256, 0, s>>>(n, sc, z, p, rv);
    }
    SPFD_LAUNCH_CHECK();
    const int g = level0_apply<R>(h, 0, true, p, nullptr, q, s, true);  // q = A p, p.q
    finalize<R>(h, g, S_PQ, F_ALPHA, s);
    k_update_r<R><<<kDotGrid, kDotThreads, 0, s>>>(n, sc, r, q, h.partials.get(), rv);
    SPFD_LAUNCH_CHECK();
    k_finalize_check<R><<<1, kFinThreads, 0, s>>>(h.partials.get(), kDotGrid, sc, h.pcg_trace.get(), hnd);
    SPFD_LAUNCH_CHECK();
}

}  // namespace

void amg_drop_graphs(Amg &h) {
    for (int R = 0; R < 3; ++R) {
        if (h.pcg_exec[R]) cudaGraphExecDestroy(h.pcg_exec[R]);
        h.pcg_exec[R] = nullptr;
        h.pcg_body_launches[R] = 0;
        h.pcg_kind[R] = -1;
        if (h.fg_exec[R]) cudaGraphExecDestroy(h.fg_exec[R]);
        h.fg_exec[R] = nullptr;
        h.fg_exec_m[R] = 0;
    }
}

namespace {

// Returns false (host-loop PCG) when the body cannot be captured; the reason
// goes to stderr with SPFD_DEBUG=1.
template <int R>
bool pcg_graph_build(Amg &h, int64_t max_iters) {
    if (!h.cap) SPFD_CUDA(cudaStreamCreateWithFlags(&h.cap, cudaStreamNonBlocking));
    if (h.pcg_trace_cap < max_iters) {
        for (auto &e : h.pcg_exec)
            if (e) { cudaGraphExecDestroy(e); e = nullptr; }
        h.pcg_trace_cap = std::max<int64_t>(max_iters, 1024);
        h.pcg_trace.alloc(h.pcg_trace_cap * 2);
    }
    if (h.pcg_exec[R] && h.pcg_kind[R] != fine_kernel_kind()) {  // kernel selection changed: recapture
        cudaGraphExecDestroy(h.pcg_exec[R]);
        h.pcg_exec[R] = nullptr;
        h.pcg_body_launches[R] = 0;
    }
    if (h.pcg_exec[R]) return true;
    if (h.pcg_body_launches[R] < 0) return false;  // capture failed before: stay on the host loop
    cudaGraph_t g = nullptr;
    SPFD_CUDA(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle hnd;
    SPFD_CUDA(cudaGraphConditionalHandleCreate(&hnd, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams np{};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = hnd;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    cudaGraphNode_t node;
    SPFD_CUDA(cudaGraphAddNode(&node, g, nullptr, 0, &np));
    cudaGraph_t body = np.conditional.phGraph_out[0];
    const int64_t l0 = launch_count();
    // relaxed: lazily loaded kernels may be loaded during the capture
    SPFD_CUDA(cudaStreamBeginCaptureToGraph(h.cap, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    std::string why;
    try {
        pcg_body<R>(h, hnd, h.cap);
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
    cudaGetLastError();  // clear a sticky capture error
    if (!why.empty()) {
        if (getenv("SPFD_DEBUG")) fprintf(stderr, "[spfd] PCG graph capture failed (%s): host loop\n", why.c_str());
        h.pcg_body_launches[R] = -1;
        return false;  // (the graph is leaked rather than destroyed half-built)
    }
    h.pcg_body_launches[R] = launch_count() - l0;
    cudaGraphDestroy(g);
    h.pcg_exec[R] = exec;
    h.pcg_kind[R] = fine_kernel_kind();
    return true;
}

template <int R>
spfd_report pcg_graph(Amg &h, const double *b, double *x_out, const spfd_config &cfg, double *h_trace,
                      cudaStream_t s) {
    spfd_report rep{};
    const int64_t n = h.lv[0].nvec;
    double *r = h.kr.get(), *p = h.kp.get(), *q = h.kq.get(), *x = h.kx.get();
    double *sc = h.scal.get();
    SPFD_CUDA(cudaMemsetAsync(x, 0, n * R * sizeof(double), s));
    SPFD_CUDA(cudaMemsetAsync(sc, 0, S_END * sizeof(double), s));
    dot<R>(h, n, b, b, S_BB, F_STORE, s);
    double hs[S_END];
    SPFD_CUDA(cudaMemcpyAsync(hs, sc, S_END * sizeof(double), cudaMemcpyDeviceToHost, s));
    SPFD_CUDA(cudaStreamSynchronize(s));
    double bnorm[2] = {std::sqrt(hs[S_BB]), R > 1 ? std::sqrt(hs[S_BB + 1]) : 0.0};
    for (int c = 0; c < R; ++c)
        if (!std::isfinite(bnorm[c])) { rep.status = SPFD_ENONFINITE; return rep; }
    bool all_zero = true;
    for (int c = 0; c < R; ++c) all_zero = all_zero && bnorm[c] == 0.0;
    if (all_zero) {
        SPFD_CUDA(cudaMemsetAsync(x_out, 0, n * R * sizeof(double), s));
        rep.converged = 1;
        return rep;
    }
    const double tol = cfg.rel_tol;
    int it = 0;
    while (true) {
        // (re)start: r = b - A x, p = 0, alpha = 0, rho initialised by the first body.
        // With x = 0 (first start) r = b bit for bit (b - (+0)); the first solve
        // still runs the stencil once so lazily built kernel data exist before
        // the capture below
        if (it == 0 && h.pcg_exec[R] && h.pcg_kind[R] == fine_kernel_kind())
            SPFD_CUDA(cudaMemcpyAsync(r, b, n * R * sizeof(double), cudaMemcpyDeviceToDevice, s));
        else
            level0_apply<R>(h, 1, false, x, b, r, s);
        // capture after the first fine-level launch: lazily built kernel data
        // (neighbour codes, z-march items) must not be built inside the graph
        if (!pcg_graph_build<R>(h, cfg.max_iters)) return pcg<R>(h, b, x_out, cfg, h_trace, s);
        SPFD_CUDA(cudaMemsetAsync(p, 0, n * R * sizeof(double), s));
        double init[S_END - S_G] = {tol, (double)cfg.max_iters, (double)it, 1.0, 0.0, 0.0, 0.0, 0.0};
        const double zero2[2] = {0.0, 0.0}, ones[2] = {1.0, 1.0};
        SPFD_CUDA(cudaMemcpyAsync(sc + S_G, init, sizeof(init), cudaMemcpyHostToDevice, s));
        SPFD_CUDA(cudaMemcpyAsync(sc + S_ALPHA, zero2, R * sizeof(double), cudaMemcpyHostToDevice, s));
        SPFD_CUDA(cudaMemcpyAsync(sc + S_ACTIVE, ones, R * sizeof(double), cudaMemcpyHostToDevice, s));
        SPFD_CUDA(cudaEventRecord(h.ev_alpha, s));          // the graph runs on the private capture
        SPFD_CUDA(cudaStreamWaitEvent(h.cap, h.ev_alpha, 0)); // stream ordered after this prologue
        SPFD_CUDA(cudaGraphLaunch(h.pcg_exec[R], h.cap));
        SPFD_CUDA(cudaEventRecord(h.ev_x, h.cap));
        SPFD_CUDA(cudaStreamWaitEvent(s, h.ev_x, 0));
        // the last iteration's x += alpha p
        k_update_x<R><<<grid_for(n, 256, 148 * 8), 256, 0, s>>>(n, sc, x, p);
        SPFD_LAUNCH_CHECK();
        SPFD_CUDA(cudaMemcpyAsync(hs, sc, S_END * sizeof(double), cudaMemcpyDeviceToHost, s));
        SPFD_CUDA(cudaStreamSynchronize(s));
        const int nit = (int)hs[S_G_IT];
        for (int64_t k = 0; k < (int64_t)(nit - it) * h.pcg_body_launches[R]; ++k) count_launch();
        if (h_trace && nit > it) {
            const int hi = std::min(nit, cfg.max_iters);
            if (hi > it)
                SPFD_CUDA(cudaMemcpy(h_trace + (int64_t)it * R, h.pcg_trace.get() + (int64_t)it * R,
                                     (size_t)(hi - it) * R * sizeof(double), cudaMemcpyDeviceToHost));
        }
        it = nit;
        if (hs[S_G_STATUS] != 0.0) {
            rep.status = SPFD_ENONFINITE;
            rep.iterations = it;
            return rep;
        }
        // true residual check (linsolve.py:296-298 semantics)
        const int gt = level0_apply<R>(h, 1, true, x, b, q, s);
        finalize<R>(h, gt, S_TMP, F_STORE, s);
        SPFD_CUDA(cudaMemcpyAsync(hs, sc, S_H * sizeof(double), cudaMemcpyDeviceToHost, s));
        SPFD_CUDA(cudaStreamSynchronize(s));
        bool ok = true;
        for (int c = 0; c < R; ++c) {
            const double rel = bnorm[c] > 0 ? std::sqrt(hs[S_TMP + c]) / bnorm[c] : 0.0;
            rep.rel_residual[c] = rel;
            if (!(rel <= tol)) ok = false;
        }
        if (ok || it >= cfg.max_iters) {
            rep.converged = ok ? 1 : 0;
            break;
        }
        // recursive residual drifted: restart from the true residual
    }
    if (x_out != x) SPFD_CUDA(cudaMemcpyAsync(x_out, x, n * R * sizeof(double), cudaMemcpyDeviceToDevice, s));
    rep.iterations = it;
    return rep;
}

}  // namespace

#include "dist.cuh"

void amg_distribute(Amg &h, Comm *comm, int64_t replicate_below, int64_t *range, cudaStream_t s) {
    amg_distribute_impl(h, comm, replicate_below, range, s);
}

void dist_range_exchange(Amg &h, double *v, int nrhs, cudaStream_t s) {
    if (h.dist) range_exchange(*h.dist, v, nrhs, s);
}

void dist_info(const Amg &h, int64_t *out) {
    const Dist &D = *h.dist;
    out[0] = D.pb; out[1] = D.pe; out[2] = D.vrow_b; out[3] = D.vrow_e;
}

Amg::~Amg() {
    delete dist;
    for (auto &e : pcg_exec)
        if (e) cudaGraphExecDestroy(e);
    for (auto &e : fg_exec)
        if (e) cudaGraphExecDestroy(e);
    if (cap) cudaStreamDestroy(cap);
    if (cap2) cudaStreamDestroy(cap2);
    if (side) cudaStreamDestroy(side);
    if (ev_alpha) cudaEventDestroy(ev_alpha);
    if (ev_x) cudaEventDestroy(ev_x);
}

// level-0 interleaved helpers used by FGMRES (R = 1)
namespace {

__global__ void k_axpy_dev(int64_t n, const double *coef, double sign, const double *x, double *y) {
    double a = sign * (*coef);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = fma(a, x[i], y[i]);
}
__global__ void k_scale_inv(int64_t n, const double *norm2, const double *x, double *y) {
    double inv = 1.0 / sqrt(*norm2);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = x[i] * inv;
}
__global__ void k_gather_col(int64_t n, int R, int c, const double *inter, double *one) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        one[i] = inter[i * R + c];
}
__global__ void k_scatter_col(int64_t n, int R, int c, const double *one, double *inter) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        inter[i * R + c] = one[i];
}
__global__ void k_combine(int64_t n, int j, const double *y, const double *zb, double *x) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double acc = 0.0;
        for (int k = 0; k < j; ++k) acc += zb[(int64_t)k * n + i] * y[k];
        x[i] += acc;
    }
}

// ---- batched FGMRES (both rhs of a pair in one Arnoldi process) ----------
// Per Arnoldi step: one V-cycle and one SpMV for both rhs (double2), then
// classical Gram-Schmidt with one re-orthogonalisation (CGS2) as block
// kernels -- k_mdot2 (<V_i, w> and <V_i, v_j> for up to 4 basis vectors per
// launch, fixed-order per-CTA partials), k_mfinal, k_gram_step, k_maxpy
// (w -= sum_i h_i V_i in order i) -- instead of the reference's MGS, which needs 3(j+1) launches
// per step and re-reads w for every basis vector.  Givens rotations, the
// least-squares solve and all convergence decisions stay per rhs on the
// host, as in fgmres1 (linsolve.py:200-298 semantics per rhs).
// Dual block dot: for k < ni, <V_{i0+k}, w> and <V_{i0+k}, v> (v = the
// newest basis vector) in one pass over the basis block; n positions, basis
// vectors ld positions apart (ld > n: a rank's own range of full-length
// vectors).  partials layout [cta][2][NI][R].
template <int R, int NI>
__global__ void __launch_bounds__(256) k_mdot2(int64_t n, int64_t ld, const double *Vb, int i0, int ni,
                                               const double *w, const double *v, double *partials) {
    using W = V<R>;
    __shared__ double red[32 * 2 * NI * R];
    double acc[2 * NI * R];
#pragma unroll
    for (int k = 0; k < 2 * NI * R; ++k) acc[k] = 0.0;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
        const typename W::T wv = W::ld(w, p), vv = W::ld(v, p);
#pragma unroll
        for (int k = 0; k < NI; ++k) {
            if (k < ni) {
                const typename W::T b = W::ld(Vb + (int64_t)(i0 + k) * ld * R, p);
#pragma unroll
                for (int c = 0; c < R; ++c) {
                    acc[k * R + c] = fma(W::comp(b, c), W::comp(wv, c), acc[k * R + c]);
                    acc[(NI + k) * R + c] = fma(W::comp(b, c), W::comp(vv, c), acc[(NI + k) * R + c]);
                }
            }
        }
    }
    block_sum<2 * NI * R>(acc, red);
    if (threadIdx.x == 0)
#pragma unroll
        for (int k = 0; k < 2 * NI * R; ++k) partials[(int64_t)blockIdx.x * 2 * NI * R + k] = acc[k];
}

// Gram-corrected CGS2 coefficients on the device (one block): store the new
// Gram column G[:, j] from the dual block dot, then hsum = h1 + (h1 - G h1)
// for every rhs; raw layout as written by k_mfinal per 4-vector block.
template <int R, int NI2>
__global__ void k_gram_step(const double *raw, int j, int m, double *gram, double *hsum) {
    const int nv = j + 1;
    for (int t = threadIdx.x; t < nv * R; t += blockDim.x) {
        const int i = t / R, c = t % R, blk = i / NI2, k = i % NI2;
        const double gij = raw[(size_t)blk * 2 * NI2 * R + (NI2 + k) * R + c];
        double *G = gram + (size_t)c * (m + 1) * (m + 1);
        G[(size_t)i * (m + 1) + j] = gij;
        G[(size_t)j * (m + 1) + i] = gij;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < nv * R; t += blockDim.x) {
        const int i = t / R, c = t % R;
        const double *G = gram + (size_t)c * (m + 1) * (m + 1);
        auto h1 = [&](int q) { return raw[(size_t)(q / NI2) * 2 * NI2 * R + (q % NI2) * R + c]; };
        double gh = 0.0;
        for (int k = 0; k < nv; ++k) gh += G[(size_t)i * (m + 1) + k] * h1(k);
        const double a = h1(i);
        hsum[(size_t)i * R + c] = a + (a - gh);
    }
}

// out[k] = sum over CTAs of partials[.][k], k < nv (one block per value, fixed order)
__global__ void __launch_bounds__(256) k_mfinal(const double *partials, int nblocks, int stride, double *out) {
    __shared__ double red[32];
    const int k = blockIdx.x;
    double s[1] = {0.0};
    const int per = (nblocks + blockDim.x - 1) / blockDim.x;
    const int b0 = threadIdx.x * per, b1 = min(nblocks, b0 + per);
    for (int b = b0; b < b1; ++b) s[0] += partials[(int64_t)b * stride + k];
    block_sum<1>(s, red);
    if (threadIdx.x == 0) out[k] = s[0];
}

// w -= sum_{i < nv} h[i] V_i  (h: [nv][R] on the device, applied in order i;
// basis vectors ld positions apart)
template <int R>
__global__ void k_maxpy(int64_t n, int64_t ld, const double *Vb, int nv, const double *hv, double *w) {
    using W = V<R>;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
        typename W::T acc = W::ld(w, p);
        for (int i = 0; i < nv; ++i) {
            double nh[R];
#pragma unroll
            for (int c = 0; c < R; ++c) nh[c] = -hv[i * R + c];
            acc = vfma<R>(nh, W::ld(Vb + (int64_t)i * ld * R, p), acc);
        }
        W::st(w, p, acc);
    }
}

// y = x * mult[c] per component
template <int R>
__global__ void k_scale_r(int64_t n, const double *mult, const double *x, double *y) {
    using W = V<R>;
    double mu[R];
#pragma unroll
    for (int c = 0; c < R; ++c) mu[c] = mult[c];
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
        typename W::T v = W::ld(x, p);
        if constexpr (R == 1) v = v * mu[0];
        else v = make_double2(v.x * mu[0], v.y * mu[1]);
        W::st(y, p, v);
    }
}

// x[:, c] += sum_{k < jc[c]} Z_k[:, c] y[c][k]  (Z_k ld positions apart)
template <int R>
__global__ void k_combine_r(int64_t n, int64_t ld, int m, const int *jc, const double *y, const double *Zb,
                            double *x) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
        for (int c = 0; c < R; ++c) {
            double acc = 0.0;
            for (int k = 0; k < jc[c]; ++k) acc += Zb[((int64_t)k * ld + p) * R + c] * y[c * m + k];
            x[p * R + c] += acc;
        }
    }
}

#include "fgmres_graph.cuh"

template <int R>
spfd_report fgmres_batch(Amg &h, const double *b, double *x, const spfd_config &cfg, double *h_trace,
                         cudaStream_t s) {
    spfd_report rep{};
    const int64_t n = h.lv[0].nvec;
    const int m = cfg.restart;
    SPFD_CHECK(m >= 1 && m <= 31, SPFD_EINVAL, "restart must be in [1, 31] for batched FGMRES");
    if (h.fg_m < m || h.fg_R < R) {
        h.fg_basis.alloc((int64_t)(m + 1) * n * R);
        h.fg_prec.alloc((int64_t)m * n * R);
        h.fg_m = m;
        h.fg_R = R;
    }
    double *Vb = h.fg_basis.get(), *Zb = h.fg_prec.get();
    double *w = h.kq.get(), *r = h.kr.get();
    double *sc = h.scal.get();
    const int G = grid_for(n, 256, 148 * 16);
    const int SH1 = S_H, SH2 = S_H + 128, SMUL = S_TMP + 2;  // pass-1 / pass-2 columns, scale factors
    SPFD_CUDA(cudaMemsetAsync(x, 0, n * R * sizeof(double), s));
    SPFD_CUDA(cudaMemsetAsync(sc, 0, S_END * sizeof(double), s));
    dot<R>(h, n, b, b, S_BB, F_STORE, s);
    double hb[R];
    SPFD_CUDA(cudaMemcpyAsync(hb, sc + S_BB, R * sizeof(double), cudaMemcpyDeviceToHost, s));
    SPFD_CUDA(cudaStreamSynchronize(s));
    double bnorm[R];
    bool done[R], all = true;
    for (int c = 0; c < R; ++c) {
        bnorm[c] = std::sqrt(hb[c]);
        if (!std::isfinite(bnorm[c])) { rep.status = SPFD_ENONFINITE; return rep; }
        done[c] = bnorm[c] == 0.0;
        all = all && done[c];
        rep.rel_residual[c] = 0.0;
    }
    if (all) { rep.converged = 1; return rep; }
    std::vector<double> H[R], cs[R], sn[R], g[R];
    fg_small_alloc(h);  // per-rhs Gram matrix, y and jc live in the hierarchy (no per-solve allocation)
    DevBuf<double> &gram = h.fg_gram;
    for (int c = 0; c < R; ++c) {
        H[c].assign((size_t)(m + 1) * m, 0.0);
        cs[c].assign(m, 0.0); sn[c].assign(m, 0.0); g[c].assign(m + 1, 0.0);
    }
    DevBuf<double> &ydev = h.fg_y;
    DevBuf<int> &jcdev = h.fg_jc;
    const int nparts = kDotGrid;
    int its = 0;
    int its_c[R];  // iterations each rhs took part in (fgmres1's count per rhs)
    for (int c = 0; c < R; ++c) its_c[c] = 0;
    while (its < cfg.max_iters) {
        // restart: true residual per rhs (linsolve.py:244-248)
        level0_apply<R>(h, 1, false, x, b, r, s);
        dot<R>(h, n, r, r, S_TMP, F_STORE, s);
        double rr[R];
        SPFD_CUDA(cudaMemcpyAsync(rr, sc + S_TMP, R * sizeof(double), cudaMemcpyDeviceToHost, s));
        SPFD_CUDA(cudaStreamSynchronize(s));
        bool active[R], any = false;
        double mult[R];
        for (int c = 0; c < R; ++c) {
            const double beta = std::sqrt(rr[c]);
            const double rel = bnorm[c] > 0 ? beta / bnorm[c] : 0.0;
            if (rel <= cfg.rel_tol) done[c] = true;  // converged on the true residual
            active[c] = !done[c];
            any = any || active[c];
            std::fill(H[c].begin(), H[c].end(), 0.0);
            std::fill(g[c].begin(), g[c].end(), 0.0);
            g[c][0] = beta;
            mult[c] = active[c] ? 1.0 / beta : 0.0;
        }
        if (!any) break;
        SPFD_CUDA(cudaMemsetAsync(gram.get(), 0, (size_t)R * (m + 1) * (m + 1) * sizeof(double), s));
        SPFD_CUDA(cudaMemcpyAsync(sc + SMUL, mult, R * sizeof(double), cudaMemcpyHostToDevice, s));
        k_scale_r<R><<<G, 256, 0, s>>>(n, sc + SMUL, r, Vb);
        int jc[R];
        for (int c = 0; c < R; ++c) jc[c] = 0;
        int j = 0;
        while (j < m && its < cfg.max_iters) {
            double *vj = Vb + (int64_t)j * n * R, *zj = Zb + (int64_t)j * n * R;
            amg_vcycle(h, vj, zj, R, s);
            level0_apply<R>(h, 0, false, zj, nullptr, w, s);
            // Gram-corrected CGS2 (two passes over the basis instead of four):
            // one dual block dot gives h1 = V^T w and the new Gram column
            // G[:, j] = V^T v_j; the re-orthogonalisation coefficients follow
            // on the host, h2 = V^T (w - V h1) = h1 - G h1, and one block
            // update forms w - V (h1 + h2) -- CGS2 in exact arithmetic.
            constexpr int NI2 = 4;
            for (int i0 = 0; i0 <= j; i0 += NI2) {
                const int ni = std::min(NI2, j + 1 - i0);
                k_mdot2<R, NI2><<<nparts, 256, 0, s>>>(n, n, Vb, i0, ni, w, vj, h.partials.get());
                k_mfinal<<<2 * NI2 * R, 256, 0, s>>>(h.partials.get(), nparts, 2 * NI2 * R, sc + SH1 + 2 * i0 * R);
                SPFD_LAUNCH_CHECK();
            }
            // the re-orthogonalisation coefficients and the Gram column on the device
            k_gram_step<R, NI2><<<1, 256, 0, s>>>(sc + SH1, j, m, gram.get(), sc + SH2);
            k_maxpy<R><<<G, 256, 0, s>>>(n, n, Vb, j + 1, sc + SH2, w);
            SPFD_LAUNCH_CHECK();
            dot<R>(h, n, w, w, S_TMP, F_STORE, s);
            std::vector<double> hcol((size_t)(j + 1) * R);
            double nn[R];
            SPFD_CUDA(cudaMemcpyAsync(hcol.data(), sc + SH2, hcol.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
            SPFD_CUDA(cudaMemcpyAsync(nn, sc + S_TMP, R * sizeof(double), cudaMemcpyDeviceToHost, s));
            SPFD_CUDA(cudaStreamSynchronize(s));
            ++its;
            bool more = false;
            for (int c = 0; c < R; ++c) {
                if (!active[c]) { mult[c] = 0.0; continue; }
                ++its_c[c];
                const double hn = std::sqrt(nn[c]);
                if (!std::isfinite(hn)) { rep.status = SPFD_ENONFINITE; rep.iterations = its; return rep; }
                auto &Hc = H[c];
                for (int i = 0; i <= j; ++i) Hc[(size_t)i * m + j] = hcol[(size_t)i * R + c];
                for (int i = 0; i < j; ++i) {
                    const double t1 = cs[c][i] * Hc[(size_t)i * m + j] + sn[c][i] * Hc[(size_t)(i + 1) * m + j];
                    const double t2 = -sn[c][i] * Hc[(size_t)i * m + j] + cs[c][i] * Hc[(size_t)(i + 1) * m + j];
                    Hc[(size_t)i * m + j] = t1;
                    Hc[(size_t)(i + 1) * m + j] = t2;
                }
                const double den = std::hypot(Hc[(size_t)j * m + j], hn);
                if (den == 0.0) { cs[c][j] = 1.0; sn[c][j] = 0.0; }
                else { cs[c][j] = Hc[(size_t)j * m + j] / den; sn[c][j] = hn / den; }
                Hc[(size_t)j * m + j] = cs[c][j] * Hc[(size_t)j * m + j] + sn[c][j] * hn;
                g[c][j + 1] = -sn[c][j] * g[c][j];
                g[c][j] = cs[c][j] * g[c][j];
                jc[c] = j + 1;
                const double est = std::fabs(g[c][j + 1]) / bnorm[c];
                if (h_trace && its <= cfg.max_iters) h_trace[(int64_t)(its - 1) * R + c] = est;
                if (hn == 0.0 || est <= cfg.rel_tol) {
                    active[c] = false;
                    mult[c] = 0.0;
                } else {
                    mult[c] = 1.0 / hn;
                    more = true;
                }
            }
            ++j;
            if (!more) break;
            if (j < m) {
                SPFD_CUDA(cudaMemcpyAsync(sc + SMUL, mult, R * sizeof(double), cudaMemcpyHostToDevice, s));
                k_scale_r<R><<<G, 256, 0, s>>>(n, sc + SMUL, w, Vb + (int64_t)j * n * R);
                SPFD_LAUNCH_CHECK();
            }
        }
        // least squares per rhs and the update x += Z y
        std::vector<double> y((size_t)R * m, 0.0);
        for (int c = 0; c < R; ++c) {
            const int jj = jc[c];
            for (int i = jj - 1; i >= 0; --i) {  // back substitution
                double acc = g[c][i];
                for (int k = i + 1; k < jj; ++k) acc -= H[c][(size_t)i * m + k] * y[(size_t)c * m + k];
                y[(size_t)c * m + i] = acc / H[c][(size_t)i * m + i];
            }
            for (int i = 0; i < jj; ++i)
                if (!std::isfinite(y[(size_t)c * m + i])) { rep.status = SPFD_ENONFINITE; rep.iterations = its; return rep; }
        }
        SPFD_CUDA(cudaMemcpyAsync(ydev.get(), y.data(), y.size() * sizeof(double), cudaMemcpyHostToDevice, s));
        SPFD_CUDA(cudaMemcpyAsync(jcdev.get(), jc, R * sizeof(int), cudaMemcpyHostToDevice, s));
        k_combine_r<R><<<G, 256, 0, s>>>(n, n, m, jcdev.get(), ydev.get(), Zb, x);
        SPFD_LAUNCH_CHECK();
    }
    // true residual at exit (linsolve.py:296-298)
    level0_apply<R>(h, 1, false, x, b, r, s);
    dot<R>(h, n, r, r, S_TMP, F_STORE, s);
    double rr[R];
    SPFD_CUDA(cudaMemcpyAsync(rr, sc + S_TMP, R * sizeof(double), cudaMemcpyDeviceToHost, s));
    SPFD_CUDA(cudaStreamSynchronize(s));
    rep.converged = 1;
    int itmax = 0;
    for (int c = 0; c < R; ++c) {
        const double rel = bnorm[c] > 0 ? std::sqrt(rr[c]) / bnorm[c] : 0.0;
        rep.rel_residual[c] = rel;
        if (!(rel <= cfg.rel_tol)) rep.converged = 0;
        itmax = std::max(itmax, its_c[c]);
    }
    rep.iterations = itmax;
    return rep;
}

// Distributed FGMRES(m) (linsolve.py:200-298) over the z-slab ranks: the
// batched Arnoldi process of fgmres_batch on each rank's own positions of
// full-length vectors.  The V-cycle and the operator are the distributed ones
// (halo exchange inside); every inner product -- the dual block dot of the
// Gram-corrected CGS2 and the norms -- is a per-rank partial, allgathered and
// summed in rank order, so every rank holds the same Hessenberg column and
// takes the same Givens / restart decisions on the host.
template <int R>
spfd_report fgmres_dist(Amg &h, const double *b, double *x, const spfd_config &cfg, double *h_trace,
                        cudaStream_t s) {
    Dist &D = *h.dist;
    spfd_report rep{};
    const int64_t n = h.lv[0].nvec;
    const int64_t no = D.pe - D.pb, off = D.pb * R;
    const int m = cfg.restart;
    SPFD_CHECK(m >= 1 && m <= 31, SPFD_EINVAL, "restart must be in [1, 31] for the distributed FGMRES");
    if (h.fg_m < m || h.fg_R < R) {
        h.fg_basis.alloc((int64_t)(m + 1) * n * R);
        h.fg_prec.alloc((int64_t)m * n * R);
        h.fg_m = m;
        h.fg_R = R;
    }
    constexpr int NI2 = 4;
    const int raw_max = (m + NI2) / NI2 * 2 * NI2 * R;  // dual-dot values of the largest column
    if ((int64_t)D.hgather.n < (int64_t)raw_max * D.size) D.hgather.alloc((int64_t)raw_max * D.size);
    double *Vb = h.fg_basis.get(), *Zb = h.fg_prec.get();
    double *w = h.kq.get(), *r = h.kr.get();
    double *sc = h.scal.get();
    const int G = grid_for(no, 256, 148 * 16);
    const int SH1 = S_H, SH2 = S_H + 128, SMUL = S_TMP + 2;
    SPFD_CUDA(cudaMemsetAsync(x, 0, n * R * sizeof(double), s));
    SPFD_CUDA(cudaMemsetAsync(sc, 0, S_END * sizeof(double), s));
    dot_dist<R>(h, b, b, S_BB, F_STORE, s);
    double hb[R];
    SPFD_CUDA(cudaMemcpyAsync(hb, sc + S_BB, R * sizeof(double), cudaMemcpyDeviceToHost, s));
    SPFD_CUDA(cudaStreamSynchronize(s));
    double bnorm[R];
    bool done[R], all = true;
    for (int c = 0; c < R; ++c) {
        bnorm[c] = std::sqrt(hb[c]);
        if (!std::isfinite(bnorm[c])) { rep.status = SPFD_ENONFINITE; return rep; }
        done[c] = bnorm[c] == 0.0;
        all = all && done[c];
    }
    if (all) { rep.converged = 1; return rep; }
    std::vector<double> H[R], cs[R], sn[R], g[R];
    fg_small_alloc(h);
    for (int c = 0; c < R; ++c) {
        H[c].assign((size_t)(m + 1) * m, 0.0);
        cs[c].assign(m, 0.0); sn[c].assign(m, 0.0); g[c].assign(m + 1, 0.0);
    }
    int its = 0, its_c[R];
    for (int c = 0; c < R; ++c) its_c[c] = 0;
    while (its < cfg.max_iters) {
        apply_dist<R>(h, 1, false, x, b, r, s);  // r = b - A x (own range)
        dot_dist<R>(h, r, r, S_TMP, F_STORE, s);
        double rr[R];
        SPFD_CUDA(cudaMemcpyAsync(rr, sc + S_TMP, R * sizeof(double), cudaMemcpyDeviceToHost, s));
        SPFD_CUDA(cudaStreamSynchronize(s));
        bool active[R], any = false;
        double mult[R];
        for (int c = 0; c < R; ++c) {
            const double beta = std::sqrt(rr[c]);
            if ((bnorm[c] > 0 ? beta / bnorm[c] : 0.0) <= cfg.rel_tol) done[c] = true;
            active[c] = !done[c];
            any = any || active[c];
            std::fill(H[c].begin(), H[c].end(), 0.0);
            std::fill(g[c].begin(), g[c].end(), 0.0);
            g[c][0] = beta;
            mult[c] = active[c] ? 1.0 / beta : 0.0;
        }
        if (!any) break;
        SPFD_CUDA(cudaMemsetAsync(h.fg_gram.get(), 0, (size_t)R * (m + 1) * (m + 1) * sizeof(double), s));
        SPFD_CUDA(cudaMemcpyAsync(sc + SMUL, mult, R * sizeof(double), cudaMemcpyHostToDevice, s));
        k_scale_r<R><<<G, 256, 0, s>>>(no, sc + SMUL, r + off, Vb + off);
        int jc[R];
        for (int c = 0; c < R; ++c) jc[c] = 0;
        int j = 0;
        while (j < m && its < cfg.max_iters) {
            double *vj = Vb + (int64_t)j * n * R, *zj = Zb + (int64_t)j * n * R;
            vcycle_dist_fine<R>(h, vj, zj, s);
            apply_dist<R>(h, 0, false, zj, nullptr, w, s);
            // per-rank dual block dots into SH2, gathered and summed in rank
            // order into SH1 (the layout k_gram_step reads)
            const int nblk = j / NI2 + 1, nraw = nblk * 2 * NI2 * R;
            for (int i0 = 0; i0 <= j; i0 += NI2) {
                const int ni = std::min(NI2, j + 1 - i0);
                k_mdot2<R, NI2><<<kDotGrid, 256, 0, s>>>(no, n, Vb + off, i0, ni, w + off, vj + off,
                                                        h.partials.get());
                k_mfinal<<<2 * NI2 * R, 256, 0, s>>>(h.partials.get(), kDotGrid, 2 * NI2 * R, sc + SH2 + 2 * i0 * R);
                SPFD_LAUNCH_CHECK();
            }
            D.comm->allgather(sc + SH2, D.hgather.get(), nraw * sizeof(double), s);
            k_rank_sum<<<1, 256, 0, s>>>(D.hgather.get(), D.size, nraw, 1, sc + SH1, nullptr, nullptr);
            k_gram_step<R, NI2><<<1, 256, 0, s>>>(sc + SH1, j, m, h.fg_gram.get(), sc + SH2);
            k_maxpy<R><<<G, 256, 0, s>>>(no, n, Vb + off, j + 1, sc + SH2, w + off);
            SPFD_LAUNCH_CHECK();
            dot_dist<R>(h, w, w, S_TMP, F_STORE, s);
            std::vector<double> hcol((size_t)(j + 1) * R);
            double nn[R];
            SPFD_CUDA(cudaMemcpyAsync(hcol.data(), sc + SH2, hcol.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
            SPFD_CUDA(cudaMemcpyAsync(nn, sc + S_TMP, R * sizeof(double), cudaMemcpyDeviceToHost, s));
            SPFD_CUDA(cudaStreamSynchronize(s));
            ++its;
            bool more = false;
            for (int c = 0; c < R; ++c) {
                if (!active[c]) { mult[c] = 0.0; continue; }
                ++its_c[c];
                const double hn = std::sqrt(nn[c]);
                if (!std::isfinite(hn)) { rep.status = SPFD_ENONFINITE; rep.iterations = its; return rep; }
                auto &Hc = H[c];
                for (int i = 0; i <= j; ++i) Hc[(size_t)i * m + j] = hcol[(size_t)i * R + c];
                for (int i = 0; i < j; ++i) {
                    const double t1 = cs[c][i] * Hc[(size_t)i * m + j] + sn[c][i] * Hc[(size_t)(i + 1) * m + j];
                    const double t2 = -sn[c][i] * Hc[(size_t)i * m + j] + cs[c][i] * Hc[(size_t)(i + 1) * m + j];
                    Hc[(size_t)i * m + j] = t1;
                    Hc[(size_t)(i + 1) * m + j] = t2;
                }
                const double den = std::hypot(Hc[(size_t)j * m + j], hn);
                if (den == 0.0) { cs[c][j] = 1.0; sn[c][j] = 0.0; }
                else { cs[c][j] = Hc[(size_t)j * m + j] / den; sn[c][j] = hn / den; }
                Hc[(size_t)j * m + j] = cs[c][j] * Hc[(size_t)j * m + j] + sn[c][j] * hn;
                g[c][j + 1] = -sn[c][j] * g[c][j];
                g[c][j] = cs[c][j] * g[c][j];
                jc[c] = j + 1;
                const double est = std::fabs(g[c][j + 1]) / bnorm[c];
                if (h_trace && its <= cfg.max_iters) h_trace[(int64_t)(its - 1) * R + c] = est;
                if (hn == 0.0 || est <= cfg.rel_tol) {
                    active[c] = false;
                    mult[c] = 0.0;
                } else {
                    mult[c] = 1.0 / hn;
                    more = true;
                }
            }
            ++j;
            if (!more) break;
            if (j < m) {
                SPFD_CUDA(cudaMemcpyAsync(sc + SMUL, mult, R * sizeof(double), cudaMemcpyHostToDevice, s));
                k_scale_r<R><<<G, 256, 0, s>>>(no, sc + SMUL, w + off, Vb + (int64_t)j * n * R + off);
                SPFD_LAUNCH_CHECK();
            }
        }
        std::vector<double> y((size_t)R * m, 0.0);
        for (int c = 0; c < R; ++c) {
            const int jj = jc[c];
            for (int i = jj - 1; i >= 0; --i) {
                double acc = g[c][i];
                for (int k = i + 1; k < jj; ++k) acc -= H[c][(size_t)i * m + k] * y[(size_t)c * m + k];
                y[(size_t)c * m + i] = acc / H[c][(size_t)i * m + i];
            }
            for (int i = 0; i < jj; ++i)
                if (!std::isfinite(y[(size_t)c * m + i])) { rep.status = SPFD_ENONFINITE; rep.iterations = its; return rep; }
        }
        SPFD_CUDA(cudaMemcpyAsync(h.fg_y.get(), y.data(), y.size() * sizeof(double), cudaMemcpyHostToDevice, s));
        SPFD_CUDA(cudaMemcpyAsync(h.fg_jc.get(), jc, R * sizeof(int), cudaMemcpyHostToDevice, s));
        k_combine_r<R><<<G, 256, 0, s>>>(no, n, m, h.fg_jc.get(), h.fg_y.get(), Zb + off, x + off);
        SPFD_LAUNCH_CHECK();
    }
    apply_dist<R>(h, 1, false, x, b, r, s);
    dot_dist<R>(h, r, r, S_TMP, F_STORE, s);
    double rr[R];
    SPFD_CUDA(cudaMemcpyAsync(rr, sc + S_TMP, R * sizeof(double), cudaMemcpyDeviceToHost, s));
    SPFD_CUDA(cudaStreamSynchronize(s));
    rep.converged = 1;
    int itmax = 0;
    for (int c = 0; c < R; ++c) {
        const double rel = bnorm[c] > 0 ? std::sqrt(rr[c]) / bnorm[c] : 0.0;
        rep.rel_residual[c] = rel;
        if (!(rel <= cfg.rel_tol)) rep.converged = 0;
        itmax = std::max(itmax, its_c[c]);
    }
    // leave x valid on the halo planes too (the E-field reads one plane beyond)
    range_exchange(D, x, R, s);
    rep.iterations = itmax;
    return rep;
}

// FGMRES(m) for one rhs in R=1 layout (linsolve.py:200-298).
spfd_report fgmres1(Amg &h, const double *b, double *x, const spfd_config &cfg, double *h_trace, cudaStream_t s) {
    spfd_report rep{};
    int64_t n = h.lv[0].nvec;
    int m = cfg.restart;
    SPFD_CHECK(m >= 1 && m <= 200, SPFD_EINVAL, "restart must be in [1, 200]");
    if (h.fg_m < m) {
        h.fg_basis.alloc((int64_t)(m + 1) * n);
        h.fg_prec.alloc((int64_t)m * n);
        h.fg_m = m;
    }
    double *V = h.fg_basis.get(), *Z = h.fg_prec.get();
    double *w = h.kq.get(), *r = h.kr.get();
    double *sc = h.scal.get();
    const int G = grid_for(n, 256, 148 * 16);
    SPFD_CUDA(cudaMemsetAsync(x, 0, n * sizeof(double), s));
    SPFD_CUDA(cudaMemsetAsync(sc, 0, (S_H + 64) * sizeof(double), s));
    double one = 1.0;
    SPFD_CUDA(cudaMemcpyAsync(sc + S_ACTIVE, &one, sizeof(double), cudaMemcpyHostToDevice, s));
    dot<1>(h, n, b, b, S_BB, F_STORE, s);
    double hb;
    SPFD_CUDA(cudaMemcpyAsync(&hb, sc + S_BB, sizeof(double), cudaMemcpyDeviceToHost, s));
    SPFD_CUDA(cudaStreamSynchronize(s));
    double bnorm = std::sqrt(hb);
    if (!std::isfinite(bnorm)) { rep.status = SPFD_ENONFINITE; return rep; }
    if (bnorm == 0.0) { rep.converged = 1; return rep; }
    std::vector<double> H((size_t)(m + 1) * m), cs(m), sn(m), g(m + 1);
    int its = 0;
    double rel = INFINITY;
    DevBuf<double> ydev;
    ydev.alloc(m + 1);
    while (its < cfg.max_iters) {
        level0_apply<1>(h, 1, false, x, b, r, s);  // r = b - A x
        dot<1>(h, n, r, r, S_TMP, F_STORE, s);
        double rr;
        SPFD_CUDA(cudaMemcpyAsync(&rr, sc + S_TMP, sizeof(double), cudaMemcpyDeviceToHost, s));
        SPFD_CUDA(cudaStreamSynchronize(s));
        double beta = std::sqrt(rr);
        rel = beta / bnorm;
        if (rel <= cfg.rel_tol) {
            rep.iterations = its; rep.rel_residual[0] = rel; rep.converged = 1;
            return rep;
        }
        std::fill(H.begin(), H.end(), 0.0);
        std::fill(g.begin(), g.end(), 0.0);
        g[0] = beta;
        k_scale_inv<<<G, 256, 0, s>>>(n, sc + S_TMP, r, V);
        int j = 0;
        while (j < m && its < cfg.max_iters) {
            double *vj = V + (int64_t)j * n, *zj = Z + (int64_t)j * n;
            amg_vcycle(h, vj, zj, 1, s);
            level0_apply<1>(h, 0, false, zj, nullptr, w, s);
            for (int i = 0; i <= j; ++i) {  // modified Gram-Schmidt
                dot<1>(h, n, V + (int64_t)i * n, w, S_H + i, F_STORE, s);
                k_axpy_dev<<<G, 256, 0, s>>>(n, sc + S_H + i, -1.0, V + (int64_t)i * n, w);
            }
            dot<1>(h, n, w, w, S_H + j + 1, F_STORE, s);
            std::vector<double> col(j + 2);
            SPFD_CUDA(cudaMemcpyAsync(col.data(), sc + S_H, (j + 2) * sizeof(double), cudaMemcpyDeviceToHost, s));
            SPFD_CUDA(cudaStreamSynchronize(s));
            double hn = std::sqrt(col[j + 1]);
            if (!std::isfinite(hn)) { rep.status = SPFD_ENONFINITE; rep.iterations = its; return rep; }
            for (int i = 0; i <= j; ++i) H[(size_t)i * m + j] = col[i];
            for (int i = 0; i < j; ++i) {
                double t1 = cs[i] * H[(size_t)i * m + j] + sn[i] * H[(size_t)(i + 1) * m + j];
                double t2 = -sn[i] * H[(size_t)i * m + j] + cs[i] * H[(size_t)(i + 1) * m + j];
                H[(size_t)i * m + j] = t1;
                H[(size_t)(i + 1) * m + j] = t2;
            }
            double den = std::hypot(H[(size_t)j * m + j], hn);
            if (den == 0.0) { cs[j] = 1.0; sn[j] = 0.0; }
            else { cs[j] = H[(size_t)j * m + j] / den; sn[j] = hn / den; }
            H[(size_t)j * m + j] = cs[j] * H[(size_t)j * m + j] + sn[j] * hn;
            g[j + 1] = -sn[j] * g[j];
            g[j] = cs[j] * g[j];
            ++its;
            ++j;
            double est = std::fabs(g[j]) / bnorm;
            if (h_trace) h_trace[its - 1] = est;
            if (hn == 0.0 || est <= cfg.rel_tol) break;
            if (j < m) k_scale_inv<<<G, 256, 0, s>>>(n, sc + S_H + j, w, V + (int64_t)j * n);
        }
        if (j > 0) {
            std::vector<double> y(j);
            for (int i = j - 1; i >= 0; --i) {  // back substitution
                double acc = g[i];
                for (int k = i + 1; k < j; ++k) acc -= H[(size_t)i * m + k] * y[k];
                y[i] = acc / H[(size_t)i * m + i];
            }
            for (double v : y)
                if (!std::isfinite(v)) { rep.status = SPFD_ENONFINITE; rep.iterations = its; return rep; }
            SPFD_CUDA(cudaMemcpyAsync(ydev.get(), y.data(), j * sizeof(double), cudaMemcpyHostToDevice, s));
            k_combine<<<G, 256, 0, s>>>(n, j, ydev.get(), Z, x);
            SPFD_LAUNCH_CHECK();
        }
    }
    level0_apply<1>(h, 1, false, x, b, r, s);
    dot<1>(h, n, r, r, S_TMP, F_STORE, s);
    double rr;
    SPFD_CUDA(cudaMemcpyAsync(&rr, sc + S_TMP, sizeof(double), cudaMemcpyDeviceToHost, s));
    SPFD_CUDA(cudaStreamSynchronize(s));
    rel = std::sqrt(rr) / bnorm;
    rep.iterations = its;
    rep.rel_residual[0] = rel;
    rep.converged = rel <= cfg.rel_tol;
    return rep;
}

}  // namespace

// Back-to-back launches of one level-0 kernel between two events on `s`
// (bench.py roofline).  Returns ms per launch; *bytes = algorithmic bytes
// per launch (each distinct array read or written once).
// Algorithmic bytes per launch of the solve's kernels (each distinct array
// counted once per launch; R = rhs batched).
namespace {
double csr_bytes(const Csr &m) { return m.rows > 0 ? 12.0 * (double)m.nnz + 8.0 * (double)(m.rows + 1) : 0.0; }

struct KernelBytes {
    double spmv = 0, presmooth = 0, postsmooth = 0, prolong = 0, aggsum = 0, blas1 = 0;
    double l1_pre = 0, l1_pp = 0;
};

KernelBytes kernel_bytes(const Amg &h, double R) {
    KernelBytes k;
    const double n = (double)h.lv[0].nvec;
    k.blas1 = n * 24.0 * R;  // r update / x update / p update: read 2, write 1
    if (h.structured) {
        const double mask = n / 8.0;
        k.spmv = n * (24.0 + 16.0 * R) + mask;          // w; x -> y
        k.presmooth = n * (32.0 + 16.0 * R) + mask;     // w, odinv; r -> d
        k.postsmooth = n * (32.0 + 24.0 * R) + mask;    // w, odinv; x, r -> x'
        if (h.lv.size() > 1) {
            const double n1 = (double)h.lv[1].n;
            k.prolong = h.lv[0].Pspan.rows
                            ? csr_bytes(h.lv[0].Pspan) + n * (8.0 + 16.0 * R) + n1 * 8.0 * R  // P; odinv; r -> x1; e_c
                            : n * (36.0 + 16.0 * R) + mask + n1 * 8.0 * R;  // w, odinv, agg; r -> x1; e_c
            k.aggsum = h.lv[0].Rspan.rows
                           ? csr_bytes(h.lv[0].Rspan) + n * 8.0 * R + n1 * (8.0 + 16.0 * R)  // R; d; od_c -> r_c, x0_c
                           : n * (4.0 + 8.0 * R) + n1 * (8.0 + 8.0 + 16.0 * R);  // members, u; ptr, od_c -> r_c, x0_c
        }
    } else {
        const Level &L = h.lv[0];
        k.spmv = csr_bytes(L.A) + n * 16.0 * R;
        k.presmooth = csr_bytes(L.A) + n * (8.0 + 16.0 * R);
        k.postsmooth = csr_bytes(L.A) + n * (8.0 + 24.0 * R);
    }
    if (h.lv.size() > 2) {
        const Level &L = h.lv[1];
        const double n1 = (double)L.n, n2 = (double)h.lv[2].n;
        k.l1_pre = csr_bytes(L.A) + n1 * 24.0 * R;                              // r, x0 -> d
        if (L.Q.rows > 0) k.l1_pp = csr_bytes(L.Q) + n1 * (8.0 + 32.0 * R) + n2 * 8.0 * R;  // Q; od, r, d -> z; e
        else if (L.AP.rows > 0) k.l1_pp = csr_bytes(L.P) + csr_bytes(L.AP) + n1 * (8.0 + 32.0 * R) + n2 * 8.0 * R;
    }
    return k;
}

// one V-cycle below level 0 (CSR levels) + the coarsest dense solve
double coarse_vcycle_bytes(const Amg &h, int l0, double R) {
    double b = 0.0;
    const int nl = (int)h.lv.size();
    for (int l = l0; l < nl - 1; ++l) {
        const Level &L = h.lv[l];
        const double n = (double)L.n, nc = (double)h.lv[l + 1].n;
        b += csr_bytes(L.A) + n * 24.0 * R;                         // pre-smooth residual
        b += csr_bytes(L.R) + n * 8.0 * R + nc * (8.0 + 16.0 * R);  // restriction (+ od r_c)
        if (L.Q.rows > 0 && h.pre == 1 && h.post == 1) b += csr_bytes(L.Q) + n * (8.0 + 32.0 * R) + nc * 8.0 * R;
        else if (L.AP.rows > 0 && h.pre == 1 && h.post == 1) b += csr_bytes(L.P) + csr_bytes(L.AP) + n * (8.0 + 32.0 * R) + nc * 8.0 * R;
        else b += csr_bytes(L.P) + csr_bytes(L.A) + n * (8.0 + 56.0 * R) + nc * 8.0 * R;
    }
    b += (double)h.nc * (double)h.nc * 8.0 + (double)h.nc * 16.0 * R;
    return b;
}
}  // namespace

double amg_iteration_bytes(const Amg &h, int nrhs) {
    const double R = nrhs;
    const KernelBytes k = kernel_bytes(h, R);
    // q = A p; r, x, p updates (x and p fused: 5 arrays instead of 6)
    double b = k.spmv + (pcg_fuse_x() ? 1.0 + 5.0 / 3.0 : 3.0) * k.blas1;
    if (h.lv.size() == 1) return b + coarse_vcycle_bytes(h, 0, R);
    const double pos = h.structured ? (double)h.op->L : 0.0;
    if (h.structured)
        b += (h.lv[0].Rspan.rows ? 1.0 : 2.0) * k.presmooth + k.aggsum + k.prolong + k.postsmooth +
             coarse_vcycle_bytes(h, 1, R);
    else b += coarse_vcycle_bytes(h, 0, R);
    return b;
}

double amg_bench_kernel(Amg &h, int which, int reps, int nrhs, double *bytes, cudaStream_t s) {
    SPFD_CHECK(nrhs >= 1 && nrhs <= h.max_nrhs && reps >= 1, SPFD_EINVAL, "bad bench arguments");
    Level &L = h.lv[0];
    int64_t n = L.nvec;
    const bool two = h.lv.size() > 1, three = h.lv.size() > 2;
    SPFD_CHECK(!(which == 4 || which == 5) || (h.structured && two), SPFD_EINVAL,
               "kernel needs a structured hierarchy with a coarse level");
    SPFD_CHECK(!(which == 6 || which == 7) || three, SPFD_EINVAL, "kernel needs three levels");
    SPFD_CHECK(which != 7 || h.lv[1].AP.rows > 0, SPFD_EINVAL, "level 1 has no fused prolongation");
    SPFD_CUDA(cudaMemsetAsync(h.kp.get(), 0x3f, n * nrhs * sizeof(double), s));
    SPFD_CUDA(cudaMemsetAsync(h.kr.get(), 0x3e, n * nrhs * sizeof(double), s));
    SPFD_CUDA(cudaMemsetAsync(h.kz.get(), 0x3e, n * nrhs * sizeof(double), s));
    SPFD_CUDA(cudaMemsetAsync(h.scal.get(), 0, S_END * sizeof(double), s));
    for (int l = 1; l < (int)h.lv.size(); ++l) {
        Level &C = h.lv[l];
        const size_t vb = (size_t)C.nvec * nrhs * sizeof(double);
        for (DevBuf<double> *v : {&C.vr, &C.vx, &C.vd, &C.vt}) SPFD_CUDA(cudaMemsetAsync(v->get(), 0x3e, vb, s));
    }
    SPFD_CHECK(which >= 0 && which < 10, SPFD_EINVAL, "unknown kernel");
    const KernelBytes kb = kernel_bytes(h, nrhs);
    const double byt[10] = {kb.spmv, kb.presmooth, kb.postsmooth, 0.0, kb.prolong, kb.aggsum, kb.l1_pre, kb.l1_pp,
                            kb.blas1, pcg_fuse_x() ? kb.blas1 * 5.0 / 3.0 : kb.blas1};
    auto launch2 = [&](auto rt) {
        constexpr int R = decltype(rt)::value;
        double *p = h.kp.get(), *r = h.kr.get(), *q = h.kq.get(), *z = h.kz.get();
        switch (which) {
            case 3: amg_vcycle(h, r, z, R, s); break;
            case 4: {
                Level &C = h.lv[1];
                if (L.Pspan.rows) {
                    launch_csr<R, 4, false>(L.Pspan, L.pspan_group, C.vx.get(), r, L.odinv.get(), nullptr, q, nullptr,
                                            s);
                } else {
                    SpanArgs sa{nullptr, r, L.odinv.get(), nullptr, C.vx.get(), L.agg_pos.get(), q, nullptr};
                    launch_fine<R, 4, false>(*h.op, sa, s);
                }
                break;
            }
            case 5: {
                Level &C = h.lv[1];
                if (L.Rspan.rows)
                    launch_csr<R, 0, false>(L.Rspan, L.rspan_group, p, nullptr, nullptr, nullptr, C.vr.get(),
                                            nullptr, s, C.odinv.get(), C.vt.get());
                else
                    k_agg_sum<R><<<grid_for(C.n, 256, 148 * 16), 256, 0, s>>>(L.mem_ptr.get(), L.mem_pos.get(), C.n,
                                                                             p, C.vr.get(), C.odinv.get(),
                                                                             C.vt.get(), 0);
                SPFD_LAUNCH_CHECK();
                break;
            }
            case 6: {
                Level &C = h.lv[1];
                launch_csr<R, 1, false>(C.A, C.a_group, C.vt.get(), C.vr.get(), C.odinv.get(), nullptr, C.vd.get(),
                                        nullptr, s);
                break;
            }
            case 7: {
                Level &C = h.lv[1];
                launch_pp<R>(C, h.lv[2].vx.get(), C.vr.get(), C.vd.get(), C.vt.get(), s);
                break;
            }
            case 8:
                k_update_r<R><<<kDotGrid, kDotThreads, 0, s>>>(n, h.scal.get(), r, q, h.partials.get(), 0);
                SPFD_LAUNCH_CHECK();
                break;
            case 9:
                if (pcg_fuse_x())
                    k_xpby_x<R><<<grid_for(n, 256, 148 * 16), 256, 0, s>>>(n, h.scal.get(), z, p, h.kx.get());
                else
                    k_xpby<R><<<grid_for(n, 256, 148 * 16), 256, 0, s>>>(n, h.scal.get(), z, p);
                SPFD_LAUNCH_CHECK();
                break;
            default: {
                const int mode = which == 0 ? 0 : (which == 1 ? 2 : 3);
                level0_apply<R>(h, mode, which != 1, p, r, q, s);
            }
        }
    };
    auto launch = [&]() {
        if (nrhs == 1) launch2(std::integral_constant<int, 1>{});
        else launch2(std::integral_constant<int, 2>{});
    };
    for (int i = 0; i < 3; ++i) launch();
    cudaEvent_t e0, e1;
    SPFD_CUDA(cudaEventCreate(&e0));
    SPFD_CUDA(cudaEventCreate(&e1));
    SPFD_CUDA(cudaEventRecord(e0, s));
    for (int i = 0; i < reps; ++i) launch();
    SPFD_CUDA(cudaEventRecord(e1, s));
    SPFD_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    SPFD_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *bytes = byt[which];
    if (which == 3) *bytes = amg_iteration_bytes(h, nrhs) - kb.spmv - (pcg_fuse_x() ? 1.0 + 5.0 / 3.0 : 3.0) * kb.blas1;
    return ms / reps;
}

spfd_report krylov_solve(Amg &h, const double *b, double *x, int nrhs, const spfd_config &cfg, double *h_trace,
                         cudaStream_t s) {
    SPFD_CHECK(nrhs >= 1 && nrhs <= h.max_nrhs, SPFD_EINVAL, "nrhs exceeds the hierarchy workspace");
    cudaEvent_t e0, e1;
    SPFD_CUDA(cudaEventCreate(&e0));
    SPFD_CUDA(cudaEventCreate(&e1));
    SPFD_CUDA(cudaEventRecord(e0, s));
    spfd_report rep{};
    if (h.dist && cfg.method == SPFD_METHOD_FGMRES) {
        rep = nrhs == 1 ? fgmres_dist<1>(h, b, x, cfg, h_trace, s) : fgmres_dist<2>(h, b, x, cfg, h_trace, s);
    } else if (cfg.method == SPFD_METHOD_FGMRES) {
        int64_t n = h.lv[0].nvec;
        // block (Gram-corrected CGS2) Arnoldi unless disabled or the restart
        // exceeds its scalar workspace; else the reference's MGS per rhs
        const bool block = !(getenv("SPFD_FGMRES_BATCH") && std::string(getenv("SPFD_FGMRES_BATCH")) == "0") &&
                           cfg.restart <= 31;
        const bool graph = block && fgmres_graph_enabled();
        if (nrhs == 1 && graph) {
            rep = fgmres_graph<1>(h, b, x, cfg, h_trace, s);
        } else if (nrhs == 1 && block) {
            rep = fgmres_batch<1>(h, b, x, cfg, h_trace, s);
        } else if (nrhs == 1) {
            rep = fgmres1(h, b, x, cfg, h_trace, s);
        } else if (graph) {
            rep = fgmres_graph<2>(h, b, x, cfg, h_trace, s);
        } else if (block) {
            rep = fgmres_batch<2>(h, b, x, cfg, h_trace, s);
        } else {
            DevBuf<double> b1, x1;
            b1.alloc(n); x1.alloc(n);
            std::vector<double> tr;
            int G = grid_for(n, 256, 148 * 16);
            rep.converged = 1;
            for (int c = 0; c < nrhs; ++c) {
                k_gather_col<<<G, 256, 0, s>>>(n, nrhs, c, b, b1.get());
                if (h_trace) tr.assign((size_t)cfg.max_iters, 0.0);
                spfd_report r1 = fgmres1(h, b1.get(), x1.get(), cfg, h_trace ? tr.data() : nullptr, s);
                k_scatter_col<<<G, 256, 0, s>>>(n, nrhs, c, x1.get(), x);
                if (h_trace)
                    for (int k = 0; k < cfg.max_iters; ++k) h_trace[(int64_t)k * nrhs + c] = tr[k];
                rep.iterations = std::max(rep.iterations, r1.iterations);
                rep.rel_residual[c] = r1.rel_residual[0];
                rep.converged = rep.converged && r1.converged;
                if (r1.status) rep.status = r1.status;
            }
        }
    } else if (h.dist) {
        rep = nrhs == 1 ? pcg_dist<1>(h, b, x, cfg, h_trace, s) : pcg_dist<2>(h, b, x, cfg, h_trace, s);
    } else {
        if (pcg_graph_enabled() && cfg.max_iters > 0)
            rep = nrhs == 1 ? pcg_graph<1>(h, b, x, cfg, h_trace, s) : pcg_graph<2>(h, b, x, cfg, h_trace, s);
        else
            rep = nrhs == 1 ? pcg<1>(h, b, x, cfg, h_trace, s) : pcg<2>(h, b, x, cfg, h_trace, s);
    }
    SPFD_CUDA(cudaEventRecord(e1, s));
    SPFD_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    SPFD_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    rep.solve_seconds = ms * 1e-3;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return rep;
}

}  // namespace spfd

// 2.5-D tiled fine-level stencil with cp.async staging (included by solve.cu).
//
// A CTA owns a 64-column x 8-row tile of the node box and marches through
// a range of z-planes.  For every plane it stages, with zero-filled
// cp.async copies, the tile plus a one-node halo of the stencil input and of
// the three edge-conductance arrays into a 4-slot shared-memory ring
// (planes k-1, k, k+1 in use, k+2 in flight), so every neighbour and every
// edge weight is a shared-memory read at a fixed offset and the HBM stream
// (positions are contiguous within a row) is read once per CTA plus the
// halo.  One warp computes one row of the tile (two positions per lane).
// The products are accumulated in the reference's sorted-column order with
// explicitly rounded operations; zero-filled neighbours add exact -0.0
// terms, so MODE 0 equals scipy's csr_matvec bit for bit.
#pragma once

constexpr int kTI = 64;                    // tile columns (i)
constexpr int kTJ = 8;                     // tile rows (j), one warp each
constexpr int kTC = kTI + 2;               // staged columns (with halo)
constexpr int kTR = kTJ + 2;               // staged rows (with halo)
constexpr int kTSlots = 4;
constexpr int kTileThreads = 32 * kTJ;

struct TileGeo {
    int NX, NY, NZ;
    int itiles, jtiles, kb, ktiles;
};

inline TileGeo tile_geo(const Operator &op, int ctas_per_sm) {
    TileGeo g;
    g.NX = (int)op.NX; g.NY = (int)op.NY; g.NZ = (int)op.NZ;
    g.itiles = (g.NX + kTI - 1) / kTI;
    g.jtiles = (g.NY + kTJ - 1) / kTJ;
    // a few waves of CTAs; the k-halo costs (kb + 2) / kb extra plane reads
    long target = 6L * 148 * (ctas_per_sm > 0 ? ctas_per_sm : 1);
    long kb = ((long)g.itiles * g.jtiles * g.NZ + target - 1) / target;
    if (kb < 8) kb = 8;
    if (kb > g.NZ) kb = g.NZ;
    g.kb = (int)kb;
    g.ktiles = (g.NZ + g.kb - 1) / g.kb;
    return g;
}

template <int R, int MODE>
struct TileSmem {
    using T = typename V<R>::T;
    // per slot: stencil input (x, r for MODE 2, e for MODE 4), wx, wy, wz,
    // and od (MODE 2) or aggregate ids (MODE 4)
    static constexpr size_t slot_x = (size_t)kTR * kTC * sizeof(T);
    static constexpr size_t slot_w = (size_t)3 * kTR * kTC * sizeof(double);
    static constexpr size_t slot_aux = MODE == 2 ? (size_t)kTR * kTC * sizeof(double)
                                     : (MODE == 4 ? (size_t)kTR * kTC * sizeof(int32_t) : 0);
    static constexpr size_t slot = slot_x + slot_w + slot_aux;
    static constexpr size_t bytes = kTSlots * slot;
};

template <int R, int MODE, bool DOT>
__global__ void __launch_bounds__(kTileThreads) k_tile(SpanView v, TileGeo g, SpanArgs a) {
    using W = V<R>;
    using T = typename W::T;
    using SM = TileSmem<R, MODE>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ double red[32 * R];
    __shared__ int any_work;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ti = blockIdx.x % g.itiles;
    const int tj = (blockIdx.x / g.itiles) % g.jtiles;
    const int tk = blockIdx.x / (g.itiles * g.jtiles);
    const int i0 = ti * kTI, j0 = tj * kTJ;
    const int k0 = tk * g.kb, k1 = min(g.NZ, k0 + g.kb);

    double dot[R];
#pragma unroll
    for (int c = 0; c < R; ++c) dot[c] = 0.0;

    // skip tiles that touch no conductive span in their planes
    if (threadIdx.x == 0) any_work = 0;
    __syncthreads();
    {
        const int j = j0 + warp;
        bool mine = false;
        if (j < g.NY)
            for (int k = k0 + lane; k < k1 && !mine; k += 32) {
                const int4 q = v.rows[j + g.NY * k];
                mine = q.z > q.y && q.y < i0 + kTI && q.z > i0;
            }
        if (__any_sync(0xffffffffu, mine) && lane == 0) any_work = 1;
    }
    __syncthreads();
    if (!any_work) {
        if (DOT && threadIdx.x < R) a.partials[blockIdx.x * R + threadIdx.x] = 0.0;
        return;
    }

    auto slot_base = [&](int kk) { return smem_raw + (size_t)((kk + kTSlots) % kTSlots) * SM::slot; };
    auto X = [&](unsigned char *b) { return reinterpret_cast<T *>(b); };
    auto WX = [&](unsigned char *b) { return reinterpret_cast<double *>(b + SM::slot_x); };
    auto WY = [&](unsigned char *b) { return WX(b) + kTR * kTC; };
    auto WZ = [&](unsigned char *b) { return WX(b) + 2 * kTR * kTC; };
    auto AUXD = [&](unsigned char *b) { return reinterpret_cast<double *>(b + SM::slot_x + SM::slot_w); };
    auto AUXI = [&](unsigned char *b) { return reinterpret_cast<int32_t *>(b + SM::slot_x + SM::slot_w); };

    // zero-filled asynchronous copy of the (kTR x kTC) halo tile of plane kk
    auto stage = [&](int kk) {
        unsigned char *b = slot_base(kk);
        for (int rr = warp; rr < kTR; rr += kTJ) {
            const int j = j0 - 1 + rr;
            int off = 0, lo = 0, hi = 0;
            if (j >= 0 && j < g.NY && kk >= 0 && kk < g.NZ) {
                const int4 q = v.rows[j + g.NY * kk];
                off = q.x; lo = q.y; hi = q.z;
            }
            for (int cc = lane; cc < kTC; cc += 32) {
                const int i = i0 - 1 + cc;
                const bool in = i >= lo && i < hi;
                const int64_t p = in ? (int64_t)off + (i - lo) : 0;
                const int e = rr * kTC + cc;
                if (MODE == 4) {
                    cp_async_zfill(AUXI(b) + e, a.aggp + p, 4, in);
                } else {
                    const double *src = MODE == 2 ? a.r : a.x;
                    cp_async_zfill(X(b) + e, src + p * R, (int)sizeof(T), in);
                }
                if (MODE == 2) cp_async_zfill(AUXD(b) + e, a.od + p, 8, in);
                cp_async_zfill(WX(b) + e, v.wx + p, 8, in);
                cp_async_zfill(WY(b) + e, v.wy + p, 8, in);
                cp_async_zfill(WZ(b) + e, v.wz + p, 8, in);
            }
        }
        cp_async_commit();
    };
    // once a slot has landed: form the stencil input in place (MODE 2: od*r,
    // MODE 4: e = T e_c gathered from the coarse vector)
    auto prepare = [&](int kk) {
        if (MODE != 2 && MODE != 4) return;
        unsigned char *b = slot_base(kk);
        for (int e = threadIdx.x; e < kTR * kTC; e += kTileThreads) {
            if (MODE == 2) X(b)[e] = W::scale(AUXD(b)[e], X(b)[e]);
            else {
                const int g1 = AUXI(b)[e];
                X(b)[e] = g1 > 0 ? W::ld(a.ec, g1 - 1) : W::zero();
            }
        }
    };

    stage(k0 - 1);
    stage(k0);
    stage(k0 + 1);
    cp_async_wait<1>();  // k0-1 and k0 landed
    __syncthreads();
    prepare(k0 - 1);
    prepare(k0);
    for (int k = k0; k < k1; ++k) {
        stage(k + 2);
        cp_async_wait<1>();  // k+1 landed
        __syncthreads();
        prepare(k + 1);
        __syncthreads();
        const int j = j0 + warp;
        if (j < g.NY) {
            const int r = j + g.NY * k;
            const int4 q = v.rows[r];
            unsigned char *bm = slot_base(k - 1), *bc = slot_base(k), *bp = slot_base(k + 1);
            const int rc = (warp + 1) * kTC;
#pragma unroll
            for (int h = 0; h < kTI / 32; ++h) {
                const int i = i0 + h * 32 + lane;
                const bool on = i >= q.y && i < q.z;
                const int cc = i - i0 + 1;
                const int e = rc + cc;
                const double wxp = WX(bc)[e], wyp = WY(bc)[e], wzp = WZ(bc)[e];
                const double wxm = WX(bc)[e - 1], wym = WY(bc)[e - kTC], wzm = WZ(bm)[e];
                const T xc = X(bc)[e];
                const double diag = add_rn(add_rn(add_rn(add_rn(add_rn(wxp, wyp), wzp), wxm), wym), wzm);
                T s = W::zero();
                s = W::axpy(-wzm, X(bm)[e], s);
                s = W::axpy(-wym, X(bc)[e - kTC], s);
                s = W::axpy(-wxm, X(bc)[e - 1], s);
                s = W::axpy(diag, xc, s);
                s = W::axpy(-wxp, X(bc)[e + 1], s);
                s = W::axpy(-wyp, X(bc)[e + kTC], s);
                s = W::axpy(-wzp, X(bp)[e], s);
                if (on) {
                    const int p = q.x + (i - q.y);
                    if (p >= a.pb && p < a.pe) {
                        T out;
                        if (MODE == 0) out = s;
                        else if (MODE == 1) out = W::sub(W::ld(a.r, p), s);
                        else if (MODE == 2) out = W::sub(W::ld(a.r, p), s);
                        else if (MODE == 3) out = W::add(xc, W::scale(a.od[p], W::sub(W::ld(a.r, p), s)));
                        else {
                            const T bb = a.base ? W::ld(a.base, p) : W::scale(a.od[p], W::ld(a.r, p));
                            out = W::sub(W::add(bb, xc), W::scale(a.od[p], s));
                        }
                        if (!mbit(v.mask, p)) out = W::zero();
                        W::st(a.y, p, out);
                        if (DOT) {
#pragma unroll
                            for (int c = 0; c < R; ++c) {
                                if (MODE == 0) dot[c] += W::dot(xc, out, c);
                                else if (MODE == 3) dot[c] += W::dot(W::ld(a.r, p), out, c);
                                else dot[c] += W::dot(out, out, c);
                            }
                        }
                    }
                }
            }
        }
        __syncthreads();
    }
    cp_async_wait<0>();
    if (DOT) {
        block_sum<R>(dot, red);
        if (threadIdx.x == 0)
#pragma unroll
            for (int c = 0; c < R; ++c) a.partials[blockIdx.x * R + c] = dot[c];
    }
}

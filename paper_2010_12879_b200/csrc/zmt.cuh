// z-marching fine-level stencil kernel staged by the bulk-copy (TMA) engine
// (included by solve.cu; rhs pairs only, R = 2).
//
// A CTA of kZtRows warps owns the 32-wide x-segment i0 .. i0+31 of the node
// rows j0 .. j0+kZtRows-1 and marches through the planes k0 .. k1-1 in
// lockstep.  For every plane kk the row segments it needs -- stencil inputs
// of the own rows and of one halo row on each side, the own rows' edge
// weights, the halo row's +y weight (the -y weight of row j0) and the mode's
// centre operands -- are fetched with one cp.async.bulk per (row, array):
// the contiguous span range [max(lo, i0-1), min(hi, i0+33)) widened to the
// enclosing 16-byte-aligned bytes, landing in a kZtSlots-deep ring of plane
// slots and completing on the slot's mbarrier (expect_tx by each warp's lane
// 0).  Nothing is zero-filled: a staged element is used only when it lies in
// its row's span (the row records travel with the slot), which is exactly
// where the flat kernel finds a neighbour.  The own column's input of plane
// k-1 and k and the -z weight stay in registers, the -x/+x neighbours come
// from lane shuffles, the -y/+y ones are the adjacent warps' rows of the
// same slot.  Per position, the warps issue ~1/32 of a copy instruction per
// array instead of one LSU load per array, and read ~100 B from shared
// memory instead of ~270 B through L1.
//
// Arithmetic and product order are k_span's (bit-identical in every mode).
#pragma once

constexpr int kZtRows = 8;                  // own rows (= warps) per CTA
constexpr int kZtThreads = 32 * kZtRows;
constexpr int kZtSlots = 4;                 // planes k, k+1 resident, k+2, k+3 in flight
constexpr int kZtRowsH = kZtRows + 2;
constexpr int kZtE = 40;                    // staged elements per row-array (34 + alignment slack)

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t *b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, unsigned parity) {
    uint32_t ok = 0;
    while (!ok) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(smem_u32(b)), "r"(parity)
            : "memory");
    }
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(b))
                 : "memory");
}

// Slot layout (bytes).  Row-arrays hold kZtE elements; element i of a row
// sits at index i - org, org = first staged x minus the alignment shift
// (per element size: 4-, 8- and 16-byte arrays shift differently).
template <int MODE>
struct ZtSlot {
    static constexpr int in_sz = MODE == 4 ? 4 : 16;
    static constexpr bool has_od = MODE == 2;
    static constexpr bool has_c = MODE == 1 || MODE == 3 || MODE == 4;
    static constexpr bool has_odc = MODE == 3 || MODE == 4;
    static constexpr int o_in = 0;                                          // [RowsH][E]
    static constexpr int o_od = o_in + kZtRowsH * kZtE * in_sz;             // [RowsH][E] (MODE 2)
    static constexpr int o_wx = o_od + (has_od ? kZtRowsH * kZtE * 8 : 0);  // [Rows][E]
    static constexpr int o_wy = o_wx + kZtRows * kZtE * 8;                  // [Rows+1][E], row 0 = halo j0-1
    static constexpr int o_wz = o_wy + (kZtRows + 1) * kZtE * 8;            // [Rows][E]
    static constexpr int o_c = o_wz + kZtRows * kZtE * 8;                   // [Rows][E] x 16 B
    static constexpr int o_odc = o_c + (has_c ? kZtRows * kZtE * 16 : 0);   // [Rows][E]
    static constexpr int o_meta = o_odc + (has_odc ? kZtRows * kZtE * 8 : 0);  // [RowsH] int4 {lo, hi, off-lo, st}
    static constexpr int bytes = o_meta + kZtRowsH * 16;
};

template <int MODE>
constexpr size_t zt_smem() { return (size_t)kZtSlots * ZtSlot<MODE>::bytes + kZtSlots * 8 + 16; }

// Issue one row-array bulk copy of span range [st, en) (element size es,
// row record q) into dst; returns the bytes it will deliver (0 if empty).
__device__ __forceinline__ unsigned zt_copy(void *dst, const void *base, int es, int4 q, int st, int en,
                                            uint64_t *bar) {
    if (en <= st) return 0;
    const int64_t p0 = (int64_t)q.x + (st - q.y);
    const uintptr_t a = (uintptr_t)base + (uintptr_t)(p0 * es);
    const uintptr_t al = a & ~(uintptr_t)15;
    const uintptr_t e = a + (uintptr_t)(en - st) * es;
    const unsigned bytes = (unsigned)(((e - al) + 15) & ~(uintptr_t)15);
    bulk_g2s(dst, (const void *)al, bytes, bar);
    return bytes;
}

template <int MODE, bool DOT>
__global__ void __launch_bounds__(kZtThreads) k_zt(SpanView v, const int4 *__restrict__ items, SpanArgs a) {
    using W = V<2>;
    using T = double2;
    using SL = ZtSlot<MODE>;
    constexpr unsigned FULL = 0xffffffffu;
    extern __shared__ __align__(128) unsigned char zt_raw[];
    __shared__ double red[64];
    uint64_t *bars = reinterpret_cast<uint64_t *>(zt_raw + kZtSlots * SL::bytes);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int4 it = items[blockIdx.x];
    const int j0 = it.x, i0 = it.y, k0 = it.z, k1 = it.w;
    const int i = i0 + lane;
    const int NY = v.NY;
    const int NZ = v.n_rows / NY;
    const int4 none = make_int4(0, 0, 0, 0);
    const int rw = warp + 1;  // slot row of the own row
    const int jh = warp == 0 ? j0 - 1 : j0 + kZtRows;
    const bool halo = warp == 0 || warp == kZtRows - 1;
    const int rh = warp == 0 ? 0 : kZtRows + 1;  // slot row of the halo row

    if (threadIdx.x == 0) {
        for (int s = 0; s < kZtSlots; ++s) mbar_init(&bars[s], kZtRows);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    auto rec = [&](int kk, int jj) -> int4 {
        return (kk >= 0 && kk < NZ && kk <= k1 && jj >= 0 && jj < NY) ? v.rows[kk * NY + jj] : none;
    };
    auto sidx = [&](int kk) { return (kk - k0 + 1) % kZtSlots; };
    auto par = [&](int kk) { return (unsigned)(((kk - k0 + 1) / kZtSlots) & 1); };
    auto slot = [&](int kk) { return zt_raw + (size_t)sidx(kk) * SL::bytes; };
    // stage plane kk (own record q, halo record h): lane 0 of every warp
    auto stage = [&](int kk, int4 q, int4 h) {
        if (lane != 0) return;
        unsigned char *sl = slot(kk);
        uint64_t *bar = &bars[sidx(kk)];
        int4 *meta = reinterpret_cast<int4 *>(sl + SL::o_meta);
        const int st = max(q.y, i0 - 1), en = min(q.z, i0 + 33);
        meta[rw] = make_int4(q.y, q.z, q.x - q.y, st);
        int hst = 0, hen = 0;
        if (halo) {
            hst = max(h.y, i0 - 1);
            hen = min(h.z, i0 + 33);
            meta[rh] = make_int4(h.y, h.z, h.x - h.y, hst);
        }
        // bytes first (expect_tx before the copies can complete)
        auto nb = [&](int es, int4 qq, int s0, int e0) -> unsigned {
            if (e0 <= s0) return 0;
            const uintptr_t aa = (uintptr_t)((int64_t)qq.x + (s0 - qq.y)) * es;
            const uintptr_t al = aa & ~(uintptr_t)15;  // (array bases are 16-byte aligned)
            return (unsigned)((((aa + (uintptr_t)(e0 - s0) * es) - al) + 15) & ~(uintptr_t)15);
        };
        unsigned tot = nb(SL::in_sz, q, st, en) * (SL::has_od ? 1 : 1);
        if (SL::has_od) tot += nb(8, q, st, en);
        tot += 3 * nb(8, q, st, en);
        if (SL::has_c) tot += nb(16, q, st, en);
        if (SL::has_odc) tot += nb(8, q, st, en);
        if (halo) {
            tot += nb(SL::in_sz, h, hst, hen);
            if (SL::has_od) tot += nb(8, h, hst, hen);
            if (warp == 0) tot += nb(8, h, hst, hen);
        }
        mbar_arrive_tx(bar, tot);
        const void *inb = MODE == 4 ? (const void *)a.aggp : (const void *)(MODE == 2 ? a.r : a.x);
        zt_copy(sl + SL::o_in + rw * kZtE * SL::in_sz, inb, SL::in_sz, q, st, en, bar);
        if (SL::has_od) zt_copy(sl + SL::o_od + rw * kZtE * 8, a.od, 8, q, st, en, bar);
        zt_copy(sl + SL::o_wx + warp * kZtE * 8, v.wx, 8, q, st, en, bar);
        zt_copy(sl + SL::o_wy + rw * kZtE * 8, v.wy, 8, q, st, en, bar);
        zt_copy(sl + SL::o_wz + warp * kZtE * 8, v.wz, 8, q, st, en, bar);
        if (SL::has_c)
            zt_copy(sl + SL::o_c + warp * kZtE * 16, (MODE == 4 && a.base) ? a.base : a.r, 16, q, st, en, bar);
        if (SL::has_odc) zt_copy(sl + SL::o_odc + warp * kZtE * 8, a.od, 8, q, st, en, bar);
        if (halo) {
            zt_copy(sl + SL::o_in + rh * kZtE * SL::in_sz, inb, SL::in_sz, h, hst, hen, bar);
            if (SL::has_od) zt_copy(sl + SL::o_od + rh * kZtE * 8, a.od, 8, h, hst, hen, bar);
            if (warp == 0) zt_copy(sl + SL::o_wy, v.wy, 8, h, hst, hen, bar);
        }
    };
    // A staged row as seen by the compute step: span test and the element
    // index of x = ii in its 16-, 8- and 4-byte arrays (aligned-superset shift)
    struct Row {
        int lo, hi, pofs, b16, b8, b4;
    };
    auto row_of = [&](const unsigned char *sl, int r) -> Row {
        const int4 m = reinterpret_cast<const int4 *>(sl + SL::o_meta)[r];
        const int p0 = m.z + m.w;  // span position of the first staged x
        return Row{m.x, m.y, m.z, -m.w, -m.w + (p0 & 1), -m.w + (p0 & 3)};
    };
    auto X = [&](const unsigned char *sl, int r, const Row &m, int ii) -> T {
        if (!(ii >= m.lo && ii < m.hi)) return W::zero();
        if (MODE == 4) {
            const int g1 = reinterpret_cast<const int32_t *>(sl + SL::o_in + r * kZtE * 4)[ii + m.b4];
            return g1 > 0 ? W::ld(a.ec, g1 - 1) : W::zero();
        }
        const T x = reinterpret_cast<const T *>(sl + SL::o_in + r * kZtE * 16)[ii + m.b16];
        if (MODE == 2) return W::scale(reinterpret_cast<const double *>(sl + SL::o_od + r * kZtE * 8)[ii + m.b8], x);
        return x;
    };
    auto D = [&](const unsigned char *sl, int off, int arow, const Row &m, int ii) -> double {
        if (!(ii >= m.lo && ii < m.hi)) return 0.0;
        return reinterpret_cast<const double *>(sl + off + arow * kZtE * 8)[ii + m.b8];
    };

    double dot[2] = {0.0, 0.0};
    // prologue: planes k0-1 .. k0+2 (slots 0..3); k0-1 and k0 are read now
    for (int kk = k0 - 1; kk <= k0 + kZtSlots - 2; ++kk) {
        if (kk <= k1) stage(kk, rec(kk, j0 + warp), halo ? rec(kk, jh) : none);
        else if (lane == 0) mbar_arrive_tx(&bars[sidx(kk)], 0);
    }
    mbar_wait(&bars[sidx(k0 - 1)], par(k0 - 1));
    mbar_wait(&bars[sidx(k0)], par(k0));
    T xm, xc;
    double wzm;
    {
        const unsigned char *s0 = slot(k0 - 1), *s1 = slot(k0);
        const Row m0 = row_of(s0, rw), m1 = row_of(s1, rw);
        xm = X(s0, rw, m0, i);
        wzm = D(s0, SL::o_wz, warp, m0, i);
        xc = X(s1, rw, m1, i);
    }
    for (int k = k0; k < k1; ++k) {
        __syncthreads();  // everyone is done with slot k-1 (read in the prologue / step k-1)
        const int kn = k + kZtSlots - 1;
        if (kn <= k1) stage(kn, rec(kn, j0 + warp), halo ? rec(kn, jh) : none);
        mbar_wait(&bars[sidx(k + 1)], par(k + 1));
        const unsigned char *sc = slot(k), *sp = slot(k + 1);
        const Row mc = row_of(sc, rw), mym = row_of(sc, rw - 1), myp = row_of(sc, rw + 1), mp = row_of(sp, rw);
        const bool on = i >= mc.lo && i < mc.hi;
        const int p = on ? mc.pofs + i : -1;
        const T xp = X(sp, rw, mp, i);
        const double wxp = D(sc, SL::o_wx, warp, mc, i);
        double wxm = __shfl_up_sync(FULL, wxp, 1);
        if (lane == 0) wxm = D(sc, SL::o_wx, warp, mc, i - 1);
        const double wyp = D(sc, SL::o_wy, rw, mc, i);
        const double wym = D(sc, SL::o_wy, warp, mym, i);
        const double wzp = D(sc, SL::o_wz, warp, mc, i);
        T xxm = shfl_up1(xc), xxp = shfl_dn1(xc);
        if (lane == 0) xxm = X(sc, rw, mc, i - 1);
        if (lane == 31) xxp = X(sc, rw, mc, i + 1);
        // reference diagonal order: tail edges x, y, z then head edges x, y, z
        const double diag = add_rn(add_rn(add_rn(add_rn(add_rn(wxp, wyp), wzp), wxm), wym), wzm);
        T s = W::zero();
        s = W::axpy(-wzm, xm, s);
        s = W::axpy(-wym, X(sc, rw - 1, mym, i), s);
        s = W::axpy(-wxm, xxm, s);
        s = W::axpy(diag, xc, s);
        s = W::axpy(-wxp, xxp, s);
        s = W::axpy(-wyp, X(sc, rw + 1, myp, i), s);
        s = W::axpy(-wzp, xp, s);
        if (on) {
            T rc = W::zero();
            double odp = 0.0;
            if (SL::has_c) rc = reinterpret_cast<const T *>(sc + SL::o_c + warp * kZtE * 16)[i + mc.b16];
            if (SL::has_odc) odp = reinterpret_cast<const double *>(sc + SL::o_odc + warp * kZtE * 8)[i + mc.b8];
            T out;
            if (MODE == 0) out = s;
            else if (MODE == 1) out = W::sub(rc, s);
            else if (MODE == 2) out = W::sub(reinterpret_cast<const T *>(sc + SL::o_in + rw * kZtE * 16)[i + mc.b16], s);
            else if (MODE == 3) out = W::add(xc, W::scale(odp, W::sub(rc, s)));
            else {
                const T b = a.base ? rc : W::scale(odp, rc);
                out = W::sub(W::add(b, xc), W::scale(odp, s));
            }
            if (!mbit(v.mask, p)) out = W::zero();
            W::st(a.y, p, out);
            if (DOT) {
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    if (MODE == 0) dot[c] += W::dot(xc, out, c);
                    else if (MODE == 3) dot[c] += W::dot(rc, out, c);
                    else dot[c] += W::dot(out, out, c);
                }
            }
        }
        xm = xc;
        xc = xp;
        wzm = wzp;
    }
    if (DOT) {
        block_sum<2>(dot, red);
        if (threadIdx.x == 0) {
            a.partials[blockIdx.x * 2] = dot[0];
            a.partials[blockIdx.x * 2 + 1] = dot[1];
        }
    }
}

// z-marching fine-level stencil kernel: a CTA of kZmRows warps owns the
// 32-wide x-segment i0 .. i0+31 of the node rows j0 .. j0+kZmRows-1 and
// marches through the planes k0 .. k1-1 in lockstep (one __syncthreads per
// plane).  Included by solve.cu after plane.cuh (cp_async_* helpers).
//
// Every operand of plane kk -- the stencil inputs of the CTA's rows plus one
// halo row on each side (with a one-element x halo on the own rows), the
// +x/+y/+z edge weights, the -y weights of the halo row, the mode's centre
// operands and the DOF-mask words -- is copied asynchronously (cp.async,
// zero-filled outside the conductive spans) into a kZmSlots-deep ring of
// plane slots in shared memory, one plane ahead of the plane being
// computed.  Each element crosses the L1/shared data path once on the way in
// and once (at most) on the way out: the own column's input of planes k-1
// and k and the -z weight stay in registers, the -x/+x neighbours and the -x
// weight come from lane shuffles, the -y/+y neighbours are the adjacent
// warps' rows of the same slot.  The flat per-position kernel gathers all
// seven inputs and six weights through L1 per position and is bound by the
// L1 data pipe (ncu: lsu data-pipe wavefronts ~70 %, DRAM ~58 %); this one
// moves ~2x fewer wavefronts per position.
//
// Arithmetic is k_span's: the same products in the reference's sorted-column
// order (-z, -y, -x, diag, +x, +y, +z).  Neighbours outside the conductive
// spans are zero-filled, so their products are exact zeros that leave the
// running sum unchanged: every mode is bit-identical to k_span, and MODE 0 to
// scipy csr_matvec.
#pragma once

constexpr int kZmRows = 8;                  // own rows (= warps) per CTA
constexpr int kZmThreads = 32 * kZmRows;
constexpr int kZmSlots = 3;                 // planes k, k+1 resident, k+2 in flight
constexpr int kZmRowsH = kZmRows + 2;       // with the -y / +y halo rows
constexpr int kZmW = 34;                    // staged x-extent of a row: i0-1 .. i0+32

__device__ __forceinline__ int zm_pos(int4 q, int i) { return (i >= q.y && i < q.z) ? q.x + (i - q.y) : -1; }

// Byte layout of one plane slot (whole CTA).
template <int R, int MODE>
struct ZmSlot {
    using T = typename V<R>::T;
    static constexpr int in_sz = MODE == 4 ? 4 : (int)sizeof(T);
    static constexpr int o_in = 0;                                          // [RowsH][34] x | r | agg+1
    static constexpr int o_od = (o_in + kZmRowsH * kZmW * in_sz + 15) & ~15; // [RowsH][34] od (MODE 2)
    static constexpr int n_od = MODE == 2 ? kZmRowsH * kZmW : 0;
    static constexpr int o_wx = (o_od + n_od * 8 + 15) & ~15;               // [Rows][34] wx at i0-1 ..
    static constexpr int o_wy = o_wx + kZmRows * kZmW * 8;                  // [Rows+1][32] row 0 = halo j0-1
    static constexpr int o_wz = o_wy + (kZmRows + 1) * 32 * 8;              // [Rows][32]
    static constexpr bool has_c = MODE == 1 || MODE == 3 || MODE == 4;      // centre r (or base)
    static constexpr bool has_odc = MODE == 3 || MODE == 4;                 // centre od
    static constexpr int o_c = o_wz + kZmRows * 32 * 8;                     // [Rows][32] T
    static constexpr int o_odc = o_c + (has_c ? kZmRows * 32 * (int)sizeof(T) : 0);
    static constexpr int o_mask = o_odc + (has_odc ? kZmRows * 32 * 8 : 0); // [Rows][32] u32
    static constexpr int o_rec = (o_mask + kZmRows * 32 * 4 + 15) & ~15;    // [Rows] own row records
    static constexpr int bytes = o_rec + kZmRows * 16;
};

template <int R, int MODE>
constexpr size_t zm_smem() { return (size_t)kZmSlots * ZmSlot<R, MODE>::bytes; }

template <int R, int MODE, bool DOT>
__global__ void __launch_bounds__(kZmThreads) k_zm(SpanView v, const int4 *__restrict__ items, SpanArgs a) {
    using W = V<R>;
    using T = typename W::T;
    using SL = ZmSlot<R, MODE>;
    constexpr unsigned FULL = 0xffffffffu;
    extern __shared__ __align__(16) unsigned char zm_raw[];
    __shared__ double red[32 * R];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int4 it = items[blockIdx.x];
    const int j0 = it.x, i0 = it.y, k0 = it.z, k1 = it.w;
    const int i = i0 + lane;
    const int NY = v.NY;
    const int NZ = v.n_rows / NY;
    const int4 none = make_int4(0, 0, 0, 0);
    const int j = j0 + warp;  // own row of this warp (may be >= NY: empty)

    auto rec = [&](int kk, int jj) -> int4 {
        return (kk >= 0 && kk < NZ && kk <= k1 && jj >= 0 && jj < NY) ? v.rows[kk * NY + jj] : none;
    };
    auto slot = [&](int kk) -> unsigned char * {
        return zm_raw + (size_t)((kk + kZmSlots) % kZmSlots) * SL::bytes;
    };
    // stage the input element at x = ii of a row (record q) into slot index e
    auto put_in = [&](unsigned char *sl, int e, int4 q, int ii) {
        const int p = zm_pos(q, ii);
        const int64_t g = p >= 0 ? p : 0;
        if (MODE == 4) {
            cp_async_zfill(sl + SL::o_in + e * 4, a.aggp + g, 4, p >= 0);
        } else if (MODE == 2) {
            cp_async_zfill(sl + SL::o_in + e * SL::in_sz, a.r + g * R, SL::in_sz, p >= 0);
            cp_async_zfill(sl + SL::o_od + e * 8, a.od + g, 8, p >= 0);
        } else {
            cp_async_zfill(sl + SL::o_in + e * SL::in_sz, a.x + g * R, SL::in_sz, p >= 0);
        }
    };
    // stage plane kk: every warp its own row (+ warp 0 the -y halo row, the
    // last warp the +y halo row); own-row records are passed in registers
    const int jh = warp == 0 ? j0 - 1 : j0 + kZmRows;  // halo row staged by warps 0 / last
    auto stage = [&](int kk, int4 q, int4 h) {
        unsigned char *sl = slot(kk);
        const int rw = warp + 1;  // slot row of the own row
        put_in(sl, rw * kZmW + lane, q, i - 1);
        if (lane < 2) put_in(sl, rw * kZmW + 32 + lane, q, i + 31);
        const int pxm = zm_pos(q, i - 1), p = zm_pos(q, i), pl = zm_pos(q, i + 31);
        double *wxs = reinterpret_cast<double *>(sl + SL::o_wx) + warp * kZmW;
        cp_async_zfill(wxs + lane, v.wx + (pxm >= 0 ? pxm : 0), 8, pxm >= 0);
        if (lane == 0) cp_async_zfill(wxs + 32, v.wx + (pl >= 0 ? pl : 0), 8, pl >= 0);
        const int64_t g = p >= 0 ? p : 0;
        cp_async_zfill(reinterpret_cast<double *>(sl + SL::o_wy) + rw * 32 + lane, v.wy + g, 8, p >= 0);
        cp_async_zfill(reinterpret_cast<double *>(sl + SL::o_wz) + warp * 32 + lane, v.wz + g, 8, p >= 0);
        if (SL::has_c) {
            const double *src = (MODE == 4 && a.base) ? a.base : a.r;
            cp_async_zfill(sl + SL::o_c + (warp * 32 + lane) * (int)sizeof(T), src + g * R, (int)sizeof(T), p >= 0);
        }
        if (SL::has_odc)
            cp_async_zfill(reinterpret_cast<double *>(sl + SL::o_odc) + warp * 32 + lane, a.od + g, 8, p >= 0);
        cp_async_zfill(reinterpret_cast<uint32_t *>(sl + SL::o_mask) + warp * 32 + lane, v.mask + (g >> 5), 4, p >= 0);
        if (lane == 0) reinterpret_cast<int4 *>(sl + SL::o_rec)[warp] = q;
        if (warp == 0) {  // -y halo row j0-1: inputs and its +y weight (= the -y weight of row j0)
            put_in(sl, 0 * kZmW + lane + 1, h, i);
            const int ph = zm_pos(h, i);
            cp_async_zfill(reinterpret_cast<double *>(sl + SL::o_wy) + lane, v.wy + (ph >= 0 ? ph : 0), 8, ph >= 0);
        }
        if (warp == kZmRows - 1) {  // +y halo row j0+Rows
            put_in(sl, (kZmRows + 1) * kZmW + lane + 1, h, i);
        }
        cp_async_commit();
    };
    auto X = [&](const unsigned char *sl, int e) -> T {
        if (MODE == 4) {
            const int g1 = reinterpret_cast<const int32_t *>(sl + SL::o_in)[e];
            return g1 > 0 ? W::ld(a.ec, g1 - 1) : W::zero();
        }
        const T x = reinterpret_cast<const T *>(sl + SL::o_in)[e];
        if (MODE == 2) return W::scale(reinterpret_cast<const double *>(sl + SL::o_od)[e], x);
        return x;
    };
    auto dsl = [&](const unsigned char *sl, int off, int e) -> double {
        return reinterpret_cast<const double *>(sl + off)[e];
    };

    double dot[R];
#pragma unroll
    for (int c = 0; c < R; ++c) dot[c] = 0.0;
    const int rw = warp + 1, e0 = rw * kZmW + lane + 1;  // slot index of the own element
    const bool halo = warp == 0 || warp == kZmRows - 1;
    // prologue: planes k0-1, k0 (resident) and k0+1 (in flight)
    for (int kk = k0 - 1; kk <= k0 + 1; ++kk) stage(kk, rec(kk, j), halo ? rec(kk, jh) : none);
    cp_async_wait<1>();
    __syncthreads();
    T xm = X(slot(k0 - 1), e0);
    double wzm = dsl(slot(k0 - 1), SL::o_wz, warp * 32 + lane);
    T xc = X(slot(k0), e0);
    int4 qn = rec(k0 + 2, j), hn = halo ? rec(k0 + 2, jh) : none;
    for (int k = k0; k < k1; ++k) {
        cp_async_wait<0>();  // plane k+1 has landed
        __syncthreads();     // ... for every thread, and every thread is done with slot k-1
        stage(k + 2, qn, hn);  // refill slot k-1 with plane k+2 (in flight during this step)
        qn = rec(k + 3, j);
        if (halo) hn = rec(k + 3, jh);
        const unsigned char *sc = slot(k), *sp = slot(k + 1);
        const int4 qc = reinterpret_cast<const int4 *>(sc + SL::o_rec)[warp];
        const int p = zm_pos(qc, i);
        const T xp = X(sp, e0);
        const double wxp = dsl(sc, SL::o_wx, warp * kZmW + lane + 1);
        double wxm = __shfl_up_sync(FULL, wxp, 1);
        if (lane == 0) wxm = dsl(sc, SL::o_wx, warp * kZmW);
        const double wyp = dsl(sc, SL::o_wy, rw * 32 + lane), wym = dsl(sc, SL::o_wy, warp * 32 + lane);
        const double wzp = dsl(sc, SL::o_wz, warp * 32 + lane);
        T xxm = shfl_up1(xc), xxp = shfl_dn1(xc);
        if (lane == 0) xxm = X(sc, rw * kZmW);
        if (lane == 31) xxp = X(sc, rw * kZmW + 33);
        // reference diagonal order: tail edges x, y, z then head edges x, y, z
        const double diag = add_rn(add_rn(add_rn(add_rn(add_rn(wxp, wyp), wzp), wxm), wym), wzm);
        T s = W::zero();
        s = W::axpy(-wzm, xm, s);
        s = W::axpy(-wym, X(sc, e0 - kZmW), s);
        s = W::axpy(-wxm, xxm, s);
        s = W::axpy(diag, xc, s);
        s = W::axpy(-wxp, xxp, s);
        s = W::axpy(-wyp, X(sc, e0 + kZmW), s);
        s = W::axpy(-wzp, xp, s);
        if (p >= 0) {
            T rc = W::zero();
            if (SL::has_c) rc = reinterpret_cast<const T *>(sc + SL::o_c)[warp * 32 + lane];
            T out;
            if (MODE == 0) out = s;
            else if (MODE == 1) out = W::sub(rc, s);
            else if (MODE == 2) out = W::sub(reinterpret_cast<const T *>(sc + SL::o_in)[e0], s);
            else if (MODE == 3) out = W::add(xc, W::scale(dsl(sc, SL::o_odc, warp * 32 + lane), W::sub(rc, s)));
            else {
                const double odp = dsl(sc, SL::o_odc, warp * 32 + lane);
                const T b = a.base ? rc : W::scale(odp, rc);
                out = W::sub(W::add(b, xc), W::scale(odp, s));
            }
            const uint32_t mw = reinterpret_cast<const uint32_t *>(sc + SL::o_mask)[warp * 32 + lane];
            if (!((mw >> (p & 31)) & 1u)) out = W::zero();
            W::st(a.y, p, out);
            if (DOT) {
#pragma unroll
                for (int c = 0; c < R; ++c) {
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
    cp_async_wait<0>();
    if (DOT) {
        block_sum<R>(dot, red);
        if (threadIdx.x == 0)
#pragma unroll
            for (int c = 0; c < R; ++c) a.partials[blockIdx.x * R + c] = dot[c];
    }
}

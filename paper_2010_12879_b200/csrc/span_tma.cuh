// Staged fine-level stencil pass (fine kernel kind 5).  A persistent CTA per
// SM walks kStage-position tiles of the span layout in a fixed round-robin
// order.  A producer warp queues, for each tile, bulk copies (cp.async.bulk:
// the TMA engine, no registers) of every window the tile's stencil reads into
// one of S shared-memory stages, completing on the stage's `full` mbarrier;
// sixteen consumer warps compute the tile from shared memory, one 32-position
// row chunk per warp at a time, and release the stage on its `empty` mbarrier.  All of a tile's HBM/L2 traffic is in
// flight at once, up to S tiles ahead of the consumers, and the per-position
// dependent chain of the flat kernel (row record -> neighbour position ->
// neighbour value in L1/L2/HBM) becomes a chain of shared-memory reads.
//
// Windows of a tile [P0, P1) (exact position ranges from Operator::stage_desc,
// widened to 16-byte boundaries):
//   C  in-plane: the tile plus its x+-1 / y+-1 neighbours  (input, wx, wy)
//   M  plane below: the z-1 neighbours                      (input, wz at z-1)
//   P  plane above: the z+1 neighbours                      (input)
//   T  the tile                                             (wz, r, omega D^-1, mask)
//   rows r0-1..r1+1 and their z-1 / z+1 rows                (row records)
// Tiles whose windows do not fit the slots (or touch the arrays' last 4
// positions) are flagged at operator build and computed by the per-position
// path from global memory, so any geometry is handled.  The per-position
// arithmetic is point_out's term for term (same bits as every other fine
// kernel); dot partials are per CTA (fixed tile assignment: bitwise
// reproducible run to run).
#pragma once

namespace stg {

constexpr int kConsumers = 512;            // 16 consumer warps
constexpr int kThreads = kConsumers + 32;  // + 1 producer warp
constexpr int kTW = kStage + 16;           // tile slot (with 16-byte slack)

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t *b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, unsigned parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(su32(b)), "r"(parity)
            : "memory");
    }
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     su32(dst)),
                 "l"(src), "r"(bytes), "r"(su32(bar))
                 : "memory");
}
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;\n" ::"n"(kConsumers) : "memory"); }

// Slots of a stage.  X = the stencil's neighbour-read input: x (modes 0, 1,
// 3), r (mode 2, with omega D^-1 in the O slots), the aggregate map (mode 4).
enum { XC = 0, XM, XP, OC, OM, OP, WX, WY, WZ, WZM, OT, RT, MK, RY, RM, RP, NSLOT };

template <int R, int MODE>
struct Layout {
    static constexpr int XE = MODE == 4 ? 4 : 8 * R;  // bytes per X element
    static constexpr bool OWIN = MODE == 2;            // omega D^-1 read at neighbours
    static constexpr bool OTILE = MODE == 3 || MODE == 4;
    static constexpr bool RTILE = MODE == 1 || MODE == 3 || MODE == 4;
    static constexpr int CW = kStageCW + 4, ZW = kStageZW + 4;  // + widening to 16 bytes
    static constexpr int oXC = 0;
    static constexpr int oXM = oXC + CW * XE;
    static constexpr int oXP = oXM + ZW * XE;
    static constexpr int oOC = oXP + ZW * XE;
    static constexpr int oOM = oOC + (OWIN ? CW * 8 : 0);
    static constexpr int oOP = oOM + (OWIN ? ZW * 8 : 0);
    static constexpr int oWX = oOP + (OWIN ? ZW * 8 : 0);
    static constexpr int oWY = oWX + kTW * 8;   // wx over [P0 - 1, P1)
    static constexpr int oWZ = oWY + CW * 8;    // wy over [C.a, P1)
    static constexpr int oWZM = oWZ + kTW * 8;
    static constexpr int oOT = oWZM + ZW * 8;
    static constexpr int oRT = oOT + (OTILE ? kTW * 8 : 0);
    static constexpr int oMK = oRT + (RTILE ? kTW * 8 * R : 0);
    static constexpr int oRY = oMK + (kStage / 32 + 4) * 4;
    static constexpr int oRM = oRY + kStageRW * 16;
    static constexpr int oRP = oRM + kStageRW * 16;
    static constexpr int STAGE = oRP + kStageRW * 16;
    static constexpr int NST = (227 * 1024 - 1024) / STAGE < 4 ? (227 * 1024 - 1024) / STAGE : 4;  // stages
    static_assert(STAGE % 16 == 0 && oXM % 16 == 0 && oXP % 16 == 0 && oOC % 16 == 0 && oOM % 16 == 0 &&
                      oOP % 16 == 0 && oWX % 16 == 0 && oWY % 16 == 0 && oWZ % 16 == 0 && oWZM % 16 == 0 &&
                      oOT % 16 == 0 && oRT % 16 == 0 && oMK % 16 == 0 && oRY % 16 == 0,
                  "16-byte aligned slots");
};

// window [a, b) of `base` (esz bytes per element) widened to 16-byte
// boundaries: first staged element index -> w0, copy size returned
__device__ __forceinline__ unsigned plan(const void *base, int esz, int64_t a, int64_t b, int &w0,
                                         const char *&src) {
    w0 = 0;
    if (!base || b <= a) return 0;
    const uintptr_t pb = reinterpret_cast<uintptr_t>(base);
    const uintptr_t s = (pb + (uintptr_t)(a * esz)) & ~(uintptr_t)15;
    const uintptr_t e = (pb + (uintptr_t)(b * esz) + 15) & ~(uintptr_t)15;
    w0 = (int)((s - pb) / esz);
    src = reinterpret_cast<const char *>(s);
    return (unsigned)(e - s);
}

}  // namespace stg

template <int R, int MODE, bool DOT, int S>
__global__ void __launch_bounds__(stg::kThreads, 1)
k_span_stg(SpanView v, SpanArgs a, const int4 *__restrict__ desc, int n_tiles) {
    using W = V<R>;
    using T = typename W::T;
    using LY = stg::Layout<R, MODE>;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t full[S], empty[S];
    __shared__ int w0s[S][stg::NSLOT];
    __shared__ int4 dsc[S][2];
    __shared__ double red[(stg::kConsumers / 32) * R];

    const int G = gridDim.x;
    const int tid = threadIdx.x;
    auto tile_of = [&](int i) -> int {
        const int tl = (int)blockIdx.x + i * G;
        if (tl >= n_tiles) return -1;
        return a.rev ? n_tiles - 1 - tl : tl;
    };

    if (tid == 0) {
        for (int k = 0; k < S; ++k) {
            stg::mbar_init(&full[k], 1);
            stg::mbar_init(&empty[k], stg::kConsumers / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    if (tid >= stg::kConsumers) {
        // ---------------- producer warp ----------------
        const int lane = tid & 31;
        const void *xs = MODE == 2 ? (const void *)a.r : MODE == 4 ? (const void *)a.aggp : (const void *)a.x;
        for (int i = 0;; ++i) {
            const int t = tile_of(i);
            if (t < 0) break;
            const int st = i % S;
            if (i >= S) stg::mbar_wait(&empty[st], (unsigned)(((i / S) - 1) & 1));
            const int4 d0 = desc[2 * t], d1 = desc[2 * t + 1];
            const bool staged = !(d1.w & kStageFlat);
            const int r0 = d1.z, r1 = d1.w & (kStageFlat - 1);
            const int64_t P0 = (int64_t)t * kStage, P1 = P0 + kStage < v.L ? P0 + kStage : v.L;
            const void *g = nullptr;
            int esz = 8, off = 0;
            int64_t wa = 0, wb = 0;
            if (staged) {
                switch (lane) {
                    case stg::XC: g = xs; esz = LY::XE; wa = d0.x; wb = d0.y; off = LY::oXC; break;
                    case stg::XM: g = xs; esz = LY::XE; wa = d0.z; wb = d0.w; off = LY::oXM; break;
                    case stg::XP: g = xs; esz = LY::XE; wa = d1.x; wb = d1.y; off = LY::oXP; break;
                    case stg::OC: if (LY::OWIN) { g = a.od; wa = d0.x; wb = d0.y; off = LY::oOC; } break;
                    case stg::OM: if (LY::OWIN) { g = a.od; wa = d0.z; wb = d0.w; off = LY::oOM; } break;
                    case stg::OP: if (LY::OWIN) { g = a.od; wa = d1.x; wb = d1.y; off = LY::oOP; } break;
                    case stg::WX: g = v.wx; wa = P0 > 0 ? P0 - 1 : 0; wb = P1; off = LY::oWX; break;
                    case stg::WY: g = v.wy; wa = d0.x < P0 ? d0.x : P0; wb = P1; off = LY::oWY; break;
                    case stg::WZ: g = v.wz; wa = P0; wb = P1; off = LY::oWZ; break;
                    case stg::WZM: g = v.wz; wa = d0.z; wb = d0.w; off = LY::oWZM; break;
                    case stg::OT: if (LY::OTILE) { g = a.od; wa = P0; wb = P1; off = LY::oOT; } break;
                    case stg::RT:
                        if (LY::RTILE) {
                            g = (MODE == 4 && a.base) ? a.base : a.r;
                            esz = 8 * R; wa = P0; wb = P1; off = LY::oRT;
                        }
                        break;
                    case stg::MK: g = v.mask; esz = 4; wa = P0 >> 5; wb = (P1 + 31) >> 5; off = LY::oMK; break;
                    case stg::RY: g = v.rows; esz = 16; wa = r0 - 1 > 0 ? r0 - 1 : 0; wb = r1 + 2; off = LY::oRY; break;
                    case stg::RM:
                        g = v.rows; esz = 16; wa = r0 - v.NY > 0 ? r0 - v.NY : 0; wb = r1 - v.NY + 1; off = LY::oRM;
                        break;
                    case stg::RP: g = v.rows; esz = 16; wa = r0 + v.NY; wb = r1 + v.NY + 1; off = LY::oRP; break;
                    default: break;
                }
            }
            int w0 = 0;
            const char *src = nullptr;
            const unsigned bytes = lane < stg::NSLOT ? stg::plan(g, esz, wa, wb, w0, src) : 0u;
            if (lane < stg::NSLOT) w0s[st][lane] = w0;
            if (lane == 0) { dsc[st][0] = d0; dsc[st][1] = d1; }
            unsigned tot = bytes;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
            __syncwarp();
            if (lane == 0) stg::mbar_expect(&full[st], tot);  // releases w0s / dsc to the consumers
            __syncwarp();
            if (bytes) stg::bulk_g2s(smem + (size_t)st * LY::STAGE + off, src, bytes, &full[st]);
        }
        return;
    }

    // ---------------- consumer warps ----------------
    double dot[R];
#pragma unroll
    for (int c = 0; c < R; ++c) dot[c] = 0.0;
    for (int i = 0;; ++i) {
        const int t = tile_of(i);
        if (t < 0) break;
        const int st = i % S;
        stg::mbar_wait(&full[st], (unsigned)((i / S) & 1));
        const int4 d1 = dsc[st][1];
        const bool staged = !(d1.w & kStageFlat);
        const int r0 = d1.z, r1 = d1.w & (kStageFlat - 1);
        const int64_t P0 = (int64_t)t * kStage, P1 = P0 + kStage < v.L ? P0 + kStage : v.L;
        if (!staged) {
            // per-position path from global memory (point_out, as k_span)
            int row = r0;
#pragma unroll 1
            for (int u = 0; u < kStage / stg::kConsumers; ++u) {
                const int p = (int)P0 + u * stg::kConsumers + tid;
                if (p >= P1) break;
                row = frow(v.rows, row, r1, p);
                const int4 q = v.rows[row];
                const Nbr n = neighbours(v, p, row, q);
                T dotv = W::zero();
                T out = point_out<R, MODE>(a, n, p, dotv);
                if (!mbit(v.mask, p)) out = W::zero();
                W::st(a.y, p, out);
                if (DOT) {
#pragma unroll
                    for (int c = 0; c < R; ++c)
                        dot[c] += (MODE == 0 || MODE == 3) ? W::dot(dotv, out, c) : W::dot(out, out, c);
                }
            }
        } else {
            const unsigned char *base = smem + (size_t)st * LY::STAGE;
            const int *w0 = w0s[st];
            const int4 *sRY = reinterpret_cast<const int4 *>(base + LY::oRY) - w0[stg::RY];
            const int4 *sRM = reinterpret_cast<const int4 *>(base + LY::oRM) - w0[stg::RM];
            const int4 *sRP = reinterpret_cast<const int4 *>(base + LY::oRP) - w0[stg::RP];
            const double *sWX = reinterpret_cast<const double *>(base + LY::oWX) - w0[stg::WX];
            const double *sWY = reinterpret_cast<const double *>(base + LY::oWY) - w0[stg::WY];
            const double *sWZ = reinterpret_cast<const double *>(base + LY::oWZ) - w0[stg::WZ];
            const double *sWZM = reinterpret_cast<const double *>(base + LY::oWZM) - w0[stg::WZM];
            const uint32_t *sMK = reinterpret_cast<const uint32_t *>(base + LY::oMK) - w0[stg::MK];
            // warp w takes the tile's 32-position row chunks w, w + 16, ...:
            // the row records and neighbour-row offsets are warp-uniform
            const int warp = tid >> 5, lane = tid & 31;
            int row = r0, cbase = 0;  // chunks of the rows before `row`
            for (int c = warp;; c += stg::kConsumers / 32) {
                int sa = 0, sb = 0;
                while (row <= r1) {
                    const int xa = sRY[row].x, xb = sRY[row + 1].x;
                    sa = xa > (int)P0 ? xa : (int)P0;
                    sb = xb < (int)P1 ? xb : (int)P1;
                    const int nch = sb > sa ? (sb - sa + 31) >> 5 : 0;
                    if (c < cbase + nch) break;
                    cbase += nch;
                    ++row;
                }
                if (row > r1) break;
                const int p = sa + ((c - cbase) << 5) + lane;
                if (p >= sb) continue;
                const int4 q = sRY[row];
                const int i_ = q.y + (p - q.x), j = q.w;
                auto sp = [&](int4 uu) { return (i_ >= uu.y && i_ < uu.z) ? uu.x + (i_ - uu.y) : -1; };
                Nbr n;
                n.pxm = (i_ > q.y) ? p - 1 : -1;
                n.pxp = (i_ + 1 < q.z) ? p + 1 : -1;
                n.pym = (j > 0) ? sp(sRY[row - 1]) : -1;
                n.pyp = (j + 1 < v.NY) ? sp(sRY[row + 1]) : -1;
                n.pzm = (row >= v.NY) ? sp(sRM[row - v.NY]) : -1;
                n.pzp = (row + v.NY < v.n_rows) ? sp(sRP[row + v.NY]) : -1;
                n.wxp = sWX[p];
                n.wyp = sWY[p];
                n.wzp = sWZ[p];
                n.wxm = n.pxm >= 0 ? sWX[n.pxm] : 0.0;
                n.wym = n.pym >= 0 ? sWY[n.pym] : 0.0;
                n.wzm = n.pzm >= 0 ? sWZM[n.pzm] : 0.0;
                n.diag = add_rn(add_rn(add_rn(add_rn(add_rn(n.wxp, n.wyp), n.wzp), n.wxm), n.wym), n.wzm);

                T xc, vzm = W::zero(), vym = W::zero(), vxm = W::zero(), vxp = W::zero(), vyp = W::zero(),
                      vzp = W::zero();
                if (MODE == 4) {
                    const int32_t *sC = reinterpret_cast<const int32_t *>(base + LY::oXC) - w0[stg::XC];
                    const int32_t *sM = reinterpret_cast<const int32_t *>(base + LY::oXM) - w0[stg::XM];
                    const int32_t *sP = reinterpret_cast<const int32_t *>(base + LY::oXP) - w0[stg::XP];
                    auto e = [&](int g1) { return g1 > 0 ? W::ld(a.ec, g1 - 1) : W::zero(); };
                    xc = e(sC[p]);
                    if (n.pzm >= 0) vzm = e(sM[n.pzm]);
                    if (n.pym >= 0) vym = e(sC[n.pym]);
                    if (n.pxm >= 0) vxm = e(sC[n.pxm]);
                    if (n.pxp >= 0) vxp = e(sC[n.pxp]);
                    if (n.pyp >= 0) vyp = e(sC[n.pyp]);
                    if (n.pzp >= 0) vzp = e(sP[n.pzp]);
                } else if (MODE == 2) {
                    const T *sC = reinterpret_cast<const T *>(base + LY::oXC) - w0[stg::XC];
                    const T *sM = reinterpret_cast<const T *>(base + LY::oXM) - w0[stg::XM];
                    const T *sP = reinterpret_cast<const T *>(base + LY::oXP) - w0[stg::XP];
                    const double *oC = reinterpret_cast<const double *>(base + LY::oOC) - w0[stg::OC];
                    const double *oM = reinterpret_cast<const double *>(base + LY::oOM) - w0[stg::OM];
                    const double *oP = reinterpret_cast<const double *>(base + LY::oOP) - w0[stg::OP];
                    xc = W::scale(oC[p], sC[p]);
                    if (n.pzm >= 0) vzm = W::scale(oM[n.pzm], sM[n.pzm]);
                    if (n.pym >= 0) vym = W::scale(oC[n.pym], sC[n.pym]);
                    if (n.pxm >= 0) vxm = W::scale(oC[n.pxm], sC[n.pxm]);
                    if (n.pxp >= 0) vxp = W::scale(oC[n.pxp], sC[n.pxp]);
                    if (n.pyp >= 0) vyp = W::scale(oC[n.pyp], sC[n.pyp]);
                    if (n.pzp >= 0) vzp = W::scale(oP[n.pzp], sP[n.pzp]);
                } else {
                    const T *sC = reinterpret_cast<const T *>(base + LY::oXC) - w0[stg::XC];
                    const T *sM = reinterpret_cast<const T *>(base + LY::oXM) - w0[stg::XM];
                    const T *sP = reinterpret_cast<const T *>(base + LY::oXP) - w0[stg::XP];
                    xc = sC[p];
                    if (n.pzm >= 0) vzm = sM[n.pzm];
                    if (n.pym >= 0) vym = sC[n.pym];
                    if (n.pxm >= 0) vxm = sC[n.pxm];
                    if (n.pxp >= 0) vxp = sC[n.pxp];
                    if (n.pyp >= 0) vyp = sC[n.pyp];
                    if (n.pzp >= 0) vzp = sP[n.pzp];
                }
                // A x in the reference's sorted-column order (apply_row)
                T s = W::zero();
                if (n.pzm >= 0) s = W::axpy(-n.wzm, vzm, s);
                if (n.pym >= 0) s = W::axpy(-n.wym, vym, s);
                if (n.pxm >= 0) s = W::axpy(-n.wxm, vxm, s);
                s = W::axpy(n.diag, xc, s);
                if (n.pxp >= 0) s = W::axpy(-n.wxp, vxp, s);
                if (n.pyp >= 0) s = W::axpy(-n.wyp, vyp, s);
                if (n.pzp >= 0) s = W::axpy(-n.wzp, vzp, s);

                T out, dotv = W::zero();
                if (MODE == 0) {
                    out = s;
                    dotv = xc;
                } else if (MODE == 2) {
                    const T *sC = reinterpret_cast<const T *>(base + LY::oXC) - w0[stg::XC];
                    out = W::sub(sC[p], s);
                } else {
                    const T *sR = reinterpret_cast<const T *>(base + LY::oRT) - w0[stg::RT];
                    const T rc = sR[p];
                    if (MODE == 1) {
                        out = W::sub(rc, s);
                    } else {
                        const double *sO = reinterpret_cast<const double *>(base + LY::oOT) - w0[stg::OT];
                        const double odc = sO[p];
                        if (MODE == 3) {
                            out = W::add(xc, W::scale(odc, W::sub(rc, s)));
                            dotv = rc;
                        } else {  // MODE 4: (base + e) - od (A e), base = od r when null
                            const T b = a.base ? rc : W::scale(odc, rc);
                            out = W::sub(W::add(b, xc), W::scale(odc, s));
                        }
                    }
                }
                if (!((sMK[p >> 5] >> (p & 31)) & 1u)) out = W::zero();
                W::st(a.y, p, out);
                if (DOT) {
#pragma unroll
                    for (int c = 0; c < R; ++c)
                        dot[c] += (MODE == 0 || MODE == 3) ? W::dot(dotv, out, c) : W::dot(out, out, c);
                }
            }
        }
        __syncwarp();
        if ((tid & 31) == 0) stg::mbar_arrive(&empty[st]);
    }
    if (DOT) {
        // consumer-only block reduction (fixed order) -> one partial per CTA
#pragma unroll
        for (int c = 0; c < R; ++c)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) dot[c] += __shfl_xor_sync(0xffffffffu, dot[c], o);
        if ((tid & 31) == 0)
#pragma unroll
            for (int c = 0; c < R; ++c) red[(tid >> 5) * R + c] = dot[c];
        stg::consumer_sync();
        if (tid == 0) {
#pragma unroll
            for (int c = 0; c < R; ++c) {
                double sum = 0.0;
                for (int w = 0; w < stg::kConsumers / 32; ++w) sum += red[w * R + c];
                a.partials[blockIdx.x * R + c] = sum;
            }
        }
    }
}

// 2.5-D z-marching stencil kernel for the fine level (included by solve.cu).
//
// A CTA owns a block of JB node rows (j0 .. j0+JB-1) and marches through a
// range of z-planes.  The stencil input of the rows j0-1 .. j0+JB of three
// consecutive planes is staged in shared memory in box coordinates (zero
// outside the conductive spans), so every +-x/+-y/+-z neighbour is a fixed
// shared-memory offset: the HBM stream is read once per CTA (plus the
// j/k halo, mostly served by L2) instead of being gathered through the row
// table per position.  One warp computes one row of the current plane;
// edge weights stream from global memory (the -y/-z ones hit L1 because
// the neighbouring warp / previous plane step just loaded them).
//
// The products are accumulated in the reference's sorted-column order with
// explicitly rounded operations (zeros outside the spans contribute exact
// -0.0 terms), so MODE 0 is bit-identical to scipy's csr_matvec.
#pragma once

constexpr int kPlaneJB = 8;                     // rows per CTA (one warp each)
constexpr int kPlaneThreads = 32 * kPlaneJB;

struct PlaneGeo {
    int NX, NY, NZ;     // node box
    int jblocks, kb;    // j-blocks, planes per CTA
    int kblocks;
};

inline PlaneGeo plane_geo(const Operator &op, int ctas_per_sm) {
    PlaneGeo g;
    g.NX = (int)op.NX; g.NY = (int)op.NY; g.NZ = (int)op.NZ;
    g.jblocks = (g.NY + kPlaneJB - 1) / kPlaneJB;
    // about two waves of CTAs: halo planes cost (kb + 2) / kb extra reads
    long target = 2L * 148 * (ctas_per_sm > 0 ? ctas_per_sm : 1);
    long kb = ((long)g.jblocks * g.NZ + target - 1) / target;
    if (kb < 4) kb = 4;
    if (kb > g.NZ) kb = g.NZ;
    g.kb = (int)kb;
    g.kblocks = (g.NZ + g.kb - 1) / g.kb;
    return g;
}

// bytes of one staged element per mode: the stencil input (x / e source),
// MODE 2 stages r and od separately, MODE 4 stages aggregate ids
template <int R, int MODE>
struct PlaneStage {
    static constexpr size_t bytes = MODE == 2 ? sizeof(typename V<R>::T) + sizeof(double)
                                  : (MODE == 4 ? sizeof(int32_t) : sizeof(typename V<R>::T));
};

constexpr int kPlaneSlots = 4;  // k-1, k, k+1 in use, k+2 in flight

template <int R, int MODE>
inline size_t plane_smem(const PlaneGeo &g) {
    return (size_t)kPlaneSlots * (kPlaneJB + 2) * g.NX * PlaneStage<R, MODE>::bytes + 64;
}

__device__ __forceinline__ void cp_async_zfill(void *smem, const void *gmem, int bytes, bool valid) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    const int n = valid ? bytes : 0;
    if (bytes == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
    else if (bytes == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <int R, int MODE, bool DOT>
__global__ void __launch_bounds__(kPlaneThreads) k_plane(SpanView v, PlaneGeo g, SpanArgs a) {
    using W = V<R>;
    using T = typename W::T;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ double red[32 * R];
    const int NX = g.NX;
    constexpr int RPS = kPlaneJB + 2;  // rows per slot (with the j halo)
    const size_t slot_elems = (size_t)RPS * NX;
    // ring layout: [slots][RPS][NX] of the primary staged array, then (MODE 2) od
    T *Sx = reinterpret_cast<T *>(smem_raw);
    double *Sod = reinterpret_cast<double *>(smem_raw + kPlaneSlots * slot_elems * sizeof(T));
    int32_t *Sag = reinterpret_cast<int32_t *>(smem_raw);
    auto slot = [&](int kk) { return (size_t)((kk + kPlaneSlots) % kPlaneSlots) * slot_elems; };

    const int jb = blockIdx.x % g.jblocks, kbk = blockIdx.x / g.jblocks;
    const int j0 = jb * kPlaneJB, k0 = kbk * g.kb, k1 = min(g.NZ, k0 + g.kb);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    double dot[R];
#pragma unroll
    for (int c = 0; c < R; ++c) dot[c] = 0.0;

    // asynchronous zero-filled copy of rows j0-1 .. j0+JB of plane kk
    auto stage = [&](int kk) {
        const size_t base = slot(kk);
        for (int rr = warp; rr < RPS; rr += kPlaneJB) {
            const int j = j0 - 1 + rr;
            int off = 0, lo = 0, hi = 0;
            if (j >= 0 && j < g.NY && kk >= 0 && kk < g.NZ) {
                const int4 q = v.rows[j + g.NY * kk];
                off = q.x; lo = q.y; hi = q.z;
            }
            const size_t rb = base + (size_t)rr * NX;
            for (int i = lane; i < NX; i += 32) {
                const bool in = i >= lo && i < hi;
                const int64_t gp = in ? (int64_t)off + (i - lo) : 0;
                if (MODE == 4) {
                    cp_async_zfill(Sag + rb + i, a.aggp + gp, 4, in);
                } else if (MODE == 2) {
                    cp_async_zfill(Sx + rb + i, a.r + gp * R, (int)sizeof(T), in);
                    cp_async_zfill(Sod + rb + i, a.od + gp, 8, in);
                } else {
                    cp_async_zfill(Sx + rb + i, a.x + gp * R, (int)sizeof(T), in);
                }
            }
        }
        cp_async_commit();
    };
    // stencil input at ring index q
    auto X = [&](size_t q) -> T {
        if (MODE == 2) return W::scale(Sod[q], Sx[q]);
        if (MODE == 4) {
            const int g1 = Sag[q];
            return g1 > 0 ? W::ld(a.ec, g1 - 1) : W::zero();
        }
        return Sx[q];
    };

    if (k0 < k1) {
        stage(k0 - 1);
        stage(k0);
        stage(k0 + 1);
    }
    for (int k = k0; k < k1; ++k) {
        stage(k + 2);
        cp_async_wait<1>();
        __syncthreads();
        const int j = j0 + warp;
        if (j < g.NY) {
            const int r = j + g.NY * k;
            const int4 q = v.rows[r];
            if (q.z > q.y) {
                const size_t bm = slot(k - 1) + (size_t)(warp + 1) * NX;
                const size_t bc = slot(k) + (size_t)(warp + 1) * NX;
                const size_t bp = slot(k + 1) + (size_t)(warp + 1) * NX;
                const int4 qy = j > 0 ? v.rows[r - 1] : make_int4(0, 0, 0, 0);
                const int4 qz = k > 0 ? v.rows[r - g.NY] : make_int4(0, 0, 0, 0);
                for (int i0 = q.y; i0 < q.z; i0 += 32) {
                    const int i = i0 + lane;
                    const bool on = i < q.z;
                    const int ic = on ? i : q.y;
                    const int ps = q.x + (ic - q.y);
                    const double wxp = v.wx[ps], wyp = v.wy[ps], wzp = v.wz[ps];
                    double wxm = __shfl_up_sync(0xffffffffu, wxp, 1);
                    if (lane == 0) wxm = ic > q.y ? v.wx[ps - 1] : 0.0;
                    if (ic == q.y) wxm = 0.0;
                    const double wym = (ic >= qy.y && ic < qy.z) ? v.wy[qy.x + (ic - qy.y)] : 0.0;
                    const double wzm = (ic >= qz.y && ic < qz.z) ? v.wz[qz.x + (ic - qz.y)] : 0.0;
                    const T xc = X(bc + ic);
                    const T xxm = ic > 0 ? X(bc + ic - 1) : W::zero();
                    const T xxp = ic + 1 < NX ? X(bc + ic + 1) : W::zero();
                    const T xym = X(bc + ic - NX);
                    const T xyp = X(bc + ic + NX);
                    const T xzm = X(bm + ic);
                    const T xzp = X(bp + ic);
                    const double diag = add_rn(add_rn(add_rn(add_rn(add_rn(wxp, wyp), wzp), wxm), wym), wzm);
                    T s = W::zero();
                    s = W::axpy(-wzm, xzm, s);
                    s = W::axpy(-wym, xym, s);
                    s = W::axpy(-wxm, xxm, s);
                    s = W::axpy(diag, xc, s);
                    s = W::axpy(-wxp, xxp, s);
                    s = W::axpy(-wyp, xyp, s);
                    s = W::axpy(-wzp, xzp, s);
                    T out;
                    if (MODE == 0) out = s;
                    else if (MODE == 1) out = W::sub(W::ld(a.r, ps), s);
                    else if (MODE == 2) out = W::sub(Sx[bc + ic], s);
                    else if (MODE == 3) out = W::add(xc, W::scale(a.od[ps], W::sub(W::ld(a.r, ps), s)));
                    else {
                        const T b = a.base ? W::ld(a.base, ps) : W::scale(a.od[ps], W::ld(a.r, ps));
                        out = W::sub(W::add(b, xc), W::scale(a.od[ps], s));
                    }
                    if (!mbit(v.mask, ps)) out = W::zero();
                    if (on) {
                        W::st(a.y, ps, out);
                        if (DOT) {
#pragma unroll
                            for (int c = 0; c < R; ++c) {
                                if (MODE == 0) dot[c] += W::dot(xc, out, c);
                                else if (MODE == 3) dot[c] += W::dot(W::ld(a.r, ps), out, c);
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

// Cooperative "tail" V-cycle for the small coarse levels (included by
// solve.cu).  Below a few hundred thousand rows the per-level kernels are
// latency-bound (a launch and a dependent-load chain each for ~5-30 us of
// work).  One cooperative launch runs the whole remaining V-cycle --
// pre-smooth + defect, restriction, the dense coarsest solve, prolongation
// and post-smooth on every tail level -- with grid-wide barriers between
// the dependent steps.  Rows are processed by fixed lane groups with a fixed
// reduction order, so the result is deterministic and equals the per-level
// kernels up to rounding.
#pragma once
#include <cooperative_groups.h>

struct TailLevel {
    CsrView A, P, R;     // P: n_l x n_{l+1}, R: n_{l+1} x n_l
    const double *od;    // omega D^-1
    double *r, *x, *d;   // level vectors (interleaved nrhs)
    int gA, gP, gR;      // lanes per row
};

constexpr int kTailMax = 8;

struct TailArgs {
    TailLevel lv[kTailMax];
    int nlev;
    const double *cinv;
    int64_t nc;
    double *rc, *zc;     // coarsest rhs / solution
};

// one CSR row-product step over the whole grid (group of G lanes per row)
// MODE 2: y = r - M(od r); 0: y = M x; 4: y = od r + M x; 3: y = x + od (r - M x)
template <int R, int MODE>
__device__ void tail_rows(const CsrView &m, int G, const double *x, const double *r, const double *od, double *y) {
    using W = V<R>;
    using T = typename W::T;
    const int lane = threadIdx.x & 31;
    const int gl = lane % G;
    const int gpw = 32 / G;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t rb = warp * gpw; rb < m.rows; rb += nwarp * gpw) {
        const int64_t row = rb + lane / G;
        const bool valid = row < m.rows;
        T acc = W::zero();
        if (valid) {
            for (int64_t q = m.ptr[row] + gl; q < m.ptr[row + 1]; q += G) {
                const int c = m.col[q];
                const T xv = MODE == 2 ? W::scale(od[c], W::ld(r, c)) : W::ld(x, c);
                acc = W::fma_(m.val[q], xv, acc);
            }
        }
        double ac[R];
#pragma unroll
        for (int cpt = 0; cpt < R; ++cpt) {
            ac[cpt] = W::comp(acc, cpt);
            for (int o = G / 2; o > 0; o >>= 1) ac[cpt] += __shfl_xor_sync(0xffffffffu, ac[cpt], o, G);
        }
        if (valid && gl == 0) {
            T sum;
            if constexpr (R == 1) sum = ac[0];
            else sum = make_double2(ac[0], ac[1]);
            T out;
            if (MODE == 0) out = sum;
            else if (MODE == 2) out = W::sub(W::ld(r, row), sum);
            else if (MODE == 4) out = W::add(W::scale(od[row], W::ld(r, row)), sum);
            else out = W::add(W::ld(x, row), W::scale(od[row], W::sub(W::ld(r, row), sum)));
            W::st(y, row, out);
        }
    }
}

template <int R>
__global__ void __launch_bounds__(256) k_tail(TailArgs t) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    // down: pre-smooth + defect, restriction
    for (int l = 0; l < t.nlev; ++l) {
        const TailLevel &L = t.lv[l];
        tail_rows<R, 2>(L.A, L.gA, nullptr, L.r, L.od, L.d);
        grid.sync();
        double *nr = l + 1 < t.nlev ? t.lv[l + 1].r : t.rc;
        tail_rows<R, 0>(L.R, L.gR, L.d, nullptr, nullptr, nr);
        grid.sync();
    }
    // coarsest: dense inverse (one warp per row)
    {
        const int lane = threadIdx.x & 31;
        const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
        const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
        for (int64_t row = warp; row < t.nc; row += nwarp) {
            double acc[R];
#pragma unroll
            for (int c = 0; c < R; ++c) acc[c] = 0.0;
            for (int64_t j = lane; j < t.nc; j += 32) {
                const double a = t.cinv[row * t.nc + j];
#pragma unroll
                for (int c = 0; c < R; ++c) acc[c] = fma(a, t.rc[j * R + c], acc[c]);
            }
#pragma unroll
            for (int c = 0; c < R; ++c)
                for (int o = 16; o > 0; o >>= 1) acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], o);
            if (lane == 0)
#pragma unroll
                for (int c = 0; c < R; ++c) t.zc[row * R + c] = acc[c];
        }
    }
    grid.sync();
    // up: prolongation + correction, post-smooth
    for (int l = t.nlev - 1; l >= 0; --l) {
        const TailLevel &L = t.lv[l];
        const double *e = l + 1 < t.nlev ? t.lv[l + 1].x : t.zc;
        tail_rows<R, 4>(L.P, L.gP, e, L.r, L.od, L.d);
        grid.sync();
        tail_rows<R, 3>(L.A, L.gA, L.d, L.r, L.od, L.x);
        if (l > 0) grid.sync();
    }
}

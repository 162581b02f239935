// SURVEY §8 rows f1-f4 on the device: the stages either side of the Poisson
// hot path that turn sampled flux densities into the edge vector potential
// and the voxel |E| into exposure statistics.
//
//   f3  coil_field (Biot-Savart, field_source.py:163-197) and
//       interpolate_to_faces (trilinear midpoint flux, field_source.py:218-272)
//   f2  divergence (build_divergence, fit_operators.py:276-286) and
//       divergence_clean (field_source.py:292-329): the l2-minimal
//       projection through an AMG-preconditioned solve on div divᵀ, reusing
//       the hot path's own setup and Krylov solver
//   f1  comb-tree gauging (gauging.py:34-71,137-172 + _kernels.py:12-76) as
//       three column prefix scans, plus the circulation residual check
//   f4  exposure statistics (dosimetry.py:119-127,195-234): nearest-rank
//       p99 / max / mean, globally and per tissue, via radix sorts
//
// Bit-exactness: interpolation, divergence, div-transpose and the gauge scans
// use explicitly rounded operations in the reference's evaluation order, so
// they equal numpy bit for bit; p99 and max are exact selections.  Norms
// (threshold tests only), means and the cleaning solve are floating-point
// reductions compared within tolerance.

#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>

#include "amg.cuh"
#include "common.cuh"
#include "field.cuh"

namespace spfd {
namespace {

// ------------------------------------------------------------- geometry --
struct Box {
    int64_t n[3];   // grid: voxels per axis; lattice: points per axis
    double h[3];
    double o[3];
};

inline Box box_of(const spfd_box &b) {
    Box r;
    for (int a = 0; a < 3; ++a) { r.n[a] = b.dims[a]; r.h[a] = b.spacing[a]; r.o[a] = b.origin[a]; }
    return r;
}

__host__ __device__ inline int64_t face_count(const Box &g, int a) {
    int64_t c = 1;
    for (int d = 0; d < 3; ++d) c *= g.n[d] + (d == a ? 1 : 0);
    return c;
}
__host__ __device__ inline int64_t edge_count(const Box &g, int a) {
    int64_t c = 1;
    for (int d = 0; d < 3; ++d) c *= g.n[d] + (d == a ? 0 : 1);
    return c;
}

// face-center coordinate along axis `d` of a face with normal `a`
// (StaggeredGrid.face_center_axes, fit_operators.py:156-165)
__host__ __device__ inline double face_coord(const Box &g, int a, int d, int64_t i) {
#ifdef __CUDA_ARCH__
    if (d == a) return __dadd_rn(g.o[d], __dmul_rn((double)i, g.h[d]));
    return __dadd_rn(g.o[d], __dmul_rn(__dadd_rn((double)i, 0.5), g.h[d]));
#else
    volatile double t = d == a ? (double)i : (double)i + 0.5;
    volatile double m = t * g.h[d];
    return g.o[d] + m;
#endif
}

// ----------------------------------------------------- f3: interpolation --
// _axis_interp_params (field_source.py:218-233): base index, local coordinate
// and the corner step (0 on a single-point axis).
struct AxisParam {
    int64_t i0;
    double t;
    int64_t s;
};

__device__ inline AxisParam axis_param(double c, double origin, double spacing, int64_t n) {
    const double u = __ddiv_rn(__dsub_rn(c, origin), spacing);
    if (n == 1) return {0, 0.0, 0};
    int64_t i0 = (int64_t)floor(u);
    i0 = i0 < 0 ? 0 : (i0 > n - 2 ? n - 2 : i0);
    return {i0, __dsub_rn(u, (double)i0), 1};
}

// The trilinear parameters of a face depend on one coordinate each, so they
// are tabulated per axis (k_axis_params: d0 + d1 + d2 entries) and the face
// kernel walks face rows (j, k) with threads along i (_trilinear +
// interpolate_to_faces, field_source.py:235-272: the sum over the 8 corners
// in (dx, dy, dz) order of ((wx*wy)*wz)*corner, times the face area), without
// per-face divisions or 64-bit div/mod.
__global__ void k_axis_params(Box g, Box lat, int a, AxisParam *tab) {
    int64_t d[3] = {g.n[0], g.n[1], g.n[2]};
    d[a] += 1;
    const int64_t tot = d[0] + d[1] + d[2];
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < tot; q += (int64_t)gridDim.x * blockDim.x) {
        const int ax = q < d[0] ? 0 : (q < d[0] + d[1] ? 1 : 2);
        const int64_t i = ax == 0 ? q : (ax == 1 ? q - d[0] : q - d[0] - d[1]);
        tab[q] = axis_param(face_coord(g, a, ax, i), lat.o[ax], lat.h[ax], lat.n[ax]);
    }
}

// One warp per face row (j, k), lanes along i; the four (dy, dz) lattice
// row offsets and weights are hoisted per row, and index math is 32-bit (the
// lattice is small).  Same corner order and products as the reference.
__global__ void __launch_bounds__(256) k_interp_rows(Box g, Box lat, int a, const AxisParam *__restrict__ tab,
                                                     const double *__restrict__ b, double area,
                                                     double *__restrict__ flux) {
    int64_t d[3] = {g.n[0], g.n[1], g.n[2]};
    d[a] += 1;
    const int nrow = (int)(d[1] * d[2]), n0 = (int)d[0], ny = (int)d[1];
    const int ln0 = (int)lat.n[0], ln1 = (int)lat.n[1];
    const AxisParam *tx = tab, *ty = tab + d[0], *tz = tab + d[0] + d[1];
    const int lane = threadIdx.x & 31;
    const int warps = gridDim.x * (blockDim.x >> 5);
    for (int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < nrow; row += warps) {
        const int j = row % ny, k = row / ny;
        const AxisParam py = ty[j], pz = tz[k];
        const double wy[2] = {__dsub_rn(1.0, py.t), py.t}, wz[2] = {__dsub_rn(1.0, pz.t), pz.t};
        int off[2][2];
#pragma unroll
        for (int dy = 0; dy < 2; ++dy)
#pragma unroll
            for (int dz = 0; dz < 2; ++dz)
                off[dy][dz] = ln0 * ((int)(py.i0 + dy * py.s) + ln1 * (int)(pz.i0 + dz * pz.s));
        double *frow = flux + (int64_t)row * n0;
        for (int i = lane; i < n0; i += 32) {
            const AxisParam px = tx[i];
            double out = 0.0;
#pragma unroll
            for (int dx = 0; dx < 2; ++dx) {
                const double wx = dx ? px.t : __dsub_rn(1.0, px.t);
                const int ix = (int)(px.i0 + dx * px.s);
#pragma unroll
                for (int dy = 0; dy < 2; ++dy) {
                    const double wxy = __dmul_rn(wx, wy[dy]);
#pragma unroll
                    for (int dz = 0; dz < 2; ++dz)
                        out = __dadd_rn(out, __dmul_rn(__dmul_rn(wxy, wz[dz]), b[3 * (ix + off[dy][dz]) + a]));
                }
            }
            frow[i] = __dmul_rn(out, area);
        }
    }
}

// Biot-Savart field of a closed polyline (coil_field, field_source.py:163-197):
// exact finite straight-wire expression per segment.  flag[0] is set when a
// point lies within `eps` of a wire segment (SingularPointError).
__global__ void k_coil_field(int64_t n, const double *__restrict__ pts, int nseg, const double *__restrict__ verts,
                             double scale, double eps2, double *__restrict__ out, int *flag) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
        const double px = pts[3 * q], py = pts[3 * q + 1], pz = pts[3 * q + 2];
        double bx = 0.0, by = 0.0, bz = 0.0;
        bool singular = false;
        for (int s = 0; s < nseg; ++s) {
            const double x1 = verts[3 * s], y1 = verts[3 * s + 1], z1 = verts[3 * s + 2];
            const double sx = verts[3 * s + 3] - x1, sy = verts[3 * s + 4] - y1, sz = verts[3 * s + 5] - z1;
            const double l2 = sx * sx + sy * sy + sz * sz;
            const double ax = px - x1, ay = py - y1, az = pz - z1;
            const double cx = ax - sx, cy = ay - sy, cz = az - sz;   // b = a - seg
            double t = (ax * sx + ay * sy + az * sz) / l2;
            t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
            const double qx = ax - t * sx, qy = ay - t * sy, qz = az - t * sz;
            if (qx * qx + qy * qy + qz * qz < eps2) singular = true;
            const double la = sqrt(ax * ax + ay * ay + az * az);
            const double lb = sqrt(cx * cx + cy * cy + cz * cz);
            const double crx = ay * cz - az * cy, cry = az * cx - ax * cz, crz = ax * cy - ay * cx;
            const double sum = la + lb;
            const double coeff = 2.0 * sum / (la * lb * (sum * sum - l2));
            bx += coeff * crx;
            by += coeff * cry;
            bz += coeff * crz;
        }
        if (singular) atomicExch(flag, 1);
        out[3 * q] = scale * bx;
        out[3 * q + 1] = scale * by;
        out[3 * q + 2] = scale * bz;
    }
}

// ------------------------------------------------------ f2: divergence --
// net outflux per cell = build_divergence(grid) @ fluxes: the six faces in
// ascending face index (x-, x+, y-, y+, z-, z+) with signs -,+,-,+,-,+,
// accumulated like scipy's csr_matvec.
__global__ void k_divergence(Box g, const double *__restrict__ f, double *__restrict__ div) {
    const int64_t nx = g.n[0], ny = g.n[1], nz = g.n[2];
    const int64_t nc = nx * ny * nz;
    const int64_t fx = (nx + 1) * ny * nz, fy = nx * (ny + 1) * nz;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nc; c += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = c % nx, j = (c / nx) % ny, k = c / (nx * ny);
        const int64_t x0 = i + (nx + 1) * (j + ny * k);
        const int64_t y0 = fx + i + nx * (j + (ny + 1) * k);
        const int64_t z0 = fx + fy + c;
        double s = 0.0;
        s = __dadd_rn(s, __dmul_rn(-1.0, f[x0]));
        s = __dadd_rn(s, f[x0 + 1]);
        s = __dadd_rn(s, __dmul_rn(-1.0, f[y0]));
        s = __dadd_rn(s, f[y0 + nx]);
        s = __dadd_rn(s, __dmul_rn(-1.0, f[z0]));
        s = __dadd_rn(s, f[z0 + nx * ny]);
        div[c] = s;
    }
}

// out = in - divᵀ phi: a face gets +phi of the cell on its low side (it is
// that cell's "+" face) and -phi of the cell on its high side, accumulated in
// ascending cell order like scipy's csc_matvec of div.T.
__global__ void k_sub_div_transpose(Box g, const double *__restrict__ phi, const double *__restrict__ in,
                                    double *__restrict__ out) {
    // 32-bit face / cell indices (the caller checks the box size)
    const int nx = (int)g.n[0], ny = (int)g.n[1], nz = (int)g.n[2];
    const int fx = (nx + 1) * ny * nz, fy = nx * (ny + 1) * nz, fz = nx * ny * (nz + 1);
    const int nf = fx + fy + fz;
    for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < nf; f += gridDim.x * blockDim.x) {
        int lo = -1, hi = -1;
        if (f < fx) {
            const int i = f % (nx + 1), r = f / (nx + 1);          // r = j + ny k
            const int c = i + nx * r;
            if (i > 0) lo = c - 1;
            if (i < nx) hi = c;
        } else if (f < fx + fy) {
            const int q = f - fx;
            const int i = q % nx, j = (q / nx) % (ny + 1), k = q / (nx * (ny + 1));
            const int c = i + nx * (j + ny * k);
            if (j > 0) lo = c - nx;
            if (j < ny) hi = c;
        } else {
            const int q = f - fx - fy;
            const int k = q / (nx * ny);
            if (k > 0) lo = q - nx * ny;
            if (k < nz) hi = q;
        }
        double y = 0.0;
        if (lo >= 0) y = __dadd_rn(y, phi[lo]);
        if (hi >= 0) y = __dadd_rn(y, __dmul_rn(-1.0, phi[hi]));
        out[f] = __dsub_rn(in[f], y);
    }
}

// div divᵀ as CSR with sorted columns (the reference sorts before setup,
// linsolve.py:131-132): diagonal 6, -1 per interior face shared with a
// neighbour cell.
__global__ void k_normal_count(Box g, int64_t *cnt) {
    const int64_t nx = g.n[0], ny = g.n[1], nz = g.n[2], nc = nx * ny * nz;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nc; c += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = c % nx, j = (c / nx) % ny, k = c / (nx * ny);
        cnt[c] = 1 + (i > 0) + (i < nx - 1) + (j > 0) + (j < ny - 1) + (k > 0) + (k < nz - 1);
    }
}

__global__ void k_normal_fill(Box g, const int64_t *__restrict__ ptr, int32_t *__restrict__ col,
                              double *__restrict__ val) {
    const int64_t nx = g.n[0], ny = g.n[1], nz = g.n[2], nc = nx * ny * nz;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nc; c += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = c % nx, j = (c / nx) % ny, k = c / (nx * ny);
        int64_t q = ptr[c];
        auto put = [&](int64_t cc, double v) { col[q] = (int32_t)cc; val[q] = v; ++q; };
        if (k > 0) put(c - nx * ny, -1.0);
        if (j > 0) put(c - nx, -1.0);
        if (i > 0) put(c - 1, -1.0);
        put(c, 6.0);
        if (i < nx - 1) put(c + 1, -1.0);
        if (j < ny - 1) put(c + nx, -1.0);
        if (k < nz - 1) put(c + nx * ny, -1.0);
    }
}

// ------------------------------------------ f2: spectral projection solve --
// div divT on the cell box is the 7-point Laplacian 6 I - adjacency with
// zeros outside the box (k_normal_fill).  Sine transforms (DST-I) along x
// and y diagonalise its x and y parts, leaving for every (x, y) mode (p, q)
// one tridiagonal system along z with diagonal mu_pq = 2 + lx_p + ly_q
// (l_p = 2 - 2 cos(pi (p+1)/(n+1))) and -1 off the diagonal:
//   phi = (4 / ((nx+1)(ny+1))) S_x S_y T_pq^-1 S_y S_x d
// with S the symmetric DST-I matrix sin(pi (a+1)(b+1)/(n+1)).  A direct
// solve to rounding error replaces the reference's AMG-FGMRES at rel_tol
// <= 1e-12 (field_source.py:315-321): the projection agrees with the
// reference to its solve tolerance.  The transforms are FP64 tiled
// products (k_dgemm_split), the z solves one Thomas sweep per mode.

// C(m, n) = sum_k A(m, k) B(k, n) in FP64, k in order (fma chain: the same
// bits as a plain loop).  The column index n is split as n = lo + nlo * hi
// with separate strides, so a batch of planes or both rhs run as one wide
// product: B(k, n) = B[k sBk + lo sBlo + hi sBhi], C(m, n) = C[m sCm + lo sClo + hi sChi].
struct GemmArgs {
    const double *A, *B;
    double *C;
    int64_t M, N, K;
    int64_t sAm, sAk;
    int64_t sBk, nlo, sBlo, sBhi;
    int64_t sCm, sClo, sChi;
};

// BM x BN tile per CTA of 256 threads, 8 x 8 outputs per thread (TM threads
// along m, TN along n); BK = 8 k per stage, the next stage prefetched into
// registers while the current one is multiplied out of shared memory.  The
// DST matrices are 160 / 112 wide at C3, so BM = 32 wastes no rows on x.
constexpr int kGBK = 8;
template <int BM>
__global__ void __launch_bounds__(256, 1) k_dgemm_split(GemmArgs g) {
    constexpr int TM = BM / 8, TN = 256 / TM, BN = TN * 8;
    constexpr int NB = kGBK * BN / 256;       // B elements per thread per stage
    constexpr int NA = (kGBK * BM + 255) / 256;
    __shared__ double As[kGBK][BM];
    __shared__ double Bs[kGBK][BN + 1];
    __shared__ int64_t boff[BN];
    const int tid = threadIdx.x, tm = tid % TM, tn = tid / TM;
    const int64_t m0 = (int64_t)blockIdx.x * BM, n0 = (int64_t)blockIdx.y * BN;
    for (int q = tid; q < BN; q += 256) {
        const int64_t n = n0 + q;
        boff[q] = n < g.N ? (n % g.nlo) * g.sBlo + (n / g.nlo) * g.sBhi : -1;
    }
    __syncthreads();
    const bool nfast = g.sBlo < g.sBk;
    double ra[NA], rb[NB];
    auto load = [&](int64_t k0) {
#pragma unroll
        for (int t = 0; t < NA; ++t) {
            const int e = tid + t * 256;
            const int mm = e % BM, kk = e / BM;
            const int64_t m = m0 + mm, k = k0 + kk;
            ra[t] = (e < kGBK * BM && m < g.M && k < g.K) ? g.A[m * g.sAm + k * g.sAk] : 0.0;
        }
#pragma unroll
        for (int t = 0; t < NB; ++t) {
            const int e = tid + t * 256;
            const int nn = nfast ? e % BN : e / kGBK, kk = nfast ? e / BN : e % kGBK;
            const int64_t o = boff[nn], k = k0 + kk;
            rb[t] = (o >= 0 && k < g.K) ? g.B[k * g.sBk + o] : 0.0;
        }
    };
    auto store = [&]() {
#pragma unroll
        for (int t = 0; t < NA; ++t) {
            const int e = tid + t * 256;
            if (e < kGBK * BM) As[e / BM][e % BM] = ra[t];
        }
#pragma unroll
        for (int t = 0; t < NB; ++t) {
            const int e = tid + t * 256;
            const int nn = nfast ? e % BN : e / kGBK, kk = nfast ? e / BN : e % kGBK;
            Bs[kk][nn] = rb[t];
        }
    };
    double acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.0;
    load(0);
    for (int64_t k0 = 0; k0 < g.K; k0 += kGBK) {
        store();
        __syncthreads();
        if (k0 + kGBK < g.K) load(k0 + kGBK);
#pragma unroll
        for (int kk = 0; kk < kGBK; ++kk) {
            double a[8], b[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = As[kk][tm + TM * i];
#pragma unroll
            for (int j = 0; j < 8; ++j) b[j] = Bs[kk][tn + TN * j];
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int64_t n = n0 + tn + TN * j;
        if (n >= g.N) continue;
        const int64_t co = (n % g.nlo) * g.sClo + (n / g.nlo) * g.sChi;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int64_t m = m0 + tm + TM * i;
            if (m < g.M) g.C[m * g.sCm + co] = acc[i][j];
        }
    }
}

// The eliminated pivots of every mode's z system depend only on the mode:
// inv_k = 1 / (mu + c_{k-1}), c_k = -inv_k, computed once per grid
// (k_tridiag_pivots); the per-snapshot solve (k_tridiag_apply) is then
// division-free, one thread per (mode, rhs):
//   forward  d'_k = (scale d_k + d'_{k-1}) inv_k
//   backward x_k  = d'_k + inv_k x_{k+1}
__global__ void k_tridiag_pivots(int64_t nx, int64_t ny, int64_t nz, const double *__restrict__ lx,
                                 const double *__restrict__ ly, double *__restrict__ inv) {
    const int64_t plane = nx * ny;
    const int64_t col = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (col >= plane) return;
    const double mu = 2.0 + lx[col % nx] + ly[col / nx];
    double c = 0.0;
    for (int64_t k = 0; k < nz; ++k) {
        const double iv = 1.0 / (mu + c);
        c = -iv;
        inv[k * plane + col] = iv;
    }
}

__global__ void k_tridiag_apply(int64_t nx, int64_t ny, int64_t nz, int nrhs, const double *__restrict__ inv,
                                double scale, double *__restrict__ d) {
    constexpr int B = 8;  // z planes per batch: all loads of a batch in flight before its recurrence steps
    const int64_t plane = nx * ny, nc = plane * nz;
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= plane * nrhs) return;
    const int64_t col = t % plane;
    double *x = d + (t / plane) * nc + col;
    const double *iv = inv + col;
    double dp = 0.0;
    for (int64_t k0 = 0; k0 < nz; k0 += B) {
        double xv[B], vv[B];
#pragma unroll
        for (int u = 0; u < B; ++u)
            if (k0 + u < nz) { xv[u] = x[(k0 + u) * plane]; vv[u] = iv[(k0 + u) * plane]; }
#pragma unroll
        for (int u = 0; u < B; ++u)
            if (k0 + u < nz) {
                dp = (xv[u] * scale + dp) * vv[u];
                x[(k0 + u) * plane] = dp;
            }
    }
    double xn = 0.0;
    for (int64_t k1 = nz; k1 > 0; k1 -= B) {
        double xv[B], vv[B];
#pragma unroll
        for (int u = 0; u < B; ++u)
            if (k1 - 1 - u >= 0) { xv[u] = x[(k1 - 1 - u) * plane]; vv[u] = iv[(k1 - 1 - u) * plane]; }
#pragma unroll
        for (int u = 0; u < B; ++u)
            if (k1 - 1 - u >= 0) {
                xn = xv[u] + vv[u] * xn;
                x[(k1 - 1 - u) * plane] = xn;
            }
    }
}

// residual d - (6 phi - sum of neighbours), summed squares per block
__global__ void k_lap_resid(Box g, const double *__restrict__ phi, const double *__restrict__ d,
                            double *__restrict__ partials) {
    const int nx = (int)g.n[0], ny = (int)g.n[1], nz = (int)g.n[2], nxy = nx * ny, nc = nxy * nz;
    double acc = 0.0;
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < nc; c += gridDim.x * blockDim.x) {
        const int i = c % nx, j = (c / nx) % ny, k = c / nxy;
        double s = 6.0 * phi[c];
        if (k > 0) s -= phi[c - nxy];
        if (j > 0) s -= phi[c - nx];
        if (i > 0) s -= phi[c - 1];
        if (i < nx - 1) s -= phi[c + 1];
        if (j < ny - 1) s -= phi[c + nx];
        if (k < nz - 1) s -= phi[c + nxy];
        const double r = d[c] - s;
        acc += r * r;
    }
    __shared__ double red[256];
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) partials[blockIdx.x] = red[0];
}

// --------------------------------------------------------- f1: gauging --
// Comb tree (gauging.py:34-71): x-edges on the line (., 0, 0), y-edges in the
// plane (., ., 0) and every z-edge carry 0.  Each remaining edge is fixed by
// one face circulation, which unrolls into running sums:
//   a_x(i, j+1, 0) = -sum_{j'<=j} b_z(i, j', 0)
//   a_x(i, j, k+1) = a_x(i, j, 0) + sum_{k'<=k} b_y(i, j, k')
//   a_y(i, j, k+1) = -sum_{k'<=k} b_x(i, j, k')
// Each running sum is sequential in the scan index (numpy cumsum order).

// a_x on the k = 0 plane: one thread per i, scanning j
__global__ void k_gauge_ax0(int64_t nx, int64_t ny, const double *__restrict__ bz, double *__restrict__ ax) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nx) return;
    ax[i] = 0.0;
    double c = 0.0;
    for (int64_t j = 0; j < ny; ++j) {
        c = __dadd_rn(c, bz[i + nx * j]);
        ax[i + nx * (j + 1)] = -c;
    }
}

// column scans along k for A*B columns: dst(col, k+1) = base(col) + c_k
// (NEG: -c_k, base unused), c_k the running sum of src(col, 0..k).  U loads
// are issued ahead of the dependent adds.
template <bool NEG, int U>
__global__ void __launch_bounds__(128) k_gauge_kscan(int64_t ncol, int64_t nk, const double *__restrict__ src,
                                                     double *__restrict__ dst) {
    const int64_t col = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (col >= ncol) return;
    const double base = NEG ? 0.0 : dst[col];
    if (NEG) dst[col] = 0.0;
    double c = 0.0;
    int64_t k = 0;
    for (; k + U <= nk; k += U) {
        double v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = __ldcs(src + col + ncol * (k + u));
#pragma unroll
        for (int u = 0; u < U; ++u) {
            c = __dadd_rn(c, v[u]);
            __stcs(dst + col + ncol * (k + u + 1), NEG ? -c : __dadd_rn(base, c));
        }
    }
    for (; k < nk; ++k) {
        c = __dadd_rn(c, src[col + ncol * k]);
        dst[col + ncol * (k + 1)] = NEG ? -c : __dadd_rn(base, c);
    }
}

// BFS tree (gauging.py:74-119) on the full node box: all x-edges, the
// y-edges of the plane i = 0 and the z-edges of the line i = j = 0 carry 0
// (level-synchronous BFS from node 0 with the +x pass first reaches every
// node with i > 0 through its -x neighbour).  The remaining edges unroll
// into running sums along x (and along j on the plane i = 0):
//   a_y(i+1, j, k) = sum_{i'<=i} b_z(i', j, k)              (z-faces)
//   a_z(0, j+1, k) = sum_{j'<=j} b_x(0, j', k)              (x-faces, i = 0)
//   a_z(i+1, j, k) = a_z(0, j, k) - sum_{i'<=i} b_y(i', j, k) (y-faces)
// one thread per row, sequential in the scan index (numpy cumsum order).
template <bool BASE>
__global__ void k_gauge_xscan(int64_t nrows, int64_t nx, const double *__restrict__ src, double *__restrict__ dst) {
    const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (row >= nrows) return;
    const double *sr = src + row * nx;
    double *dr = dst + row * (nx + 1);
    const double base = BASE ? dr[0] : 0.0;
    if (!BASE) dr[0] = 0.0;
    double c = 0.0;
    for (int64_t i = 0; i < nx; ++i) {
        c = __dadd_rn(c, sr[i]);
        dr[i + 1] = BASE ? __dsub_rn(base, c) : c;
    }
}

// a_z on the plane i = 0: one thread per k, scanning j
__global__ void k_gauge_bfs_az0(int64_t nx, int64_t ny, int64_t nz, const double *__restrict__ bx,
                                double *__restrict__ az) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= nz) return;
    az[(nx + 1) * (ny + 1) * k] = 0.0;
    double c = 0.0;
    for (int64_t j = 0; j < ny; ++j) {
        c = __dadd_rn(c, bx[(nx + 1) * (j + ny * k)]);
        az[(nx + 1) * (j + 1 + (ny + 1) * k)] = c;
    }
}

__global__ void k_zero(int64_t n, double *p) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
        p[q] = 0.0;
}

// per-face circulation defect (gauging.py:127-134, right-handed boundary
// +e1(base) +e2(base+e1) -e1(base+e2) -e2(base), fit_operators.py:186-224)
__global__ void k_circulation(Box g, const double *__restrict__ a, const double *__restrict__ flux,
                              double *__restrict__ defect) {
    const int64_t nx = g.n[0], ny = g.n[1], nz = g.n[2];
    const int64_t F0 = (nx + 1) * ny * nz, F1 = nx * (ny + 1) * nz, F2 = nx * ny * (nz + 1);
    const int64_t E0 = nx * (ny + 1) * (nz + 1), E1 = (nx + 1) * ny * (nz + 1);
    const int64_t nf = F0 + F1 + F2;
    for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < nf; f += (int64_t)gridDim.x * blockDim.x) {
        int ax;
        int64_t q;
        if (f < F0) { ax = 0; q = f; }
        else if (f < F0 + F1) { ax = 1; q = f - F0; }
        else { ax = 2; q = f - F0 - F1; }
        int64_t fd[3] = {nx, ny, nz};
        fd[ax] += 1;
        int64_t c[3] = {q % fd[0], (q / fd[0]) % fd[1], q / (fd[0] * fd[1])};
        auto edge = [&](int e, int64_t i, int64_t j, int64_t k) -> double {
            int64_t ed[3] = {nx + 1, ny + 1, nz + 1};
            ed[e] -= 1;
            const int64_t off = e == 0 ? 0 : (e == 1 ? E0 : E0 + E1);
            return a[off + i + ed[0] * (j + ed[1] * k)];
        };
        const int e1 = (ax + 1) % 3, e2 = (ax + 2) % 3;
        int64_t s1[3] = {c[0], c[1], c[2]}, s2[3] = {c[0], c[1], c[2]};
        s1[e1] += 1;
        s2[e2] += 1;
        double circ = edge(e1, c[0], c[1], c[2]);
        circ += edge(e2, s1[0], s1[1], s1[2]);
        circ -= edge(e1, s2[0], s2[1], s2[2]);
        circ -= edge(e2, c[0], c[1], c[2]);
        defect[f] = circ - flux[f];
    }
}

// ------------------------------------------------- deterministic norms --
constexpr int kRedThreads = 256;
constexpr int kRedBlocks = 148 * 4;

__global__ void __launch_bounds__(kRedThreads) k_sumsq_partial(int64_t n, const double *__restrict__ x,
                                                               double *__restrict__ part) {
    __shared__ double red[32];
    double v[1] = {0.0};
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
        v[0] = fma(x[q], x[q], v[0]);
    block_sum<1>(v, red);
    if (threadIdx.x == 0) part[blockIdx.x] = v[0];
}

// Sum of squares of the circulation defect (k_circulation) without storing
// it: blocks walk face rows (axis, j, k) with threads along i, so the face
// index needs one division per row instead of 64-bit div/mod per face;
// per-block partials, summed on the host in block order.
// Sum of squared circulation defects over every face (gauging.py:167-171):
// one warp per face row, lanes along the row, 32-bit index math (a box axis
// holds < 2^31 edges; checked by the caller).
__global__ void __launch_bounds__(kRedThreads) k_circ_sumsq(Box g, const double *__restrict__ a,
                                                            const double *__restrict__ flux,
                                                            double *__restrict__ part) {
    __shared__ double red[32];
    const int nx = (int)g.n[0], ny = (int)g.n[1], nz = (int)g.n[2];
    const int64_t E0 = (int64_t)nx * (ny + 1) * (nz + 1), E1 = (int64_t)(nx + 1) * ny * (nz + 1);
    const int64_t eoff[3] = {0, E0, E0 + E1};
    const int lane = threadIdx.x & 31;
    const int warp = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), warps = gridDim.x * (blockDim.x >> 5);
    double v[1] = {0.0};
    int64_t fbase = 0;
    for (int ax = 0; ax < 3; ++ax) {
        int fd[3] = {nx, ny, nz};
        fd[ax] += 1;
        const int nrow = fd[1] * fd[2];
        const int e1 = (ax + 1) % 3, e2 = (ax + 2) % 3;
        int ed1[3] = {nx + 1, ny + 1, nz + 1}, ed2[3] = {nx + 1, ny + 1, nz + 1};
        ed1[e1] -= 1;
        ed2[e2] -= 1;
        // unit steps of the two edge arrays along e1 / e2 and along i
        const int st1[3] = {1, ed1[0], ed1[0] * ed1[1]}, st2[3] = {1, ed2[0], ed2[0] * ed2[1]};
        const double *A1 = a + eoff[e1], *A2 = a + eoff[e2];
        for (int row = warp; row < nrow; row += warps) {
            const int j = row % fd[1], k = row / fd[1];
            // edge e1 at c and c + e2, edge e2 at c and c + e1, for c = (0, j, k)
            const int b1 = ed1[0] * (j + ed1[1] * k), b2 = ed2[0] * (j + ed2[1] * k);
            const double *frow = flux + fbase + (int64_t)row * fd[0];
            for (int i = lane; i < fd[0]; i += 32) {
                const int q1 = b1 + i, q2 = b2 + i;
                double circ = A1[q1];
                circ += A2[q2 + st2[e1]];
                circ -= A1[q1 + st1[e2]];
                circ -= A2[q2];
                const double dd = circ - frow[i];
                v[0] = fma(dd, dd, v[0]);
            }
        }
        fbase += (int64_t)nrow * fd[0];
    }
    block_sum<1>(v, red);
    if (threadIdx.x == 0) part[blockIdx.x] = v[0];
}

// lowest index of the largest |x| (np.argmax(np.abs(x)))
__global__ void __launch_bounds__(kRedThreads) k_argmax_partial(int64_t n, const double *__restrict__ x,
                                                                double *__restrict__ pv, int64_t *__restrict__ pi) {
    __shared__ double sv[kRedThreads];
    __shared__ int64_t si[kRedThreads];
    double bv = -1.0;
    int64_t bi = -1;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
        const double a = fabs(x[q]);
        if (a > bv) { bv = a; bi = q; }
    }
    sv[threadIdx.x] = bv;
    si[threadIdx.x] = bi;
    __syncthreads();
    for (int o = kRedThreads / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            const double ov = sv[threadIdx.x + o];
            const int64_t oi = si[threadIdx.x + o];
            if (ov > sv[threadIdx.x] || (ov == sv[threadIdx.x] && oi >= 0 && (si[threadIdx.x] < 0 || oi < si[threadIdx.x]))) {
                sv[threadIdx.x] = ov;
                si[threadIdx.x] = oi;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) { pv[blockIdx.x] = sv[0]; pi[blockIdx.x] = si[0]; }
}

// --------------------------------------------------- f4: statistics --
__global__ void k_stats_prep(int64_t n, const double *__restrict__ values, double scale,
                             const int64_t *__restrict__ vox_index, const uint16_t *__restrict__ ids_box, int32_t n_ids,
                             double *__restrict__ scaled, int32_t *__restrict__ ids, int64_t *__restrict__ counts) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
        scaled[q] = __dmul_rn(values[q], scale);
        int32_t id = ids_box[vox_index[q]];
        ids[q] = id;
        if (id >= n_ids) id = n_ids;   // overflow slot: reported as an error
        atomicAdd(reinterpret_cast<unsigned long long *>(counts + id), 1ull);
    }
}

// per-id nearest-rank p99 (index ceil(0.99 c) - 1) and max of the
// value-sorted segments; row n_ids holds the global statistics
__global__ void k_stats_pick(int32_t n_ids, const int64_t *__restrict__ off, const int64_t *__restrict__ cnt,
                             const double *__restrict__ seg_vals, const double *__restrict__ sorted_vals, int64_t n,
                             double *__restrict__ p99, double *__restrict__ mx) {
    const int32_t id = blockIdx.x * blockDim.x + threadIdx.x;
    if (id > n_ids) return;
    const int64_t c = id < n_ids ? cnt[id] : n;
    const double *v = id < n_ids ? seg_vals + off[id] : sorted_vals;
    if (c == 0) { p99[id] = 0.0; mx[id] = 0.0; return; }
    const int64_t rank = (99 * c + 99) / 100;   // ceil(0.99 c) = -((-99 c) // 100)
    p99[id] = v[rank - 1];
    mx[id] = v[c - 1];
}

}  // namespace

// ======================================================================= host

struct Field {
    Box g;
    spfd_config cfg;
    DevBuf<double> part;      // reduction partials
    DevBuf<int64_t> parti;
    DevBuf<double> wc, wf;    // cell / face workspaces
    DevBuf<AxisParam> wt;     // per-axis trilinear parameters (field_interpolate)
    Amg *clean_amg = nullptr; // AMG on div divᵀ (built on first use; SPFD_CLEAN_SOLVER=amg)
    double clean_setup_seconds = 0.0;
    DevBuf<double> sx, sy, lx, ly;  // spectral projection: DST-I matrices and 1-D eigenvalues
    DevBuf<double> spec_ws;         // [2][nc] transform ping-pong
    DevBuf<double> spec_inv;        // [nc] eliminated pivots of the z systems (per mode, k)
    ~Field() { delete clean_amg; }
    int64_t n_cells() const { return g.n[0] * g.n[1] * g.n[2]; }
    int64_t n_faces() const { return face_count(g, 0) + face_count(g, 1) + face_count(g, 2); }
    int64_t n_edges() const { return edge_count(g, 0) + edge_count(g, 1) + edge_count(g, 2); }
};

namespace {

double sumsq(Field &F, const double *x, int64_t n, cudaStream_t s) {
    if (n == 0) return 0.0;
    k_sumsq_partial<<<kRedBlocks, kRedThreads, 0, s>>>(n, x, F.part.get());
    SPFD_LAUNCH_CHECK();
    std::vector<double> h(kRedBlocks);
    SPFD_CUDA(cudaMemcpyAsync(h.data(), F.part.get(), kRedBlocks * sizeof(double), cudaMemcpyDeviceToHost, s));
    SPFD_CUDA(cudaStreamSynchronize(s));
    double t = 0.0;
    for (double v : h) t += v;  // fixed order
    return t;
}

int64_t argmax_abs(Field &F, const double *x, int64_t n, double *h_val, cudaStream_t s) {
    k_argmax_partial<<<kRedBlocks, kRedThreads, 0, s>>>(n, x, F.part.get(), F.parti.get());
    SPFD_LAUNCH_CHECK();
    std::vector<double> v(kRedBlocks);
    std::vector<int64_t> ix(kRedBlocks);
    SPFD_CUDA(cudaMemcpyAsync(v.data(), F.part.get(), kRedBlocks * sizeof(double), cudaMemcpyDeviceToHost, s));
    SPFD_CUDA(cudaMemcpyAsync(ix.data(), F.parti.get(), kRedBlocks * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    SPFD_CUDA(cudaStreamSynchronize(s));
    double bv = -1.0;
    int64_t bi = -1;
    for (int b = 0; b < kRedBlocks; ++b)
        if (ix[b] >= 0 && (v[b] > bv || (v[b] == bv && ix[b] < bi))) { bv = v[b]; bi = ix[b]; }
    if (bi >= 0 && h_val) SPFD_CUDA(cudaMemcpy(h_val, x + bi, sizeof(double), cudaMemcpyDeviceToHost));
    return bi;
}

inline int blocks(int64_t n, int t = 256) { return grid_for(n, t, 148 * 32); }

}  // namespace

Field *field_create(const spfd_box &grid, const spfd_config &cfg) {
    auto *F = new Field();
    F->g = box_of(grid);
    F->cfg = cfg;
    F->part.alloc(kRedBlocks);
    F->parti.alloc(kRedBlocks);
    return F;
}

void field_destroy(Field *F) { delete F; }

void field_check_lattice(const Field &F, const spfd_box &lat) {
    const Box L = box_of(lat);
    for (int a = 0; a < 3; ++a) {
        SPFD_CHECK(L.n[a] >= 1, SPFD_EINVAL, "lattice dims must be >= 1");
        SPFD_CHECK(L.h[a] > 0.0, SPFD_EINVAL, "lattice spacing must be positive");
    }
    // a single-point lattice axis supports only queries on that plane
    for (int d = 0; d < 3; ++d) {
        if (L.n[d] != 1) continue;
        for (int a = 0; a < 3; ++a) {
            const int64_t m = F.g.n[d] + (d == a ? 1 : 0);
            for (int64_t i = 0; i < m; ++i)
                SPFD_CHECK(std::fabs(face_coord(F.g, a, d, i) - L.o[d]) <= 1e-9, SPFD_ELATTICE,
                           "lattice has a single point along an axis that requires interpolation");
        }
    }
}

void field_interpolate(Field &F, const spfd_box &lat, const double *b, double *flux, cudaStream_t s) {
    field_check_lattice(F, lat);
    const Box L = box_of(lat);
    int64_t off = 0;
    for (int a = 0; a < 3; ++a) {
        const int t0 = a == 0 ? 1 : 0, t1 = a == 2 ? 1 : 2;
        const double area = F.g.h[t0] * F.g.h[t1];
        const int64_t nf = face_count(F.g, a);
        if (nf) {
            int64_t d[3] = {F.g.n[0], F.g.n[1], F.g.n[2]};
            d[a] += 1;
            const int64_t nt = d[0] + d[1] + d[2];
            if (F.wt.n < (size_t)nt) F.wt.alloc(nt);
            k_axis_params<<<blocks(nt), 256, 0, s>>>(F.g, L, a, F.wt.get());
            const int grid = (int)std::min<int64_t>((d[1] * d[2] + 7) / 8, 148 * 16);  // 8 warps = 8 rows
            k_interp_rows<<<grid, 256, 0, s>>>(F.g, L, a, F.wt.get(), b, area, flux + off);
            SPFD_LAUNCH_CHECK();
        }
        off += nf;
    }
}

void coil_field(int64_t n, const double *pts, int nseg, const double *verts, double scale, double *out,
                cudaStream_t s) {
    DevBuf<int> flag;
    flag.alloc(1);
    SPFD_CUDA(cudaMemsetAsync(flag.get(), 0, sizeof(int), s));
    if (n) {
        k_coil_field<<<blocks(n, 128), 128, 0, s>>>(n, pts, nseg, verts, scale, 1e-24, out, flag.get());
        SPFD_LAUNCH_CHECK();
    }
    int h = 0;
    SPFD_CUDA(cudaMemcpyAsync(&h, flag.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
    SPFD_CUDA(cudaStreamSynchronize(s));
    SPFD_CHECK(!h, SPFD_ESINGULAR, "evaluation point lies on the coil wire");
}

void field_divergence(Field &F, const double *flux, double *div, cudaStream_t s) {
    const int64_t nc = F.n_cells();
    if (!nc) return;
    k_divergence<<<blocks(nc), 256, 0, s>>>(F.g, flux, div);
    SPFD_LAUNCH_CHECK();
}

static void ensure_clean_amg(Field &F, cudaStream_t s) {
    if (F.clean_amg) return;
    const int64_t nc = F.n_cells();
    DevBuf<int64_t> ptr;
    ptr.alloc(nc + 1);
    k_normal_count<<<blocks(nc), 256, 0, s>>>(F.g, ptr.get() + 1);
    SPFD_LAUNCH_CHECK();
    SPFD_CUDA(cudaMemsetAsync(ptr.get(), 0, sizeof(int64_t), s));
    size_t tb = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tb, ptr.get() + 1, ptr.get() + 1, nc, s);
    DevBuf<unsigned char> tmp;
    tmp.alloc(tb);
    cub::DeviceScan::InclusiveSum(tmp.get(), tb, ptr.get() + 1, ptr.get() + 1, nc, s);
    SPFD_LAUNCH_CHECK();
    int64_t nnz = 0;
    SPFD_CUDA(cudaMemcpyAsync(&nnz, ptr.get() + nc, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    SPFD_CUDA(cudaStreamSynchronize(s));
    DevBuf<int32_t> col;
    DevBuf<double> val;
    col.alloc(nnz);
    val.alloc(nnz);
    k_normal_fill<<<blocks(nc), 256, 0, s>>>(F.g, ptr.get(), col.get(), val.get());
    SPFD_LAUNCH_CHECK();
    spfd_config c = F.cfg;
    c.max_nrhs = 2;   // re/im sample sets batched (field_clean)
    F.clean_amg = amg_setup_csr(nc, nnz, ptr.get(), col.get(), val.get(), c, s);
    F.clean_setup_seconds = F.clean_amg->setup_seconds;
    // level 0 is the constant-coefficient cell Laplacian: matrix-free
    // (SPFD_CLEAN_BOX=0 keeps the CSR path for A/B)
    const bool box = !(getenv("SPFD_CLEAN_BOX") && std::string(getenv("SPFD_CLEAN_BOX")) == "0");
    if (box) amg_set_box_level0(*F.clean_amg, F.g.n, s);
    pool_trim();
}

// cleaning solver: spectral (default) or the AMG hierarchy (SPFD_CLEAN_SOLVER=amg,
// the reference's method, kept for A/B and the hierarchy parity tests)
static bool clean_spectral() {
    const char *e = getenv("SPFD_CLEAN_SOLVER");
    return !(e && std::string(e) == "amg");
}

static void ensure_spectral(Field &F, cudaStream_t s) {
    if (F.sx.n) return;
    const int64_t nx = F.g.n[0], ny = F.g.n[1];
    auto build = [&](int64_t n, DevBuf<double> &S, DevBuf<double> &L) {
        std::vector<double> hs((size_t)(n * n)), hl((size_t)n);
        const int64_t period = 2 * (n + 1);
        for (int64_t a = 0; a < n; ++a) {
            hl[a] = 2.0 - 2.0 * std::cos(M_PI * (double)(a + 1) / (double)(n + 1));
            for (int64_t b = 0; b < n; ++b) {
                const int64_t t = ((a + 1) * (b + 1)) % period;  // exact argument reduction
                hs[a * n + b] = std::sin(M_PI * (double)t / (double)(n + 1));
            }
        }
        S.alloc(n * n);
        L.alloc(n);
        SPFD_CUDA(cudaMemcpyAsync(S.get(), hs.data(), hs.size() * sizeof(double), cudaMemcpyHostToDevice, s));
        SPFD_CUDA(cudaMemcpyAsync(L.get(), hl.data(), hl.size() * sizeof(double), cudaMemcpyHostToDevice, s));
        SPFD_CUDA(cudaStreamSynchronize(s));
    };
    build(nx, F.sx, F.lx);
    build(ny, F.sy, F.ly);
    F.spec_ws.alloc(2 * F.n_cells());
    F.spec_inv.alloc(F.n_cells());
    const int64_t plane = nx * ny;
    k_tridiag_pivots<<<(unsigned)((plane + 127) / 128), 128, 0, s>>>(nx, ny, F.g.n[2], F.lx.get(), F.ly.get(),
                                                                    F.spec_inv.get());
    SPFD_LAUNCH_CHECK();
}

// The same product on the FP64 tensor cores (mma.sync m8n8k4 f64): a CTA
// tile of 32 x 256, each of the 8 warps 32 x 32 as 4 x 4 m8n8k4 blocks.  The
// k order inside an MMA is the hardware's, so the bits can differ from the
// FFMA chain in the last place (the spectral solve is tolerance-checked).
__device__ __forceinline__ void dmma_m8n8k4(double &d0, double &d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(double *dst, const double *src, bool valid) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    const int n = valid ? 8 : 0;  // zero-fill outside the operand
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(valid ? src : dst), "r"(n) : "memory");
}

// kDmmaStages-deep cp.async pipeline of BK = 8 slices (dynamic shared memory)
constexpr int kDmmaStages = 4, kDmmaBM = 32, kDmmaBN = 256, kDmmaPA = kDmmaBM + 4, kDmmaPB = kDmmaBN + 4;
constexpr size_t kDmmaSmem = (size_t)kDmmaStages * kGBK * (kDmmaPA + kDmmaPB) * sizeof(double) + kDmmaBN * sizeof(int64_t);

__global__ void __launch_bounds__(256) k_dgemm_mma(GemmArgs g) {
    constexpr int BM = kDmmaBM, BN = kDmmaBN, PA = kDmmaPA, PB = kDmmaPB, ST = kDmmaStages;
    constexpr int NB = kGBK * BN / 256, NA = (kGBK * BM + 255) / 256;
    extern __shared__ __align__(16) double dsm[];
    double *As = dsm;                              // [ST][BK][PA]
    double *Bs = dsm + ST * kGBK * PA;             // [ST][BK][PB]
    int64_t *boff = reinterpret_cast<int64_t *>(Bs + ST * kGBK * PB);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t m0 = (int64_t)blockIdx.x * BM, n0 = (int64_t)blockIdx.y * BN;
    for (int q = tid; q < BN; q += 256) {
        const int64_t n = n0 + q;
        boff[q] = n < g.N ? (n % g.nlo) * g.sBlo + (n / g.nlo) * g.sBhi : -1;
    }
    __syncthreads();
    const bool nfast = g.sBlo < g.sBk;
    const int nk = (int)((g.K + kGBK - 1) / kGBK);
    auto issue = [&](int kt) {
        if (kt < nk) {
            const int st = kt % ST;
            const int64_t k0 = (int64_t)kt * kGBK;
#pragma unroll
            for (int t = 0; t < NA; ++t) {
                const int e = tid + t * 256;
                if (e < kGBK * BM) {
                    const int mm = e % BM, kk = e / BM;
                    const int64_t m = m0 + mm, k = k0 + kk;
                    const bool ok = m < g.M && k < g.K;
                    cp_async8(&As[(st * kGBK + kk) * PA + mm], ok ? g.A + m * g.sAm + k * g.sAk : nullptr, ok);
                }
            }
#pragma unroll
            for (int t = 0; t < NB; ++t) {
                const int e = tid + t * 256;
                const int nn = nfast ? e % BN : e / kGBK, kk = nfast ? e / BN : e % kGBK;
                const int64_t o = boff[nn], k = k0 + kk;
                const bool ok = o >= 0 && k < g.K;
                cp_async8(&Bs[(st * kGBK + kk) * PB + nn], ok ? g.B + k * g.sBk + o : nullptr, ok);
            }
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    const int fr = lane & 3, fc = lane >> 2;  // fragment row (k) / column (m or n)
#pragma unroll
    for (int s0 = 0; s0 < ST - 1; ++s0) issue(s0);
    for (int kt = 0; kt < nk; ++kt) {
        asm volatile("cp.async.wait_group %0;\n" ::"n"(ST - 2) : "memory");
        __syncthreads();
        issue(kt + ST - 1);  // refills the stage computed in iteration kt - 1
        const double *A = As + (kt % ST) * kGBK * PA, *B = Bs + (kt % ST) * kGBK * PB;
#pragma unroll
        for (int kq = 0; kq < kGBK; kq += 4) {
            double a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = A[(kq + fr) * PA + i * 8 + fc];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = B[(kq + fr) * PB + warp * 32 + j * 8 + fc];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma_m8n8k4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
        }
    }
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int64_t n = n0 + warp * 32 + j * 8 + fr * 2 + h;
            if (n >= g.N) continue;
            const int64_t co = (n % g.nlo) * g.sClo + (n / g.nlo) * g.sChi;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int64_t m = m0 + i * 8 + fc;
                if (m < g.M) g.C[m * g.sCm + co] = acc[i][j][h];
            }
        }
}

static void gemm(const GemmArgs &g, cudaStream_t s) {
    constexpr int BM = 32;
    const bool mma = !(getenv("SPFD_DGEMM_MMA") && std::string(getenv("SPFD_DGEMM_MMA")) == "0");  // read per call
    const int BN = mma ? 256 : 8 * (256 / (BM / 8));
    SPFD_CHECK((g.N + BN - 1) / BN <= 65535, SPFD_EINVAL, "grid too large for the spectral solve");
    const dim3 grid((unsigned)((g.M + BM - 1) / BM), (unsigned)((g.N + BN - 1) / BN));
    if (mma) {
        static bool attr = false;
        if (!attr) {
            SPFD_CUDA(cudaFuncSetAttribute(k_dgemm_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDmmaSmem));
            attr = true;
        }
        k_dgemm_mma<<<grid, 256, kDmmaSmem, s>>>(g);
    }
    else k_dgemm_split<BM><<<grid, 256, 0, s>>>(g);
    SPFD_LAUNCH_CHECK();
}

// phi = (div divT)^-1 d for na planar right-hand sides [na][nc] (d kept)
static void spectral_solve(Field &F, int na, const double *d, double *phi, cudaStream_t s) {
    ensure_spectral(F, s);
    const int64_t nx = F.g.n[0], ny = F.g.n[1], nz = F.g.n[2], plane = nx * ny, nc = plane * nz;
    double *buf = F.spec_ws.get();
    const double *Sx = F.sx.get(), *Sy = F.sy.get();
    // along x: out(p, col) = sum_i Sx(p, i) in(i, col), col = (j, k)
    auto along_x = [&](const double *in, double *out) {
        // A = Sx (p, i); B(i, n) = in[i + nx col + nc rhs], n = col + ny nz rhs
        gemm(GemmArgs{Sx, in, out, nx, ny * nz * na, nx, nx, 1, 1, ny * nz, nx, nc, 1, nx, nc}, s);
    };
    // along y: out(i, q, kz) = sum_j Sy(q, j) in(i, j, kz) as one product,
    // A = Sy (q, j); B(j, n) = in[i + nx j + plane kz'], n = i + nx kz' (kz' runs over nz na planes)
    auto along_y = [&](const double *in, double *out) {
        gemm(GemmArgs{Sy, in, out, ny, nx * nz * na, ny, ny, 1, nx, nx, 1, plane, nx, 1, plane}, s);
    };
    along_x(d, buf);
    along_y(buf, phi);
    k_tridiag_apply<<<(unsigned)((plane * na + 127) / 128), 128, 0, s>>>(
        nx, ny, nz, na, F.spec_inv.get(), 4.0 / ((double)(nx + 1) * (double)(ny + 1)), phi);
    SPFD_LAUNCH_CHECK();
    along_y(phi, buf);
    along_x(buf, phi);
}

static double lap_resid_sq(Field &F, const double *phi, const double *d, cudaStream_t s) {
    k_lap_resid<<<kRedBlocks, 256, 0, s>>>(F.g, phi, d, F.part.get());
    SPFD_LAUNCH_CHECK();
    std::vector<double> h(kRedBlocks);
    SPFD_CUDA(cudaMemcpyAsync(h.data(), F.part.get(), kRedBlocks * sizeof(double), cudaMemcpyDeviceToHost, s));
    SPFD_CUDA(cudaStreamSynchronize(s));
    double t = 0.0;
    for (double v : h) t += v;
    return t;
}

// Batched projection of nrhs (1 or 2, e.g. the real and imaginary sample
// sets of a snapshot) face-flux vectors, planar [nrhs][n_faces]: the
// per-vector decisions of field_source.py:292-329 (skip when already
// solenoidal, tolerance min(1e-12, 0.25 tol / rel)), one Krylov solve for
// the vectors that need it (the stricter tolerance of the two; each then
// meets its own), and the same post-check per vector.
void field_clean(Field &F, int nrhs, const double *in, double *out, double tol, spfd_clean_info *info,
                 cudaStream_t s) {
    SPFD_CHECK(nrhs == 1 || nrhs == 2, SPFD_EINVAL, "nrhs must be 1 or 2");
    const int64_t nc = F.n_cells(), nf = F.n_faces();
    SPFD_CHECK(nf < (int64_t)1 << 30, SPFD_EINVAL, "grid too large for 32-bit face indexing");
    if (F.wc.n < (size_t)(4 * nc)) F.wc.alloc(4 * nc);  // [2][nc] divergences + [nc][2] interleaved
    double *divp = F.wc.get(), *inter = F.wc.get() + 2 * nc;
    double fnorm[2] = {0.0, 0.0};
    int act[2], na = 0;
    double rtol = 1e-12;
    for (int c = 0; c < nrhs; ++c) {
        info[c] = spfd_clean_info{};
        const double *ic = in + (int64_t)c * nf;
        double *oc = out + (int64_t)c * nf;
        // a skipped rhs is passed through; a cleaned one is written by
        // k_sub_div_transpose from `in`, so it needs no copy
        auto pass = [&] {
            if (oc != ic) SPFD_CUDA(cudaMemcpyAsync(oc, ic, nf * sizeof(double), cudaMemcpyDeviceToDevice, s));
        };
        fnorm[c] = std::sqrt(sumsq(F, ic, nf, s));
        if (fnorm[c] == 0.0 || nc == 0) { pass(); continue; }
        field_divergence(F, ic, divp + (int64_t)na * nc, s);
        const double rel = std::sqrt(sumsq(F, divp + (int64_t)na * nc, nc, s)) / fnorm[c];
        info[c].rel_before = rel;
        info[c].rel_after = rel;
        if (rel <= tol) { pass(); continue; }
        rtol = std::min(rtol, std::min(1e-12, 0.25 * tol / rel));
        act[na++] = c;
    }
    if (na == 0) return;
    if (clean_spectral()) {
        // direct solve (rounding-level residual, reported), then the same
        // correction and post-check as the Krylov path
        double *phi = inter;  // [na][nc]
        spectral_solve(F, na, divp, phi, s);
        for (int k = 0; k < na; ++k) {
            const int c = act[k];
            spfd_clean_info &ic = info[c];
            ic.solved = 1;
            ic.iterations = 0;
            const double dn = ic.rel_before * fnorm[c];
            ic.solve_rel_residual = std::sqrt(lap_resid_sq(F, phi + (int64_t)k * nc, divp + (int64_t)k * nc, s)) / dn;
            // a direct solve: its residual is the rounding floor, reported (the
            // projection's acceptance is the post-check below)
            SPFD_CHECK(std::isfinite(ic.solve_rel_residual), SPFD_ENONFINITE, "non-finite value in the projection solve");
            k_sub_div_transpose<<<blocks(nf), 256, 0, s>>>(F.g, phi + (int64_t)k * nc, in + (int64_t)c * nf,
                                                           out + (int64_t)c * nf);
            SPFD_LAUNCH_CHECK();
        }
        for (int k = 0; k < na; ++k) {
            const int c = act[k];
            double *div = divp;  // scratch (the divergences are no longer needed)
            field_divergence(F, out + (int64_t)c * nf, div, s);
            info[c].rel_after = std::sqrt(sumsq(F, div, nc, s)) / fnorm[c];
            if (info[c].rel_after > tol) {
                char msg[160];
                snprintf(msg, sizeof msg, "divergence cleaning left relative defect %.3e > %.3e", info[c].rel_after, tol);
                throw Error(SPFD_EPROJECTION, msg);
            }
        }
        return;
    }
    ensure_clean_amg(F, s);
    spfd_config cfg = F.cfg;
    cfg.rel_tol = rtol;
    cfg.max_nrhs = 2;
    Amg &h = *F.clean_amg;
    amg_to_level0(h, divp, inter, na, s);
    spfd_report rep = krylov_solve(h, inter, h.kx.get(), na, cfg, nullptr, s);
    SPFD_CUDA(cudaStreamSynchronize(s));
    SPFD_CHECK(rep.status != SPFD_ENONFINITE, SPFD_ENONFINITE, "non-finite value in the projection solve");
    amg_from_level0(h, h.kx.get(), divp, na, s);   // potentials, planar [na][nc]
    for (int k = 0; k < na; ++k) {
        const int c = act[k];
        spfd_clean_info &ic = info[c];
        ic.solved = 1;
        ic.iterations = rep.iterations;
        ic.solve_rel_residual = rep.rel_residual[k];
        ic.setup_seconds = F.clean_setup_seconds;
        if (!rep.converged) {
            char msg[160];
            snprintf(msg, sizeof msg, "divergence projection did not converge (residual %.3e)", rep.rel_residual[k]);
            throw Error(SPFD_EPROJECTION, msg);
        }
        k_sub_div_transpose<<<blocks(nf), 256, 0, s>>>(F.g, divp + (int64_t)k * nc, in + (int64_t)c * nf,
                                                       out + (int64_t)c * nf);
        SPFD_LAUNCH_CHECK();
    }
    for (int k = 0; k < na; ++k) {
        const int c = act[k];
        double *div = inter;  // scratch
        field_divergence(F, out + (int64_t)c * nf, div, s);
        info[c].rel_after = std::sqrt(sumsq(F, div, nc, s)) / fnorm[c];
        if (info[c].rel_after > tol) {
            char msg[160];
            snprintf(msg, sizeof msg, "divergence cleaning left relative defect %.3e > %.3e", info[c].rel_after, tol);
            throw Error(SPFD_EPROJECTION, msg);
        }
    }
}

void field_circulation(Field &F, const double *a, const double *flux, double *defect, cudaStream_t s) {
    const int64_t nf = F.n_faces();
    if (!nf) return;
    k_circulation<<<blocks(nf), 256, 0, s>>>(F.g, a, flux, defect);
    SPFD_LAUNCH_CHECK();
}

void field_gauge(Field &F, int tree, const double *flux, double *a, double tol, spfd_gauge_info *info, cudaStream_t s) {
    const int64_t nx = F.g.n[0], ny = F.g.n[1], nz = F.g.n[2];
    const int64_t F0 = face_count(F.g, 0), F1 = face_count(F.g, 1);
    const int64_t E0 = edge_count(F.g, 0), E1 = edge_count(F.g, 1), E2 = edge_count(F.g, 2);
    const int64_t nf = F.n_faces();
    *info = spfd_gauge_info{};
    info->worst_face = -1;
    double *ax = a, *ay = a + E0, *az = a + E0 + E1;
    const double fnorm = std::sqrt(sumsq(F, flux, nf, s));
    if (fnorm == 0.0) {
        k_zero<<<blocks(E0 + E1 + E2), 256, 0, s>>>(E0 + E1 + E2, a);
        SPFD_LAUNCH_CHECK();
        return;
    }
    const double *bx = flux, *by = flux + F0, *bz = flux + F0 + F1;
    if (tree == 1) {  // BFS tree: x-scans
        k_zero<<<blocks(E0), 256, 0, s>>>(E0, ax);
        SPFD_LAUNCH_CHECK();
        if (ny > 0) {
            const int64_t nrow = ny * (nz + 1);
            k_gauge_xscan<false><<<(int)((nrow + 127) / 128), 128, 0, s>>>(nrow, nx, bz, ay);
            SPFD_LAUNCH_CHECK();
        }
        if (nz > 0) {
            k_gauge_bfs_az0<<<(int)((nz + 127) / 128), 128, 0, s>>>(nx, ny, nz, bx, az);
            SPFD_LAUNCH_CHECK();
            const int64_t nrow = (ny + 1) * nz;
            k_gauge_xscan<true><<<(int)((nrow + 127) / 128), 128, 0, s>>>(nrow, nx, by, az);
            SPFD_LAUNCH_CHECK();
        }
    } else {
        // a_x: k = 0 plane, then the k scans (nx * (ny+1) columns)
        if (nx > 0) {
            k_gauge_ax0<<<(int)((nx + 127) / 128), 128, 0, s>>>(nx, ny, bz, ax);
            SPFD_LAUNCH_CHECK();
            const int64_t ncol = nx * (ny + 1);
            k_gauge_kscan<false, 16><<<(int)((ncol + 127) / 128), 128, 0, s>>>(ncol, nz, by, ax);
            SPFD_LAUNCH_CHECK();
        }
        if (ny > 0) {
            const int64_t ncol = (nx + 1) * ny;
            k_gauge_kscan<true, 16><<<(int)((ncol + 127) / 128), 128, 0, s>>>(ncol, nz, bx, ay);
            SPFD_LAUNCH_CHECK();
        }
        if (E2) {
            k_zero<<<blocks(E2), 256, 0, s>>>(E2, az);
            SPFD_LAUNCH_CHECK();
        }
    }
    // postcondition: circulation residual over every face (gauging.py:167-171);
    // the defect array is only materialised to locate the worst face
    SPFD_CHECK((F.g.n[0] + 1) * (F.g.n[1] + 1) * (F.g.n[2] + 1) < (int64_t)INT32_MAX, SPFD_EINVAL,
               "grid too large for 32-bit face indexing");
    k_circ_sumsq<<<kRedBlocks, kRedThreads, 0, s>>>(F.g, a, flux, F.part.get());
    SPFD_LAUNCH_CHECK();
    {
        std::vector<double> h(kRedBlocks);
        SPFD_CUDA(cudaMemcpyAsync(h.data(), F.part.get(), kRedBlocks * sizeof(double), cudaMemcpyDeviceToHost, s));
        SPFD_CUDA(cudaStreamSynchronize(s));
        double t = 0.0;
        for (double v : h) t += v;  // fixed order
        info->rel_residual = std::sqrt(t) / fnorm;
    }
    if (info->rel_residual > tol) {
        if (F.wf.n < (size_t)nf) F.wf.alloc(nf);
        field_circulation(F, a, flux, F.wf.get(), s);
        info->worst_face = argmax_abs(F, F.wf.get(), nf, &info->worst_defect, s);
        char msg[200];
        snprintf(msg, sizeof msg, "incompatible fluxes: relative circulation residual %.3e (worst face %lld, defect %.3e)",
                 info->rel_residual, (long long)info->worst_face, info->worst_defect);
        throw Error(SPFD_EINCOMPAT, msg);
    }
}

void exposure_stats(const double *values, int64_t n, double scale, const int64_t *vox_index, const uint16_t *ids_box,
                    int32_t n_ids, double *scaled, int64_t *h_count, double *h_mean, double *h_max, double *h_p99,
                    double *h_global, cudaStream_t s) {
    SPFD_CHECK(n >= 1, SPFD_EINVAL, "percentile of an empty array");
    SPFD_CHECK(n_ids >= 1 && n_ids <= 65536, SPFD_EINVAL, "n_ids must be in [1, 65536]");
    DevBuf<int32_t> ids, ids_sorted, seg_ids;
    DevBuf<double> sorted, seg_vals, sums, p99, mx;
    DevBuf<int64_t> cnt, off;
    ids.alloc(n); ids_sorted.alloc(n); seg_ids.alloc(n);
    sorted.alloc(n); seg_vals.alloc(n);
    cnt.alloc(n_ids + 1); off.alloc(n_ids + 1);
    sums.alloc(n_ids); p99.alloc(n_ids + 1); mx.alloc(n_ids + 1);
    SPFD_CUDA(cudaMemsetAsync(cnt.get(), 0, (n_ids + 1) * sizeof(int64_t), s));
    k_stats_prep<<<blocks(n), 256, 0, s>>>(n, values, scale, vox_index, ids_box, n_ids, scaled, ids.get(), cnt.get());
    SPFD_LAUNCH_CHECK();
    int end_bit = 1;
    while ((1 << end_bit) < n_ids) ++end_bit;
    size_t t1 = 0, t2 = 0, t3 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, t1, scaled, sorted.get(), ids.get(), ids_sorted.get(), n, 0, 64, s);
    cub::DeviceRadixSort::SortPairs(nullptr, t2, ids_sorted.get(), seg_ids.get(), sorted.get(), seg_vals.get(), n, 0,
                                    end_bit, s);
    cub::DeviceSegmentedReduce::Sum(nullptr, t3, seg_vals.get(), sums.get(), n_ids, off.get(), off.get() + 1, s);
    DevBuf<unsigned char> tmp;
    tmp.alloc(std::max(t1, std::max(t2, t3)));
    size_t tb = tmp.bytes();
    // 1) by value (global p99 / max); 2) stable by tissue id -> per-id value-sorted segments
    SPFD_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), tb, scaled, sorted.get(), ids.get(), ids_sorted.get(), n, 0,
                                              64, s));
    tb = tmp.bytes();
    SPFD_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), tb, ids_sorted.get(), seg_ids.get(), sorted.get(),
                                              seg_vals.get(), n, 0, end_bit, s));
    count_launch();
    std::vector<int64_t> hc(n_ids + 1), ho(n_ids + 1, 0);
    SPFD_CUDA(cudaMemcpyAsync(hc.data(), cnt.get(), (n_ids + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    SPFD_CUDA(cudaStreamSynchronize(s));
    SPFD_CHECK(hc[n_ids] == 0, SPFD_EINVAL, "tissue id >= n_ids");
    for (int32_t i = 0; i < n_ids; ++i) ho[i + 1] = ho[i] + hc[i];
    SPFD_CUDA(cudaMemcpyAsync(off.get(), ho.data(), (n_ids + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    tb = tmp.bytes();
    SPFD_CUDA(cub::DeviceSegmentedReduce::Sum(tmp.get(), tb, seg_vals.get(), sums.get(), n_ids, off.get(),
                                              off.get() + 1, s));
    k_stats_pick<<<(n_ids + 1 + 127) / 128, 128, 0, s>>>(n_ids, off.get(), cnt.get(), seg_vals.get(), sorted.get(), n,
                                                         p99.get(), mx.get());
    SPFD_LAUNCH_CHECK();
    std::vector<double> hs(n_ids), hp(n_ids + 1), hm(n_ids + 1);
    SPFD_CUDA(cudaMemcpyAsync(hs.data(), sums.get(), n_ids * sizeof(double), cudaMemcpyDeviceToHost, s));
    SPFD_CUDA(cudaMemcpyAsync(hp.data(), p99.get(), (n_ids + 1) * sizeof(double), cudaMemcpyDeviceToHost, s));
    SPFD_CUDA(cudaMemcpyAsync(hm.data(), mx.get(), (n_ids + 1) * sizeof(double), cudaMemcpyDeviceToHost, s));
    SPFD_CUDA(cudaStreamSynchronize(s));
    for (int32_t i = 0; i < n_ids; ++i) {
        h_count[i] = hc[i];
        h_mean[i] = hc[i] ? hs[i] / (double)hc[i] : 0.0;
        h_max[i] = hm[i];
        h_p99[i] = hp[i];
    }
    h_global[0] = hp[n_ids];
    h_global[1] = hm[n_ids];
}

}  // namespace spfd

// Field sources, divergence cleaning, comb-tree gauging and exposure
// statistics; implementation in field.cu.
#pragma once
#include "common.cuh"

namespace spfd {

struct Field;  // per-grid workspace (+ the cleaning hierarchy)

Field *field_create(const spfd_box &grid, const spfd_config &cfg);
void field_destroy(Field *F);
void field_interpolate(Field &F, const spfd_box &lattice, const double *b, double *flux, cudaStream_t s);
void field_divergence(Field &F, const double *flux, double *div, cudaStream_t s);
void field_clean(Field &F, int nrhs, const double *in, double *out, double tol, spfd_clean_info *info,
                 cudaStream_t s);
// tree: 0 = comb (gauging.py:34-71), 1 = BFS (gauging.py:74-119)
void field_gauge(Field &F, int tree, const double *flux, double *a, double tol, spfd_gauge_info *info, cudaStream_t s);
void field_circulation(Field &F, const double *a, const double *flux, double *defect, cudaStream_t s);
void coil_field(int64_t n, const double *pts, int nseg, const double *verts, double scale, double *out,
                cudaStream_t s);
void exposure_stats(const double *values, int64_t n, double scale, const int64_t *vox_index, const uint16_t *ids_box,
                    int32_t n_ids, double *scaled, int64_t *h_count, double *h_mean, double *h_max, double *h_p99,
                    double *h_global, cudaStream_t s);

}  // namespace spfd

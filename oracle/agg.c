/*
 * CPU oracle (TEST INFRASTRUCTURE ONLY — never linked into the product).
 *
 * Restatement of the reference's greedy root-node aggregation
 * (/root/reference/pkg/src/spfd/_kernels.py:79-120, `plain_aggregation`).
 * The reference JIT-compiles it with numba; this is the same serial algorithm
 * in plain C so the oracle does not depend on numba.
 *
 *   pass 1 (index order): a node that is still free and whose strong
 *           neighbours are all free becomes a root; it and its strong
 *           neighbours form a new aggregate.
 *   pass 2 (index order): every still-free node joins the aggregate of its
 *           strongest already-assigned strong neighbour (strict '>', so the
 *           first maximum in CSR order wins, starting from strength 0.0);
 *           nodes without one become singletons.
 *
 * Returns the number of aggregates; agg[] receives the aggregate id per node.
 */
#include <stdint.h>

int64_t oracle_plain_aggregation(const int64_t *indptr, const int64_t *indices,
                                 const double *strengths, int64_t n,
                                 int32_t *agg) {
    int64_t next_id = 0;
    for (int64_t v = 0; v < n; ++v) agg[v] = -1;

    for (int64_t v = 0; v < n; ++v) {
        if (agg[v] >= 0) continue;
        int blocked = 0;
        for (int64_t q = indptr[v]; q < indptr[v + 1]; ++q) {
            if (agg[indices[q]] >= 0) { blocked = 1; break; }
        }
        if (blocked) continue;
        agg[v] = (int32_t)next_id;
        for (int64_t q = indptr[v]; q < indptr[v + 1]; ++q) agg[indices[q]] = (int32_t)next_id;
        ++next_id;
    }

    for (int64_t v = 0; v < n; ++v) {
        if (agg[v] >= 0) continue;
        int64_t pick = -1;
        double top = 0.0;
        for (int64_t q = indptr[v]; q < indptr[v + 1]; ++q) {
            int64_t u = indices[q];
            if (agg[u] >= 0 && strengths[q] > top) { top = strengths[q]; pick = u; }
        }
        if (pick >= 0) {
            agg[v] = agg[pick];
        } else {
            agg[v] = (int32_t)next_id;
            ++next_id;
        }
    }
    return next_id;
}

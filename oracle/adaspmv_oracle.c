/*
 * adaspmv_oracle.c -- CPU ORACLE (test infrastructure, NOT product code).
 * See adaspmv_oracle.h for the contract and the pinning status.
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off, no -ffast-math).
 */
#include "adaspmv_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* partition.hpp:30-33: std::upper_bound(offsets, pos) - 1 */
int64_t or_segment_of(const int64_t* offsets, int64_t n_offsets, int64_t pos) {
    int64_t lo = 0, hi = n_offsets; /* first index with offsets[i] > pos */
    while (lo < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        if (offsets[mid] <= pos) lo = mid + 1;
        else hi = mid;
    }
    return lo - 1;
}

/* partition.hpp:37-56 */
int or_make_partition(const int64_t* offsets, int64_t n_offsets, int64_t total_items, int workers,
                      int64_t* out) {
    if (workers <= 0) return -1;
    if (n_offsets <= 0 || offsets[n_offsets - 1] != total_items) return -1;
    for (int w = 0; w < workers; ++w) {
        int64_t ib = total_items * w / workers;
        int64_t ie = total_items * (w + 1) / workers;
        out[4 * w + 0] = ib;
        out[4 * w + 1] = ie;
        if (ib >= ie) {
            out[4 * w + 2] = out[4 * w + 3] = 0;
            continue;
        }
        out[4 * w + 2] = or_segment_of(offsets, n_offsets, ib);
        out[4 * w + 3] = or_segment_of(offsets, n_offsets, ie - 1) + 1;
    }
    return 0;
}

/* parallel.hpp:153-157 */
void or_chunk_range(int64_t n, int chunks, int c, int64_t* lo, int64_t* hi) {
    *lo = n * c / chunks;
    *hi = n * (c + 1) / chunks;
}

/* sparse.hpp:333-337 (BitMask::set sparse.hpp:140: LSB-first in u64 words) */
void or_build_bitmask_sparse(int64_t n, int64_t nnz, const int64_t* idx, uint64_t* words) {
    for (int64_t w = 0; w < (n + 63) / 64; ++w) words[w] = 0;
    for (int64_t k = 0; k < nnz; ++k) words[idx[k] >> 6] |= (uint64_t)1 << (idx[k] & 63);
}

/* sparse.hpp:348-359 */
int64_t or_effective_nnz(const int64_t* col_offsets, int64_t nnz_x, const int64_t* idx) {
    int64_t acc = 0;
    for (int64_t i = 0; i < nnz_x; ++i) acc += col_offsets[idx[i] + 1] - col_offsets[idx[i]];
    return acc;
}

/* sparse.hpp:44-63 */
int or_csr_validate(int64_t rows, int64_t cols, const int64_t* ro, const int64_t* ci) {
    if (ro[0] != 0) return -1;
    for (int64_t r = 0; r < rows; ++r) {
        if (ro[r + 1] < ro[r]) return -2;
        for (int64_t k = ro[r]; k < ro[r + 1]; ++k) {
            if (ci[k] < 0 || ci[k] >= cols) return -3;
            if (k > ro[r] && ci[k] <= ci[k - 1]) return -4;
        }
    }
    return 0;
}

static int cmp_i64(const void* a, const void* b) {
    int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}

/* G = (2*sum_{i=1..k} i*d_(i)) / (k*sum d) - (k+1)/k, 0 if sum d == 0. */
double or_gini_coefficient(int64_t k, const int64_t* degrees) {
    if (k <= 0) return 0.0;
    int64_t* d = (int64_t*)malloc(sizeof(int64_t) * (size_t)k);
    memcpy(d, degrees, sizeof(int64_t) * (size_t)k);
    qsort(d, (size_t)k, sizeof(int64_t), cmp_i64);
    /* exact integer accumulation (sum i*d_(i) <= k * sum d fits in u64 for the
     * configs' sizes), converted to double once */
    unsigned __int128 wsum = 0;
    unsigned __int128 total = 0;
    for (int64_t i = 0; i < k; ++i) {
        wsum += (unsigned __int128)(i + 1) * (unsigned __int128)d[i];
        total += (unsigned __int128)d[i];
    }
    free(d);
    if (total == 0) return 0.0;
    return (2.0 * (double)wsum) / ((double)k * (double)total) - ((double)k + 1.0) / (double)k;
}

/* sum_i sum_j |d_i - d_j| / (2 k sum d) */
double or_gini_pairwise(int64_t k, const int64_t* d) {
    double total = 0, acc = 0;
    for (int64_t i = 0; i < k; ++i) total += (double)d[i];
    if (k <= 0 || total == 0) return 0.0;
    for (int64_t i = 0; i < k; ++i)
        for (int64_t j = 0; j < k; ++j) acc += fabs((double)d[i] - (double)d[j]);
    return acc / (2.0 * (double)k * total);
}

/* SPEC.md:217-219, 235-243, 281 (population std) */
int or_matrix_features(int64_t rows, int64_t cols, const int64_t* ro, double* out) {
    if (rows <= 0) return -1;
    const int64_t nnz = ro[rows];
    int64_t mx = 0, mn = INT64_MAX;
    int64_t* deg = (int64_t*)malloc(sizeof(int64_t) * (size_t)rows);
    for (int64_t r = 0; r < rows; ++r) {
        deg[r] = ro[r + 1] - ro[r];
        if (deg[r] > mx) mx = deg[r];
        if (deg[r] < mn) mn = deg[r];
    }
    const double avg = (double)nnz / (double)rows;
    /* population variance from exact integer moments: E[d^2] - avg^2 */
    unsigned __int128 sq = 0;
    for (int64_t r = 0; r < rows; ++r) sq += (unsigned __int128)deg[r] * (unsigned __int128)deg[r];
    double var = (double)sq / (double)rows - avg * avg;
    if (var < 0) var = 0;
    out[0] = (double)rows;
    out[1] = (double)cols;
    out[2] = (double)nnz;
    out[3] = (double)mx;
    out[4] = (double)mn;
    out[5] = avg;
    out[6] = cols > 0 ? (double)(mx - mn) / (double)cols : 0.0;
    out[7] = sqrt(var);
    out[8] = or_gini_coefficient(rows, deg);
    free(deg);
    return 0;
}

/* SPEC.md:301 routing: value <= threshold -> left; leaf when feature < 0. */
int or_tree_predict(const int32_t* feature, const double* threshold, const int32_t* left,
                    const int32_t* right, const int32_t* leaf, const double* f13) {
    int32_t i = 0;
    while (feature[i] >= 0) i = f13[feature[i]] <= threshold[i] ? left[i] : right[i];
    return leaf[i];
}

/* SPEC.md:489-497 level-synchronous semantics checked by a queue BFS: the
 * multiply y = A x reaches row r from frontier column c for every stored
 * (r, c); so neighbours of c are the row ids of CSC column c. */
int64_t or_bfs_queue(int64_t n, const int64_t* co, const int64_t* ri, int64_t source,
                     int64_t* levels) {
    for (int64_t i = 0; i < n; ++i) levels[i] = -1;
    if (source < 0 || source >= n) return 0;
    int64_t* q = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    int64_t head = 0, tail = 0, nlev = 0;
    levels[source] = 0;
    q[tail++] = source;
    while (head < tail) {
        int64_t c = q[head++];
        if (levels[c] + 1 > nlev) nlev = levels[c] + 1;
        for (int64_t k = co[c]; k < co[c + 1]; ++k) {
            int64_t r = ri[k];
            if (levels[r] < 0) {
                levels[r] = levels[c] + 1;
                q[tail++] = r;
            }
        }
    }
    free(q);
    return nlev;
}

/* or_bfs_queue over int32 row indices (the device layout): the same queue
 * BFS for graphs whose int64 index copy would not fit host memory (C5). */
int64_t or_bfs_queue_i32(int64_t n, const int64_t* co, const int32_t* ri, int64_t source,
                         int64_t* levels) {
    for (int64_t i = 0; i < n; ++i) levels[i] = -1;
    if (source < 0 || source >= n) return 0;
    int32_t* q = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    int64_t head = 0, tail = 0, nlev = 0;
    levels[source] = 0;
    q[tail++] = (int32_t)source;
    while (head < tail) {
        int64_t c = q[head++];
        if (levels[c] + 1 > nlev) nlev = levels[c] + 1;
        for (int64_t k = co[c]; k < co[c + 1]; ++k) {
            int64_t r = ri[k];
            if (levels[r] < 0) {
                levels[r] = levels[c] + 1;
                q[tail++] = (int32_t)r;
            }
        }
    }
    free(q);
    return nlev;
}

/* SPEC.md:498-506 incremental PageRank (delta propagation with pruning),
 * pinned only by SPEC's examples and by dense power iteration (tests).
 * delta' = d * A^T_colnorm * delta, i.e. P = A^T with column j
 * scaled by 1/outdeg(j).  The caller passes A's CSR as (co, ri): entry e of
 * "column" j below is an edge j -> ri[e] of A and outdeg(j) = co[j+1]-co[j]
 * (dangling vertices propagate nothing).
 * rank = 0, delta = 1/n; while delta != {} and it < max_iters:
 *   rank += delta; y = P delta; delta = {d*y_i : |d*y_i| >= prune, != 0}.
 * Products are formed as (1/deg_j) * delta_j, like a multiply by P's values.
 * Returns the number of multiplies. */
int64_t or_pagerank_incremental(int64_t n, const int64_t* co, const int64_t* ri, double damping,
                                double prune, int64_t max_iters, double* rank) {
    double* dv = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    double* y = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    int64_t* di = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    int64_t nd = n, it = 0;
    for (int64_t i = 0; i < n; ++i) {
        rank[i] = 0.0;
        di[i] = i;
        dv[i] = 1.0 / (double)n;
    }
    while (nd > 0 && it < max_iters) {
        for (int64_t k = 0; k < nd; ++k) rank[di[k]] += dv[k];
        for (int64_t i = 0; i < n; ++i) y[i] = 0.0;
        for (int64_t k = 0; k < nd; ++k) {
            const int64_t j = di[k];
            const int64_t deg = co[j + 1] - co[j];
            if (deg == 0) continue;
            const double w = 1.0 / (double)deg;
            for (int64_t e = co[j]; e < co[j + 1]; ++e) y[ri[e]] += w * dv[k];
        }
        nd = 0;
        for (int64_t i = 0; i < n; ++i) {
            const double v = damping * y[i];
            if (v != 0.0 && fabs(v) >= prune) {
                di[nd] = i;
                dv[nd] = v;
                ++nd;
            }
        }
        ++it;
    }
    free(dv);
    free(y);
    free(di);
    return it;
}

void or_vector_features_sparse(int64_t n, int64_t nnz, const int64_t* co, int64_t nnz_x,
                               const int64_t* xi, double* out4) {
    int64_t ns = or_effective_nnz(co, nnz_x, xi);
    out4[0] = (double)nnz_x;
    out4[1] = n > 0 ? (double)nnz_x / (double)n : 0.0;
    out4[2] = (double)ns;
    out4[3] = nnz > 0 ? (double)ns / (double)nnz : 0.0;
}

#define REAL double
#define SFX _f64
#include "oracle_impl.inc"
#undef REAL
#undef SFX

#define REAL float
#define SFX _f32
#include "oracle_impl.inc"
#undef REAL
#undef SFX

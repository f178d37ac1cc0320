/*
 * adaspmv_oracle.h -- CPU ORACLE (test infrastructure, NOT product code).
 *
 * A plain-C, single-threaded restatement of the reference algorithms of
 * arXiv 2006.16767's adaptive SpMV/SpMSpV path, used only as the checker by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg.  Nothing in
 * the product library (paper_2006_16767_b200/) links, loads or calls it.
 *
 * Each function cites the reference file:line it restates.  Paths are
 * relative to the reference root (proj/include/adaspmv/ headers, SPEC.md).
 *
 * Parity pinning: the kernel / conversion / partition / I/O functions are
 * pinned against the reference itself (oracle/_ref, compiled from the
 * unmodified reference headers by oracle/Makefile) and against the golden
 * fixtures in tests/golden/ generated from it (tests/golden/make_golden.py).
 * The SPEC-only functions (features, Gini, tree routing, BFS) have no
 * reference code; they are pinned only by SPEC.md's known-answer examples
 * ("parity unpinned" beyond those).
 *
 * Index type is int64 as in types.hpp:9.  Every value-typed function exists
 * in a _f64 (double) and a _f32 (float, the reference's ADASPMV_REAL32) form.
 */
#ifndef ADASPMV_ORACLE_H
#define ADASPMV_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- partition.hpp ---------------------------------------------------- */
/* partition.hpp:30-33: largest s with offsets[s] <= pos. */
int64_t or_segment_of(const int64_t* offsets, int64_t n_offsets, int64_t pos);
/* partition.hpp:37-56: out[4*w..4*w+3] = item_begin,item_end,span_begin,span_end.
 * Returns 0, or -1 for workers <= 0 / offsets not covering total. */
int or_make_partition(const int64_t* offsets, int64_t n_offsets, int64_t total_items,
                      int workers, int64_t* out);
/* parallel.hpp:153-157 */
void or_chunk_range(int64_t n, int chunks, int c, int64_t* lo, int64_t* hi);

/* ---- sparse.hpp (index-only) ------------------------------------------ */
/* sparse.hpp:333-337: words must hold (n+63)/64 u64, zeroed by the callee. */
void or_build_bitmask_sparse(int64_t n, int64_t nnz, const int64_t* idx, uint64_t* words);
/* sparse.hpp:348-359 */
int64_t or_effective_nnz(const int64_t* col_offsets, int64_t nnz_x, const int64_t* idx);
/* sparse.hpp:44-63 CsrMatrix::validate; returns 0 ok, else a negative code. */
int or_csr_validate(int64_t rows, int64_t cols, const int64_t* ro, const int64_t* ci);

/* ---- SPEC-only: features ----------------------------- */
/* SPEC.md:244-252 sorted identity; degrees need not be sorted (copied). */
double or_gini_coefficient(int64_t k, const int64_t* degrees);
/* SPEC.md:251 pairwise O(k^2) definition, used to check the sorted form. */
double or_gini_pairwise(int64_t k, const int64_t* degrees);
/* out[0..8] = m,n,nnz,max_row,min_row,avg_row,
 * relative_range,var_nnz_row(population std),gc.  Returns -1 if rows == 0. */
int or_matrix_features(int64_t rows, int64_t cols, const int64_t* ro, double* out9);

/* ---- SPEC-only: selector tree routing ------- */
/* Node arrays: feature[i] < 0 marks a leaf whose class is leaf[i].
 * Routing: value <= threshold -> left. */
int or_tree_predict(const int32_t* feature, const double* threshold, const int32_t* left,
                    const int32_t* right, const int32_t* leaf, const double* features13);

/* ---- SPEC-only: BFS ---------------------------------- */
/* Queue BFS over the pattern of A (edge r->c for every stored (r,c) read as
 * y = A x: vertex r is reached from frontier vertex c).  levels[i] = -1
 * when unreached.  Returns the number of levels (iterations). */
/* SPEC.md:498-506 incremental PageRank (see adaspmv_oracle.c); rank[n]. */
int64_t or_pagerank_incremental(int64_t n, const int64_t* co, const int64_t* ri, double damping,
                                double prune, int64_t max_iters, double* rank);
int64_t or_bfs_queue(int64_t n, const int64_t* col_offsets, const int64_t* row_indices,
                     int64_t source, int64_t* levels);
int64_t or_bfs_queue_i32(int64_t n, const int64_t* col_offsets, const int32_t* row_indices,
                         int64_t source, int64_t* levels);

#define OR_DECLARE(REAL, SFX)                                                                  \
    /* kernels.hpp:197-209 */                                                                  \
    void or_reference_multiply##SFX(int64_t rows, const int64_t* ro, const int64_t* ci,        \
                                    const REAL* vals, const REAL* x, REAL* y);                 \
    /* semirings of SPEC.md:489-497 (0 plus-times, 1 or-and, 2 min-plus) */                   \
    void or_semiring_multiply##SFX(int64_t rows, const int64_t* ro, const int64_t* ci,         \
                                   const REAL* vals, const REAL* x, int sr, REAL* y);          \
    /* kernels.hpp:219-286 (validate = RowSpMSpV with mask, else SpMV) */                     \
    void or_row_major_multiply##SFX(int64_t rows, const int64_t* ro, const int64_t* ci,        \
                                    const REAL* vals, const REAL* x, const uint64_t* mask,     \
                                    int load_balanced, int workers, REAL* y);                  \
    /* kernels.hpp:377-514.  Atomic: writes dense y[rows], returns -1.  Sort: writes the    \
     * sparse y (capacity rows) and returns nnz_y.  private_acc = kernels.hpp:452-478. */    \
    int64_t or_spmspv_col##SFX(int64_t rows, const int64_t* co, const int64_t* ri,            \
                               const REAL* vals, int64_t nnz_x, const int64_t* xi,             \
                               const REAL* xv, int load_balanced, int sort, int workers,       \
                               int private_acc, REAL* y_dense, int64_t* y_idx, REAL* y_val);   \
    /* kernels.hpp:341-345 + 323-337: stable sort by row, sum runs, drop exact zeros. */      \
    int64_t or_sort_reduce_pairs##SFX(int64_t npairs, const int64_t* rows_in,                  \
                                      const REAL* vals_in, int64_t* out_idx, REAL* out_val);   \
    /* sparse.hpp:157-178 */                                                                   \
    void or_csr_to_csc##SFX(int64_t rows, int64_t cols, const int64_t* ro, const int64_t* ci,  \
                            const REAL* vals, int64_t* co, int64_t* ri, REAL* cvals);          \
    /* sparse.hpp:283-321 (drops exact zeros; -0.0 == 0) */                                    \
    int64_t or_dense_to_sparse##SFX(int64_t n, const REAL* v, int64_t* idx, REAL* val);        \
    /* sparse.hpp:323-331; returns -1 on an out-of-range index (std::out_of_range) */          \
    int or_sparse_to_dense##SFX(int64_t n, int64_t nnz, const int64_t* idx, const REAL* val,   \
                                REAL* out);                                                    \
    /* sparse.hpp:339-344 */                                                                   \
    void or_build_bitmask_dense##SFX(int64_t n, const REAL* v, uint64_t* words);               \
    /* out[0..3] = nnz_x, x_sparsity, nnz_s, m_sparsity (dense input:     \
     * nnz_x counts nonzero entries) */                                                        \
    void or_vector_features_dense##SFX(int64_t n, int64_t nnz, const int64_t* co,              \
                                       const REAL* x, double* out4);

OR_DECLARE(double, _f64)
OR_DECLARE(float, _f32)

/* SPEC.md:253-261 for a sparse input (values irrelevant). */
void or_vector_features_sparse(int64_t n, int64_t nnz, const int64_t* co, int64_t nnz_x,
                               const int64_t* xi, double* out4);

#ifdef __cplusplus
}
#endif

#endif

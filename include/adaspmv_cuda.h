/*
 * adaspmv_cuda.h -- C-ABI of the B200-native adaptive SpMV/SpMSpV library
 * (libadaspmv_cuda.so, built from paper_2006_16767_b200/csrc/).
 *
 * This is the drop-in boundary for the reference's hot path
 * (arXiv 2006.16767 reference, header-only C++ `namespace adaspmv`).  Every
 * entry point below cites the reference interface it replaces.  Conventions:
 *
 *  - plain pointers and sizes only; no C++ or torch types cross the ABI;
 *  - every function returns an adaspmv_status; no exception crosses the ABI.
 *    The C++ wrapper (adaspmv_cuda.hpp) maps the codes back to the
 *    reference's exception types: ADASPMV_ERR_INVALID_ARGUMENT ->
 *    std::invalid_argument, ADASPMV_ERR_OUT_OF_RANGE -> std::out_of_range,
 *    ADASPMV_ERR_PARSE -> adaspmv::ParseError, ADASPMV_ERR_FORMAT ->
 *    adaspmv::FormatError (types.hpp:21-36);
 *  - host arrays use the reference's layout (int64 indices, types.hpp:9;
 *    values double or float, types.hpp:13-17 selected per object by dtype);
 *    the device keeps int64 offsets, int32 indices;
 *  - one context = one device + one CUDA stream; calls on a context are
 *    serialised (as the reference's ThreadPool serialises jobs,
 *    parallel.hpp:41,143).  Objects are bound to the context that made them.
 */
#ifndef ADASPMV_CUDA_H
#define ADASPMV_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    ADASPMV_OK = 0,
    ADASPMV_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument (kernels.hpp:198, sparse.hpp:44-96) */
    ADASPMV_ERR_OUT_OF_RANGE = 2,     /* std::out_of_range (sparse.hpp:326-327) */
    ADASPMV_ERR_PARSE = 3,            /* ParseError (types.hpp:21-30) */
    ADASPMV_ERR_FORMAT = 4,           /* FormatError (types.hpp:33-36) */
    ADASPMV_ERR_CUDA = 5,             /* CUDA runtime / launch failure */
    ADASPMV_ERR_NOMEM = 6,            /* device or host allocation failure */
    ADASPMV_ERR_INTERNAL = 7
} adaspmv_status;

typedef enum { ADASPMV_F64 = 0, ADASPMV_F32 = 1 } adaspmv_dtype; /* real_t, types.hpp:13-17 */

/* Semiring of a multiply.  PLUS_TIMES is the reference arithmetic
 * (kernels.hpp:236); OR_AND (pattern only, values ignored) and MIN_PLUS are
 * the BFS semirings of BASELINE.json's north_star (SPEC.md:489-497 drives BFS
 * with plus-times; see DESIGN.md for the equivalence). */
typedef enum {
    ADASPMV_PLUS_TIMES = 0,
    ADASPMV_OR_AND = 1,
    ADASPMV_MIN_PLUS = 2
} adaspmv_semiring;

/* KernelId::index() order, kernels.hpp:52-60 / names kernels.hpp:77-79. */
typedef enum {
    ADASPMV_SPMV_DIRECT = 0,
    ADASPMV_SPMV_LB = 1,
    ADASPMV_ROW_DIRECT = 2,
    ADASPMV_ROW_LB = 3,
    ADASPMV_COL_DIRECT_ATOMIC = 4,
    ADASPMV_COL_DIRECT_SORT = 5,
    ADASPMV_COL_LB_ATOMIC = 6,
    ADASPMV_COL_LB_SORT = 7
} adaspmv_kernel;

/* Feature ids, frozen order of SPEC.md:226. */
enum {
    ADASPMV_F_M = 0, ADASPMV_F_N, ADASPMV_F_NNZ, ADASPMV_F_MAX_ROW, ADASPMV_F_MIN_ROW,
    ADASPMV_F_AVG_ROW, ADASPMV_F_RELATIVE_RANGE, ADASPMV_F_VAR_NNZ_ROW, ADASPMV_F_GC,
    ADASPMV_F_NNZ_X, ADASPMV_F_X_SPARSITY, ADASPMV_F_NNZ_S, ADASPMV_F_M_SPARSITY,
    ADASPMV_NUM_FEATURES
};

typedef struct adaspmv_ctx adaspmv_ctx;
typedef struct adaspmv_matrix adaspmv_matrix;
typedef struct adaspmv_vector adaspmv_vector;
typedef struct adaspmv_output adaspmv_output;
typedef struct adaspmv_bundle adaspmv_bundle;

/* KernelConfig (kernels.hpp:154-162) plus device knobs.  Zero-initialise for
 * defaults.  `workers` is accepted for API parity; the GPU split is a
 * function of the input alone (tile sizes), so results never depend on it. */
typedef struct {
    int32_t workers;                     /* kernels.hpp:155-158 */
    int32_t atomic_private_accumulators; /* kernels.hpp:161: CTA-private accumulators */
    int32_t semiring;                    /* adaspmv_semiring */
    int32_t lanes_per_row;               /* 0 = auto; direct kernels' lanes per row/column */
    /* Execution of the Direct row-major kernels K0/K2: 0 = auto (row bins when
     * the matrix's x gathers are scattered), 1 = CSR
     * gather, 2 = row bins (column-sorted entries, shared-memory y segment). */
    int32_t row_layout;
    int32_t bin_rows;                    /* rows per bin override (0 = auto) */
    int64_t bin_tile_nnz;                /* entries per bin tile override (0 = auto) */
    /* CTAs per bin tile: 1 = one CTA owns a bin tile; 2 = a thread-block
     * cluster pair shares it (twice the rows per bin, the pair's shared-memory
     * y segments combined over DSMEM); 0 = auto. */
    int32_t bin_cluster;
    /* x bytes per column panel of the row bins, KiB (<= 0 = one panel, the
     * default): the bins stream x panel by panel, their y segments
     * accumulating across panels (opt-in). */
    int32_t bin_panel_kib;
} adaspmv_config;

enum { ADASPMV_ROW_LAYOUT_AUTO = 0, ADASPMV_ROW_LAYOUT_CSR = 1, ADASPMV_ROW_LAYOUT_BINNED = 2 };

/* ---- context -------------------------------------------------------------- */
/* Binds `device` and a stream (NULL = a new non-blocking stream owned by the
 * context; else the caller's cudaStream_t, borrowed). */
int adaspmv_ctx_create(int device, void* stream, adaspmv_ctx** out);
int adaspmv_ctx_destroy(adaspmv_ctx* ctx);
int adaspmv_ctx_synchronize(adaspmv_ctx* ctx);
/* cudaStream_t of the context. */
void* adaspmv_ctx_stream(adaspmv_ctx* ctx);
/* Message of the last failed call on this thread (never NULL). */
const char* adaspmv_last_error(void);
/* Number of kernels this library launched on `ctx` so far (bench evidence). */
int64_t adaspmv_ctx_launch_count(adaspmv_ctx* ctx);
/* When enabled, every run is bracketed by CUDA events on the context stream
 * (device time of the multiply incl. conversions it triggers, excluding host
 * time before the first launch); read with adaspmv_output_elapsed. */
int adaspmv_ctx_set_timing(adaspmv_ctx* ctx, int enable);
/* BFS level loop of adaspmv_bfs: 1 = the host-driven loop (one
 * synchronisation per level); 0 (default) = device-resident where it applies
 * (membership-only levels -- OR_AND, or a pattern matrix -- under the
 * built-in policy or a selector bundle): the whole traversal is one
 * cooperative persistent kernel (grid barriers between levels; the level
 * decisions, frontier updates and the selector's tree walk on the device;
 * one launch and one host synchronisation per traversal -- C3 R-MAT 22:
 * 0.19 ms vs 0.52 ms for the host loop), or, with ADASPMV_BFS_PERSIST=0 in
 * the environment, one CUDA graph whose WHILE / SWITCH conditional nodes run
 * only the chosen branch of each level.  Forced kernels and values-dependent
 * semirings on weighted matrices always use the host loop. */
int adaspmv_ctx_set_bfs_loop(adaspmv_ctx* ctx, int host_loop);
const char* adaspmv_version(void);

/* ---- matrices: DualMatrix (sparse.hpp:204-259) ------------------------------ */
/* DualMatrix::from_csr (sparse.hpp:212-217): validates like CsrMatrix::validate
 * (sparse.hpp:44-63), copies the host CSR to the device (vals == NULL means a
 * pattern matrix, every value 1.0), builds the CSC on the device with the
 * reference's stable order (csr_to_csc, sparse.hpp:157-178) and the matrix
 * features.  Host arrays are borrowed for the call only. */
int adaspmv_matrix_create_csr(adaspmv_ctx* ctx, int64_t rows, int64_t cols,
                              const int64_t* row_offsets, const int64_t* col_indices,
                              const void* values, int dtype, adaspmv_matrix** out);
/* Same from device-resident CSR (int64 offsets, int32 indices); validated on
 * the device like the host path (CsrMatrix::validate, one synchronisation),
 * then copied. */
int adaspmv_matrix_create_csr_device(adaspmv_ctx* ctx, int64_t rows, int64_t cols, int64_t nnz,
                                     const int64_t* d_row_offsets, const int32_t* d_col_indices,
                                     const void* d_values, int dtype, adaspmv_matrix** out);
/* DualMatrix::from_triplets (sparse.hpp:220-258): sorts, sums duplicates. */
int adaspmv_matrix_from_triplets(adaspmv_ctx* ctx, int64_t rows, int64_t cols, int64_t count,
                                 const int64_t* t_rows, const int64_t* t_cols,
                                 const void* t_values, int dtype, adaspmv_matrix** out);
/* load_matrix (matrix_market.hpp:228-238): ASPMVBIN v1 or Matrix Market. */
int adaspmv_matrix_load(adaspmv_ctx* ctx, const char* path, int dtype, adaspmv_matrix** out);
/* write_matrix_market (matrix_market.hpp:132-146) / save_binary (:160-182). */
int adaspmv_matrix_write_matrix_market(adaspmv_ctx* ctx, const adaspmv_matrix* m, const char* path);
int adaspmv_matrix_save_binary(adaspmv_ctx* ctx, const adaspmv_matrix* m, const char* path);
/* transpose (sparse.hpp:262-275): swaps the two layouts on the device. */
int adaspmv_matrix_transpose(adaspmv_ctx* ctx, const adaspmv_matrix* m, adaspmv_matrix** out);
int adaspmv_matrix_destroy(adaspmv_matrix* m);
int adaspmv_matrix_dims(const adaspmv_matrix* m, int64_t* rows, int64_t* cols, int64_t* nnz,
                        int* dtype);
/* Copies the device CSR / CSC back in the reference layout (int64 indices).
 * Any pointer may be NULL. */
int adaspmv_matrix_download(adaspmv_ctx* ctx, const adaspmv_matrix* m, int64_t* row_offsets,
                            int64_t* col_indices, void* values, int64_t* col_offsets,
                            int64_t* row_indices, void* csc_values);
/* Matrix features ids 0..8, computed once at creation. */
int adaspmv_matrix_features(const adaspmv_matrix* m, double out9[9]);
/* Mean |col - row*cols/rows| over the nonzeros, in columns: how scattered the
 * x gathers of the row-major kernels are (drives row_layout = AUTO). */
int adaspmv_matrix_gather_spread(const adaspmv_matrix* m, double* out);

/* ---- vectors (DenseVector / SparseVector / BitMask, sparse.hpp:99-151) ------ */
/* A vector is one logical operand x of length n with a device cache of the
 * representations kernels need (OperandViews, kernels.hpp:171-175); each is
 * built at most once per set_* call, only when a kernel or feature asks. */
int adaspmv_vector_create(adaspmv_ctx* ctx, int64_t length, int dtype, adaspmv_vector** out);
int adaspmv_vector_destroy(adaspmv_vector* v);
/* SparseVector (sparse.hpp:113-130): indices strictly increasing and < n
 * (validated, SparseVector::validate :120-129); explicit zeros are kept. */
int adaspmv_vector_set_sparse(adaspmv_ctx* ctx, adaspmv_vector* v, int64_t nnz,
                              const int64_t* indices, const void* values);
/* DenseVector (sparse.hpp:99-109): n values. */
int adaspmv_vector_set_dense(adaspmv_ctx* ctx, adaspmv_vector* v, const void* values);
/* Device-resident inputs (e.g. a previous y or a BFS frontier): copied.  The
 * sparse form's int32 indices are validated on the device first
 * (SparseVector::validate, one synchronisation). */
int adaspmv_vector_set_sparse_device(adaspmv_ctx* ctx, adaspmv_vector* v, int64_t nnz,
                                     const int32_t* d_indices, const void* d_values);
int adaspmv_vector_set_dense_device(adaspmv_ctx* ctx, adaspmv_vector* v, const void* d_values);
/* x := a previous multiply's output, without leaving the device. */
int adaspmv_vector_set_output(adaspmv_ctx* ctx, adaspmv_vector* v, adaspmv_output* y);
/* Builds the representation(s) kernel `kernel_index` needs (SPEC.md:398-399,
 * 413): dense for SpMV, dense + bitmask for RowSpMSpV, sparse for ColSpMSpV.
 * Conversions: sparse_to_dense (sparse.hpp:323-331), dense_to_sparse
 * (:283-321), build_bitmask (:333-344).  Optional; run() does it lazily. */
int adaspmv_vector_prepare(adaspmv_ctx* ctx, adaspmv_vector* v, int kernel_index);
/* Host copies of the cached representations (testing / interop). */
int adaspmv_vector_nnz(adaspmv_ctx* ctx, adaspmv_vector* v, int64_t* nnz);
int adaspmv_vector_get_sparse(adaspmv_ctx* ctx, adaspmv_vector* v, int64_t capacity,
                              int64_t* indices, void* values, int64_t* nnz);
int adaspmv_vector_get_dense(adaspmv_ctx* ctx, adaspmv_vector* v, void* values);
int adaspmv_vector_get_bitmask(adaspmv_ctx* ctx, adaspmv_vector* v, uint64_t* words);
/* effective_nnz (sparse.hpp:348-359) of v against m's CSC. */
int adaspmv_effective_nnz(adaspmv_ctx* ctx, const adaspmv_matrix* m, adaspmv_vector* v,
                          int64_t* out);

/* ---- features + selector hook ---------------------------- */
/* Lazily computes the features whose bit is set in `mask` (bit i = feature id
 * i); others are left untouched.  Only nnz_s / m_sparsity (and
 * nnz_x of a dense input) touch the device. */
int adaspmv_features(adaspmv_ctx* ctx, const adaspmv_matrix* m, adaspmv_vector* v,
                     uint32_t mask, double out13[13]);
/* SelectorBundle from a model file (SPEC.md:383 schema,
 * text form documented in DESIGN.md) or from node arrays (tree 0 = pattern,
 * 1 = workload, 2 = write-back; feature < 0 marks a leaf with class `leaf`). */
int adaspmv_bundle_load(const char* path, adaspmv_bundle** out);
int adaspmv_bundle_create(const int32_t n_nodes[3], const int32_t* const feature[3],
                          const double* const threshold[3], const int32_t* const left[3],
                          const int32_t* const right[3], const int32_t* const leaf[3],
                          adaspmv_bundle** out);
int adaspmv_bundle_destroy(adaspmv_bundle* b);
/* predict_kernel: pattern tree -> workload tree ->
 * write-back tree iff ColSpMSpV, pulling features lazily.  Writes the chosen
 * KernelId::index(); `features_used` (optional) gets the mask of features
 * evaluated, `trees_evaluated` (optional) the number of trees walked. */
int adaspmv_select(adaspmv_ctx* ctx, const adaspmv_matrix* m, adaspmv_vector* v,
                   const adaspmv_bundle* b, int* kernel_index, uint32_t* features_used,
                   int* trees_evaluated);

/* ---- multiply: run_kernel (kernels.hpp:520-535) ---------------------------- */
int adaspmv_output_create(adaspmv_ctx* ctx, adaspmv_output** out);
int adaspmv_output_destroy(adaspmv_output* y);
/* y = A x with kernel `kernel_index` (0..7, KernelId::index()).  `cfg` may be
 * NULL.  Missing representations are built first (the reference throws
 * std::invalid_argument instead, kernels.hpp:524-534; prepare() beforehand to
 * exclude conversion from the kernel time).  Asynchronous on the context
 * stream; the output keeps the representation the kernel produced (sort
 * write-back: sparse; else dense, kernels.hpp:113-115). */
int adaspmv_run(adaspmv_ctx* ctx, const adaspmv_matrix* m, adaspmv_vector* x, int kernel_index,
                const adaspmv_config* cfg, adaspmv_output* y);
/* Adaptive: select (bundle != NULL) then run; `chosen` optional. */
int adaspmv_run_adaptive(adaspmv_ctx* ctx, const adaspmv_matrix* m, adaspmv_vector* x,
                         const adaspmv_bundle* b, const adaspmv_config* cfg, adaspmv_output* y,
                         int* chosen);
/* ---- batched multiplies from host buffers (serving path) ------------------ */
/* One operand x in the reference's host layout: nnz < 0 = DenseVector
 * (sparse.hpp:99-109, `values` holds n reals); else SparseVector
 * (sparse.hpp:113-130, nnz int64 indices strictly increasing and < n). */
typedef struct {
    int64_t nnz;
    const int64_t* indices;
    const void* values;
} adaspmv_host_operand;

/* Result form of a batched multiply. */
enum {
    ADASPMV_RESULT_DENSE = 0,  /* MultiplyOutput::dense(): m values */
    ADASPMV_RESULT_SPARSE = 1, /* MultiplyOutput::sparse(): int64 indices + values, zeros dropped */
    ADASPMV_RESULT_AUTO = 2    /* the smaller of the two (sparse when the sort kernels produced it or
                                  nnz_s bounds nnz_y below the dense size); `form` reports which */
};

/* One result in host memory.  In: form, capacity (sparse entries the
 * indices/values buffers hold), indices (int64, may be NULL for DENSE),
 * values (m reals for DENSE / AUTO, `capacity` reals for SPARSE).  Out: form
 * written, kernel run (KernelId::index()), nnz_y (SPARSE; -1 for DENSE). */
typedef struct {
    int32_t form;
    int32_t kernel;
    int64_t capacity;
    int64_t* indices;
    void* values;
    int64_t nnz_y;
} adaspmv_host_result;

/* `count` independent multiplies y_k = A x_k, each exactly what
 * vector_set_* -> run_adaptive (or run with `forced_kernel` >= 0) ->
 * output_dense/sparse does, pipelined over `lanes` (0 = 3) streams of the
 * device: one vector's host-to-device copy, another's multiply and a third's
 * device-to-host copy overlap.  Pinned host buffers make the copies
 * asynchronous.  Returns after every result is in host memory; the first
 * failure (e.g. an invalid operand) stops the batch and is reported. */
int adaspmv_run_batch(adaspmv_ctx* ctx, const adaspmv_matrix* m, const adaspmv_bundle* b,
                      int forced_kernel, const adaspmv_config* cfg, int64_t count,
                      const adaspmv_host_operand* xs, adaspmv_host_result* ys, int lanes);

/* MultiplyOutput (kernels.hpp:116-152). */
int adaspmv_output_info(adaspmv_output* y, int64_t* length, int* has_dense, int* has_sparse,
                        int* dtype);
/* dense() view (kernels.hpp:136-139), materialised lazily; copies m values
 * to host memory `values` (may be NULL to only materialise). */
int adaspmv_output_dense(adaspmv_ctx* ctx, adaspmv_output* y, void* values);
/* sparse() view (kernels.hpp:141-144): exact zeros dropped (sparse.hpp:291).
 * Writes nnz_y; copies up to `capacity` entries when indices/values != NULL. */
int adaspmv_output_sparse(adaspmv_ctx* ctx, adaspmv_output* y, int64_t capacity,
                          int64_t* indices, void* values, int64_t* nnz_y);
/* KernelCounters (kernels.hpp:106-111; the reference's ADASPMV_ENABLE_COUNTERS
 * build): while enabled on a context, every run records out3[0] values_read
 * (matrix entries consumed -- a product formed), out3[1] pairs_emitted (sort
 * write-back) and out3[2] cas_retries (always 0: hardware atomics). */
int adaspmv_ctx_set_counters(adaspmv_ctx* ctx, int enable);
int adaspmv_output_counters(adaspmv_ctx* ctx, adaspmv_output* y, uint64_t out3[3]);
/* Seconds between the events of the last timed run of `y` (synchronises). */
int adaspmv_output_elapsed(adaspmv_ctx* ctx, adaspmv_output* y, double* seconds);
/* Device pointers of the views (materialised on demand). */
int adaspmv_output_device_dense(adaspmv_ctx* ctx, adaspmv_output* y, const void** d_values);
int adaspmv_output_device_sparse(adaspmv_ctx* ctx, adaspmv_output* y, const int32_t** d_indices,
                                 const void** d_values, int64_t* nnz_y);

/* ---- primitives (partition.hpp, kernels.hpp:323-345) ------------------------ */
/* make_partition (partition.hpp:37-56) on the host: out[4w..4w+3] =
 * item_begin, item_end, span_begin, span_end. */
int adaspmv_make_partition(const int64_t* offsets, int64_t n_offsets, int64_t total_items,
                           int workers, int64_t* out);
/* sort_reduce_pairs (kernels.hpp:341-345) on the device: stable by row, exact
 * zero sums dropped.  Host in/out; returns nnz via *nnz_out. */
int adaspmv_sort_reduce_pairs(adaspmv_ctx* ctx, int64_t npairs, const int64_t* rows,
                              const void* values, int dtype, int64_t nrows, int64_t* out_indices,
                              void* out_values, int64_t* nnz_out);
/* nnz-balanced row cut for the row-partitioned multi-GPU mode: cuts[0..g] with
 * cuts[0] = 0, cuts[g] = rows, cut i = segment_of(row_offsets, i*nnz/g)
 * snapped so no row is split (partition.hpp:30-33 search). */
int adaspmv_shard_rows(const int64_t* row_offsets, int64_t rows, int nshards, int64_t* cuts);

/* ---- row-partitioned multi-GPU mode, one process ---- */
/* The matrix (host CSR, as adaspmv_matrix_create_csr) is cut into `ngpu`
 * contiguous row blocks of ~nnz/ngpu nonzeros (adaspmv_shard_rows); block g
 * lives on devices[g] (NULL: device g) as its own DualMatrix.  A run sends x
 * (nnz_x < 0: dense, `values` = n reals; else int64-indexed sparse) to every
 * block, each block selects (bundle, or `forced_kernel` >= 0) and multiplies,
 * and y (m reals, host) receives every block at its row offset; `kernels`
 * (optional, ngpu ints) gets each block's KernelId::index(). */
typedef struct adaspmv_multi adaspmv_multi;
int adaspmv_multi_create(int ngpu, const int* devices, int64_t rows, int64_t cols,
                         const int64_t* row_offsets, const int64_t* col_indices, const void* values,
                         int dtype, adaspmv_multi** out);
int adaspmv_multi_cuts(const adaspmv_multi* mm, int64_t* cuts); /* ngpu + 1 row cuts */
int adaspmv_multi_run(adaspmv_multi* mm, const adaspmv_bundle* b, int forced_kernel,
                      const adaspmv_config* cfg, int64_t nnz_x, const int64_t* indices,
                      const void* values, void* y, int* kernels);
int adaspmv_multi_destroy(adaspmv_multi* mm);

/* ---- BFS driver ------------------------------------------ */
typedef struct {
    int64_t iteration;
    int64_t nnz_x;      /* frontier size */
    int32_t kernel;     /* KernelId::index() selected (or forced) */
    int32_t exec_mode;  /* how it ran: ADASPMV_EXEC_* (BFS fuses some choices) */
    double feature_s, predict_s, convert_s, kernel_s; /* IterationReport */
} adaspmv_iteration_report;

/* adaspmv_iteration_report::exec_mode.  BFS runs a row-major choice as the
 * output-masked pull (K2/K3, and K0/K1 under OR_AND) and, when frontier
 * membership does not depend on values, a column-major choice as the fused
 * top-down push over K6's load-balanced tiles (claims rows, appends the next
 * frontier; no dense y): `kernel` then names the selection, `exec_mode` what
 * actually ran. */
#define ADASPMV_EXEC_AS_SELECTED 0
#define ADASPMV_EXEC_MASKED_PULL 1
#define ADASPMV_EXEC_FUSED_PUSH_LB 2

/* execute_iteration: lazy features -> predict_kernel (or
 * `forced_kernel` >= 0) -> convert x iff the kernel needs another format ->
 * run.  Fills `report` (IterationReport): host seconds of
 * the feature pulls and the tree walk, device seconds of the conversion and
 * of the multiply (CUDA events; synchronises once at the end). */
int adaspmv_execute_iteration(adaspmv_ctx* ctx, const adaspmv_matrix* m, adaspmv_vector* x,
                              const adaspmv_bundle* b, int forced_kernel, const adaspmv_config* cfg,
                              adaspmv_output* y, adaspmv_iteration_report* report);

/* Level-synchronous BFS from `source` over y = A x (A as stored, square).
 * `semiring` selects the multiply's algebra; `bundle` (may be NULL) selects
 * a kernel per level, else `forced_kernel` (0..7) is used for every level,
 * or -1 = built-in direction heuristic.  levels[n] gets the level or -1
 * (levels may be NULL: traversal only, no device-to-host copy).
 * reports (optional, capacity max_reports) gets one row per level. */
int adaspmv_bfs(adaspmv_ctx* ctx, const adaspmv_matrix* m, int64_t source, int semiring,
                const adaspmv_bundle* b, int forced_kernel, int64_t* levels, int64_t* n_levels,
                adaspmv_iteration_report* reports, int64_t max_reports);

/* Incremental (delta-propagation) PageRank: P = A^T with
 * column j scaled by 1/outdeg(j), outdeg(j) = stored entries of row j of A
 * (SPEC.md:500 delta' = damping * A^T_colnorm * delta: edge i -> j moves
 * mass from i to j; pattern; dangling vertices propagate nothing,
 * SPEC.md:543), built once per matrix on the device.  rank = 0,
 * delta = 1/n; repeat { rank += delta; delta = {d*(P delta)_i : |.| >= prune,
 * != 0} } until delta is empty or `max_iters` multiplies were done.  Kernel
 * per iteration: `bundle`, else `forced_kernel` (0..7), else (-1) the
 * built-in bytes model.  rank[n] (host, may be NULL) gets the ranks widened
 * to double; reports as adaspmv_bfs. */
int adaspmv_pagerank(adaspmv_ctx* ctx, const adaspmv_matrix* m, double damping, double prune,
                     int64_t max_iters, const adaspmv_bundle* b, int forced_kernel, double* rank,
                     int64_t* n_iters, adaspmv_iteration_report* reports, int64_t max_reports);

/* ---- row-partitioned mode, one process per GPU ----------- */
/* Rank g of `world` holds the row block [cuts[g], cuts[g+1]) of the matrix
 * (adaspmv_shard_rows) as its own adaspmv_matrix on its context's device
 * (all n columns, so every kernel runs locally and each rank selects its own
 * kernel: nnz_s differs per block).  The library performs the exchanges on
 * the context's stream, device to device:
 *   x broadcast from a root rank (adaspmv_dist_bcast_vector),
 *   the y blocks into a full y on every rank (adaspmv_dist_allgather_output),
 *   the BFS frontier lists all-gathered every level (adaspmv_dist_bfs).
 * Transport: NCCL (adaspmv_dist_create_nccl; rank 0 makes the id with
 * adaspmv_dist_unique_id and the caller hands it to every rank, e.g. over
 * torch.distributed; NVLink / NVSwitch between B200s), or the caller's host
 * all-gather (adaspmv_dist_create_host: tests, ranks sharing a GPU).
 * Collective: every rank makes the same sequence of dist calls. */
typedef struct adaspmv_dist adaspmv_dist;
/* Host all-gather: every rank contributes `nbytes` (the same on all ranks);
 * recv gets world * nbytes in rank order.  Returns 0 on success. */
typedef int (*adaspmv_allgather_fn)(void* user, const void* send, int64_t nbytes, void* recv);
int adaspmv_dist_unique_id(void* id128);  /* ncclUniqueId, 128 bytes */
int adaspmv_dist_create_nccl(adaspmv_ctx* ctx, int rank, int world, const void* id128, adaspmv_dist** out);
int adaspmv_dist_create_host(adaspmv_ctx* ctx, int rank, int world, adaspmv_allgather_fn fn, void* user,
                             adaspmv_dist** out);
int adaspmv_dist_destroy(adaspmv_dist* d);
/* x of rank `root` (set sparse or dense) into x of every rank (same length). */
int adaspmv_dist_bcast_vector(adaspmv_dist* d, adaspmv_vector* x, int root);
/* Every rank's dense y block, in rank order, into y_full (device, sum of the
 * blocks' rows values); *total gets that sum. */
/* A full-y buffer of `bytes` bytes on this rank's device, IPC-shared with
 * every rank (collective).  adaspmv_dist_allgather_output into it writes each
 * rank's block straight into every rank's buffer with peer stores over
 * NVLink / NVSwitch (csrc/peer.cu) instead of NCCL broadcasts.  Freed with
 * the dist.  Replaces: the y all-gather after a row-partitioned multiply
 * (partition.hpp:30-56 row blocks). */
int adaspmv_dist_alloc_peer_output(adaspmv_dist* d, int64_t bytes, void** y_full_device);
/* Kernel `kernel_index` on this rank's row block AND the y all-gather in one
 * call: the row-bin K0/K2 store epilogue writes every row into every rank's
 * peer output as it finishes it (the transfer overlaps the multiply bin by
 * bin); other kernels are followed by the put kernel.  y also receives the
 * local block.  *fused (optional) = 1 when the epilogue did it.  Collective. */
int adaspmv_dist_run_allgather(adaspmv_dist* d, const adaspmv_matrix* block, adaspmv_vector* x, int kernel_index,
                               const adaspmv_config* cfg, adaspmv_output* y, void* y_full_device, int64_t* total,
                               int* fused);
int adaspmv_dist_allgather_output(adaspmv_dist* d, adaspmv_output* y, void* y_full_device, int64_t* total);
/* BFS (as adaspmv_bfs) over the square matrix whose rows row0 .. row0 +
 * rows(block) - 1 this rank holds; every level each rank multiplies its block
 * with its own kernel choice (bundle / forced / heuristic, decided on its
 * block), forms the next frontier among its rows and the frontier lists are
 * all-gathered.  levels (optional) gets this rank's rows' levels; n_levels
 * and reports (this rank's levels) as adaspmv_bfs. */
int adaspmv_dist_bfs(adaspmv_dist* d, const adaspmv_matrix* block, int64_t row0, int64_t source, int semiring,
                     const adaspmv_bundle* b, int forced_kernel, int64_t* levels, int64_t* n_levels,
                     adaspmv_iteration_report* reports, int64_t max_reports);

#ifdef __cplusplus
}
#endif

#endif /* ADASPMV_CUDA_H */

// internal.hpp -- host-side object model of libadaspmv_cuda (not installed).
//
// Objects behind the C-ABI handles of include/adaspmv_cuda.h:
//   Context  one device + one stream + grow-only scratch (parallel.hpp's
//            ThreadPool is replaced by CUDA grids on this stream)
//   Matrix   device-resident DualMatrix (sparse.hpp:204-259): CSR + CSC,
//            int64 offsets, int32 indices, fp32/fp64 values; matrix-static
//            LB tile heads; the 9 matrix features
//   Vector   one operand x with its lazily-built representations
//            (OperandViews, kernels.hpp:171-175)
//   Output   MultiplyOutput (kernels.hpp:116-152)
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <atomic>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/adaspmv_cuda.h"

namespace ada {

// Status-carrying exception; converted to adaspmv_status at the C-ABI.
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void invalid(const std::string& m) { throw Error(ADASPMV_ERR_INVALID_ARGUMENT, m); }
[[noreturn]] inline void out_of_range(const std::string& m) { throw Error(ADASPMV_ERR_OUT_OF_RANGE, m); }

#define ADA_CUDA(expr)                                                                      \
    do {                                                                                    \
        cudaError_t e_ = (expr);                                                            \
        if (e_ != cudaSuccess)                                                              \
            throw ::ada::Error(e_ == cudaErrorMemoryAllocation ? ADASPMV_ERR_NOMEM          \
                                                               : ADASPMV_ERR_CUDA,          \
                               std::string(#expr) + ": " + cudaGetErrorString(e_));        \
    } while (0)

// After every kernel launch: catches configuration errors immediately.
#define ADA_LAUNCHED(ctx)                                                                   \
    do {                                                                                    \
        ADA_CUDA(cudaGetLastError());                                                       \
        (ctx).launches++;                                                                   \
    } while (0)

inline int value_bytes(int dtype) { return dtype == ADASPMV_F64 ? 8 : 4; }

// Stream of the context bound by the current C-ABI call: device memory is
// stream-ordered (cudaMallocAsync from the device's pool, release threshold
// raised at context creation), so temporaries and growth never synchronise
// the device or return memory to the driver.
inline thread_local cudaStream_t g_alloc_stream = nullptr;

// Grow-only device allocation.
struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaStream_t s = nullptr;  // stream the allocation is ordered on
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), cap(o.cap), s(o.s) { o.p = nullptr; o.cap = 0; }
    ~DevBuf() { release(); }
    void release() {
        if (p) cudaFreeAsync(p, s);
        p = nullptr;
        cap = 0;
    }
    void* ensure(size_t bytes) {
        if (bytes <= cap && p) return p;
        release();
        size_t want = bytes < 256 ? 256 : bytes;
        s = g_alloc_stream;
        ADA_CUDA(cudaMallocAsync(&p, want, s));
        cap = want;
        return p;
    }
    template <class T>
    T* as() const { return static_cast<T*>(p); }
};

struct BatchLane;  // batch.cpp: one pipelined stream of adaspmv_run_batch
struct BfsPlan;    // bfs_graph.cu: a captured device-resident BFS level loop
struct BfsPlanDeleter {
    void operator()(BfsPlan* p) const;
};

struct Context {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int sm_count = 148;
    int64_t launches = 0;
    bool timing = false;  // bracket every run with CUDA events (adaspmv_output_elapsed)
    bool counters = false;  // KernelCounters per run (adaspmv_ctx_set_counters)
    bool bfs_host_loop = false;  // adaspmv_ctx_set_bfs_loop: host-driven BFS level loop, or the device graph (default)
    unsigned long long* ctr = nullptr;  // the running output's device counters (kernels' last argument)
    // fused distributed y all-gather (peer.cu dist_run_allgather): while set,
    // a kernel whose store epilogue supports it also writes each row to every
    // rank's full y (peer_dst[world], at row peer_row0 + row) and sets peer_fused
    char* const* peer_dst = nullptr;
    int peer_world = 0;
    int64_t peer_row0 = 0;
    bool peer_fused = false;
    // general scratch (reused by every call; calls on a context are serialised)
    // [0..3] sort write-back keys/values (double buffered), [4] vector scans,
    // [5] matrix build scans, [6..9] radix counts / scan / segment sums / flags
    DevBuf scratch[10];
    // pinned, device-mapped host scalars for counts (nnz_s, nnz_y, ...): a
    // one-thread kernel stores them over PCIe (scalars_to_host) instead of a
    // copy-engine transfer, which would queue behind other streams' large
    // device-to-host copies (adaspmv_run_batch lanes)
    int64_t* h_scalars = nullptr;
    int64_t* h_scalars_dev = nullptr;  // device alias of h_scalars
    DevBuf d_scalars;  // 64 int64 slots
    // per-tile head/tail partials of the LB row kernels (kernels_row.cu):
    // context-owned so that contexts sharing a matrix never share them
    DevBuf lb_partials;
    // pinned staging for host vector uploads
    void* h_stage = nullptr;
    size_t h_stage_cap = 0;
    // lanes of adaspmv_run_batch, created on first use and kept
    std::vector<std::unique_ptr<BatchLane>> lanes;
    void* stage(size_t bytes);  // pinned host buffer of >= bytes
    void sync() { ADA_CUDA(cudaStreamSynchronize(stream)); }
    int64_t* dscal(int i) { return d_scalars.as<int64_t>() + i; }
    // D2H one device int64 (synchronises the stream)
    int64_t fetch_scalar(const int64_t* d);
    // h_scalars[0..n) = d[0..n) (synchronises the stream)
    void fetch_scalars(const int64_t* d, int n);

};

// LB tiles of the row-major kernels: fixed kRowTile nonzeros per warp
// (make_partition's equal-item split, partition.hpp:37-56, W = ceil(nnz/kRowTile)).
constexpr int kRowTile = 256;

// Row-bin layout of the binned K0/K2 execution (kernels_binned.cu): the CSC
// order stably partitioned by bins of R rows; entry = (col & (2^cw-1)) <<
// rbits | row - bin*R; each (bin, chunk = col >> cw) run padded to a multiple
// of 128 entries (padding entry: row slot 2^rbits - 1, value 0) and stored
// interleaved in 128-entry groups; chunk_off[b*nchunks + c] = first (padded)
// entry of the run ([nbins*nchunks] = n_padded).  Tiles: CTA work units.
struct BinLayout {
    bool built = false;
    int dtype = -1;
    int64_t force_rows = 0;   // rows-per-bin override it was built with
    int cluster_req = 0;      // bin_cluster request it was built with
    int cluster = 1;          // CTAs per bin tile (1, or 2 = cluster pair)
    int64_t R = 0, nbins = 0, nchunks = 0;  // R = rows of the tallest bin (shared-memory segment)
    int rbits = 0, cw = 0;
    DevBuf bin_r0;                  // int64 [nbins+1]: first row of each bin (variable-height bins)
    DevBuf pk, bv, chunk_off;
    std::vector<int64_t> bin_start;  // host: first entry of each bin, [nbins] = nnz
    std::vector<int64_t> h_chunk_off;  // host copy of chunk_off (panel tile planning)
    int64_t tile_cap = -1, tile_cap_req = -1, ntiles = 0, panel_chunks = -1;
    std::vector<int64_t> panel_tile0;  // first tile of each column panel, [npanels] = ntiles
    bool multi = false;       // some bin is split into several tiles
    // heavy rows (degree > heavy_min) leave the light bins (contiguous row
    // ranges, bins [0, nlight)) for heavy bins of up to rh rows each (bins
    // [nlight, nbins)): hrows = the heavy rows ascending (int32), hbits = their
    // bitmap (the light bins' write-back skips them)
    int64_t heavy_min = 0, nheavy = 0, nlight = 0, n_binned = 0, n_padded = 0;
    int rh = 1;
    DevBuf hrows, hbits;
    DevBuf tiles, tile_bin, tile_multi;
};

// Heavy-column segment table of the row-segmented column write-back
// (kernels_colseg.cu): columns with >= lmin entries, and for each of them the
// absolute CSC position where each R-row segment starts.
struct ColSegs {
    bool built = false;
    int64_t R = 0, nseg = 0, nheavy = 0, lmin = 0, heavy_nnz = 0;  // heavy_nnz: entries in heavy columns
    DevBuf hid;    // int32 [cols]: heavy id, or -1
    DevBuf hcols;  // int32 [nheavy]: heavy id -> column
    DevBuf cnt;    // build scratch
    DevBuf tab;    // int64 [(nseg + 1) * nheavy]: tab[b * nheavy + h]
};

struct Matrix {
    Context* ctx = nullptr;
    int64_t rows = 0, cols = 0, nnz = 0;
    int dtype = ADASPMV_F64;
    uint64_t id = 0;
    DevBuf row_off, col_idx, vals;   // CSR
    DevBuf col_off, row_idx, cvals;  // CSC
    // fp32 matrices: the CSC entries again as interleaved (row, value bits)
    // 8-byte pairs, so the direct column kernel (K4) reads a support column's
    // entries as one contiguous run (random columns: half the DRAM bursts of
    // two separate arrays)
    DevBuf cpairs;
    int64_t n_row_tiles = 0;
    // int64 [n_row_tiles+2]: [t] = first row of tile t's row window: the row
    // holding item t*kRowTile, or the first row starting there (so empty rows
    // starting at the tile boundary are inside the window); [n] = rows;
    // [n+1] = first row starting at nnz (trailing empty rows)
    DevBuf tile_head;
    DevBuf empty_rows;        // int32 ids of rows with no entries (written by the LB fix-up)
    int64_t n_empty = 0;
    // guards the lazily-built structures (row-bin layout) when several
    // contexts (adaspmv_run_batch lanes) multiply with the same matrix
    mutable std::mutex lazy;
    double feat[9] = {0};
    int64_t max_col_deg = 0;
    double avg_col = 0;
    // column degrees, distinct values ascending with prefix counts / sums
    // (host): sum of the k smallest / largest degrees bounds nnz_s of any
    // operand with k distinct stored indices, so the selector can settle an
    // nnz_s / m_sparsity split without the device reduction (selector.cpp)
    std::vector<int64_t> cdeg, cdeg_cnt, cdeg_sum;  // cnt/sum: prefix over cdeg[< i]
    int64_t nnz_s_lower(int64_t k) const;
    int64_t nnz_s_upper(int64_t k) const;
    bool pattern = false;   // created without values (all 1.0)
    float amin = 1.0f;      // fp32: smallest nonzero |a| (the atomic write-backs' subnormal-range check)
    double gather_spread = 0;  // mean |col - row*n/m| over the nonzeros (columns)
    mutable std::unique_ptr<BinLayout> bins{new BinLayout()};
    mutable std::unique_ptr<ColSegs> csegs{new ColSegs()};  // row-segmented K6 (built on first use)
    // column-normalised pattern copy for PageRank (pagerank.cu), built once
    mutable std::unique_ptr<Matrix> colnorm;
    // captured device-resident BFS loop (bfs_graph.cu), built on first use
    mutable std::unique_ptr<BfsPlan, BfsPlanDeleter> bfs_plan;
    int vbytes() const { return value_bytes(dtype); }
};

struct Vector {
    Context* ctx = nullptr;
    int64_t n = 0;
    int dtype = ADASPMV_F64;
    uint64_t version = 0;
    // representations (kernels.hpp:171-175)
    DevBuf dense;   bool has_dense = false;
    int dense_fill = -1;  // semiring whose identity filled absent entries (-1: user dense)
    DevBuf sp_idx;  DevBuf sp_val; bool has_sparse = false;
    int64_t nnz = -1;  // |supp x| when known on host (sparse input, or counted)
    DevBuf mask;    bool has_mask = false;   // (n+31)/32 u32 words == (n+63)/64 u64 LSB-first
    // For a user-dense x the sparse and mask views depend on what "absent"
    // means under the multiply's semiring: 0 (plus-times, or-and) or +inf
    // (min-plus, where 0 is a real value).  absent_of(semiring) they were
    // derived with; -1 = not derived from the dense values (user sparse x).
    int sparse_absent = -1, mask_absent = -1;
    // effective-nnz prefix (eff_offsets, kernels.hpp:400-404) for one matrix
    DevBuf eff;     uint64_t eff_matrix = 0; bool has_eff = false;
    int64_t nnz_s = -1; uint64_t nnz_s_matrix = 0;
    DevBuf stage_idx;  // int64 staging for host index uploads
    void invalidate() {
        has_dense = has_sparse = has_mask = has_eff = false;
        dense_fill = -1;
        sparse_absent = mask_absent = -1;
        nnz = -1;
        nnz_s = -1;
        nnz_s_matrix = 0;
        eff_matrix = 0;
        ++version;
    }
};

struct Output {
    Context* ctx = nullptr;
    int64_t n = 0;
    int dtype = ADASPMV_F64;
    DevBuf dense;   bool has_dense = false;
    DevBuf sp_idx;  DevBuf sp_val; bool has_sparse = false;
    int64_t nnz = -1;      // host-known nnz_y (-1 = only on device, slot d_nnz)
    DevBuf d_nnz;          // device int64 nnz_y
    int semiring = ADASPMV_PLUS_TIMES;  // identity of absent entries
    // KernelCounters of the last run (kernels.hpp:106-111), when the context
    // counts: [0] values_read, [1] pairs_emitted
    DevBuf d_ctr;
    bool has_ctr = false;
    // device-time bracket of the last run (recorded when Context::timing)
    cudaEvent_t ev[2] = {nullptr, nullptr};
    bool timed = false;
    ~Output() {
        if (ev[0]) cudaEventDestroy(ev[0]);
        if (ev[1]) cudaEventDestroy(ev[1]);
    }
    void reset(int64_t len, int dt) {
        n = len;
        dtype = dt;
        has_dense = has_sparse = false;
        nnz = -1;
    }
};

// One lane of a batched multiply: its own stream (context), operand and
// output, so that lanes overlap their copies and kernels.
struct BatchLane {
    Context c;
    Vector v;
    Output y;
    ~BatchLane();
};

// One shard of the single-process row-partitioned mode (multi.cpp): its
// device context, its row block as a matrix, an operand and an output.
struct MultiShard {
    Context ctx;
    Matrix* m = nullptr;
    Vector v;
    Output y;
    ~MultiShard();
};
struct Multi {
    int64_t rows = 0, cols = 0;
    int dtype = ADASPMV_F64;
    std::vector<int64_t> cuts;  // [G+1] row cuts
    std::vector<std::unique_ptr<MultiShard>> shards;
};

// The one-process-per-GPU row-partitioned mode's exchange (dist.cpp): NCCL
// communicator, or the caller's host all-gather callback.
struct Dist {
    Context* ctx = nullptr;
    int rank = 0, world = 1;
    void* comm = nullptr;  // ncclComm_t
    adaspmv_allgather_fn host_fn = nullptr;
    void* host_user = nullptr;
    std::vector<int64_t> counts;  // per-rank counts of the last allgatherv
    DevBuf d_cnt;
    std::vector<char> h_send, h_recv;
    DevBuf d_bytes;
    // peer transport of the y all-gather (peer.cu): this rank's full-y buffer
    // (cudaMalloc, IPC-exported) and every rank's, mapped here
    void* peer_buf = nullptr;
    int64_t peer_bytes = 0;
    std::vector<void*> peer_ptrs;
    std::vector<char> peer_opened;  // 1: opened from another process's IPC handle
    DevBuf d_peers;                 // device copy of peer_ptrs
    ~Dist();
    void host_allgather(const void* send, size_t bytes, void* recv);
    // every rank's `bytes` host bytes, in rank order (synchronises)
    void allgather_bytes(const void* send, size_t bytes, void* recv);
    // every rank's `mine` (host; synchronises)
    void allgather_count(int64_t mine, std::vector<int64_t>& all);
    // concatenation in rank order of every rank's `count` elements of `elem`
    // bytes into the device buffer `recv`; returns the total count
    int64_t allgatherv(const void* send, int64_t count, size_t elem, void* recv);
    void broadcast(void* buf, int64_t bytes, int root);
};

// peer.cu: the y all-gather as direct peer stores (CUDA IPC over NVLink)
void* dist_alloc_peer_output(Dist& d, int64_t bytes);  // collective
void dist_release_peers(Dist& d);
int64_t dist_peer_allgatherv(Dist& d, const void* send, int64_t count, size_t elem);
// kernel `k` on this rank's row block, its y rows stored into every rank's
// full y (the peer output) by the kernel's own epilogue where it can (the
// row-bin K0/K2), else by the put kernel; *fused reports which
int64_t dist_run_allgather(Dist& d, const Matrix& m, Vector& x, int k, const adaspmv_config& cfg, Output& y,
                           void* y_full, int* fused);

// One decision tree: flat node array.
struct Tree {
    int target = 0;          // 0 pattern, 1 workload, 2 write-back
    uint32_t mask = 0x1fff;  // features the tree may read
    std::vector<int32_t> feature, left, right, leaf;
    std::vector<double> threshold;
};

inline uint64_t next_object_id() {
    static std::atomic<uint64_t> n{1};
    return n.fetch_add(1);
}

struct Bundle {
    uint64_t id = next_object_id();  // identity for device-side caches (immutable after creation)
    int schema_version = 1;
    std::string hardware_tag;
    std::string feature_order_hash;
    // [0] pattern, [1] workload, [2] write-back; schema 2 adds [3] the
    // ColSpMSpV family's own workload tree (has_col)
    Tree trees[4];
    bool has_col = false;
};

// ---- entry points implemented in the .cu/.cpp files ------------------------
// context set-up / tear-down (capi.cpp): stream (own unless given), pinned
// scalars, device pool release threshold
void context_init(Context& ctx, int device, cudaStream_t stream);
void context_release(Context& ctx);

// BFS push over K6's LB tiles (kernels_col.cu), boolean semiring
template <class V>
void bfs_push_lb(Context& ctx, const Matrix& m, Vector& x, int32_t* lv, int32_t level, int32_t* next_idx,
                 V* next_val, V value, unsigned long long* cnt);

// row-partitioned multi-GPU mode (multi.cpp)
void shard_cuts(const int64_t* ro, int64_t rows, int g, int64_t* cuts);
Multi* multi_create(int ngpu, const int* devices, int64_t rows, int64_t cols, const int64_t* ro,
                    const int64_t* ci, const void* vals, int dtype);
void multi_run(Multi& mm, const Bundle* b, int forced, const adaspmv_config& cfg, int64_t nnz_x,
               const int64_t* idx, const void* vals, void* y_host, int* kernels);

// adaspmv_run_batch (batch.cpp)
void run_batch(Context& ctx, const Matrix& m, const Bundle* b, int forced, const adaspmv_config& cfg,
               int64_t count, const adaspmv_host_operand* xs, adaspmv_host_result* ys, int lanes);

Matrix* matrix_create_device(Context& ctx, int64_t rows, int64_t cols, int64_t nnz,
                             const int64_t* d_ro, const int32_t* d_ci, const void* d_vals,
                             int dtype, bool pattern);
Matrix* matrix_transpose(Context& ctx, const Matrix& m);

void vector_set_dense_device(Context& ctx, Vector& v, const void* d_vals);
// validate: check the indices on the device first (one synchronisation;
// the C-ABI entry validates caller arrays, internal producers skip it)
void vector_set_sparse_device(Context& ctx, Vector& v, int64_t nnz, const int32_t* d_idx,
                              const void* d_vals, bool validate = false);
// CsrMatrix::validate on caller device arrays (one synchronisation)
void validate_device_csr(Context& ctx, int64_t rows, int64_t cols, int64_t nnz, const int64_t* d_ro,
                         const int32_t* d_ci);
// host int64 indices (the reference's index_t) + values: H2D, then validated
// and narrowed on the device (one synchronisation for the verdict)
void vector_set_sparse_host(Context& ctx, Vector& v, int64_t nnz, const int64_t* h_idx, const void* h_vals);
// the same without waiting for the verdict: indices out of range are stored
// as 0 meanwhile; vector_check_deferred (synchronises) throws the reference's
// error.  Used by the batch lanes, whose next synchronisation (nnz_s for the
// selector) then carries the verdict too.
constexpr int kVerdictSlot = 16;  // in Context::h_scalars
// the per-iteration frontier / delta scans of BFS and PageRank store their
// total directly into this mapped slot (no copy kernel before the read)
constexpr int kScanTotalSlot = 20;
void vector_set_sparse_host_deferred(Context& ctx, Vector& v, int64_t nnz, const int64_t* h_idx,
                                     const void* h_vals);
void vector_check_deferred(Context& ctx, Vector& v);
// dense view; entries absent from a sparse input hold the identity of
// `semiring` (0 for plus-times / or-and, +inf for min-plus)
void vector_ensure_dense(Context& ctx, Vector& v, int semiring = ADASPMV_PLUS_TIMES);
// what an absent entry of x holds under a semiring: 0 = zero, 1 = +inf
inline int absent_of(int semiring) { return semiring == ADASPMV_MIN_PLUS ? 1 : 0; }
// sparse / bitmask views; for a user-dense x, entries equal to the
// semiring's identity are absent (semiring-keyed cache)
void vector_ensure_sparse(Context& ctx, Vector& v, int semiring = ADASPMV_PLUS_TIMES);
void vector_ensure_mask(Context& ctx, Vector& v, int semiring = ADASPMV_PLUS_TIMES);
void vector_ensure_eff(Context& ctx, Vector& v, const Matrix& m, int semiring = ADASPMV_PLUS_TIMES);  // also sparse
int64_t vector_nnz(Context& ctx, Vector& v);
int64_t vector_nnz_s(Context& ctx, Vector& v, const Matrix& m);
// dst[i] = src[i], i < n <= 64, by one thread on ctx's stream (dst: mapped host)
void copy_scalars_kernel_launch(Context& ctx, const int64_t* src, int64_t* dst, int n);
// out[k] = in[k] (int32 device indices -> int64), on ctx's stream
void widen_indices(Context& ctx, int64_t n, const int32_t* in, int64_t* out);

void run_kernel(Context& ctx, const Matrix& m, Vector& x, int kernel, const adaspmv_config& cfg,
                Output& y);
// binned K0/K2 (kernels_binned.cu)
double matrix_gather_spread(Context& ctx, const Matrix& m);
bool binned_preferred(const Matrix& m);
// dist.cpp
void dist_unique_id(void* out128);
Dist* dist_create_nccl(Context& ctx, int rank, int world, const void* id128);
Dist* dist_create_host(Context& ctx, int rank, int world, adaspmv_allgather_fn fn, void* user);
void dist_bcast_vector(Dist& d, Vector& x, int root);
int64_t dist_allgather_output(Dist& d, Output& y, void* y_full);
// bfs.cu: BFS over a row block of a square matrix (rows row0 .. row0 +
// m.rows - 1 of an m.cols x m.cols graph), frontiers exchanged through `d`
void bfs_dist(Context& ctx, const Matrix& m, Dist& d, int64_t row0, int64_t source, int semiring, const Bundle* b,
              int forced, int64_t* levels, int64_t* n_levels, adaspmv_iteration_report* reports,
              int64_t max_reports);
void output_ensure_dense(Context& ctx, Output& y);
void output_ensure_sparse(Context& ctx, Output& y);
int64_t output_nnz(Context& ctx, Output& y);

// device sort_reduce_pairs: keys int32 rows in [0, nrows); returns nnz
int64_t sort_reduce_pairs_device(Context& ctx, int64_t npairs, const int32_t* d_rows,
                                 const void* d_vals, int dtype, int64_t nrows, int32_t* d_out_idx,
                                 void* d_out_val);

// features / selector (selector.cpp)
void features(Context& ctx, const Matrix& m, Vector& v, uint32_t mask, double* out13);
int predict(Context& ctx, const Matrix& m, Vector& v, const Bundle& b, uint32_t* used,
            int* trees, double* feature_s = nullptr);
Bundle* bundle_load(const std::string& path);

// host I/O (mmio.cpp): CSR in the reference layout
struct HostCsr {
    int64_t rows = 0, cols = 0;
    std::vector<int64_t> row_offsets, col_indices;
    std::vector<double> values;  // widened; narrowed per dtype at upload
};
// Matrix Market coordinate entries in file order (symmetric entries
// mirrored right after their source), 0-based, values as parsed (double)
struct HostTriplets {
    int64_t rows = 0, cols = 0;
    std::vector<int64_t> r, c;
    std::vector<double> v;
};
struct HostMatrixFile {
    bool is_csr = false;  // ASPMVBIN: csr; Matrix Market: trip
    HostCsr csr;
    HostTriplets trip;
};
HostTriplets load_mm(const std::string& path);  // parallel, serial on any irregularity
HostMatrixFile load_matrix_file(const std::string& path, int dtype);
// DualMatrix::from_triplets (sparse.hpp:220-258) on the device (ingest.cu);
// h_v holds `count` values of `dtype`
Matrix* matrix_from_triplets_device(Context& ctx, int64_t rows, int64_t cols, int64_t count, const int64_t* h_r,
                                    const int64_t* h_c, const void* h_v, int dtype);
void write_matrix_market_file(const std::string& path, int64_t rows, int64_t cols,
                              const std::vector<int64_t>& ro, const std::vector<int64_t>& ci,
                              const std::vector<double>& vals);
void save_binary_file(const std::string& path, int64_t rows, int64_t cols,
                      const std::vector<int64_t>& ro, const std::vector<int64_t>& ci,
                      const void* vals, int dtype);

// BFS (bfs.cu)
void bfs(Context& ctx, const Matrix& m, int64_t source, int semiring, const Bundle* b,
         int forced, int64_t* levels, int64_t* n_levels, adaspmv_iteration_report* reports,
         int64_t max_reports);

// device-resident BFS (bfs_graph.cu): membership-only levels, heuristic or
// selector policy; levels / reports as bfs()
bool bfs_graph_applicable(const Matrix& m, int semiring, int forced);
void bfs_graph(Context& ctx, const Matrix& m, int64_t source, const Bundle* b, int64_t* levels, int64_t* n_levels,
               adaspmv_iteration_report* reports, int64_t max_reports);
// out[i] = lv[i] (int32 levels -> int64), on ctx's stream
void widen_levels(Context& ctx, const int32_t* lv, int64_t n, int64_t* out);

// incremental PageRank (pagerank.cu)
void pagerank(Context& ctx, const Matrix& m, double damping, double prune, int64_t max_iters,
              const Bundle* b, int forced, double* rank, int64_t* n_iters,
              adaspmv_iteration_report* reports, int64_t max_reports);

}  // namespace ada

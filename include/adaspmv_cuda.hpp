// adaspmv_cuda.hpp -- C++ drop-in for the reference's `namespace adaspmv`
// hot path, over the C-ABI of libadaspmv_cuda.so (adaspmv_cuda.h).
//
// Same names, argument meaning and exception types as the reference headers
// (proj/include/adaspmv/{types,partition,sparse,kernels,matrix_market}.hpp):
//   index_t / real_t (types.hpp:9-17; ADASPMV_REAL32 selects float)
//   ParseError / FormatError (types.hpp:21-36)
//   Pattern / Workload / Writeback / KernelId (kernels.hpp:35-100)
//   WorkerRange / WorkPartition / segment_of / make_partition (partition.hpp)
//   DenseVector / SparseVector / BitMask (sparse.hpp:99-151) -- host values
//   DualMatrix (sparse.hpp:204-259) -- here device resident (CSR + CSC)
//   KernelConfig / OperandViews / MultiplyOutput / run_kernel / spmv /
//   spmspv_row / spmspv_col (kernels.hpp:116-535)
//   load_matrix / write_matrix_market / save_binary (matrix_market.hpp)
// plus the selector hook and the BFS driver.
// Status codes map back to std::invalid_argument, std::out_of_range,
// ParseError and FormatError; CUDA failures throw std::runtime_error.
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "adaspmv_cuda.h"

namespace adaspmv::cuda {

using index_t = std::int64_t;
#ifdef ADASPMV_REAL32
using real_t = float;
inline constexpr int kDtype = ADASPMV_F32;
#else
using real_t = double;
inline constexpr int kDtype = ADASPMV_F64;
#endif

class ParseError : public std::runtime_error {
public:
    ParseError(const std::string& what, long line) : std::runtime_error(what), line_(line) {}
    long line() const { return line_; }

private:
    long line_;
};

class FormatError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

inline void check(int status) {
    if (status == ADASPMV_OK) return;
    const std::string msg = adaspmv_last_error();
    switch (status) {
        case ADASPMV_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case ADASPMV_ERR_OUT_OF_RANGE: throw std::out_of_range(msg);
        case ADASPMV_ERR_PARSE: {
            long line = 0;
            const auto p = msg.rfind("(line ");
            if (p != std::string::npos) line = std::strtol(msg.c_str() + p + 6, nullptr, 10);
            throw ParseError(msg, line);
        }
        case ADASPMV_ERR_FORMAT: throw FormatError(msg);
        case ADASPMV_ERR_NOMEM: throw std::bad_alloc();
        default: throw std::runtime_error(msg);
    }
}

// ---- kernel identity (kernels.hpp:35-100) ----------------------------------
enum class Pattern : std::uint8_t { ColSpMSpV = 0, RowSpMSpV = 1, SpMV = 2 };
enum class Workload : std::uint8_t { Direct = 0, LoadBalanced = 1 };
enum class Writeback : std::uint8_t { Atomic = 0, Sort = 1 };

struct KernelId {
    Pattern pattern = Pattern::SpMV;
    Workload workload = Workload::Direct;
    Writeback writeback = Writeback::Atomic;
    static constexpr int kCount = 8;

    constexpr int index() const {
        const int lb = workload == Workload::LoadBalanced ? 1 : 0;
        switch (pattern) {
            case Pattern::SpMV: return lb;
            case Pattern::RowSpMSpV: return 2 + lb;
            case Pattern::ColSpMSpV: return 4 + 2 * lb + (writeback == Writeback::Sort ? 1 : 0);
        }
        return -1;
    }
    static constexpr KernelId from_index(int i) {
        if (i < 0 || i > 7) throw std::invalid_argument("kernel index out of range");
        if (i < 2) return {Pattern::SpMV, i == 1 ? Workload::LoadBalanced : Workload::Direct, Writeback::Atomic};
        if (i < 4) return {Pattern::RowSpMSpV, i == 3 ? Workload::LoadBalanced : Workload::Direct, Writeback::Atomic};
        return {Pattern::ColSpMSpV, i >= 6 ? Workload::LoadBalanced : Workload::Direct,
                (i & 1) ? Writeback::Sort : Writeback::Atomic};
    }
    std::string_view name() const {
        static constexpr std::array<std::string_view, 8> names = {
            "spmv_direct", "spmv_lb", "row_direct", "row_lb",
            "col_direct_atomic", "col_direct_sort", "col_lb_atomic", "col_lb_sort"};
        return names[static_cast<size_t>(index())];
    }
    static std::optional<KernelId> parse(std::string_view s) {
        for (int i = 0; i < kCount; ++i)
            if (from_index(i).name() == s) return from_index(i);
        return std::nullopt;
    }
    friend constexpr bool operator==(KernelId a, KernelId b) {
        if (a.pattern != b.pattern || a.workload != b.workload) return false;
        return a.pattern != Pattern::ColSpMSpV || a.writeback == b.writeback;
    }
};

// ---- partition.hpp -----------------------------------------------------------
struct WorkerRange {
    index_t item_begin = 0, item_end = 0, span_begin = 0, span_end = 0;
    bool empty() const { return item_begin >= item_end; }
};
struct WorkPartition {
    std::vector<WorkerRange> worker_ranges;
};
inline index_t segment_of(std::span<const index_t> offsets, index_t pos) {
    return static_cast<index_t>(std::upper_bound(offsets.begin(), offsets.end(), pos) - offsets.begin()) - 1;
}
inline WorkPartition make_partition(std::span<const index_t> offsets, index_t total, int workers) {
    std::vector<int64_t> raw(4 * static_cast<size_t>(std::max(workers, 1)));
    check(adaspmv_make_partition(offsets.data(), static_cast<int64_t>(offsets.size()), total, workers, raw.data()));
    WorkPartition p;
    p.worker_ranges.resize(static_cast<size_t>(workers));
    for (int w = 0; w < workers; ++w)
        p.worker_ranges[static_cast<size_t>(w)] = {raw[4 * w], raw[4 * w + 1], raw[4 * w + 2], raw[4 * w + 3]};
    return p;
}

// KernelCounters (kernels.hpp:106-111)
struct KernelCounters {
    std::uint64_t values_read = 0;    // matrix entries consumed
    std::uint64_t pairs_emitted = 0;  // (row, product) pairs on the sort path
    std::uint64_t cas_retries = 0;    // 0 on the device: hardware atomics
};

// ---- host value types (sparse.hpp:99-151) ---------------------------------------
struct DenseVector {
    std::vector<real_t> values;
    DenseVector() = default;
    explicit DenseVector(index_t n, real_t fill = 0) : values(static_cast<size_t>(n), fill) {}
    explicit DenseVector(std::vector<real_t> v) : values(std::move(v)) {}
    index_t size() const { return static_cast<index_t>(values.size()); }
    real_t operator[](index_t i) const { return values[static_cast<size_t>(i)]; }
    real_t& operator[](index_t i) { return values[static_cast<size_t>(i)]; }
};

struct SparseVector {
    index_t length = 0;
    std::vector<index_t> indices;
    std::vector<real_t> values;
    index_t nnz() const { return static_cast<index_t>(indices.size()); }
};

struct BitMask {
    index_t length = 0;
    std::vector<std::uint64_t> words;
    explicit BitMask(index_t n = 0) : length(n), words(static_cast<size_t>((n + 63) / 64), 0) {}
    bool test(index_t i) const { return (words[static_cast<size_t>(i >> 6)] >> (i & 63)) & 1u; }
};

struct KernelConfig {
    int workers = 0;
    bool atomic_private_accumulators = false;
    int semiring = ADASPMV_PLUS_TIMES;
    int lanes_per_row = 0;
    int row_layout = ADASPMV_ROW_LAYOUT_AUTO;  // K0/K2 execution (adaspmv_cuda.h)
    int bin_rows = 0;
    long long bin_tile_nnz = 0;
    int bin_cluster = 0;  // CTAs per bin tile (1 single, 2 cluster pair, 0 auto)
    int bin_panel_kib = 0;  // x bytes per column panel of the row bins (<= 0: one panel)
    adaspmv_config c() const {
        adaspmv_config r{};
        r.workers = workers;
        r.atomic_private_accumulators = atomic_private_accumulators ? 1 : 0;
        r.semiring = semiring;
        r.lanes_per_row = lanes_per_row;
        r.row_layout = row_layout;
        r.bin_rows = bin_rows;
        r.bin_tile_nnz = bin_tile_nnz;
        r.bin_cluster = bin_cluster;
        r.bin_panel_kib = bin_panel_kib;
        return r;
    }
};

struct OperandViews {
    const DenseVector* dense = nullptr;
    const SparseVector* sparse = nullptr;
    const BitMask* mask = nullptr;
};

// ---- device objects --------------------------------------------------------------
class Context {
public:
    explicit Context(int device = 0, void* stream = nullptr) {
        check(adaspmv_ctx_create(device, stream, &h_));
    }
    ~Context() { adaspmv_ctx_destroy(h_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    adaspmv_ctx* get() const { return h_; }
    void synchronize() { check(adaspmv_ctx_synchronize(h_)); }
    void set_counters(bool enable) { check(adaspmv_ctx_set_counters(h_, enable ? 1 : 0)); }

private:
    adaspmv_ctx* h_ = nullptr;
};

class DualMatrix {
public:
    DualMatrix(Context& ctx, adaspmv_matrix* h) : ctx_(&ctx), h_(h, adaspmv_matrix_destroy) {}
    // DualMatrix::from_csr (sparse.hpp:212-217)
    static DualMatrix from_csr(Context& ctx, index_t rows, index_t cols, std::span<const index_t> row_offsets,
                               std::span<const index_t> col_indices, std::span<const real_t> values) {
        if (row_offsets.size() != static_cast<size_t>(rows) + 1)
            throw std::invalid_argument("csr: row_offsets length != rows+1");
        adaspmv_matrix* h = nullptr;
        check(adaspmv_matrix_create_csr(ctx.get(), rows, cols, row_offsets.data(), col_indices.data(),
                                        values.data(), kDtype, &h));
        return DualMatrix(ctx, h);
    }
    index_t rows() const { return dims()[0]; }
    index_t cols() const { return dims()[1]; }
    index_t nnz() const { return dims()[2]; }
    adaspmv_matrix* get() const { return h_.get(); }
    Context& context() const { return *ctx_; }

private:
    std::array<index_t, 3> dims() const {
        std::array<index_t, 3> d{};
        check(adaspmv_matrix_dims(h_.get(), &d[0], &d[1], &d[2], nullptr));
        return d;
    }
    Context* ctx_;
    std::shared_ptr<adaspmv_matrix> h_;
};

inline DualMatrix load_matrix(Context& ctx, const std::string& path) {
    adaspmv_matrix* h = nullptr;
    check(adaspmv_matrix_load(ctx.get(), path.c_str(), kDtype, &h));
    return DualMatrix(ctx, h);
}
inline DualMatrix transpose(const DualMatrix& m) {
    adaspmv_matrix* h = nullptr;
    check(adaspmv_matrix_transpose(m.context().get(), m.get(), &h));
    return DualMatrix(m.context(), h);
}
inline void write_matrix_market(const DualMatrix& m, const std::string& path) {
    check(adaspmv_matrix_write_matrix_market(m.context().get(), m.get(), path.c_str()));
}
inline void save_binary(const DualMatrix& m, const std::string& path) {
    check(adaspmv_matrix_save_binary(m.context().get(), m.get(), path.c_str()));
}

// MultiplyOutput (kernels.hpp:116-152): views materialise lazily on the host.
class MultiplyOutput {
public:
    explicit MultiplyOutput(Context& ctx) : ctx_(&ctx) {
        adaspmv_output* y = nullptr;
        check(adaspmv_output_create(ctx.get(), &y));
        h_.reset(y, adaspmv_output_destroy);
    }
    index_t size() const {
        int64_t n = 0;
        check(adaspmv_output_info(h_.get(), &n, nullptr, nullptr, nullptr));
        return n;
    }
    bool has_dense() const { return info(1); }
    bool has_sparse() const { return info(2); }
    const DenseVector& dense() const {
        if (!dense_) {
            DenseVector d(size());
            check(adaspmv_output_dense(ctx_->get(), h_.get(), d.values.data()));
            dense_ = std::move(d);
        }
        return *dense_;
    }
    const SparseVector& sparse() const {
        if (!sparse_) {
            SparseVector s;
            s.length = size();
            int64_t k = 0;
            check(adaspmv_output_sparse(ctx_->get(), h_.get(), 0, nullptr, nullptr, &k));
            s.indices.resize(static_cast<size_t>(k));
            s.values.resize(static_cast<size_t>(k));
            check(adaspmv_output_sparse(ctx_->get(), h_.get(), k, s.indices.data(), s.values.data(), &k));
            sparse_ = std::move(s);
        }
        return *sparse_;
    }
    adaspmv_output* get() const { return h_.get(); }
    // KernelCounters (kernels.hpp:106-111) of the run, when the context counts
    // (Context::set_counters); std::invalid_argument otherwise
    KernelCounters counters() const {
        std::uint64_t c[3] = {0, 0, 0};
        check(adaspmv_output_counters(ctx_->get(), h_.get(), c));
        return KernelCounters{c[0], c[1], c[2]};
    }

private:
    bool info(int which) const {
        int d = 0, s = 0;
        check(adaspmv_output_info(h_.get(), nullptr, &d, &s, nullptr));
        return which == 1 ? d != 0 : s != 0;
    }
    Context* ctx_;
    std::shared_ptr<adaspmv_output> h_;
    mutable std::optional<DenseVector> dense_;
    mutable std::optional<SparseVector> sparse_;
};

namespace detail {
struct DeviceOperand {
    std::shared_ptr<adaspmv_vector> h;
    DeviceOperand(Context& ctx, index_t n) {
        adaspmv_vector* v = nullptr;
        check(adaspmv_vector_create(ctx.get(), n, kDtype, &v));
        h.reset(v, adaspmv_vector_destroy);
    }
};
}  // namespace detail

// run_kernel (kernels.hpp:520-535): same operand checks, then the CUDA kernel.
inline MultiplyOutput run_kernel(const DualMatrix& m, KernelId id, const OperandViews& views,
                                 const KernelConfig& cfg = {}) {
    Context& ctx = m.context();
    detail::DeviceOperand x(ctx, m.cols());
    switch (id.pattern) {
        case Pattern::SpMV:
            if (!views.dense) throw std::invalid_argument("SpMV requires a dense operand");
            break;
        case Pattern::RowSpMSpV:
            if (!views.dense || !views.mask)
                throw std::invalid_argument("RowSpMSpV requires dense values and a bitmask");
            break;
        case Pattern::ColSpMSpV:
            if (!views.sparse) throw std::invalid_argument("ColSpMSpV requires a sparse operand");
            break;
    }
    if (id.pattern == Pattern::ColSpMSpV) {
        if (views.sparse->length != m.cols())
            throw std::invalid_argument("spmspv_col: vector length != matrix columns");
        check(adaspmv_vector_set_sparse(ctx.get(), x.h.get(), views.sparse->nnz(), views.sparse->indices.data(),
                                        views.sparse->values.data()));
    } else {
        if (views.dense->size() != m.cols())
            throw std::invalid_argument("multiply: vector length != matrix columns");
        check(adaspmv_vector_set_dense(ctx.get(), x.h.get(), views.dense->values.data()));
    }
    MultiplyOutput out(ctx);
    const adaspmv_config c = cfg.c();
    check(adaspmv_run(ctx.get(), m.get(), x.h.get(), id.index(), &c, out.get()));
    return out;
}

inline MultiplyOutput spmv(const DualMatrix& m, const DenseVector& x, Workload w, const KernelConfig& cfg = {}) {
    OperandViews v;
    v.dense = &x;
    return run_kernel(m, {Pattern::SpMV, w, Writeback::Atomic}, v, cfg);
}

inline MultiplyOutput spmspv_row(const DualMatrix& m, const DenseVector& x_values, const BitMask& mask,
                                 Workload w, const KernelConfig& cfg = {}) {
    if (mask.length != m.cols()) throw std::invalid_argument("spmspv_row: mask length != matrix columns");
    OperandViews v;
    v.dense = &x_values;
    v.mask = &mask;
    return run_kernel(m, {Pattern::RowSpMSpV, w, Writeback::Atomic}, v, cfg);
}

inline MultiplyOutput spmspv_col(const DualMatrix& m, const SparseVector& x, Workload w, Writeback wb,
                                 const KernelConfig& cfg = {}) {
    OperandViews v;
    v.sparse = &x;
    return run_kernel(m, {Pattern::ColSpMSpV, w, wb}, v, cfg);
}

// ---- selector hook ------------------------------------------------
class SelectorBundle {
public:
    static SelectorBundle load(const std::string& path) {
        adaspmv_bundle* b = nullptr;
        check(adaspmv_bundle_load(path.c_str(), &b));
        return SelectorBundle(b);
    }
    adaspmv_bundle* get() const { return h_.get(); }

private:
    explicit SelectorBundle(adaspmv_bundle* b) : h_(b, adaspmv_bundle_destroy) {}
    std::shared_ptr<adaspmv_bundle> h_;
};

inline KernelId predict_kernel(const DualMatrix& m, const SparseVector& x, const SelectorBundle& b) {
    detail::DeviceOperand v(m.context(), m.cols());
    check(adaspmv_vector_set_sparse(m.context().get(), v.h.get(), x.nnz(), x.indices.data(), x.values.data()));
    int k = 0;
    check(adaspmv_select(m.context().get(), m.get(), v.h.get(), b.get(), &k, nullptr, nullptr));
    return KernelId::from_index(k);
}

// ---- batched multiplies from host vectors (adaspmv_run_batch) ------------------------
// One operand of a batch: a DenseVector or a SparseVector (the other empty).
struct BatchOperand {
    const DenseVector* dense = nullptr;
    const SparseVector* sparse = nullptr;
};

// Result of one batched multiply: the dense or the sparse form of y
// (MultiplyOutput::dense()/sparse(), kernels.hpp:136-144) and the kernel run.
struct BatchResult {
    KernelId kernel;
    bool is_sparse = false;
    DenseVector dense;
    SparseVector sparse;
};

// y_k = A x_k for every operand, selected by `b` (or `forced_kernel` >= 0),
// pipelined over `lanes` streams; `form` = ADASPMV_RESULT_DENSE / SPARSE / AUTO.
inline std::vector<BatchResult> run_batch(const DualMatrix& m, const std::vector<BatchOperand>& xs,
                                          const SelectorBundle* b, int forced_kernel = -1,
                                          int form = ADASPMV_RESULT_AUTO, const KernelConfig& cfg = {},
                                          int lanes = 0) {
    const size_t n = xs.size();
    std::vector<adaspmv_host_operand> ops(n);
    std::vector<adaspmv_host_result> res(n);
    std::vector<BatchResult> out(n);
    const index_t rows = m.rows();
    for (size_t k = 0; k < n; ++k) {
        if (xs[k].sparse) {
            if (xs[k].sparse->length != m.cols()) throw std::invalid_argument("run_batch: vector length != matrix columns");
            ops[k] = {xs[k].sparse->nnz(), xs[k].sparse->indices.data(), xs[k].sparse->values.data()};
        } else if (xs[k].dense) {
            if (xs[k].dense->size() != m.cols()) throw std::invalid_argument("run_batch: vector length != matrix columns");
            ops[k] = {-1, nullptr, xs[k].dense->values.data()};
        } else {
            throw std::invalid_argument("run_batch: empty operand");
        }
        // buffers for either form (AUTO decides on the device side)
        out[k].dense.values.resize(static_cast<size_t>(rows));
        res[k].form = form;
        res[k].values = out[k].dense.values.data();
        if (form != ADASPMV_RESULT_DENSE) {
            out[k].sparse.length = rows;
            out[k].sparse.indices.resize(static_cast<size_t>(rows));
            out[k].sparse.values.resize(static_cast<size_t>(rows));
            res[k].capacity = rows;
            res[k].indices = out[k].sparse.indices.data();
            if (form == ADASPMV_RESULT_SPARSE) res[k].values = out[k].sparse.values.data();
        }
    }
    const adaspmv_config c = cfg.c();
    check(adaspmv_run_batch(m.context().get(), m.get(), b ? b->get() : nullptr, forced_kernel, &c,
                            static_cast<int64_t>(n), ops.data(), res.data(), lanes));
    for (size_t k = 0; k < n; ++k) {
        out[k].kernel = KernelId::from_index(res[k].kernel);
        out[k].is_sparse = res[k].form == ADASPMV_RESULT_SPARSE;
        if (out[k].is_sparse) {
            const size_t nz = static_cast<size_t>(res[k].nnz_y);
            if (form == ADASPMV_RESULT_AUTO)  // values landed in the dense buffer
                out[k].sparse.values.assign(out[k].dense.values.begin(), out[k].dense.values.begin() + nz);
            out[k].sparse.indices.resize(nz);
            out[k].sparse.values.resize(nz);
            out[k].dense.values.clear();
        } else {
            out[k].sparse = SparseVector{};
        }
    }
    return out;
}

// ---- row-partitioned mode in one process (adaspmv_multi_*) ------------------------------
class MultiMatrix {
public:
    // rows of the host CSR cut into devices.size() blocks of ~nnz/G nonzeros
    MultiMatrix(const std::vector<int>& devices, index_t rows, index_t cols, const std::vector<index_t>& row_offsets,
                const std::vector<index_t>& col_indices, const std::vector<real_t>& values)
        : rows_(rows), g_(static_cast<int>(devices.size())) {
        adaspmv_multi* h = nullptr;
        check(adaspmv_multi_create(g_, devices.data(), rows, cols, row_offsets.data(), col_indices.data(),
                                   values.empty() ? nullptr : values.data(), kDtype, &h));
        h_.reset(h, adaspmv_multi_destroy);
    }
    // y = A x (dense x); the per-block kernel choices go to `kernels` if given
    DenseVector multiply(const DenseVector& x, const SelectorBundle* b, int forced_kernel = -1,
                         std::vector<int>* kernels = nullptr) const {
        DenseVector y(rows_);
        std::vector<int> ks(static_cast<size_t>(g_));
        check(adaspmv_multi_run(h_.get(), b ? b->get() : nullptr, forced_kernel, nullptr, -1, nullptr,
                                x.values.data(), y.values.data(), ks.data()));
        if (kernels) *kernels = ks;
        return y;
    }
    DenseVector multiply(const SparseVector& x, const SelectorBundle* b, int forced_kernel = -1,
                         std::vector<int>* kernels = nullptr) const {
        DenseVector y(rows_);
        std::vector<int> ks(static_cast<size_t>(g_));
        check(adaspmv_multi_run(h_.get(), b ? b->get() : nullptr, forced_kernel, nullptr, x.nnz(), x.indices.data(),
                                x.values.data(), y.values.data(), ks.data()));
        if (kernels) *kernels = ks;
        return y;
    }

private:
    index_t rows_;
    int g_;
    std::shared_ptr<adaspmv_multi> h_;
};

// ---- BFS driver --------------------------------------------------------
inline std::vector<index_t> bfs(const DualMatrix& m, index_t source, int semiring = ADASPMV_OR_AND,
                                const SelectorBundle* b = nullptr, int forced_kernel = -1) {
    std::vector<index_t> levels(static_cast<size_t>(m.rows()));
    int64_t n_levels = 0;
    check(adaspmv_bfs(m.context().get(), m.get(), source, semiring, b ? b->get() : nullptr, forced_kernel,
                      levels.data(), &n_levels, nullptr, 0));
    return levels;
}

// ---- incremental PageRank -------------------------------------------------
inline std::vector<double> pagerank_incremental(const DualMatrix& m, double damping = 0.85,
                                                double prune = 1e-6, int64_t max_iters = 300,
                                                const SelectorBundle* b = nullptr, int forced_kernel = -1,
                                                int64_t* n_iters = nullptr) {
    std::vector<double> rank(static_cast<size_t>(m.rows()));
    int64_t it = 0;
    check(adaspmv_pagerank(m.context().get(), m.get(), damping, prune, max_iters, b ? b->get() : nullptr,
                           forced_kernel, rank.data(), &it, nullptr, 0));
    if (n_iters) *n_iters = it;
    return rank;
}

}  // namespace adaspmv::cuda

// batch.cpp -- adaspmv_run_batch: many independent multiplies y_k = A x_k
// from host buffers, pipelined over several streams of one device.
//
// Each x_k goes through exactly the single-vector path of the C-ABI
// (vector_set_* -> predict_kernel or a forced KernelId ->
// run_kernel (kernels.hpp:520-535) -> MultiplyOutput::dense()/sparse()
// (kernels.hpp:136-144)); what the batch adds is concurrency.  A lane is one
// host thread driving its own stream, operand and output.  A lane blocks on
// its own stream only (operand validation verdict, nnz_s for the selector,
// nnz_y of a sparse result, the final copy), so while one lane copies x_k in
// over PCIe another multiplies and a third copies its y out: the host<->device
// copies of a serving loop overlap each other and the kernels.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <mutex>
#include <thread>
#include <vector>

#include "internal.hpp"

namespace ada {

BatchLane::~BatchLane() {
    cudaSetDevice(c.device);
    g_alloc_stream = c.stream;
    v.dense.release();
    v.sp_idx.release();
    v.sp_val.release();
    v.mask.release();
    v.eff.release();
    v.stage_idx.release();
    y.dense.release();
    y.sp_idx.release();
    y.sp_val.release();
    y.d_nnz.release();
    context_release(c);
}

namespace {

void set_operand(Context& c, Vector& v, const adaspmv_host_operand& x) {
    if (x.nnz < 0) {  // DenseVector: n values (adaspmv_vector_set_dense)
        if (v.n > 0 && !x.values) invalid("run_batch: dense operand without values");
        v.invalidate();
        const size_t bytes = static_cast<size_t>(value_bytes(v.dtype)) * static_cast<size_t>(v.n);
        v.dense.ensure(std::max<size_t>(bytes, 1));
        if (bytes) ADA_CUDA(cudaMemcpyAsync(v.dense.p, x.values, bytes, cudaMemcpyHostToDevice, c.stream));
        v.has_dense = true;
    } else {
        if (x.nnz > 0 && (!x.indices || !x.values)) invalid("run_batch: sparse operand without indices/values");
        vector_set_sparse_host_deferred(c, v, x.nnz, x.indices, x.values);
    }
}

// Writes y to r in the requested (or the smaller) form.
void fetch_result(Context& c, const Matrix& m, Vector& v, Output& y, int kernel, adaspmv_host_result& r) {
    const int64_t vb = m.vbytes();
    bool sparse = r.form == ADASPMV_RESULT_SPARSE;
    if (r.form == ADASPMV_RESULT_AUTO) {
        // sparse costs 8 + V bytes per entry, dense V per row
        int64_t bound = -1;  // an upper bound of nnz_y
        if (kernel == 5 || kernel == 7) bound = output_nnz(c, y);
        else if (kernel >= 4) {  // nnz_s bounds nnz_y; the degree profile's bound first (no device trip)
            const int64_t ub = v.nnz >= 0 ? m.nnz_s_upper(v.nnz) : -1;
            if (v.nnz_s >= 0 && v.nnz_s_matrix == m.id) bound = v.nnz_s;
            else if (ub >= 0 && ub * (8 + vb) < m.rows * vb && ub <= r.capacity) bound = ub;
            else bound = vector_nnz_s(c, v, m);
        }
        else if (v.nnz_s >= 0 && v.nnz_s_matrix == m.id) bound = v.nnz_s;
        sparse = r.indices && bound >= 0 && bound * (8 + vb) < m.rows * vb && bound <= r.capacity;
        if (sparse && !(kernel == 5 || kernel == 7)) {
            const int64_t nnz = output_nnz(c, y);  // compaction of the dense result
            sparse = nnz <= r.capacity;
        }
    }
    if (sparse) {
        const int64_t nnz = output_nnz(c, y);
        const int64_t n = std::min(r.capacity, nnz);
        if (n > 0) {
            if (!r.values) invalid("run_batch: sparse result without a values buffer");
            if (r.indices) {  // int64 index_t, widened on the device, one copy
                int64_t* d64 = static_cast<int64_t*>(c.scratch[7].ensure(sizeof(int64_t) * static_cast<size_t>(n)));
                widen_indices(c, n, y.sp_idx.as<int32_t>(), d64);
                ADA_CUDA(cudaMemcpyAsync(r.indices, d64, sizeof(int64_t) * static_cast<size_t>(n),
                                         cudaMemcpyDeviceToHost, c.stream));
            }
            ADA_CUDA(cudaMemcpyAsync(r.values, y.sp_val.p, static_cast<size_t>(vb * n), cudaMemcpyDeviceToHost,
                                     c.stream));
        }
        r.form = ADASPMV_RESULT_SPARSE;
        r.nnz_y = nnz;
    } else {
        output_ensure_dense(c, y);
        if (m.rows > 0) {
            if (!r.values) invalid("run_batch: dense result without a values buffer");
            ADA_CUDA(cudaMemcpyAsync(r.values, y.dense.p, static_cast<size_t>(vb * m.rows), cudaMemcpyDeviceToHost,
                                     c.stream));
        }
        r.form = ADASPMV_RESULT_DENSE;
        r.nnz_y = -1;
    }
    r.kernel = kernel;
    c.sync();
}

}  // namespace

void run_batch(Context& ctx, const Matrix& m, const Bundle* b, int forced, const adaspmv_config& cfg,
               int64_t count, const adaspmv_host_operand* xs, adaspmv_host_result* ys, int lanes) {
    if (count == 0) return;
    for (int64_t k = 0; k < count; ++k)
        if (ys[k].form < ADASPMV_RESULT_DENSE || ys[k].form > ADASPMV_RESULT_AUTO)
            invalid("run_batch: unknown result form");
    const int L = static_cast<int>(std::min<int64_t>(lanes, count));
    // work already queued on the caller's stream (e.g. the matrix build)
    // completes before the lanes' streams read the matrix
    ctx.sync();
    while (static_cast<int>(ctx.lanes.size()) < L) {
        auto lane = std::make_unique<BatchLane>();
        context_init(lane->c, ctx.device, nullptr);
        ctx.lanes.push_back(std::move(lane));
    }
    for (int i = 0; i < L; ++i) {
        BatchLane& ln = *ctx.lanes[static_cast<size_t>(i)];
        ln.c.sm_count = ctx.sm_count;
        ln.c.timing = false;
        if (ln.v.n != m.cols || ln.v.dtype != m.dtype) {
            ln.v.ctx = &ln.c;
            ln.v.n = m.cols;
            ln.v.dtype = m.dtype;
        }
        ln.v.invalidate();
        ln.y.ctx = &ln.c;
    }
    // ADASPMV_BATCH_TRACE=1: per-operand host timeline on stderr (ms since start)
    const bool trace = std::getenv("ADASPMV_BATCH_TRACE") != nullptr;
    const auto start = std::chrono::steady_clock::now();
    auto now = [&] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - start).count(); };
    // Order: the batch is a two-stage flow shop (host-to-device copy, then
    // multiply + device-to-host copy; the two copy directions run
    // concurrently, each FIFO across streams).  Johnson's rule minimises its
    // makespan: operands whose input is smaller than their result first, by
    // increasing input bytes, then the rest by decreasing result bytes.
    // Results are written by index, so the order is not observable.
    const double vb = m.vbytes();
    const double avg_col = m.cols > 0 ? static_cast<double>(m.nnz) / static_cast<double>(m.cols) : 0.0;
    std::vector<int64_t> order(static_cast<size_t>(count));
    std::vector<double> in_b(static_cast<size_t>(count)), out_b(static_cast<size_t>(count));
    for (int64_t k = 0; k < count; ++k) {
        const adaspmv_host_operand& x = xs[k];
        const size_t i = static_cast<size_t>(k);
        order[i] = k;
        const double dense_out = static_cast<double>(m.rows) * vb;
        in_b[i] = x.nnz < 0 ? static_cast<double>(m.cols) * vb : static_cast<double>(x.nnz) * (8 + vb);
        // nnz_y <= nnz_s ~ nnz_x * mean column degree
        const double sp_out = x.nnz < 0 ? dense_out : std::min(static_cast<double>(m.rows), x.nnz * avg_col) * (8 + vb);
        out_b[i] = ys[k].form == ADASPMV_RESULT_DENSE ? dense_out
                   : ys[k].form == ADASPMV_RESULT_SPARSE ? sp_out : std::min(sp_out, dense_out);
    }
    // Operands whose copies are small (< 2 MB both ways) are cheap for the
    // copy engines but still hold a lane for a few synchronisations: they go
    // after the large ones so the large transfers start at once.
    constexpr double kSmall = 2.0 * (1 << 20);
    std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
        const size_t i = static_cast<size_t>(a), j = static_cast<size_t>(b);
        const bool sa = in_b[i] + out_b[i] < kSmall, sb = in_b[j] + out_b[j] < kSmall;
        if (sa != sb) return sb;
        const bool fa = in_b[i] < out_b[i], fb = in_b[j] < out_b[j];
        if (fa != fb) return fa;
        // ties (equal keys) go to the operand that frees the other copy
        // direction sooner: the smaller input in the second group, the
        // larger result in the first
        if (fa) return in_b[i] != in_b[j] ? in_b[i] < in_b[j] : out_b[i] > out_b[j];
        return out_b[i] != out_b[j] ? out_b[i] > out_b[j] : in_b[i] < in_b[j];
    });
    std::atomic<int64_t> next{0};
    std::atomic<bool> stop{false};
    std::mutex err_mu;
    std::exception_ptr first;
    int64_t first_k = -1;
    auto worker = [&](int li) {
        BatchLane& ln = *ctx.lanes[static_cast<size_t>(li)];
        try {
            ADA_CUDA(cudaSetDevice(ln.c.device));
            g_alloc_stream = ln.c.stream;
            for (;;) {
                if (stop.load(std::memory_order_relaxed)) return;
                const int64_t j = next.fetch_add(1);
                if (j >= count) return;
                const int64_t k = order[static_cast<size_t>(j)];
                try {
                    const double t0 = trace ? now() : 0;
                    set_operand(ln.c, ln.v, xs[k]);
                    const double t1 = trace ? now() : 0;
                    const int kern = forced >= 0 ? forced : predict(ln.c, m, ln.v, *b, nullptr, nullptr);
                    // the operand's validation verdict (usually already here:
                    // the selector's nnz_s read synchronised the stream)
                    if (xs[k].nnz >= 0) vector_check_deferred(ln.c, ln.v);
                    const double t2 = trace ? now() : 0;
                    run_kernel(ln.c, m, ln.v, kern, cfg, ln.y);
                    fetch_result(ln.c, m, ln.v, ln.y, kern, ys[k]);
                    if (trace)
                        std::fprintf(stderr, "run_batch lane %d op %lld kernel %d: set %.3f-%.3f select -%.3f "
                                     "run+fetch -%.3f ms\n", li, static_cast<long long>(k), kern, t0, t1, t2, now());
                } catch (...) {
                    std::lock_guard<std::mutex> g(err_mu);
                    if (!first || k < first_k) {
                        first = std::current_exception();
                        first_k = k;
                    }
                    stop = true;
                    cudaStreamSynchronize(ln.c.stream);
                    return;
                }
            }
        } catch (...) {
            std::lock_guard<std::mutex> g(err_mu);
            if (!first) first = std::current_exception();
            stop = true;
        }
    };
    const int64_t l0 = [&] {
        int64_t s = 0;
        for (int i = 0; i < L; ++i) s += ctx.lanes[static_cast<size_t>(i)]->c.launches;
        return s;
    }();
    std::vector<std::thread> th;
    th.reserve(static_cast<size_t>(L - 1));
    for (int i = 1; i < L; ++i) th.emplace_back(worker, i);
    worker(0);
    for (auto& t : th) t.join();
    // the caller's thread keeps the caller's allocation stream
    g_alloc_stream = ctx.stream;
    ADA_CUDA(cudaSetDevice(ctx.device));
    int64_t l1 = 0;
    for (int i = 0; i < L; ++i) l1 += ctx.lanes[static_cast<size_t>(i)]->c.launches;
    ctx.launches += l1 - l0;
    if (first) {
        try {
            std::rethrow_exception(first);
        } catch (const Error& e) {
            throw Error(e.code, "run_batch: operand " + std::to_string(first_k) + ": " + e.what());
        }
    }
}

}  // namespace ada

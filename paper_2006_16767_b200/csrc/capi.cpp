// capi.cpp -- the extern "C" boundary (include/adaspmv_cuda.h).  Every entry
// point catches exceptions and returns an adaspmv_status; the message of the
// last failure is kept per thread (adaspmv_last_error).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/adaspmv_cuda.h"
#include "internal.hpp"

namespace ada {
void validate_bundle(const Bundle& b);
}

struct adaspmv_ctx : ada::Context {};
struct adaspmv_matrix : ada::Matrix {};
struct adaspmv_vector : ada::Vector {};
struct adaspmv_output : ada::Output {};
struct adaspmv_bundle : ada::Bundle {};
struct adaspmv_multi : ada::Multi {};
struct adaspmv_dist : ada::Dist {};

namespace {

thread_local std::string g_error;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return ADASPMV_OK;
    } catch (const ada::Error& e) {
        g_error = e.what();
        return e.code;
    } catch (const std::bad_alloc& e) {
        g_error = "host allocation failed";
        return ADASPMV_ERR_NOMEM;
    } catch (const std::exception& e) {
        g_error = e.what();
        return ADASPMV_ERR_INTERNAL;
    } catch (...) {
        g_error = "unknown error";
        return ADASPMV_ERR_INTERNAL;
    }
}

void need(const void* p, const char* what) {
    if (!p) ada::invalid(std::string(what) + " is NULL");
}

void bind(ada::Context* ctx) {
    need(ctx, "context");
    ADA_CUDA(cudaSetDevice(ctx->device));
    ada::g_alloc_stream = ctx->stream;
}

// Objects are freed on the stream of the context that made them.
void bind_quiet(ada::Context* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    ada::g_alloc_stream = ctx->stream;
}

// Blocking copy ordered on the context stream (device memory is allocated
// stream-ordered on it, see DevBuf).
cudaError_t copy_sync(ada::Context& c, void* dst, const void* src, size_t bytes, cudaMemcpyKind kind) {
    cudaError_t e = cudaMemcpyAsync(dst, src, bytes, kind, c.stream);
    return e != cudaSuccess ? e : cudaStreamSynchronize(c.stream);
}
cudaError_t copy_sync(ada::Context* c, void* dst, const void* src, size_t bytes, cudaMemcpyKind kind) {
    return copy_sync(*c, dst, src, bytes, kind);
}

void check_dtype(int dtype) {
    if (dtype != ADASPMV_F64 && dtype != ADASPMV_F32) ada::invalid("unknown dtype");
}

// CsrMatrix::validate (sparse.hpp:44-63) on borrowed host arrays.
void validate_host_csr(int64_t rows, int64_t cols, const int64_t* ro, const int64_t* ci) {
    if (rows < 0 || cols < 0) ada::invalid("negative matrix dimension");
    if (ro[0] != 0) ada::invalid("csr: row_offsets[0] != 0");
    for (int64_t r = 0; r < rows; ++r) {
        if (ro[r + 1] < ro[r]) ada::invalid("csr: row_offsets not nondecreasing");
        for (int64_t k = ro[r]; k < ro[r + 1]; ++k) {
            if (ci[k] < 0 || ci[k] >= cols) ada::invalid("csr: column index out of range");
            if (k > ro[r] && ci[k] <= ci[k - 1])
                ada::invalid("csr: columns not strictly increasing in row " + std::to_string(r));
        }
    }
}

ada::Matrix* upload_host_csr(ada::Context& ctx, int64_t rows, int64_t cols, const int64_t* ro,
                             const int64_t* ci, const void* vals, int dtype) {
    const int64_t nnz = ro[rows];
    std::vector<int32_t> ci32(static_cast<size_t>(nnz));
    for (int64_t k = 0; k < nnz; ++k) ci32[static_cast<size_t>(k)] = static_cast<int32_t>(ci[k]);
    ada::DevBuf d_ro, d_ci, d_v;
    const size_t vb = static_cast<size_t>(ada::value_bytes(dtype));
    d_ro.ensure(sizeof(int64_t) * static_cast<size_t>(rows + 1));
    d_ci.ensure(sizeof(int32_t) * static_cast<size_t>(std::max<int64_t>(nnz, 1)));
    d_v.ensure(vb * static_cast<size_t>(std::max<int64_t>(nnz, 1)));
    ADA_CUDA(copy_sync(ctx, d_ro.p, ro, sizeof(int64_t) * static_cast<size_t>(rows + 1), cudaMemcpyHostToDevice));
    if (nnz > 0) {
        ADA_CUDA(copy_sync(ctx, d_ci.p, ci32.data(), sizeof(int32_t) * ci32.size(), cudaMemcpyHostToDevice));
        if (vals) ADA_CUDA(copy_sync(ctx, d_v.p, vals, vb * static_cast<size_t>(nnz), cudaMemcpyHostToDevice));
    }
    return ada::matrix_create_device(ctx, rows, cols, nnz, d_ro.as<int64_t>(), d_ci.as<int32_t>(),
                                     vals ? d_v.p : nullptr, dtype, vals == nullptr);
}

template <class T>
void to_host_vals(const std::vector<double>& src, void* dst) {
    T* d = static_cast<T*>(dst);
    for (size_t i = 0; i < src.size(); ++i) d[i] = static_cast<T>(src[i]);
}

}  // namespace

namespace ada {

void* Context::stage(size_t bytes) {
    if (bytes > h_stage_cap) {
        ADA_CUDA(cudaStreamSynchronize(stream));
        if (h_stage) cudaFreeHost(h_stage);
        h_stage = nullptr;
        h_stage_cap = 0;
        ADA_CUDA(cudaHostAlloc(&h_stage, bytes, cudaHostAllocDefault));
        h_stage_cap = bytes;
    }
    return h_stage;
}

void context_init(Context& ctx, int device, cudaStream_t stream) {
    ctx.device = device;
    ADA_CUDA(cudaSetDevice(device));
    ADA_CUDA(cudaFree(nullptr));
    if (stream) {
        ctx.stream = stream;
    } else {
        ADA_CUDA(cudaStreamCreateWithFlags(&ctx.stream, cudaStreamNonBlocking));
        ctx.own_stream = true;
    }
    ADA_CUDA(cudaDeviceGetAttribute(&ctx.sm_count, cudaDevAttrMultiProcessorCount, device));
    ADA_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&ctx.h_scalars), 64 * sizeof(int64_t), cudaHostAllocMapped));
    ADA_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&ctx.h_scalars_dev), ctx.h_scalars, 0));
    // keep freed blocks in the device's default pool instead of returning
    // them to the driver at every synchronisation
    cudaMemPool_t pool;
    ADA_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t threshold = UINT64_MAX;
    ADA_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold));
    g_alloc_stream = ctx.stream;
    ctx.d_scalars.ensure(64 * sizeof(int64_t));
    // slots 10-12 are the accumulators of the one-launch reductions
    // (vector.cu: reduce2_to_host), which expect them zero between calls
    ADA_CUDA(cudaMemsetAsync(ctx.d_scalars.p, 0, 64 * sizeof(int64_t), ctx.stream));
}

void context_release(Context& ctx) {
    ctx.lanes.clear();
    cudaSetDevice(ctx.device);
    g_alloc_stream = ctx.stream;
    cudaStreamSynchronize(ctx.stream);
    for (auto& b : ctx.scratch) b.release();
    ctx.d_scalars.release();
    ctx.lb_partials.release();
    if (ctx.h_scalars) cudaFreeHost(ctx.h_scalars);
    if (ctx.h_stage) cudaFreeHost(ctx.h_stage);
    ctx.h_scalars = nullptr;
    ctx.h_stage = nullptr;
    if (ctx.own_stream) {
        cudaStreamSynchronize(ctx.stream);  // the releases above are ordered on it
        cudaStreamDestroy(ctx.stream);
    }
    ctx.stream = nullptr;
    ctx.own_stream = false;
}

void Context::fetch_scalars(const int64_t* d, int n) {
    copy_scalars_kernel_launch(*this, d, h_scalars_dev, n);
    ADA_CUDA(cudaStreamSynchronize(stream));
}

int64_t Context::fetch_scalar(const int64_t* d) {
    fetch_scalars(d, 1);
    return h_scalars[0];
}

}  // namespace ada

extern "C" {

const char* adaspmv_version(void) { return "adaspmv-b200 0.1 (sm_100a)"; }
const char* adaspmv_last_error(void) { return g_error.c_str(); }

int adaspmv_ctx_create(int device, void* stream, adaspmv_ctx** out) {
    return guarded([&] {
        need(out, "out");
        auto ctx = std::make_unique<adaspmv_ctx>();
        ada::context_init(*ctx, device, static_cast<cudaStream_t>(stream));
        *out = ctx.release();
    });
}

int adaspmv_ctx_destroy(adaspmv_ctx* ctx) {
    if (!ctx) return ADASPMV_OK;
    return guarded([&] {
        ada::context_release(*ctx);
        delete ctx;
    });
}

int adaspmv_ctx_synchronize(adaspmv_ctx* ctx) {
    return guarded([&] {
        bind(ctx);
        ctx->sync();
    });
}

void* adaspmv_ctx_stream(adaspmv_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

int64_t adaspmv_ctx_launch_count(adaspmv_ctx* ctx) { return ctx ? ctx->launches : 0; }

int adaspmv_ctx_set_timing(adaspmv_ctx* ctx, int enable) {
    return guarded([&] {
        need(ctx, "context");
        ctx->timing = enable != 0;
    });
}

int adaspmv_ctx_set_bfs_loop(adaspmv_ctx* ctx, int host_loop) {
    return guarded([&] {
        need(ctx, "context");
        ctx->bfs_host_loop = host_loop != 0;
    });
}

int adaspmv_ctx_set_counters(adaspmv_ctx* ctx, int enable) {
    return guarded([&] {
        need(ctx, "context");
        ctx->counters = enable != 0;
    });
}

int adaspmv_output_counters(adaspmv_ctx* ctx, adaspmv_output* y, uint64_t out3[3]) {
    return guarded([&] {
        bind(ctx);
        need(y, "output");
        need(out3, "out");
        if (!y->has_ctr) ada::invalid("output_counters: the run was not counted (adaspmv_ctx_set_counters)");
        unsigned long long h[2] = {0, 0};
        ADA_CUDA(copy_sync(ctx, h, y->d_ctr.p, sizeof(h), cudaMemcpyDeviceToHost));
        out3[0] = h[0];
        out3[1] = h[1];
        out3[2] = 0;  // hardware atomics: no counted CAS retries
    });
}

int adaspmv_output_elapsed(adaspmv_ctx* ctx, adaspmv_output* y, double* seconds) {
    return guarded([&] {
        bind(ctx);
        need(y, "output");
        need(seconds, "out");
        if (!y->timed || !y->ev[0] || !y->ev[1]) ada::invalid("output was not produced by a timed run");
        ADA_CUDA(cudaEventSynchronize(y->ev[1]));
        float ms = 0;
        ADA_CUDA(cudaEventElapsedTime(&ms, y->ev[0], y->ev[1]));
        *seconds = static_cast<double>(ms) * 1e-3;
    });
}

// ---- matrices -------------------------------------------------------------------
int adaspmv_matrix_create_csr(adaspmv_ctx* ctx, int64_t rows, int64_t cols,
                              const int64_t* row_offsets, const int64_t* col_indices,
                              const void* values, int dtype, adaspmv_matrix** out) {
    return guarded([&] {
        bind(ctx);
        need(out, "out");
        need(row_offsets, "row_offsets");
        check_dtype(dtype);
        if (rows < 0 || cols < 0) ada::invalid("negative matrix dimension");
        if (row_offsets[rows] > 0) need(col_indices, "col_indices");
        validate_host_csr(rows, cols, row_offsets, col_indices);
        ada::Matrix* m = upload_host_csr(*ctx, rows, cols, row_offsets, col_indices, values, dtype);
        *out = static_cast<adaspmv_matrix*>(m);
    });
}

int adaspmv_matrix_create_csr_device(adaspmv_ctx* ctx, int64_t rows, int64_t cols, int64_t nnz,
                                     const int64_t* d_row_offsets, const int32_t* d_col_indices,
                                     const void* d_values, int dtype, adaspmv_matrix** out) {
    return guarded([&] {
        bind(ctx);
        need(out, "out");
        need(d_row_offsets, "row_offsets");
        check_dtype(dtype);
        if (nnz < 0) ada::invalid("negative nnz");
        ada::validate_device_csr(*ctx, rows, cols, nnz, d_row_offsets, d_col_indices);
        *out = static_cast<adaspmv_matrix*>(ada::matrix_create_device(
            *ctx, rows, cols, nnz, d_row_offsets, d_col_indices, d_values, dtype, d_values == nullptr));
    });
}

static adaspmv_matrix* from_host(ada::Context& ctx, const ada::HostCsr& h, int dtype) {
    const size_t nnz = h.col_indices.size();
    std::vector<unsigned char> vals(nnz * static_cast<size_t>(ada::value_bytes(dtype)));
    if (dtype == ADASPMV_F64) to_host_vals<double>(h.values, vals.data());
    else to_host_vals<float>(h.values, vals.data());
    return static_cast<adaspmv_matrix*>(upload_host_csr(ctx, h.rows, h.cols, h.row_offsets.data(),
                                                        h.col_indices.data(), vals.data(), dtype));
}

int adaspmv_matrix_from_triplets(adaspmv_ctx* ctx, int64_t rows, int64_t cols, int64_t count,
                                 const int64_t* t_rows, const int64_t* t_cols,
                                 const void* t_values, int dtype, adaspmv_matrix** out) {
    return guarded([&] {
        bind(ctx);
        need(out, "out");
        check_dtype(dtype);
        if (count < 0) ada::invalid("negative triplet count");
        if (count > 0) {
            need(t_rows, "rows");
            need(t_cols, "cols");
            need(t_values, "values");
        }
        *out = static_cast<adaspmv_matrix*>(
            ada::matrix_from_triplets_device(*ctx, rows, cols, count, t_rows, t_cols, t_values, dtype));
    });
}

int adaspmv_matrix_load(adaspmv_ctx* ctx, const char* path, int dtype, adaspmv_matrix** out) {
    return guarded([&] {
        bind(ctx);
        need(out, "out");
        need(path, "path");
        check_dtype(dtype);
        ada::HostMatrixFile h = ada::load_matrix_file(path, dtype);
        if (h.is_csr) {
            *out = from_host(*ctx, h.csr, dtype);
            return;
        }
        ada::HostTriplets& t = h.trip;
        const int64_t n = static_cast<int64_t>(t.r.size());
        if (dtype == ADASPMV_F64) {
            *out = static_cast<adaspmv_matrix*>(
                ada::matrix_from_triplets_device(*ctx, t.rows, t.cols, n, t.r.data(), t.c.data(), t.v.data(), dtype));
        } else {  // real_t = float: the parsed double narrowed once, as the reference's float build
            std::vector<float> v32(t.v.begin(), t.v.end());
            *out = static_cast<adaspmv_matrix*>(
                ada::matrix_from_triplets_device(*ctx, t.rows, t.cols, n, t.r.data(), t.c.data(), v32.data(), dtype));
        }
    });
}

static void download_csr(ada::Context& ctx, const ada::Matrix& m, std::vector<int64_t>& ro,
                         std::vector<int64_t>& ci, std::vector<double>& vals) {
    ro.resize(static_cast<size_t>(m.rows + 1));
    ci.resize(static_cast<size_t>(m.nnz));
    vals.resize(static_cast<size_t>(m.nnz));
    std::vector<int32_t> c32(static_cast<size_t>(m.nnz));
    std::vector<unsigned char> v(static_cast<size_t>(m.nnz) * static_cast<size_t>(m.vbytes()));
    ADA_CUDA(cudaMemcpyAsync(ro.data(), m.row_off.p, sizeof(int64_t) * ro.size(), cudaMemcpyDeviceToHost, ctx.stream));
    if (m.nnz > 0) {
        ADA_CUDA(cudaMemcpyAsync(c32.data(), m.col_idx.p, sizeof(int32_t) * c32.size(), cudaMemcpyDeviceToHost, ctx.stream));
        ADA_CUDA(cudaMemcpyAsync(v.data(), m.vals.p, v.size(), cudaMemcpyDeviceToHost, ctx.stream));
    }
    ctx.sync();
    for (size_t k = 0; k < c32.size(); ++k) ci[k] = c32[k];
    for (size_t k = 0; k < vals.size(); ++k)
        vals[k] = m.dtype == ADASPMV_F64 ? reinterpret_cast<double*>(v.data())[k]
                                         : reinterpret_cast<float*>(v.data())[k];
}

int adaspmv_matrix_write_matrix_market(adaspmv_ctx* ctx, const adaspmv_matrix* m, const char* path) {
    return guarded([&] {
        bind(ctx);
        need(m, "matrix");
        need(path, "path");
        std::vector<int64_t> ro, ci;
        std::vector<double> vals;
        download_csr(*ctx, *m, ro, ci, vals);
        ada::write_matrix_market_file(path, m->rows, m->cols, ro, ci, vals);
    });
}

int adaspmv_matrix_save_binary(adaspmv_ctx* ctx, const adaspmv_matrix* m, const char* path) {
    return guarded([&] {
        bind(ctx);
        need(m, "matrix");
        need(path, "path");
        std::vector<int64_t> ro, ci;
        std::vector<double> vals;
        download_csr(*ctx, *m, ro, ci, vals);
        std::vector<unsigned char> raw(vals.size() * static_cast<size_t>(m->vbytes()));
        if (m->dtype == ADASPMV_F64) to_host_vals<double>(vals, raw.data());
        else to_host_vals<float>(vals, raw.data());
        ada::save_binary_file(path, m->rows, m->cols, ro, ci, raw.data(), m->dtype);
    });
}

int adaspmv_matrix_transpose(adaspmv_ctx* ctx, const adaspmv_matrix* m, adaspmv_matrix** out) {
    return guarded([&] {
        bind(ctx);
        need(m, "matrix");
        need(out, "out");
        *out = static_cast<adaspmv_matrix*>(ada::matrix_transpose(*ctx, *m));
    });
}

int adaspmv_matrix_destroy(adaspmv_matrix* m) {
    if (!m) return ADASPMV_OK;
    return guarded([&] {
        if (m->ctx) {
            bind_quiet(m->ctx);
            cudaStreamSynchronize(m->ctx->stream);
        }
        delete static_cast<ada::Matrix*>(m);
    });
}

int adaspmv_matrix_dims(const adaspmv_matrix* m, int64_t* rows, int64_t* cols, int64_t* nnz, int* dtype) {
    return guarded([&] {
        need(m, "matrix");
        if (rows) *rows = m->rows;
        if (cols) *cols = m->cols;
        if (nnz) *nnz = m->nnz;
        if (dtype) *dtype = m->dtype;
    });
}

int adaspmv_matrix_download(adaspmv_ctx* ctx, const adaspmv_matrix* m, int64_t* row_offsets,
                            int64_t* col_indices, void* values, int64_t* col_offsets,
                            int64_t* row_indices, void* csc_values) {
    return guarded([&] {
        bind(ctx);
        need(m, "matrix");
        const size_t z = static_cast<size_t>(m->nnz);
        const size_t vb = static_cast<size_t>(m->vbytes());
        std::vector<int32_t> tmp(z);
        if (row_offsets)
            ADA_CUDA(copy_sync(ctx, row_offsets, m->row_off.p, sizeof(int64_t) * static_cast<size_t>(m->rows + 1), cudaMemcpyDeviceToHost));
        if (col_offsets)
            ADA_CUDA(copy_sync(ctx, col_offsets, m->col_off.p, sizeof(int64_t) * static_cast<size_t>(m->cols + 1), cudaMemcpyDeviceToHost));
        if (z == 0) return;
        if (col_indices) {
            ADA_CUDA(copy_sync(ctx, tmp.data(), m->col_idx.p, sizeof(int32_t) * z, cudaMemcpyDeviceToHost));
            for (size_t k = 0; k < z; ++k) col_indices[k] = tmp[k];
        }
        if (row_indices) {
            ADA_CUDA(copy_sync(ctx, tmp.data(), m->row_idx.p, sizeof(int32_t) * z, cudaMemcpyDeviceToHost));
            for (size_t k = 0; k < z; ++k) row_indices[k] = tmp[k];
        }
        if (values) ADA_CUDA(copy_sync(ctx, values, m->vals.p, vb * z, cudaMemcpyDeviceToHost));
        if (csc_values) ADA_CUDA(copy_sync(ctx, csc_values, m->cvals.p, vb * z, cudaMemcpyDeviceToHost));
    });
}

int adaspmv_matrix_features(const adaspmv_matrix* m, double out9[9]) {
    return guarded([&] {
        need(m, "matrix");
        need(out9, "out");
        std::copy(m->feat, m->feat + 9, out9);
    });
}

int adaspmv_matrix_gather_spread(const adaspmv_matrix* m, double* out) {
    return guarded([&] {
        need(m, "matrix");
        need(out, "out");
        *out = m->gather_spread;
    });
}

// ---- vectors ----------------------------------------------------------------------
int adaspmv_vector_create(adaspmv_ctx* ctx, int64_t length, int dtype, adaspmv_vector** out) {
    return guarded([&] {
        bind(ctx);
        need(out, "out");
        check_dtype(dtype);
        if (length < 0) ada::invalid("negative vector length");
        if (length >= (int64_t(1) << 31)) ada::invalid("vector length exceeds the device index range");
        auto* v = new adaspmv_vector();
        v->ctx = ctx;
        v->n = length;
        v->dtype = dtype;
        *out = v;
    });
}

int adaspmv_vector_destroy(adaspmv_vector* v) {
    if (!v) return ADASPMV_OK;
    return guarded([&] {
        if (v->ctx) {
            bind_quiet(v->ctx);
            cudaStreamSynchronize(v->ctx->stream);
        }
        delete v;
    });
}

int adaspmv_vector_set_sparse(adaspmv_ctx* ctx, adaspmv_vector* v, int64_t nnz,
                              const int64_t* indices, const void* values) {
    return guarded([&] {
        bind(ctx);
        need(v, "vector");
        if (nnz < 0) ada::invalid("sparse vector: negative nnz");
        if (nnz > 0) {
            need(indices, "indices");
            need(values, "values");
        }
        ada::vector_set_sparse_host(*ctx, *v, nnz, indices, values);
    });
}

int adaspmv_vector_set_dense(adaspmv_ctx* ctx, adaspmv_vector* v, const void* values) {
    return guarded([&] {
        bind(ctx);
        need(v, "vector");
        if (v->n > 0) need(values, "values");
        v->invalidate();
        const size_t bytes = static_cast<size_t>(ada::value_bytes(v->dtype)) * static_cast<size_t>(v->n);
        v->dense.ensure(std::max<size_t>(bytes, 1));
        if (bytes) ADA_CUDA(cudaMemcpyAsync(v->dense.p, values, bytes, cudaMemcpyHostToDevice, ctx->stream));
        v->has_dense = true;
    });
}

int adaspmv_vector_set_sparse_device(adaspmv_ctx* ctx, adaspmv_vector* v, int64_t nnz,
                                     const int32_t* d_indices, const void* d_values) {
    return guarded([&] {
        bind(ctx);
        need(v, "vector");
        ada::vector_set_sparse_device(*ctx, *v, nnz, d_indices, d_values, true);
    });
}

int adaspmv_vector_set_dense_device(adaspmv_ctx* ctx, adaspmv_vector* v, const void* d_values) {
    return guarded([&] {
        bind(ctx);
        need(v, "vector");
        ada::vector_set_dense_device(*ctx, *v, d_values);
    });
}

int adaspmv_vector_set_output(adaspmv_ctx* ctx, adaspmv_vector* v, adaspmv_output* y) {
    return guarded([&] {
        bind(ctx);
        need(v, "vector");
        need(y, "output");
        if (y->n != v->n) ada::invalid("output length != vector length");
        if (y->dtype != v->dtype) ada::invalid("output dtype != vector dtype");
        if (y->has_sparse) {
            const int64_t nnz = ada::output_nnz(*ctx, *y);
            ada::vector_set_sparse_device(*ctx, *v, nnz, y->sp_idx.as<int32_t>(), y->sp_val.p);
        } else {
            ada::output_ensure_dense(*ctx, *y);
            ada::vector_set_dense_device(*ctx, *v, y->dense.p);
        }
    });
}

int adaspmv_vector_prepare(adaspmv_ctx* ctx, adaspmv_vector* v, int kernel_index) {
    return guarded([&] {
        bind(ctx);
        need(v, "vector");
        if (kernel_index < 0 || kernel_index > 7) ada::invalid("kernel index out of range");
        if (kernel_index <= 3) {
            ada::vector_ensure_dense(*ctx, *v);
            if (kernel_index >= 2) ada::vector_ensure_mask(*ctx, *v);
        } else {
            ada::vector_ensure_sparse(*ctx, *v);
        }
    });
}

int adaspmv_vector_nnz(adaspmv_ctx* ctx, adaspmv_vector* v, int64_t* nnz) {
    return guarded([&] {
        bind(ctx);
        need(v, "vector");
        need(nnz, "out");
        *nnz = ada::vector_nnz(*ctx, *v);
    });
}

int adaspmv_vector_get_sparse(adaspmv_ctx* ctx, adaspmv_vector* v, int64_t capacity,
                              int64_t* indices, void* values, int64_t* nnz) {
    return guarded([&] {
        bind(ctx);
        need(v, "vector");
        ada::vector_ensure_sparse(*ctx, *v);
        ctx->sync();
        if (nnz) *nnz = v->nnz;
        const int64_t n = std::min(capacity, v->nnz);
        if (n <= 0) return;
        if (indices) {
            ada::DevBuf& w = ctx->scratch[7];
            int64_t* d64 = static_cast<int64_t*>(w.ensure(sizeof(int64_t) * static_cast<size_t>(n)));
            ada::widen_indices(*ctx, n, v->sp_idx.as<int32_t>(), d64);
            ADA_CUDA(copy_sync(ctx, indices, d64, sizeof(int64_t) * static_cast<size_t>(n), cudaMemcpyDeviceToHost));
        }
        if (values)
            ADA_CUDA(copy_sync(ctx, values, v->sp_val.p, static_cast<size_t>(ada::value_bytes(v->dtype)) * static_cast<size_t>(n),
                                cudaMemcpyDeviceToHost));
    });
}

int adaspmv_vector_get_dense(adaspmv_ctx* ctx, adaspmv_vector* v, void* values) {
    return guarded([&] {
        bind(ctx);
        need(v, "vector");
        ada::vector_ensure_dense(*ctx, *v);
        ctx->sync();
        if (values && v->n > 0)
            ADA_CUDA(copy_sync(ctx, values, v->dense.p, static_cast<size_t>(ada::value_bytes(v->dtype)) * static_cast<size_t>(v->n),
                                cudaMemcpyDeviceToHost));
    });
}

int adaspmv_vector_get_bitmask(adaspmv_ctx* ctx, adaspmv_vector* v, uint64_t* words) {
    return guarded([&] {
        bind(ctx);
        need(v, "vector");
        ada::vector_ensure_mask(*ctx, *v);
        ctx->sync();
        const size_t nw = static_cast<size_t>((v->n + 63) / 64);
        if (words && nw) ADA_CUDA(copy_sync(ctx, words, v->mask.p, sizeof(uint64_t) * nw, cudaMemcpyDeviceToHost));
    });
}

int adaspmv_effective_nnz(adaspmv_ctx* ctx, const adaspmv_matrix* m, adaspmv_vector* v, int64_t* out) {
    return guarded([&] {
        bind(ctx);
        need(m, "matrix");
        need(v, "vector");
        need(out, "out");
        if (v->n != m->cols) ada::invalid("effective_nnz: vector length != matrix columns");
        *out = ada::vector_nnz_s(*ctx, *v, *m);
    });
}

// ---- features / selector -----------------------------------------------------
int adaspmv_features(adaspmv_ctx* ctx, const adaspmv_matrix* m, adaspmv_vector* v, uint32_t mask,
                     double out13[13]) {
    return guarded([&] {
        bind(ctx);
        need(m, "matrix");
        need(out13, "out");
        if (mask >> 9) {
            need(v, "vector");
            if (v->n != m->cols) ada::invalid("features: vector length != matrix columns");
        }
        ada::features(*ctx, *m, *v, mask, out13);
    });
}

int adaspmv_bundle_load(const char* path, adaspmv_bundle** out) {
    return guarded([&] {
        need(path, "path");
        need(out, "out");
        std::unique_ptr<ada::Bundle> b(ada::bundle_load(path));
        auto* r = new adaspmv_bundle();
        static_cast<ada::Bundle&>(*r) = std::move(*b);
        *out = r;
    });
}

int adaspmv_bundle_create(const int32_t n_nodes[3], const int32_t* const feature[3],
                          const double* const threshold[3], const int32_t* const left[3],
                          const int32_t* const right[3], const int32_t* const leaf[3],
                          adaspmv_bundle** out) {
    return guarded([&] {
        need(out, "out");
        auto b = std::make_unique<adaspmv_bundle>();
        static const uint32_t masks[3] = {0x1fffu, 0x1ffu, (1u << 0) | (1u << 1) | (1u << 2) | (1u << 9) |
                                                               (1u << 10) | (1u << 11) | (1u << 12)};
        for (int t = 0; t < 3; ++t) {
            const int32_t n = n_nodes[t];
            if (n <= 0) ada::invalid("tree without nodes");
            ada::Tree& tr = b->trees[t];
            tr.target = t;
            tr.mask = masks[t];
            tr.feature.assign(feature[t], feature[t] + n);
            tr.threshold.assign(threshold[t], threshold[t] + n);
            tr.left.assign(left[t], left[t] + n);
            tr.right.assign(right[t], right[t] + n);
            tr.leaf.assign(leaf[t], leaf[t] + n);
        }
        try {
            ada::validate_bundle(*b);
        } catch (const ada::Error& e) {
            throw ada::Error(ADASPMV_ERR_INVALID_ARGUMENT, e.what());
        }
        *out = b.release();
    });
}

int adaspmv_bundle_destroy(adaspmv_bundle* b) {
    delete b;
    return ADASPMV_OK;
}

int adaspmv_select(adaspmv_ctx* ctx, const adaspmv_matrix* m, adaspmv_vector* v,
                   const adaspmv_bundle* b, int* kernel_index, uint32_t* features_used,
                   int* trees_evaluated) {
    return guarded([&] {
        bind(ctx);
        need(m, "matrix");
        need(v, "vector");
        need(b, "bundle");
        need(kernel_index, "out");
        if (v->n != m->cols) ada::invalid("select: vector length != matrix columns");
        *kernel_index = ada::predict(*ctx, *m, *v, *b, features_used, trees_evaluated);
    });
}

// ---- multiply ------------------------------------------------------------------
int adaspmv_output_create(adaspmv_ctx* ctx, adaspmv_output** out) {
    return guarded([&] {
        bind(ctx);
        need(out, "out");
        auto* y = new adaspmv_output();
        y->ctx = ctx;
        *out = y;
    });
}

int adaspmv_output_destroy(adaspmv_output* y) {
    if (!y) return ADASPMV_OK;
    return guarded([&] {
        if (y->ctx) {
            bind_quiet(y->ctx);
            cudaStreamSynchronize(y->ctx->stream);
        }
        delete y;
    });
}

int adaspmv_run(adaspmv_ctx* ctx, const adaspmv_matrix* m, adaspmv_vector* x, int kernel_index,
                const adaspmv_config* cfg, adaspmv_output* y) {
    return guarded([&] {
        bind(ctx);
        need(m, "matrix");
        need(x, "vector");
        need(y, "output");
        adaspmv_config c{};
        if (cfg) c = *cfg;
        ada::run_kernel(*ctx, *m, *x, kernel_index, c, *y);
    });
}

int adaspmv_run_adaptive(adaspmv_ctx* ctx, const adaspmv_matrix* m, adaspmv_vector* x,
                         const adaspmv_bundle* b, const adaspmv_config* cfg, adaspmv_output* y,
                         int* chosen) {
    return guarded([&] {
        bind(ctx);
        need(m, "matrix");
        need(x, "vector");
        need(y, "output");
        need(b, "bundle");
        if (x->n != m->cols) ada::invalid("multiply: vector length != matrix columns");
        const int k = ada::predict(*ctx, *m, *x, *b, nullptr, nullptr);
        adaspmv_config c{};
        if (cfg) c = *cfg;
        ada::run_kernel(*ctx, *m, *x, k, c, *y);
        if (chosen) *chosen = k;
    });
}

int adaspmv_execute_iteration(adaspmv_ctx* ctx, const adaspmv_matrix* m, adaspmv_vector* x,
                              const adaspmv_bundle* b, int forced_kernel, const adaspmv_config* cfg,
                              adaspmv_output* y, adaspmv_iteration_report* report) {
    return guarded([&] {
        bind(ctx);
        need(m, "matrix");
        need(x, "vector");
        need(y, "output");
        if (x->n != m->cols) ada::invalid("execute_iteration: vector length != matrix columns");
        if (forced_kernel < 0 && !b) ada::invalid("execute_iteration: untrained bundle without override");
        if (forced_kernel > 7) ada::invalid("kernel index out of range");
        using clk = std::chrono::steady_clock;
        double feature_s = 0;
        const auto t0 = clk::now();
        const int k = forced_kernel >= 0 ? forced_kernel
                                         : ada::predict(*ctx, *m, *x, *b, nullptr, nullptr, &feature_s);
        const double select_s = std::chrono::duration<double>(clk::now() - t0).count();
        cudaEvent_t ev[3];
        for (auto& e : ev) ADA_CUDA(cudaEventCreate(&e));
        struct Guard {
            cudaEvent_t* e;
            ~Guard() {
                for (int i = 0; i < 3; ++i) cudaEventDestroy(e[i]);
            }
        } guard{ev};
        adaspmv_config c{};
        if (cfg) c = *cfg;
        ADA_CUDA(cudaEventRecord(ev[0], ctx->stream));
        // convert iff the kernel needs another representation
        if (k <= 3) {
            ada::vector_ensure_dense(*ctx, *x, c.semiring);
            if (k >= 2) ada::vector_ensure_mask(*ctx, *x, c.semiring);
        } else {
            ada::vector_ensure_sparse(*ctx, *x, c.semiring);
            if (k == 6 || k == 7) ada::vector_ensure_eff(*ctx, *x, *m, c.semiring);
        }
        ADA_CUDA(cudaEventRecord(ev[1], ctx->stream));
        ada::run_kernel(*ctx, *m, *x, k, c, *y);
        ADA_CUDA(cudaEventRecord(ev[2], ctx->stream));
        ADA_CUDA(cudaEventSynchronize(ev[2]));
        float conv_ms = 0, kern_ms = 0;
        ADA_CUDA(cudaEventElapsedTime(&conv_ms, ev[0], ev[1]));
        ADA_CUDA(cudaEventElapsedTime(&kern_ms, ev[1], ev[2]));
        if (report) {
            report->iteration = 0;
            report->nnz_x = x->nnz;
            report->kernel = k;
            report->exec_mode = ADASPMV_EXEC_AS_SELECTED;
            report->feature_s = feature_s;
            report->predict_s = select_s - feature_s;
            report->convert_s = conv_ms * 1e-3;
            report->kernel_s = kern_ms * 1e-3;
        }
    });
}

int adaspmv_run_batch(adaspmv_ctx* ctx, const adaspmv_matrix* m, const adaspmv_bundle* b,
                      int forced_kernel, const adaspmv_config* cfg, int64_t count,
                      const adaspmv_host_operand* xs, adaspmv_host_result* ys, int lanes) {
    return guarded([&] {
        bind(ctx);
        need(m, "matrix");
        if (count < 0) ada::invalid("run_batch: negative count");
        if (count > 0) {
            need(xs, "operands");
            need(ys, "results");
        }
        if (forced_kernel > 7) ada::invalid("kernel index out of range");
        if (forced_kernel < 0 && !b) ada::invalid("run_batch: no bundle and no forced kernel");
        if (lanes < 0 || lanes > 16) ada::invalid("run_batch: lanes must be in [0, 16]");
        adaspmv_config c{};
        if (cfg) c = *cfg;
        ada::run_batch(*ctx, *m, b, forced_kernel, c, count, xs, ys, lanes == 0 ? 3 : lanes);
    });
}

int adaspmv_output_info(adaspmv_output* y, int64_t* length, int* has_dense, int* has_sparse, int* dtype) {
    return guarded([&] {
        need(y, "output");
        if (length) *length = y->n;
        if (has_dense) *has_dense = y->has_dense;
        if (has_sparse) *has_sparse = y->has_sparse;
        if (dtype) *dtype = y->dtype;
    });
}

int adaspmv_output_dense(adaspmv_ctx* ctx, adaspmv_output* y, void* values) {
    return guarded([&] {
        bind(ctx);
        need(y, "output");
        ada::output_ensure_dense(*ctx, *y);
        if (values && y->n > 0)
            ADA_CUDA(cudaMemcpyAsync(values, y->dense.p, static_cast<size_t>(ada::value_bytes(y->dtype)) * static_cast<size_t>(y->n),
                                     cudaMemcpyDeviceToHost, ctx->stream));
        ctx->sync();
    });
}

int adaspmv_output_sparse(adaspmv_ctx* ctx, adaspmv_output* y, int64_t capacity, int64_t* indices,
                          void* values, int64_t* nnz_y) {
    return guarded([&] {
        bind(ctx);
        need(y, "output");
        const int64_t nnz = ada::output_nnz(*ctx, *y);
        if (nnz_y) *nnz_y = nnz;
        const int64_t n = std::min(capacity, nnz);
        if (n <= 0) return;
        if (indices) {  // widened to the reference's int64 index_t on the device, one D2H
            ada::DevBuf& w = ctx->scratch[7];
            int64_t* d64 = static_cast<int64_t*>(w.ensure(sizeof(int64_t) * static_cast<size_t>(n)));
            ada::widen_indices(*ctx, n, y->sp_idx.as<int32_t>(), d64);
            ADA_CUDA(cudaMemcpyAsync(indices, d64, sizeof(int64_t) * static_cast<size_t>(n), cudaMemcpyDeviceToHost,
                                     ctx->stream));
        }
        if (values)
            ADA_CUDA(cudaMemcpyAsync(values, y->sp_val.p, static_cast<size_t>(ada::value_bytes(y->dtype)) * static_cast<size_t>(n),
                                     cudaMemcpyDeviceToHost, ctx->stream));
        ctx->sync();
    });
}

int adaspmv_output_device_dense(adaspmv_ctx* ctx, adaspmv_output* y, const void** d_values) {
    return guarded([&] {
        bind(ctx);
        need(y, "output");
        need(d_values, "out");
        ada::output_ensure_dense(*ctx, *y);
        *d_values = y->dense.p;
    });
}

int adaspmv_output_device_sparse(adaspmv_ctx* ctx, adaspmv_output* y, const int32_t** d_indices,
                                 const void** d_values, int64_t* nnz_y) {
    return guarded([&] {
        bind(ctx);
        need(y, "output");
        const int64_t nnz = ada::output_nnz(*ctx, *y);
        if (d_indices) *d_indices = y->sp_idx.as<int32_t>();
        if (d_values) *d_values = y->sp_val.p;
        if (nnz_y) *nnz_y = nnz;
    });
}

// ---- primitives -----------------------------------------------------------------
int adaspmv_make_partition(const int64_t* offsets, int64_t n_offsets, int64_t total_items,
                           int workers, int64_t* out) {
    return guarded([&] {
        if (workers <= 0) ada::invalid("make_partition: workers must be positive");
        if (!offsets || n_offsets <= 0 || offsets[n_offsets - 1] != total_items)
            ada::invalid("make_partition: offsets do not cover total_items");
        need(out, "out");
        auto seg = [&](int64_t pos) {  // partition.hpp:30-33
            return static_cast<int64_t>(std::upper_bound(offsets, offsets + n_offsets, pos) - offsets) - 1;
        };
        for (int w = 0; w < workers; ++w) {
            const int64_t ib = total_items * w / workers, ie = total_items * (w + 1) / workers;
            out[4 * w] = ib;
            out[4 * w + 1] = ie;
            if (ib >= ie) {
                out[4 * w + 2] = out[4 * w + 3] = 0;
                continue;
            }
            out[4 * w + 2] = seg(ib);
            out[4 * w + 3] = seg(ie - 1) + 1;
        }
    });
}

int adaspmv_sort_reduce_pairs(adaspmv_ctx* ctx, int64_t npairs, const int64_t* rows,
                              const void* values, int dtype, int64_t nrows, int64_t* out_indices,
                              void* out_values, int64_t* nnz_out) {
    return guarded([&] {
        bind(ctx);
        check_dtype(dtype);
        need(nnz_out, "out");
        if (npairs < 0) ada::invalid("negative pair count");
        if (nrows < 0 || nrows >= (int64_t(1) << 31)) ada::invalid("row count out of range");
        std::vector<int32_t> r32(static_cast<size_t>(npairs));
        for (int64_t i = 0; i < npairs; ++i) {
            if (rows[i] < 0 || rows[i] >= nrows) ada::out_of_range("pair row out of range");
            r32[static_cast<size_t>(i)] = static_cast<int32_t>(rows[i]);
        }
        const size_t vb = static_cast<size_t>(ada::value_bytes(dtype));
        ada::DevBuf dr, dv, oi, ov;
        dr.ensure(sizeof(int32_t) * std::max<size_t>(r32.size(), 1));
        dv.ensure(vb * std::max<size_t>(r32.size(), 1));
        oi.ensure(sizeof(int32_t) * std::max<size_t>(r32.size(), 1));
        ov.ensure(vb * std::max<size_t>(r32.size(), 1));
        if (npairs > 0) {
            ADA_CUDA(copy_sync(ctx, dr.p, r32.data(), sizeof(int32_t) * r32.size(), cudaMemcpyHostToDevice));
            ADA_CUDA(copy_sync(ctx, dv.p, values, vb * r32.size(), cudaMemcpyHostToDevice));
        }
        const int64_t k = ada::sort_reduce_pairs_device(*ctx, npairs, dr.as<int32_t>(), dv.p, dtype, nrows,
                                                        oi.as<int32_t>(), ov.p);
        *nnz_out = k;
        if (k > 0) {
            std::vector<int32_t> t(static_cast<size_t>(k));
            ADA_CUDA(copy_sync(ctx, t.data(), oi.p, sizeof(int32_t) * t.size(), cudaMemcpyDeviceToHost));
            for (int64_t i = 0; i < k; ++i) out_indices[i] = t[static_cast<size_t>(i)];
            ADA_CUDA(copy_sync(ctx, out_values, ov.p, vb * static_cast<size_t>(k), cudaMemcpyDeviceToHost));
        }
    });
}

int adaspmv_shard_rows(const int64_t* row_offsets, int64_t rows, int nshards, int64_t* cuts) {
    return guarded([&] {
        need(row_offsets, "row_offsets");
        need(cuts, "cuts");
        if (nshards <= 0) ada::invalid("shard_rows: nshards must be positive");
        if (rows < 0) ada::invalid("shard_rows: negative rows");
        ada::shard_cuts(row_offsets, rows, nshards, cuts);
    });
}

int adaspmv_multi_create(int ngpu, const int* devices, int64_t rows, int64_t cols, const int64_t* row_offsets,
                         const int64_t* col_indices, const void* values, int dtype, adaspmv_multi** out) {
    return guarded([&] {
        need(out, "out");
        need(row_offsets, "row_offsets");
        check_dtype(dtype);
        if (ngpu <= 0 || ngpu > 64) ada::invalid("multi: ngpu must be in [1, 64]");
        if (rows < 0 || cols < 0) ada::invalid("negative matrix dimension");
        if (row_offsets[rows] > 0) need(col_indices, "col_indices");
        validate_host_csr(rows, cols, row_offsets, col_indices);
        *out = static_cast<adaspmv_multi*>(
            ada::multi_create(ngpu, devices, rows, cols, row_offsets, col_indices, values, dtype));
    });
}

int adaspmv_multi_cuts(const adaspmv_multi* mm, int64_t* cuts) {
    return guarded([&] {
        need(mm, "multi");
        need(cuts, "cuts");
        std::copy(mm->cuts.begin(), mm->cuts.end(), cuts);
    });
}

int adaspmv_multi_run(adaspmv_multi* mm, const adaspmv_bundle* b, int forced_kernel, const adaspmv_config* cfg,
                      int64_t nnz_x, const int64_t* indices, const void* values, void* y, int* kernels) {
    return guarded([&] {
        need(mm, "multi");
        if (forced_kernel > 7) ada::invalid("kernel index out of range");
        if (forced_kernel < 0 && !b) ada::invalid("multi_run: no bundle and no forced kernel");
        if (nnz_x > 0 || (nnz_x < 0 && mm->cols > 0)) need(values, "values");
        if (nnz_x > 0) need(indices, "indices");
        adaspmv_config c{};
        if (cfg) c = *cfg;
        ada::multi_run(*mm, b, forced_kernel, c, nnz_x, indices, values, y, kernels);
    });
}

int adaspmv_multi_destroy(adaspmv_multi* mm) {
    if (!mm) return ADASPMV_OK;
    return guarded([&] { delete static_cast<ada::Multi*>(mm); });
}

int adaspmv_bfs(adaspmv_ctx* ctx, const adaspmv_matrix* m, int64_t source, int semiring,
                const adaspmv_bundle* b, int forced_kernel, int64_t* levels, int64_t* n_levels,
                adaspmv_iteration_report* reports, int64_t max_reports) {
    return guarded([&] {
        bind(ctx);
        need(m, "matrix");
        need(n_levels, "n_levels");
        ada::bfs(*ctx, *m, source, semiring, b, forced_kernel, levels, n_levels, reports, max_reports);
    });
}

int adaspmv_pagerank(adaspmv_ctx* ctx, const adaspmv_matrix* m, double damping, double prune,
                     int64_t max_iters, const adaspmv_bundle* b, int forced_kernel, double* rank,
                     int64_t* n_iters, adaspmv_iteration_report* reports, int64_t max_reports) {
    return guarded([&] {
        bind(ctx);
        need(m, "matrix");
        need(n_iters, "n_iters");
        ada::pagerank(*ctx, *m, damping, prune, max_iters, b, forced_kernel, rank, n_iters, reports,
                      max_reports);
    });
}

// ---- row-partitioned mode, one process per GPU (dist.cpp) ------------------
int adaspmv_dist_unique_id(void* id128) {
    return guarded([&] {
        need(id128, "id");
        ada::dist_unique_id(id128);
    });
}

int adaspmv_dist_create_nccl(adaspmv_ctx* ctx, int rank, int world, const void* id128, adaspmv_dist** out) {
    return guarded([&] {
        bind(ctx);
        need(id128, "id");
        need(out, "out");
        *out = static_cast<adaspmv_dist*>(ada::dist_create_nccl(*ctx, rank, world, id128));
    });
}

int adaspmv_dist_create_host(adaspmv_ctx* ctx, int rank, int world, adaspmv_allgather_fn fn, void* user,
                             adaspmv_dist** out) {
    return guarded([&] {
        bind(ctx);
        need(out, "out");
        *out = static_cast<adaspmv_dist*>(ada::dist_create_host(*ctx, rank, world, fn, user));
    });
}

int adaspmv_dist_destroy(adaspmv_dist* d) {
    if (!d) return ADASPMV_OK;
    return guarded([&] {
        bind(d->ctx);
        delete static_cast<ada::Dist*>(d);
    });
}

int adaspmv_dist_bcast_vector(adaspmv_dist* d, adaspmv_vector* x, int root) {
    return guarded([&] {
        need(d, "dist");
        need(x, "vector");
        bind(d->ctx);
        if (x->ctx != d->ctx) ada::invalid("dist_bcast_vector: the vector belongs to another context");
        ada::dist_bcast_vector(*d, *x, root);
    });
}

int adaspmv_dist_alloc_peer_output(adaspmv_dist* d, int64_t bytes, void** y_full_device) {
    return guarded([&] {
        need(d, "dist");
        need(y_full_device, "y_full_device");
        bind(d->ctx);
        *y_full_device = ada::dist_alloc_peer_output(*d, bytes);
    });
}

int adaspmv_dist_run_allgather(adaspmv_dist* d, const adaspmv_matrix* block, adaspmv_vector* x, int kernel_index,
                               const adaspmv_config* cfg, adaspmv_output* y, void* y_full_device, int64_t* total,
                               int* fused) {
    return guarded([&] {
        need(d, "dist");
        need(block, "matrix");
        need(x, "vector");
        need(y, "output");
        need(y_full_device, "y_full");
        bind(d->ctx);
        adaspmv_config c{};
        if (cfg) c = *cfg;
        const int64_t t = ada::dist_run_allgather(*d, *block, *x, kernel_index, c, *y, y_full_device, fused);
        if (total) *total = t;
    });
}

int adaspmv_dist_allgather_output(adaspmv_dist* d, adaspmv_output* y, void* y_full_device, int64_t* total) {
    return guarded([&] {
        need(d, "dist");
        need(y, "output");
        need(y_full_device, "y_full");
        bind(d->ctx);
        const int64_t t = ada::dist_allgather_output(*d, *y, y_full_device);
        if (total) *total = t;
    });
}

int adaspmv_dist_bfs(adaspmv_dist* d, const adaspmv_matrix* block, int64_t row0, int64_t source, int semiring,
                     const adaspmv_bundle* b, int forced_kernel, int64_t* levels, int64_t* n_levels,
                     adaspmv_iteration_report* reports, int64_t max_reports) {
    return guarded([&] {
        need(d, "dist");
        need(block, "matrix");
        need(n_levels, "n_levels");
        bind(d->ctx);
        ada::bfs_dist(*d->ctx, *block, *d, row0, source, semiring, b, forced_kernel, levels, n_levels, reports,
                      max_reports);
    });
}

}  // extern "C"

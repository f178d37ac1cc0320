// run.cu -- run_kernel dispatch (kernels.hpp:520-535) and the lazy second
// representation of MultiplyOutput (kernels.hpp:116-152).
#include <algorithm>

#include "device.cuh"
#include "internal.hpp"
#include "kernels.hpp"
#include "prims.cuh"

namespace ada {

namespace {

template <class V>
__global__ void out_scatter_kernel(int64_t nnz, const int32_t* __restrict__ idx,
                                   const V* __restrict__ val, V* __restrict__ out) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < nnz) out[idx[i]] = val[i];
}

template <class V, int SR>
struct NotIdentityIn {
    const V* y;
    __device__ int64_t operator()(int64_t i) const { return y[i] != Semiring<SR, V>::zero() ? 1 : 0; }
};

template <class V>
struct CompactOut {
    const V* y;
    int32_t* idx;
    V* val;
    __device__ void operator()(int64_t i, int64_t p, int64_t v) const {
        if (v) {
            idx[p] = static_cast<int32_t>(i);
            val[p] = y[i];
        }
    }
};

template <class V, int SR>
void run_t(Context& ctx, const Matrix& m, Vector& x, int kernel, const adaspmv_config& cfg,
           Output& y) {
    const int lanes = cfg.lanes_per_row;
    const size_t rows = static_cast<size_t>(std::max<int64_t>(m.rows, 1));
    switch (kernel) {
        case 0:
        case 1:
        case 2:
        case 3: {
            vector_ensure_dense(ctx, x, SR);
            const uint32_t* mask = nullptr;
            if (kernel >= 2) {
                vector_ensure_mask(ctx, x, SR);
                mask = x.mask.as<uint32_t>();
            }
            V* yd = static_cast<V*>(y.dense.ensure(sizeof(V) * rows));
            const bool direct = kernel == 0 || kernel == 2;
            const bool binned = direct && (cfg.row_layout == ADASPMV_ROW_LAYOUT_BINNED ||
                                           (cfg.row_layout == ADASPMV_ROW_LAYOUT_AUTO && binned_preferred(m)));
            if (cfg.row_layout < 0 || cfg.row_layout > 2) invalid("unknown row_layout");
            if (binned)
                run_row_binned<V, SR>(ctx, m, x.dense.as<V>(), mask, yd, cfg.bin_rows, cfg.bin_tile_nnz,
                                      cfg.bin_cluster, cfg.bin_panel_kib);
            else if (m.rows > 0)
                run_row_major<V, SR>(ctx, m, x.dense.as<V>(), mask, kernel == 1 || kernel == 3,
                                     lanes, yd);
            y.has_dense = true;
            break;
        }
        default: {
            const bool lb = kernel >= 6;
            const bool sort = kernel == 5 || kernel == 7;
            if (!sort) {
                V* yd = static_cast<V*>(y.dense.ensure(sizeof(V) * rows));
                int64_t dummy;
                run_col_major<V, SR>(ctx, m, x, lb, false, cfg.atomic_private_accumulators != 0,
                                     lanes, yd, nullptr, nullptr, nullptr, &dummy);
                y.has_dense = true;
            } else {
                int32_t* yi = static_cast<int32_t*>(y.sp_idx.ensure(sizeof(int32_t) * rows));
                V* yv = static_cast<V*>(y.sp_val.ensure(sizeof(V) * rows));
                int64_t* dn = static_cast<int64_t*>(y.d_nnz.ensure(sizeof(int64_t)));
                int64_t hn = -1;
                run_col_major<V, SR>(ctx, m, x, lb, true, false, lanes, nullptr, yi, yv, dn, &hn);
                y.nnz = hn;
                y.has_sparse = true;
            }
        }
    }
}

template <class V>
void run_v(Context& ctx, const Matrix& m, Vector& x, int kernel, const adaspmv_config& cfg,
           Output& y) {
    switch (cfg.semiring) {
        case ADASPMV_PLUS_TIMES: run_t<V, SR_PLUS_TIMES>(ctx, m, x, kernel, cfg, y); break;
        case ADASPMV_OR_AND: run_t<V, SR_OR_AND>(ctx, m, x, kernel, cfg, y); break;
        case ADASPMV_MIN_PLUS: run_t<V, SR_MIN_PLUS>(ctx, m, x, kernel, cfg, y); break;
        default: invalid("unknown semiring");
    }
}

template <class V, int SR>
void dense_from_sparse(Context& ctx, Output& y) {
    V* d = static_cast<V*>(y.dense.ensure(sizeof(V) * static_cast<size_t>(std::max<int64_t>(y.n, 1))));
    fill_value<V, SR>(ctx, d, y.n);
    const int64_t nnz = output_nnz(ctx, y);
    if (nnz > 0) {
        out_scatter_kernel<V><<<static_cast<unsigned>((nnz + 255) / 256), 256, 0, ctx.stream>>>(
            nnz, y.sp_idx.as<int32_t>(), y.sp_val.as<V>(), d);
        ADA_LAUNCHED(ctx);
    }
}

template <class V, int SR>
void sparse_from_dense(Context& ctx, Output& y) {
    const size_t cap = static_cast<size_t>(std::max<int64_t>(y.n, 1));
    int32_t* yi = static_cast<int32_t*>(y.sp_idx.ensure(sizeof(int32_t) * cap));
    V* yv = static_cast<V*>(y.sp_val.ensure(sizeof(V) * cap));
    int64_t* dn = static_cast<int64_t*>(y.d_nnz.ensure(sizeof(int64_t)));
    const V* d = y.dense.as<V>();
    scan3(ctx, y.n, NotIdentityIn<V, SR>{d}, CompactOut<V>{d, yi, yv}, dn, ctx.scratch[4]);
    y.nnz = -1;
}

}  // namespace

void run_kernel(Context& ctx, const Matrix& m, Vector& x, int kernel, const adaspmv_config& cfg,
                Output& y) {
    if (kernel < 0 || kernel > 7) invalid("kernel index out of range");
    if (x.n != m.cols) invalid("multiply: vector length != matrix columns");
    if (x.dtype != m.dtype) invalid("multiply: vector dtype != matrix dtype");
    if (!x.has_dense && !x.has_sparse) invalid("multiply: vector has no value set");
    y.ctx = &ctx;
    y.reset(m.rows, m.dtype);
    y.semiring = cfg.semiring;
    y.timed = ctx.timing;
    if (y.timed) {
        for (auto& e : y.ev)
            if (!e) ADA_CUDA(cudaEventCreate(&e));
        ADA_CUDA(cudaEventRecord(y.ev[0], ctx.stream));
    }
    y.has_ctr = ctx.counters;
    if (ctx.counters) {
        ctx.ctr = static_cast<unsigned long long*>(y.d_ctr.ensure(2 * sizeof(unsigned long long)));
        ADA_CUDA(cudaMemsetAsync(ctx.ctr, 0, 2 * sizeof(unsigned long long), ctx.stream));
    }
    struct CtrReset {
        Context& c;
        ~CtrReset() { c.ctr = nullptr; }
    } ctr_reset{ctx};
    if (m.dtype == ADASPMV_F64) run_v<double>(ctx, m, x, kernel, cfg, y);
    else run_v<float>(ctx, m, x, kernel, cfg, y);
    if (y.timed) ADA_CUDA(cudaEventRecord(y.ev[1], ctx.stream));
}

int64_t output_nnz(Context& ctx, Output& y) {
    if (!y.has_sparse) output_ensure_sparse(ctx, y);
    if (y.nnz < 0) y.nnz = ctx.fetch_scalar(y.d_nnz.as<int64_t>());
    return y.nnz;
}

void output_ensure_dense(Context& ctx, Output& y) {
    if (y.has_dense) return;
    if (!y.has_sparse) invalid("output holds no result");
    const bool f64 = y.dtype == ADASPMV_F64;
    switch (y.semiring) {
        case ADASPMV_MIN_PLUS:
            f64 ? dense_from_sparse<double, SR_MIN_PLUS>(ctx, y) : dense_from_sparse<float, SR_MIN_PLUS>(ctx, y);
            break;
        default:
            f64 ? dense_from_sparse<double, SR_PLUS_TIMES>(ctx, y) : dense_from_sparse<float, SR_PLUS_TIMES>(ctx, y);
    }
    y.has_dense = true;
}

void output_ensure_sparse(Context& ctx, Output& y) {
    if (y.has_sparse) return;
    if (!y.has_dense) invalid("output holds no result");
    const bool f64 = y.dtype == ADASPMV_F64;
    switch (y.semiring) {
        case ADASPMV_MIN_PLUS:
            f64 ? sparse_from_dense<double, SR_MIN_PLUS>(ctx, y) : sparse_from_dense<float, SR_MIN_PLUS>(ctx, y);
            break;
        default:
            f64 ? sparse_from_dense<double, SR_PLUS_TIMES>(ctx, y) : sparse_from_dense<float, SR_PLUS_TIMES>(ctx, y);
    }
    y.has_sparse = true;
}

}  // namespace ada

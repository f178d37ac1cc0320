// pagerank.cu -- incremental (delta-propagation) PageRank driver over the
// adaspmv multiply: the paper's second
// varied-sparsity workload.
//
//   P        = A^T with column j scaled by 1 / outdeg(j), outdeg(j) = the
//              stored entries of row j of A (values ignored, "graph"
//              semantics): SPEC.md:500's delta' = damping * A^T_colnorm *
//              delta, so an edge i -> j (A_ij stored) moves i's mass to j.
//              P's CSR is A's CSC (already on the device), built once; rows
//              with no entries (dangling vertices) propagate nothing
//              (SPEC.md:543).
//   rank     = 0, delta = 1/n everywhere
//   repeat   rank += delta;  y = P delta (adaptive kernel);
//            delta' = {i : |d*y_i| >= prune and d*y_i != 0} with d*y_i
//   until    delta' empty or max_iters multiplies.
//
// The prune + rank accumulation + compaction of the next delta is ONE fused
// scan pass over y (dense or sparse view), like the BFS frontier update
// (bfs.cu); only the next delta's size crosses to the host per iteration.
#include <algorithm>
#include <chrono>
#include <memory>

#include "device.cuh"
#include "internal.hpp"
#include "kernels.hpp"
#include "prims.cuh"

namespace ada {

namespace {

unsigned grid_for(const Context& ctx, int64_t work, int threads) {  // grid-stride, <= 32 CTAs / SM
    const int64_t g = std::min<int64_t>((work + threads - 1) / threads, static_cast<int64_t>(ctx.sm_count) * 32);
    return static_cast<unsigned>(std::max<int64_t>(g, 1));
}

using clk = std::chrono::steady_clock;

double secs(clk::time_point a, clk::time_point b) { return std::chrono::duration<double>(b - a).count(); }

// vals[k] = 1 / outdeg(ri[k]): entry k of A's CSC (row ri[k]) becomes entry
// k of P's CSR, scaled by the out-degree (row length in A) of its source
template <class V>
__global__ void outdeg_values_kernel(const int32_t* __restrict__ ri, const int64_t* __restrict__ ro,
                                     int64_t nnz, V* __restrict__ vals) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < nnz; k += stride) {
        const int32_t r = ri[k];
        vals[k] = V(1) / static_cast<V>(ro[r + 1] - ro[r]);
    }
}

// rank[i] = delta.val = 1/n; delta.idx = i
template <class V>
__global__ void pr_init_kernel(int64_t n, V inv_n, V rank0, V* __restrict__ rank, int32_t* __restrict__ xi,
                               V* __restrict__ xv) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride) {
        rank[i] = rank0;
        xi[i] = static_cast<int32_t>(i);
        xv[i] = inv_n;
    }
}

template <class V>
__device__ __forceinline__ bool keep(V v, V prune) {
    return v != V(0) && fabs(v) >= prune;
}

// Items pack (kept ? 1 : 0) << kCntShift | deg_col(row) when `co` is set:
// the prefix is each kept row's delta slot and its effective-nnz offset, the
// total gives nnz_x and nnz_s in one read (as the BFS frontier update).
constexpr int kCntShift = 36;

template <class V>
struct DenseDeltaIn {
    const V* y;
    V d, prune;
    const int64_t* co;
    __device__ int64_t operator()(int64_t i) const {
        if (!keep(d * y[i], prune)) return 0;
        return co ? (int64_t(1) << kCntShift) | (co[i + 1] - co[i]) : 1;
    }
};

template <class V>
struct SparseDeltaIn {
    const int32_t* yi;
    const V* yv;
    V d, prune;
    const int64_t* co;
    __device__ int64_t operator()(int64_t k) const {
        if (!keep(d * yv[k], prune)) return 0;
        const int32_t r = yi[k];
        return co ? (int64_t(1) << kCntShift) | (co[r + 1] - co[r]) : 1;
    }
};

template <class V>
struct DeltaEpi {
    const int32_t* yi;  // null for the dense view
    const V* yv;
    V d;
    V* rank;  // null: do not accumulate (the multiply budget is spent)
    int32_t* xi;
    V* xv;
    int64_t* eff;  // null: plain 0/1 items
    __device__ void operator()(int64_t i, int64_t p, int64_t v) const {
        if (!v) return;
        const int32_t row = yi ? yi[i] : static_cast<int32_t>(i);
        const V dv = d * yv[i];
        if (rank) rank[row] += dv;  // rank += delta' (the next iteration's first step, fused)
        const int64_t slot = eff ? p >> kCntShift : p;
        xi[slot] = row;
        xv[slot] = dv;
        if (eff) eff[slot] = p & ((int64_t(1) << kCntShift) - 1);
    }
};

__global__ void set_i64_kernel(int64_t* p, int64_t v) { *p = v; }

template <class V>
int64_t next_delta(Context& ctx, const Matrix& m, Output& y, Vector& x, V* rank, V d, V prune) {  // rank may be null
    x.invalidate();
    int32_t* xi = static_cast<int32_t*>(x.sp_idx.ensure(sizeof(int32_t) * static_cast<size_t>(x.n)));
    V* xv = static_cast<V*>(x.sp_val.ensure(sizeof(V) * static_cast<size_t>(x.n)));
    const bool fused = m.nnz < (int64_t(1) << kCntShift) && x.n < (int64_t(1) << (63 - kCntShift));
    const int64_t* co = fused ? m.col_off.as<int64_t>() : nullptr;
    int64_t* eff = fused ? static_cast<int64_t*>(x.eff.ensure(sizeof(int64_t) * static_cast<size_t>(x.n + 1))) : nullptr;
    if (y.has_sparse) {
        const int64_t nnz = output_nnz(ctx, y);
        scan3(ctx, nnz, SparseDeltaIn<V>{y.sp_idx.as<int32_t>(), y.sp_val.as<V>(), d, prune, co},
              DeltaEpi<V>{y.sp_idx.as<int32_t>(), y.sp_val.as<V>(), d, rank, xi, xv, eff}, ctx.h_scalars_dev + kScanTotalSlot,
              ctx.scratch[4]);
    } else {
        scan3(ctx, y.n, DenseDeltaIn<V>{y.dense.as<V>(), d, prune, co},
              DeltaEpi<V>{nullptr, y.dense.as<V>(), d, rank, xi, xv, eff}, ctx.h_scalars_dev + kScanTotalSlot, ctx.scratch[4]);
    }
    // the scan's total was stored straight into the mapped scalars
    ctx.sync();
    const int64_t tot = ctx.h_scalars[kScanTotalSlot];
    x.nnz = fused ? tot >> kCntShift : tot;
    x.has_sparse = true;
    if (fused) {
        const int64_t nnz_s = tot & ((int64_t(1) << kCntShift) - 1);
        set_i64_kernel<<<1, 1, 0, ctx.stream>>>(eff + x.nnz, nnz_s);  // eff[nnz_x] = nnz_s
        ADA_LAUNCHED(ctx);
        x.has_eff = true;
        x.eff_matrix = m.id;
        x.nnz_s = nnz_s;
        x.nnz_s_matrix = m.id;
    }
    return x.nnz;
}

// Default policy without a bundle: the algorithmic-bytes model of SURVEY.md
// 8(d) -- column scatter (K6/K7 family) against a full row pass (K0/K1) --
// with each scattered entry priced at 4x its bytes: an L2 atomic per entry
// (measured on B200: C2 K6 84 us for 6.7 M entries vs K0 ~165 us for 67 M).
int heuristic_kernel(Context& ctx, const Matrix& m, Vector& x) {
    const int64_t nnz_s = vector_nnz_s(ctx, x, m);
    const double vb = m.vbytes();
    constexpr double kAtomic = 4.0;
    const double col = static_cast<double>(x.nnz) * (20.0 + vb) + kAtomic * static_cast<double>(nnz_s) * (4.0 + vb) +
                       (nnz_s <= 4096 ? 0.0 : static_cast<double>(m.rows) * vb);
    const double row = static_cast<double>(m.rows + 1) * 8.0 + static_cast<double>(m.nnz) * (4.0 + vb) +
                       static_cast<double>(m.cols + m.rows) * vb;
    if (col <= row) return nnz_s <= 4096 ? 7 : 6;
    // skewed rows (Gini) -> load-balanced, unless the row-bin layout (which
    // splits the heavy rows out) runs the direct kernel
    return m.feat[8] > 0.5 && !binned_preferred(m) ? 1 : 0;
}

template <class V>
void pagerank_t(Context& ctx, const Matrix& g, double damping, double prune, int64_t max_iters,
                const Bundle* b, int forced, double* rank_out, int64_t* n_iters,
                adaspmv_iteration_report* reports, int64_t max_reports) {
    const int64_t n = g.rows;
    // P = A^T, column-normalised by out-degree (pattern values): its CSR is
    // A's CSC; cached on the graph matrix (structure-only, immutable)
    if (!g.colnorm) {
        DevBuf pv;
        V* vals = static_cast<V*>(pv.ensure(sizeof(V) * static_cast<size_t>(std::max<int64_t>(g.nnz, 1))));
        if (g.nnz > 0) {
            outdeg_values_kernel<V><<<grid_for(ctx, g.nnz, 256), 256, 0, ctx.stream>>>(
                g.row_idx.as<int32_t>(), g.row_off.as<int64_t>(), g.nnz, vals);
            ADA_LAUNCHED(ctx);
        }
        g.colnorm.reset(matrix_create_device(ctx, g.cols, g.rows, g.nnz, g.col_off.as<int64_t>(),
                                             g.row_idx.as<int32_t>(), vals, g.dtype, false));
    }
    const Matrix* P = g.colnorm.get();
    DevBuf rb;
    V* rank = static_cast<V*>(rb.ensure(sizeof(V) * static_cast<size_t>(std::max<int64_t>(n, 1))));
    Vector x;
    x.ctx = &ctx;
    x.n = n;
    x.dtype = g.dtype;
    {
        int32_t* xi = static_cast<int32_t*>(x.sp_idx.ensure(sizeof(int32_t) * static_cast<size_t>(std::max<int64_t>(n, 1))));
        V* xv = static_cast<V*>(x.sp_val.ensure(sizeof(V) * static_cast<size_t>(std::max<int64_t>(n, 1))));
        if (n > 0) {
            const V inv_n = V(1) / static_cast<V>(n);
            // rank += delta_0 is fused here unless no multiply is allowed
            pr_init_kernel<V><<<grid_for(ctx, n, 256), 256, 0, ctx.stream>>>(n, inv_n, max_iters > 0 ? inv_n : V(0),
                                                                              rank, xi, xv);
            ADA_LAUNCHED(ctx);
        }
        x.nnz = n;
        x.has_sparse = true;
    }
    Output y;
    y.ctx = &ctx;
    adaspmv_config cfg{};
    cfg.semiring = ADASPMV_PLUS_TIMES;
    cudaEvent_t ev[3];
    for (auto& e : ev) ADA_CUDA(cudaEventCreate(&e));
    struct EvGuard {
        cudaEvent_t* e;
        ~EvGuard() {
            for (int i = 0; i < 3; ++i) cudaEventDestroy(e[i]);
        }
    } guard{ev};
    int64_t it = 0;
    while (x.nnz > 0 && it < max_iters) {
        const auto t0 = clk::now();
        int k;
        if (b) k = predict(ctx, *P, x, *b, nullptr, nullptr);
        else if (forced >= 0) k = forced;
        else k = heuristic_kernel(ctx, *P, x);
        const auto t1 = clk::now();
        ADA_CUDA(cudaEventRecord(ev[0], ctx.stream));
        if (k <= 3) {
            vector_ensure_dense(ctx, x, ADASPMV_PLUS_TIMES);
            if (k >= 2) vector_ensure_mask(ctx, x);
        } else if (k == 6 || k == 7) {
            vector_ensure_eff(ctx, x, *P);
        }
        ADA_CUDA(cudaEventRecord(ev[1], ctx.stream));
        const int64_t nnz_x = x.nnz;
        run_kernel(ctx, *P, x, k, cfg, y);
        ADA_CUDA(cudaEventRecord(ev[2], ctx.stream));
        // delta' joins rank only if another multiply may follow (SPEC.md:498-506:
        // rank holds exactly the deltas that were propagated or are final)
        next_delta<V>(ctx, *P, y, x, it + 1 < max_iters ? rank : nullptr, static_cast<V>(damping),
                      static_cast<V>(prune));  // syncs
        if (reports && it < max_reports) {
            float c_ms = 0, k_ms = 0;
            ADA_CUDA(cudaEventElapsedTime(&c_ms, ev[0], ev[1]));
            ADA_CUDA(cudaEventElapsedTime(&k_ms, ev[1], ev[2]));
            adaspmv_iteration_report& r = reports[it];
            r.iteration = it;
            r.nnz_x = nnz_x;
            r.kernel = k;
            r.exec_mode = ADASPMV_EXEC_AS_SELECTED;
            r.predict_s = secs(t0, t1);
            r.feature_s = 0;
            r.convert_s = c_ms * 1e-3;
            r.kernel_s = k_ms * 1e-3;
        }
        ++it;
    }
    *n_iters = it;
    if (rank_out && n > 0) {
        if (sizeof(V) == sizeof(double)) {
            ADA_CUDA(cudaMemcpyAsync(rank_out, rank, sizeof(double) * static_cast<size_t>(n),
                                     cudaMemcpyDeviceToHost, ctx.stream));
            ctx.sync();
        } else {
            std::vector<V> h(static_cast<size_t>(n));
            ADA_CUDA(cudaMemcpyAsync(h.data(), rank, sizeof(V) * static_cast<size_t>(n), cudaMemcpyDeviceToHost,
                                     ctx.stream));
            ctx.sync();
            for (int64_t i = 0; i < n; ++i) rank_out[i] = static_cast<double>(h[static_cast<size_t>(i)]);
        }
    }
    ctx.sync();
}

}  // namespace

void pagerank(Context& ctx, const Matrix& m, double damping, double prune, int64_t max_iters,
              const Bundle* b, int forced, double* rank, int64_t* n_iters,
              adaspmv_iteration_report* reports, int64_t max_reports) {
    if (m.rows != m.cols) invalid("pagerank: matrix must be square");
    if (!(damping > 0.0 && damping < 1.0)) invalid("pagerank: damping must be in (0, 1)");
    if (!(prune >= 0.0)) invalid("pagerank: prune must be >= 0");
    if (max_iters < 0) invalid("pagerank: max_iters must be >= 0");
    if (forced < -1 || forced > 7) invalid("pagerank: forced kernel out of range");
    if (m.dtype == ADASPMV_F64)
        pagerank_t<double>(ctx, m, damping, prune, max_iters, b, forced, rank, n_iters, reports, max_reports);
    else
        pagerank_t<float>(ctx, m, damping, prune, max_iters, b, forced, rank, n_iters, reports, max_reports);
}

}  // namespace ada

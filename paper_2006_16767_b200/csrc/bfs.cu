// bfs.cu -- level-synchronous BFS driver over the adaptive
// multiply: x = frontier, y = A x (A as stored), next frontier =
// {i : y_i != identity and level[i] unset}.  The frontier update is one fused
// compaction kernel over y (dense or sparse view) that writes the next
// frontier's index list + values and the levels in the same pass; only the
// frontier size crosses to the host per level.
//
// Semirings: PLUS_TIMES with frontier values 1.0 is the reference-spec
// driver; OR_AND is the pattern-only boolean BFS; MIN_PLUS
// carries levels as values (y_i = min_j level_j + a_ij).
#include <algorithm>
#include <chrono>

#include "device.cuh"
#include "internal.hpp"
#include "kernels.hpp"
#include "prims.cuh"

namespace ada {

namespace {

using clk = std::chrono::steady_clock;

double secs(clk::time_point a, clk::time_point b) { return std::chrono::duration<double>(b - a).count(); }

__global__ void widen_levels_kernel(const int32_t* __restrict__ lv, int64_t n, int64_t* __restrict__ out) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < n) out[i] = lv[i];
}

// The frontier update is one scan whose items pack (kept ? 1 : 0) << kCntShift
// | deg_col(row): the prefix gives each kept row its frontier slot AND its
// effective-nnz offset (kernels.hpp:400-404's eff_offsets of the next x), and
// the total gives nnz_x and nnz_s in one device-to-host read.
constexpr int kCntShift = 36;  // fused packing: nnz_s < 2^36 and frontier < 2^27

template <class V, int SR>
struct DenseFrontierIn {
    const V* y;
    const int32_t* lv;
    const int64_t* co;  // null: plain 0/1 items (no packing)
    __device__ int64_t operator()(int64_t i) const {
        if (!(y[i] != Semiring<SR, V>::zero() && lv[i] < 0)) return 0;
        return co ? (int64_t(1) << kCntShift) | (co[i + 1] - co[i]) : 1;
    }
};

template <class V, int SR>
struct SparseFrontierIn {
    const int32_t* yi;
    const V* yv;
    const int32_t* lv;
    const int64_t* co;
    __device__ int64_t operator()(int64_t k) const {
        const int32_t r = yi[k];
        if (!(yv[k] != Semiring<SR, V>::zero() && lv[r] < 0)) return 0;
        return co ? (int64_t(1) << kCntShift) | (co[r + 1] - co[r]) : 1;
    }
};

template <class V>
struct FrontierEpi {
    const int32_t* yi;  // null for the dense view (row = i)
    int32_t* lv;
    int32_t* xi;
    V* xv;
    int64_t* eff;       // null: no effective-nnz offsets
    int32_t level;
    V value;
    __device__ void operator()(int64_t i, int64_t p, int64_t v) const {
        if (!v) return;
        const int32_t row = yi ? yi[i] : static_cast<int32_t>(i);
        const int64_t slot = eff ? p >> kCntShift : p;
        lv[row] = level;
        xi[slot] = row;
        xv[slot] = value;
        if (eff) eff[slot] = p & ((int64_t(1) << kCntShift) - 1);
    }
};

__global__ void set_i64_kernel(int64_t* p, int64_t v) { *p = v; }

// row block -> global vertex ids (dist BFS: the block's rows start at row0)
__global__ void add_offset_kernel(int32_t* __restrict__ ids, int64_t n, int64_t off) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < n) ids[i] = static_cast<int32_t>(ids[i] + off);
}

template <class V>
__global__ void fill_kernel(V* __restrict__ p, int64_t n, V v) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < n) p[i] = v;
}

// levels of this block's rows (-1 = unvisited), and the first frontier
// {source} with its value (no host copy, no synchronisation)
template <class V>
__global__ void init_block_levels_kernel(int32_t* lv, int64_t nr, int64_t src_local, int32_t* xi, V* xv,
                                         int32_t source, V one, const int64_t* __restrict__ co,
                                         volatile int64_t* host_nnz_s) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < nr) lv[i] = i == src_local ? 0 : -1;
    if (i == 0) {
        xi[0] = source;
        xv[0] = one;
        *host_nnz_s = co[source + 1] - co[source];  // the first frontier's nnz_s (selector feature)
    }
}

template <class V, int SR>
int64_t next_frontier(Context& ctx, const Matrix& m, Output& y, Vector& x, int32_t* lv, int32_t level,
                      bool local_ids = false) {
    x.invalidate();
    int32_t* xi = static_cast<int32_t*>(x.sp_idx.ensure(sizeof(int32_t) * static_cast<size_t>(x.n)));
    V* xv = static_cast<V*>(x.sp_val.ensure(sizeof(V) * static_cast<size_t>(x.n)));
    const V value = SR == SR_MIN_PLUS ? V(level) : V(1);
    // fused nnz_s / eff offsets when the packing cannot overflow (x.n = cols)
    // and the row ids are the column ids (not on a row block: local_ids)
    const bool fused = !local_ids && m.nnz < (int64_t(1) << kCntShift) && x.n < (int64_t(1) << (63 - kCntShift));
    const int64_t* co = fused ? m.col_off.as<int64_t>() : nullptr;
    int64_t* eff = fused ? static_cast<int64_t*>(x.eff.ensure(sizeof(int64_t) * static_cast<size_t>(x.n + 1))) : nullptr;
    if (y.has_sparse) {
        const int64_t nnz = output_nnz(ctx, y);
        scan3(ctx, nnz, SparseFrontierIn<V, SR>{y.sp_idx.as<int32_t>(), y.sp_val.as<V>(), lv, co},
              FrontierEpi<V>{y.sp_idx.as<int32_t>(), lv, xi, xv, eff, level, value}, ctx.h_scalars_dev + kScanTotalSlot,
              ctx.scratch[4]);
    } else {
        scan3(ctx, y.n, DenseFrontierIn<V, SR>{y.dense.as<V>(), lv, co},
              FrontierEpi<V>{nullptr, lv, xi, xv, eff, level, value}, ctx.h_scalars_dev + kScanTotalSlot, ctx.scratch[4]);
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

// Output-masked pull: the fused BFS extension of K2/K3.
// Rows already visited are skipped before any index is loaded; with the
// boolean semiring, or any semiring on a pattern matrix (only membership of
// the next frontier is used), a lane stops at its first frontier neighbour.
// Only unvisited rows are written; the frontier update reads y only there.
template <class V, int G, int SR, bool EARLY>
__global__ void __launch_bounds__(256) bfs_pull_kernel(int64_t rows, const int64_t* __restrict__ ro,
                                                       const int32_t* __restrict__ ci,
                                                       const V* __restrict__ vals,
                                                       const V* __restrict__ x,
                                                       const uint32_t* __restrict__ fmask,
                                                       const int32_t* __restrict__ lv,
                                                       V* __restrict__ y) {
    using S = Semiring<SR, V>;
    constexpr int kU = 4;
    const int64_t gid = static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x;
    const int64_t row = gid / G;
    const int lg = threadIdx.x & (G - 1);
    const bool live = row < rows && __ldg(lv + row) < 0;
    const int64_t b = live ? __ldg(ro + row) : 0, e = live ? __ldg(ro + row + 1) : 0;
    V acc = S::zero();
    for (int64_t k0 = b + lg; k0 < e; k0 += G * kU) {
        int c[kU];
        bool hit[kU];
#pragma unroll
        for (int j = 0; j < kU; ++j) {
            const int64_t k = k0 + j * G;
            c[j] = k < e ? __ldg(ci + k) : -1;
        }
#pragma unroll
        for (int j = 0; j < kU; ++j)
            hit[j] = c[j] >= 0 && ((__ldg(fmask + (c[j] >> 5)) >> (c[j] & 31)) & 1u);
#pragma unroll
        for (int j = 0; j < kU; ++j)
            // OR_AND: a frontier hit is the whole answer (x holds 1 there), no x load
            if (hit[j])
                acc = SR == SR_OR_AND ? V(1)
                                      : S::fma(S::kUsesValues ? __ldg(vals + k0 + j * G) : V(1), __ldg(x + c[j]), acc);
        if (EARLY && acc != S::zero()) break;
    }
#pragma unroll
    for (int d = G / 2; d > 0; d >>= 1) acc = S::add(acc, __shfl_xor_sync(kFull, acc, d, G));
    if (live && lg == 0) y[row] = acc;
}

template <class V, int SR, bool EARLY>
void launch_pull_e(Context& ctx, const Matrix& m, const Vector& x, const int32_t* lv, V* y) {
    // early exit: a row usually stops within its first few entries, so fewer
    // lanes per row (R-MAT 22 BFS, G = 1/2/4/8/16/32: 0.70/0.73/0.82/0.96/
    // 1.28/1.85 ms); full sums keep the SpMV lane rule
    const int G = EARLY ? std::max(1, default_lanes_per_row(m.feat[5]) / 8) : default_lanes_per_row(m.feat[5]);
    const unsigned blocks = static_cast<unsigned>((m.rows * G + 255) / 256);
    if (!blocks) return;
#define ADA_G(GG)                                                                               \
    case GG:                                                                                    \
        bfs_pull_kernel<V, GG, SR, EARLY><<<blocks, 256, 0, ctx.stream>>>(                      \
            m.rows, m.row_off.as<int64_t>(), m.col_idx.as<int32_t>(), m.vals.as<V>(),           \
            SR == SR_OR_AND ? nullptr : x.dense.as<V>(), x.mask.as<uint32_t>(), lv, y);         \
        break;
    switch (G) { ADA_G(1) ADA_G(2) ADA_G(4) ADA_G(8) ADA_G(16) ADA_G(32) default: invalid("lanes"); }
#undef ADA_G
    ADA_LAUNCHED(ctx);
}

template <class V, int SR>
void launch_pull(Context& ctx, const Matrix& m, const Vector& x, const int32_t* lv, Output& y) {
    V* yd = static_cast<V*>(y.dense.ensure(sizeof(V) * static_cast<size_t>(std::max<int64_t>(m.rows, 1))));
    // membership only: on a pattern matrix any frontier neighbour decides
    // (plus-times sums of 1s, min-plus of 1 + level), as with the boolean one
    const bool early = SR == SR_OR_AND || m.pattern;
    if (early) launch_pull_e<V, SR, true>(ctx, m, x, lv, yd);
    else launch_pull_e<V, SR, false>(ctx, m, x, lv, yd);
    y.reset(m.rows, m.dtype);
    y.semiring = SR;
    y.has_dense = true;
}

// One fused push level (boolean semiring): the column-major choices (K4-K7)
// run K6's load-balanced tiles, and instead of an atomic write into a dense y
// each unvisited row is claimed once (atomicCAS on its level) and appended
// to the next frontier with its column degree -- no dense y to clear, no scan
// over all n rows.  x becomes the next frontier; returns its size.
template <class V>
int64_t push_level(Context& ctx, const Matrix& m, Vector& x, int32_t* lv, int32_t level, V value, DevBuf& nidx,
                   DevBuf& nval, cudaEvent_t done) {
    const size_t n = static_cast<size_t>(std::max<int64_t>(x.n, 1));
    int32_t* ni = static_cast<int32_t*>(nidx.ensure(sizeof(int32_t) * n));
    V* nv = static_cast<V*>(nval.ensure(sizeof(V) * n));
    unsigned long long* cnt = reinterpret_cast<unsigned long long*>(ctx.dscal(13));
    ADA_CUDA(cudaMemsetAsync(cnt, 0, 2 * sizeof(unsigned long long), ctx.stream));
    bfs_push_lb<V>(ctx, m, x, lv, level, ni, nv, value, cnt);
    ADA_CUDA(cudaEventRecord(done, ctx.stream));
    ctx.fetch_scalars(reinterpret_cast<const int64_t*>(cnt), 2);
    const int64_t nx = ctx.h_scalars[0], ns = ctx.h_scalars[1];
    x.invalidate();
    std::swap(x.sp_idx.p, nidx.p);
    std::swap(x.sp_idx.cap, nidx.cap);
    std::swap(x.sp_idx.s, nidx.s);
    std::swap(x.sp_val.p, nval.p);
    std::swap(x.sp_val.cap, nval.cap);
    std::swap(x.sp_val.s, nval.s);
    x.nnz = nx;
    x.has_sparse = true;
    x.nnz_s = ns;
    x.nnz_s_matrix = m.id;
    return nx;
}

// Push vs pull by the algorithmic-bytes model of SURVEY.md section 8(d):
// column-major reads ~ nnz_s entries, row-major (validated) reads every index.
// The pull is output-masked (bfs_pull_kernel): only the ~unvisited share of
// the index stream is read.
int heuristic_kernel(Context& ctx, const Matrix& m, Vector& x, int64_t visited) {
    const int64_t nnz_s = vector_nnz_s(ctx, x, m);
    const double vb = m.vbytes();
    const double unvisited = m.rows > 0 ? 1.0 - static_cast<double>(visited) / static_cast<double>(m.rows) : 0.0;
    const double push = static_cast<double>(x.nnz) * 20.0 + static_cast<double>(nnz_s) * (4.0 + vb) +
                        (nnz_s <= 4096 ? 0.0 : static_cast<double>(m.rows) * vb);
    const double pull = static_cast<double>(m.rows + 1) * 8.0 + static_cast<double>(m.nnz) * 4.0 * unvisited +
                        static_cast<double>(m.cols) / 8.0 + static_cast<double>(m.rows) * vb * unvisited;
    if (push <= pull) return nnz_s <= 4096 ? 7 : 6;
    return 2;
}

// The frontier this rank formed among its rows (block-local ids in
// x.sp_idx[0 .. x.nnz)) -> the global frontier: ids shifted to vertex ids,
// every rank's list all-gathered in rank order (= ascending vertex order:
// blocks are contiguous), values refilled.  Returns the global size.
template <class V>
int64_t gather_frontier(Context& ctx, Dist& d, Vector& x, int64_t row0, V value, DevBuf& gathered) {
    const int64_t cnt = std::max<int64_t>(x.nnz, 0);
    if (cnt > 0 && row0 != 0) {
        add_offset_kernel<<<static_cast<unsigned>((cnt + 255) / 256), 256, 0, ctx.stream>>>(x.sp_idx.as<int32_t>(),
                                                                                           cnt, row0);
        ADA_LAUNCHED(ctx);
    }
    gathered.ensure(sizeof(int32_t) * static_cast<size_t>(std::max<int64_t>(x.n, 1)));
    const int64_t total = d.allgatherv(x.sp_idx.p, cnt, sizeof(int32_t), gathered.p);
    x.invalidate();
    std::swap(x.sp_idx.p, gathered.p);
    std::swap(x.sp_idx.cap, gathered.cap);
    std::swap(x.sp_idx.s, gathered.s);
    V* xv = static_cast<V*>(x.sp_val.ensure(sizeof(V) * static_cast<size_t>(std::max<int64_t>(x.n, 1))));
    if (total > 0) {
        fill_kernel<V><<<static_cast<unsigned>((total + 255) / 256), 256, 0, ctx.stream>>>(xv, total, value);
        ADA_LAUNCHED(ctx);
    }
    x.nnz = total;
    x.has_sparse = true;
    return total;
}

// Level-synchronous BFS.  dist == nullptr: the whole
// square matrix on this device.  dist != nullptr: m is the row block
// [row0, row0 + m.rows) of an m.cols-vertex graph; levels
// and the kernel decisions are per block, the frontier is exchanged.
template <class V, int SR>
void bfs_t(Context& ctx, const Matrix& m, int64_t source, const Bundle* b, int forced,
           int64_t* levels, int64_t* n_levels, adaspmv_iteration_report* reports,
           int64_t max_reports, Dist* dist = nullptr, int64_t row0 = 0) {
    const int64_t n = m.cols;   // vertices (= rows of the whole matrix)
    const int64_t nr = m.rows;  // rows held here
    DevBuf lvb, gathered;
    int32_t* lv = static_cast<int32_t*>(lvb.ensure(sizeof(int32_t) * static_cast<size_t>(std::max<int64_t>(nr, 1))));
    const int64_t src_local = source - row0;  // outside [0, nr): another rank's row
    Vector x;
    x.ctx = &ctx;
    x.n = n;
    x.dtype = m.dtype;
    {
        int32_t* xi = static_cast<int32_t*>(x.sp_idx.ensure(sizeof(int32_t) * static_cast<size_t>(n)));
        V* xv = static_cast<V*>(x.sp_val.ensure(sizeof(V) * static_cast<size_t>(n)));
        const V one = SR == SR_MIN_PLUS ? V(0) : V(1);
        init_block_levels_kernel<V><<<static_cast<unsigned>(std::max<int64_t>((nr + 255) / 256, 1)), 256, 0,
                                      ctx.stream>>>(lv, nr, src_local, xi, xv, static_cast<int32_t>(source), one,
                                                    m.col_off.as<int64_t>(), ctx.h_scalars_dev + kScanTotalSlot);
        ADA_LAUNCHED(ctx);
        ctx.sync();
        x.nnz = 1;
        x.has_sparse = true;
        x.nnz_s = ctx.h_scalars[kScanTotalSlot];
        x.nnz_s_matrix = m.id;
    }
    Output y;
    y.ctx = &ctx;
    DevBuf next_idx, next_val;  // the fused push's next frontier (swapped into x)
    adaspmv_config cfg{};
    cfg.semiring = SR;
    int64_t it = 0;
    int64_t visited = src_local >= 0 && src_local < nr ? 1 : 0;  // of this block's rows
    // device-side phase timing without extra synchronisation: events around
    // the conversion and the multiply, read after the frontier-size fetch
    cudaEvent_t ev[3];
    for (auto& e : ev) ADA_CUDA(cudaEventCreate(&e));
    struct EvGuard {
        cudaEvent_t* e;
        ~EvGuard() {
            for (int i = 0; i < 3; ++i) cudaEventDestroy(e[i]);
        }
    } guard{ev};
    while (x.nnz > 0) {
        const auto t0 = clk::now();
        int k;
        if (b) k = predict(ctx, m, x, *b, nullptr, nullptr);
        else if (forced >= 0) k = forced;
        else k = heuristic_kernel(ctx, m, x, visited);
        const auto t1 = clk::now();
        ADA_CUDA(cudaEventRecord(ev[0], ctx.stream));
        // RowSpMSpV (K2/K3) runs as the output-masked pull: a row already
        // visited cannot join the next frontier, so skipping it
        // changes no level.  With the boolean semiring SpMV (K0/K1) does
        // too: non-frontier entries of x are false and add nothing (with
        // values, an Inf * 0 of the plain SpMV could differ, so those keep
        // the unmasked multiply).
        const bool pull = k == 2 || k == 3 || (SR == SR_OR_AND && k <= 1);
        // the column choices run as the fused push when membership of the
        // next frontier does not depend on values: the boolean semiring, or a
        // pattern matrix (plus-times sums of 1s are >= 1; min-plus of 1 +
        // level is finite)
        // (a frontier reaching more entries than there are rows -- forced
        // column kernels on a fat level -- keeps the atomic multiply + scan,
        // which is faster there than claiming row by row)
        const bool push = k >= 4 && (SR == SR_OR_AND || m.pattern) && vector_nnz_s(ctx, x, m) <= m.rows;
        if (pull) {  // output-masked pull: the mask, and x values unless OR_AND
            vector_ensure_mask(ctx, x, SR);
            if (SR != SR_OR_AND) vector_ensure_dense(ctx, x, SR);
        } else if (k <= 1) {
            vector_ensure_dense(ctx, x, SR);
        } else if (k == 6 || k == 7 || push) {
            vector_ensure_eff(ctx, x, m, SR);
        }
        ADA_CUDA(cudaEventRecord(ev[1], ctx.stream));
        const int64_t nnz_x = x.nnz;
        const V value = SR == SR_MIN_PLUS ? V(it + 1) : V(1);  // as next_frontier writes
        if (push) {  // multiply + frontier update in one pass (syncs)
            visited += push_level<V>(ctx, m, x, lv, static_cast<int32_t>(it + 1), value, next_idx, next_val, ev[2]);
        } else {
            if (pull) launch_pull<V, SR>(ctx, m, x, lv, y);  // row-major, output-masked
            else run_kernel(ctx, m, x, k, cfg, y);
            ADA_CUDA(cudaEventRecord(ev[2], ctx.stream));
            visited += next_frontier<V, SR>(ctx, m, y, x, lv, static_cast<int32_t>(it + 1), dist != nullptr);
        }
        if (dist) gather_frontier<V>(ctx, *dist, x, row0, value, gathered);  // the next x on every rank
        if (reports && it < max_reports) {
            float c_ms = 0, k_ms = 0;
            ADA_CUDA(cudaEventElapsedTime(&c_ms, ev[0], ev[1]));
            ADA_CUDA(cudaEventElapsedTime(&k_ms, ev[1], ev[2]));
            adaspmv_iteration_report& r = reports[it];
            r.iteration = it;
            r.nnz_x = nnz_x;
            r.kernel = k;
            r.exec_mode = push ? ADASPMV_EXEC_FUSED_PUSH_LB : (pull ? ADASPMV_EXEC_MASKED_PULL : ADASPMV_EXEC_AS_SELECTED);
            r.predict_s = secs(t0, t1);  // host: tree walk + lazy features (nnz_s fetch)
            r.feature_s = 0;             // folded into predict_s (features pulled lazily)
            r.convert_s = c_ms * 1e-3;
            r.kernel_s = k_ms * 1e-3;
        }
        ++it;
    }
    *n_levels = it;
    if (!levels) return;  // traversal only (levels stay on the device)
    // widen on the device, one D2H of the caller's int64 array
    DevBuf l64;
    if (nr <= 0) return;
    int64_t* d64 = static_cast<int64_t*>(l64.ensure(sizeof(int64_t) * static_cast<size_t>(nr)));
    widen_levels_kernel<<<static_cast<unsigned>((nr + 255) / 256), 256, 0, ctx.stream>>>(lv, nr, d64);
    ADA_LAUNCHED(ctx);
    ADA_CUDA(cudaMemcpyAsync(levels, d64, sizeof(int64_t) * static_cast<size_t>(nr), cudaMemcpyDeviceToHost,
                             ctx.stream));
    ctx.sync();
}

}  // namespace

void widen_levels(Context& ctx, const int32_t* lv, int64_t n, int64_t* out) {
    if (n <= 0) return;
    widen_levels_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, ctx.stream>>>(lv, n, out);
    ADA_LAUNCHED(ctx);
}

void bfs(Context& ctx, const Matrix& m, int64_t source, int semiring, const Bundle* b, int forced,
         int64_t* levels, int64_t* n_levels, adaspmv_iteration_report* reports,
         int64_t max_reports) {
    if (m.rows != m.cols) invalid("bfs: matrix must be square");
    if (source < 0 || source >= m.rows) invalid("bfs: source out of range");
    if (forced < -1 || forced > 7) invalid("bfs: forced kernel out of range");
    if (semiring < ADASPMV_PLUS_TIMES || semiring > ADASPMV_MIN_PLUS) invalid("unknown semiring");
    if (!ctx.bfs_host_loop && bfs_graph_applicable(m, semiring, forced)) {
        bfs_graph(ctx, m, source, b, levels, n_levels, reports, max_reports);
        return;
    }
    const bool f64 = m.dtype == ADASPMV_F64;
    switch (semiring) {
        case ADASPMV_PLUS_TIMES:
            f64 ? bfs_t<double, SR_PLUS_TIMES>(ctx, m, source, b, forced, levels, n_levels, reports, max_reports)
                : bfs_t<float, SR_PLUS_TIMES>(ctx, m, source, b, forced, levels, n_levels, reports, max_reports);
            break;
        case ADASPMV_OR_AND:
            f64 ? bfs_t<double, SR_OR_AND>(ctx, m, source, b, forced, levels, n_levels, reports, max_reports)
                : bfs_t<float, SR_OR_AND>(ctx, m, source, b, forced, levels, n_levels, reports, max_reports);
            break;
        case ADASPMV_MIN_PLUS:
            f64 ? bfs_t<double, SR_MIN_PLUS>(ctx, m, source, b, forced, levels, n_levels, reports, max_reports)
                : bfs_t<float, SR_MIN_PLUS>(ctx, m, source, b, forced, levels, n_levels, reports, max_reports);
            break;
        default: invalid("unknown semiring");
    }
}

void bfs_dist(Context& ctx, const Matrix& m, Dist& d, int64_t row0, int64_t source, int semiring, const Bundle* b,
              int forced, int64_t* levels, int64_t* n_levels, adaspmv_iteration_report* reports,
              int64_t max_reports) {
    if (row0 < 0 || row0 + m.rows > m.cols) invalid("dist_bfs: the row block is outside the square matrix");
    if (source < 0 || source >= m.cols) invalid("bfs: source out of range");
    if (forced < -1 || forced > 7) invalid("bfs: forced kernel out of range");
    const bool f64 = m.dtype == ADASPMV_F64;
    switch (semiring) {
        case ADASPMV_PLUS_TIMES:
            f64 ? bfs_t<double, SR_PLUS_TIMES>(ctx, m, source, b, forced, levels, n_levels, reports, max_reports, &d, row0)
                : bfs_t<float, SR_PLUS_TIMES>(ctx, m, source, b, forced, levels, n_levels, reports, max_reports, &d, row0);
            break;
        case ADASPMV_OR_AND:
            f64 ? bfs_t<double, SR_OR_AND>(ctx, m, source, b, forced, levels, n_levels, reports, max_reports, &d, row0)
                : bfs_t<float, SR_OR_AND>(ctx, m, source, b, forced, levels, n_levels, reports, max_reports, &d, row0);
            break;
        case ADASPMV_MIN_PLUS:
            f64 ? bfs_t<double, SR_MIN_PLUS>(ctx, m, source, b, forced, levels, n_levels, reports, max_reports, &d, row0)
                : bfs_t<float, SR_MIN_PLUS>(ctx, m, source, b, forced, levels, n_levels, reports, max_reports, &d, row0);
            break;
        default: invalid("unknown semiring");
    }
}

}  // namespace ada

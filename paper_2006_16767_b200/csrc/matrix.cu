// matrix.cu -- device-resident DualMatrix (sparse.hpp:204-259).
//
// Upload keeps the CSR as given (int64 offsets, indices narrowed to int32)
// and builds the CSC on the device with the reference's stable order
// (csr_to_csc, sparse.hpp:157-178: rows ascending within each column) by a
// stable LSD radix sort of (column, (row, value)) in CSR order.  The matrix
// features and the LB tile heads (partition.hpp:30-33) are
// computed once here ("computed only once at the beginning").
#include <algorithm>
#include <string>
#include <atomic>
#include <cmath>
#include <cstring>
#include <vector>

#include "device.cuh"
#include "internal.hpp"
#include "prims.cuh"

namespace ada {

namespace {

std::atomic<uint64_t> g_matrix_ids{1};

template <class V>
struct RowVal {
    int32_t row;
    V val;
};

__global__ void fill_ones_kernel(void* vals, int64_t n, int vbytes) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t k = i; k < n; k += stride) {
        if (vbytes == 8) static_cast<double*>(vals)[k] = 1.0;
        else static_cast<float*>(vals)[k] = 1.0f;
    }
}

// one warp per row: keys = column, payload = (row, value) in CSR order
template <class V>
__global__ void csr_expand_kernel(const int64_t* __restrict__ ro, const int32_t* __restrict__ ci,
                                  const V* __restrict__ vals, int64_t rows,
                                  uint32_t* __restrict__ keys, RowVal<V>* __restrict__ pay) {
    const int64_t warp = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int64_t r = warp; r < rows; r += nwarps) {
        const int64_t b = ro[r], e = ro[r + 1];
        for (int64_t k = b + lane; k < e; k += 32) {
            keys[k] = static_cast<uint32_t>(ci[k]);
            pay[k] = RowVal<V>{static_cast<int32_t>(r), vals[k]};
        }
    }
}

template <class V>
__global__ void csc_unpack_kernel(const RowVal<V>* __restrict__ pay, int64_t nnz,
                                  int32_t* __restrict__ ri, V* __restrict__ cv) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t k = i; k < nnz; k += stride) {
        RowVal<V> p = pay[k];
        ri[k] = p.row;
        cv[k] = p.val;
    }
}

__global__ void col_count_kernel(const int32_t* __restrict__ ci, int64_t nnz,
                                 unsigned long long* __restrict__ counts) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t k = i; k < nnz; k += stride) atomicAdd(counts + ci[k], 1ull);
}

struct U64In {
    const unsigned long long* c;
    __device__ int64_t operator()(int64_t i) const { return static_cast<int64_t>(c[i]); }
};

// lower_bound: first index i in [0, rows] with ro[i] >= pos
__device__ int64_t lower_row(const int64_t* __restrict__ ro, int64_t rows, int64_t pos) {
    int64_t lo = 0, hi = rows + 1;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (ro[mid] < pos) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// Row window start of each LB warp tile (see Matrix::tile_head): the row that
// holds item t*kRowTile when the tile starts mid-row, else the first row
// starting at the tile boundary (empty rows there are owned by this tile).
__global__ void tile_head_kernel(const int64_t* __restrict__ ro, int64_t rows, int64_t nnz,
                                 int64_t ntiles, int64_t* __restrict__ head) {
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (t > ntiles + 1) return;
    if (t == ntiles) {
        head[t] = rows;
        return;
    }
    if (t == ntiles + 1) {
        head[t] = lower_row(ro, rows, nnz);
        return;
    }
    const int64_t pos = t * static_cast<int64_t>(kRowTile);
    const int64_t lb = lower_row(ro, rows, pos);
    head[t] = (lb <= rows && ro[lb] == pos) ? lb : lb - 1;
}

struct EmptyRowIn {
    const int64_t* ro;
    __device__ int64_t operator()(int64_t r) const { return ro[r] == ro[r + 1] ? 1 : 0; }
};
struct EmptyRowEpi {
    int32_t* out;
    __device__ void operator()(int64_t r, int64_t p, int64_t v) const {
        if (v) out[p] = static_cast<int32_t>(r);
    }
};

void build_tiles(Context& ctx, Matrix& m) {
    m.n_row_tiles = (m.nnz + kRowTile - 1) / kRowTile;
    const size_t n = static_cast<size_t>(m.n_row_tiles + 2);
    m.tile_head.ensure(sizeof(int64_t) * n);
    tile_head_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, ctx.stream>>>(
        m.row_off.as<int64_t>(), m.rows, m.nnz, m.n_row_tiles, m.tile_head.as<int64_t>());
    ADA_LAUNCHED(ctx);
    // list of empty rows (the LB kernels never see them; the fix-up writes them)
    m.empty_rows.ensure(sizeof(int32_t) * static_cast<size_t>(std::max<int64_t>(m.rows, 1)));
    scan3(ctx, m.rows, EmptyRowIn{m.row_off.as<int64_t>()}, EmptyRowEpi{m.empty_rows.as<int32_t>()},
          ctx.dscal(3), ctx.scratch[5]);
    m.n_empty = ctx.fetch_scalar(ctx.dscal(3));
}

// degree statistics: slot[0] = max, [1] = min, [2] = sum of squares (u64)
__global__ void degree_stats_kernel(const int64_t* __restrict__ off, int64_t n,
                                    unsigned long long* __restrict__ slot) {
    unsigned long long mx = 0, mn = ~0ull, sq = 0;
    const int64_t i0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t r = i0; r < n; r += stride) {
        const unsigned long long d = static_cast<unsigned long long>(off[r + 1] - off[r]);
        mx = d > mx ? d : mx;
        mn = d < mn ? d : mn;
        sq += d * d;
    }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
        mx = max(mx, __shfl_xor_sync(kFull, mx, s));
        mn = min(mn, __shfl_xor_sync(kFull, mn, s));
        sq += __shfl_xor_sync(kFull, sq, s);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(slot + 0, mx);
        atomicMin(slot + 1, mn);
        atomicAdd(slot + 2, sq);
    }
}

// histogram of row degrees (for the Gini coefficient by the sorted identity)
constexpr int kHistSmem = 2048;
__global__ void degree_hist_kernel(const int64_t* __restrict__ off, int64_t n, int64_t nbins,
                                   unsigned long long* __restrict__ hist) {
    __shared__ unsigned int sh[kHistSmem];
    for (int i = threadIdx.x; i < kHistSmem; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    const int64_t i0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t r = i0; r < n; r += stride) {
        const int64_t d = off[r + 1] - off[r];
        if (d < kHistSmem) atomicAdd(&sh[d], 1u);
        else atomicAdd(hist + d, 1ull);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kHistSmem && i < nbins; i += blockDim.x)
        if (sh[i]) atomicAdd(hist + i, static_cast<unsigned long long>(sh[i]));
}

int grid_for(const Context& ctx, int64_t work, int threads) {
    int64_t g = (work + threads - 1) / threads;
    const int64_t cap = static_cast<int64_t>(ctx.sm_count) * 32;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return static_cast<int>(g);
}

template <class V>
void build_csc(Context& ctx, Matrix& m) {
    const int64_t nnz = m.nnz;
    m.col_off.ensure(sizeof(int64_t) * static_cast<size_t>(m.cols + 1));
    m.row_idx.ensure(sizeof(int32_t) * static_cast<size_t>(std::max<int64_t>(nnz, 1)));
    m.cvals.ensure(sizeof(V) * static_cast<size_t>(std::max<int64_t>(nnz, 1)));
    // column counts -> col_offsets (exclusive scan; [cols] = nnz)
    DevBuf counts;
    counts.ensure(sizeof(unsigned long long) * static_cast<size_t>(std::max<int64_t>(m.cols, 1)));
    ADA_CUDA(cudaMemsetAsync(counts.p, 0, sizeof(unsigned long long) * static_cast<size_t>(m.cols),
                             ctx.stream));
    if (nnz > 0) {
        col_count_kernel<<<grid_for(ctx, nnz, 256), 256, 0, ctx.stream>>>(
            m.col_idx.as<int32_t>(), nnz, counts.as<unsigned long long>());
        ADA_LAUNCHED(ctx);
    }
    int64_t* co = m.col_off.as<int64_t>();
    scan3(ctx, m.cols, U64In{counts.as<unsigned long long>()}, WriteExclusive{co}, co + m.cols,
          ctx.scratch[5]);
    if (m.cols == 0) ADA_CUDA(cudaMemsetAsync(co, 0, sizeof(int64_t), ctx.stream));
    if (nnz == 0) return;
    // stable sort of CSR-order entries by column
    DevBuf k0, k1, p0, p1, cnt;
    k0.ensure(sizeof(uint32_t) * static_cast<size_t>(nnz));
    k1.ensure(sizeof(uint32_t) * static_cast<size_t>(nnz));
    p0.ensure(sizeof(RowVal<V>) * static_cast<size_t>(nnz));
    p1.ensure(sizeof(RowVal<V>) * static_cast<size_t>(nnz));
    csr_expand_kernel<V><<<grid_for(ctx, m.rows * 32, 256), 256, 0, ctx.stream>>>(
        m.row_off.as<int64_t>(), m.col_idx.as<int32_t>(), m.vals.as<V>(), m.rows,
        k0.as<uint32_t>(), p0.as<RowVal<V>>());
    ADA_LAUNCHED(ctx);
    const int which = radix_sort_pairs<RowVal<V>>(ctx, k0.as<uint32_t>(), p0.as<RowVal<V>>(),
                                                  k1.as<uint32_t>(), p1.as<RowVal<V>>(), nnz,
                                                  bits_for(m.cols), cnt, ctx.scratch[5]);
    const RowVal<V>* sorted = which ? p1.as<RowVal<V>>() : p0.as<RowVal<V>>();
    csc_unpack_kernel<V><<<grid_for(ctx, nnz, 256), 256, 0, ctx.stream>>>(
        sorted, nnz, m.row_idx.as<int32_t>(), m.cvals.as<V>());
    ADA_LAUNCHED(ctx);
    ctx.sync();  // scratch buffers are released on return
}

// Matrix features.
void compute_features(Context& ctx, Matrix& m) {
    double* f = m.feat;
    f[0] = static_cast<double>(m.rows);
    f[1] = static_cast<double>(m.cols);
    f[2] = static_cast<double>(m.nnz);
    if (m.rows == 0) {
        for (int i = 3; i < 9; ++i) f[i] = 0;
        return;
    }
    DevBuf slots;
    slots.ensure(sizeof(unsigned long long) * 8);
    unsigned long long init[8] = {0, ~0ull, 0, 0, 0, ~0ull, 0, 0};
    ADA_CUDA(cudaMemcpyAsync(slots.p, init, sizeof(init), cudaMemcpyHostToDevice, ctx.stream));
    degree_stats_kernel<<<grid_for(ctx, m.rows, 256), 256, 0, ctx.stream>>>(
        m.row_off.as<int64_t>(), m.rows, slots.as<unsigned long long>());
    ADA_LAUNCHED(ctx);
    if (m.cols > 0) {  // column degree max (slot 4) for the column kernels' sizing
        degree_stats_kernel<<<grid_for(ctx, m.cols, 256), 256, 0, ctx.stream>>>(
            m.col_off.as<int64_t>(), m.cols, slots.as<unsigned long long>() + 4);
        ADA_LAUNCHED(ctx);
    }
    unsigned long long h[8];
    ADA_CUDA(cudaMemcpyAsync(h, slots.p, sizeof(h), cudaMemcpyDeviceToHost, ctx.stream));
    ctx.sync();
    const uint64_t mx = h[0], mn = h[1], sq = h[2];
    m.max_col_deg = m.cols > 0 ? static_cast<int64_t>(h[4]) : 0;
    m.avg_col = m.cols > 0 ? static_cast<double>(m.nnz) / static_cast<double>(m.cols) : 0.0;
    const double avg = static_cast<double>(m.nnz) / static_cast<double>(m.rows);
    double var = static_cast<double>(sq) / static_cast<double>(m.rows) - avg * avg;
    if (var < 0) var = 0;
    f[3] = static_cast<double>(mx);
    f[4] = static_cast<double>(mn);
    f[5] = avg;
    f[6] = m.cols > 0 ? static_cast<double>(mx - mn) / static_cast<double>(m.cols) : 0.0;
    f[7] = std::sqrt(var);
    // Gini: G = 2*sum_i i*d_(i) / (k*sum d) - (k+1)/k with d sorted ascending.
    // From the degree histogram c_v: positions C_<v + 1 .. C_<v + c_v carry v.
    // column degree profile (selector bounds on nnz_s)
    m.cdeg.clear();
    m.cdeg_cnt.assign(1, 0);
    m.cdeg_sum.assign(1, 0);
    if (m.cols > 0) {
        const int64_t nb = m.max_col_deg + 1;
        DevBuf ch;
        ch.ensure(sizeof(unsigned long long) * static_cast<size_t>(nb));
        ADA_CUDA(cudaMemsetAsync(ch.p, 0, sizeof(unsigned long long) * static_cast<size_t>(nb), ctx.stream));
        degree_hist_kernel<<<grid_for(ctx, m.cols, 256), 256, 0, ctx.stream>>>(
            m.col_off.as<int64_t>(), m.cols, nb, ch.as<unsigned long long>());
        ADA_LAUNCHED(ctx);
        std::vector<unsigned long long> hc(static_cast<size_t>(nb));
        ADA_CUDA(cudaMemcpyAsync(hc.data(), ch.p, sizeof(unsigned long long) * hc.size(), cudaMemcpyDeviceToHost,
                                 ctx.stream));
        ctx.sync();
        for (int64_t d = 0; d < nb; ++d) {
            const int64_t c = static_cast<int64_t>(hc[static_cast<size_t>(d)]);
            if (!c) continue;
            m.cdeg.push_back(d);
            m.cdeg_cnt.push_back(m.cdeg_cnt.back() + c);
            m.cdeg_sum.push_back(m.cdeg_sum.back() + c * d);
        }
    }
    const int64_t nbins = static_cast<int64_t>(mx) + 1;
    DevBuf hist;
    hist.ensure(sizeof(unsigned long long) * static_cast<size_t>(nbins));
    ADA_CUDA(cudaMemsetAsync(hist.p, 0, sizeof(unsigned long long) * static_cast<size_t>(nbins),
                             ctx.stream));
    degree_hist_kernel<<<grid_for(ctx, m.rows, 256), 256, 0, ctx.stream>>>(
        m.row_off.as<int64_t>(), m.rows, nbins, hist.as<unsigned long long>());
    ADA_LAUNCHED(ctx);
    std::vector<unsigned long long> hh(static_cast<size_t>(nbins));
    ADA_CUDA(cudaMemcpyAsync(hh.data(), hist.p, sizeof(unsigned long long) * hh.size(),
                             cudaMemcpyDeviceToHost, ctx.stream));
    ctx.sync();
    unsigned __int128 wsum = 0, total = 0, before = 0;
    for (int64_t v = 0; v < nbins; ++v) {
        const unsigned __int128 c = hh[static_cast<size_t>(v)];
        if (!c) continue;
        // sum of positions before+1 .. before+c
        const unsigned __int128 pos_sum = c * before + c * (c + 1) / 2;
        wsum += pos_sum * static_cast<unsigned __int128>(v);
        total += c * static_cast<unsigned __int128>(v);
        before += c;
    }
    const double k = static_cast<double>(m.rows);
    f[8] = total == 0 ? 0.0
                      : (2.0 * static_cast<double>(wsum)) / (k * static_cast<double>(total)) -
                            (k + 1.0) / k;
}

__global__ void csc_pairs_kernel(int64_t nnz, const int32_t* __restrict__ ri, const float* __restrict__ cv,
                                 uint2* __restrict__ out) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < nnz; k += stride)
        out[k] = make_uint2(static_cast<uint32_t>(ri[k]), __float_as_uint(cv[k]));
}

// smallest nonzero |v| as float bits (positive floats order like their bits)
__global__ void min_abs_nonzero_kernel(int64_t n, const float* __restrict__ v, unsigned* __restrict__ out) {
    unsigned best = 0x7f800000u;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n; k += stride) {
        const unsigned b = __float_as_uint(fabsf(v[k]));
        if (b != 0u && b < best) best = b;
    }
    best = __reduce_min_sync(0xffffffffu, best);
    if ((threadIdx.x & 31) == 0) atomicMin(out, best);
}

// Matrix::cpairs of an fp32 matrix from its CSC, and Matrix::amin
void build_pairs(Context& ctx, Matrix& m) {
    if (m.dtype != ADASPMV_F32 || m.nnz <= 0) return;
    uint2* p = static_cast<uint2*>(m.cpairs.ensure(sizeof(uint2) * static_cast<size_t>(m.nnz)));
    csc_pairs_kernel<<<grid_for(ctx, m.nnz, 256), 256, 0, ctx.stream>>>(m.nnz, m.row_idx.as<int32_t>(),
                                                                       m.cvals.as<float>(), p);
    ADA_LAUNCHED(ctx);
    DevBuf mb;
    unsigned* d = static_cast<unsigned*>(mb.ensure(sizeof(unsigned)));
    const unsigned inf = 0x7f800000u;
    ADA_CUDA(cudaMemcpyAsync(d, &inf, sizeof(unsigned), cudaMemcpyHostToDevice, ctx.stream));
    min_abs_nonzero_kernel<<<grid_for(ctx, m.nnz, 256), 256, 0, ctx.stream>>>(m.nnz, m.cvals.as<float>(), d);
    ADA_LAUNCHED(ctx);
    unsigned h = inf;
    ADA_CUDA(cudaMemcpyAsync(&h, d, sizeof(unsigned), cudaMemcpyDeviceToHost, ctx.stream));
    ctx.sync();
    float a;
    std::memcpy(&a, &h, sizeof(a));
    m.amin = h >= inf ? 3.0e38f : a;  // no nonzero value: nothing to check
}

template <class V>
void finish_matrix(Context& ctx, Matrix& m) {
    build_csc<V>(ctx, m);
    build_pairs(ctx, m);
    build_tiles(ctx, m);
    compute_features(ctx, m);
    m.gather_spread = matrix_gather_spread(ctx, m);
}

}  // namespace

namespace {
// CsrMatrix::validate (sparse.hpp:44-63) on caller-owned device arrays, one
// thread per row (grid-stride).  err = min over violations of (kind << 56 |
// row): the lowest failing kind, then the lowest row, as one verdict.
//   kind 0 row_offsets[0] != 0 / row_offsets[rows] != nnz
//   kind 1 row_offsets decreasing at row r
//   kind 2 column index out of range in row r
//   kind 3 columns not strictly increasing in row r
__global__ void csr_validate_kernel(int64_t rows, int64_t cols, int64_t nnz, const int64_t* __restrict__ ro,
                                    const int32_t* __restrict__ ci, unsigned long long* __restrict__ err) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int64_t t0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (t0 == 0 && (ro[0] != 0 || ro[rows] != nnz)) atomicMin(err, 0ull);
    for (int64_t r = t0; r < rows; r += stride) {
        const int64_t b = ro[r], e = ro[r + 1];
        unsigned long long v = ~0ull;
        if (e < b || b < 0 || e > nnz) {
            v = (1ull << 56) | static_cast<unsigned long long>(r);
        } else {
            int32_t prev = -1;
            for (int64_t k = b; k < e; ++k) {
                const int32_t c = ci[k];
                if (c < 0 || c >= cols) { v = (2ull << 56) | static_cast<unsigned long long>(r); break; }
                if (c <= prev) { v = (3ull << 56) | static_cast<unsigned long long>(r); break; }
                prev = c;
            }
        }
        if (v != ~0ull) atomicMin(err, v);
    }
}
}  // namespace

void validate_device_csr(Context& ctx, int64_t rows, int64_t cols, int64_t nnz, const int64_t* d_ro,
                         const int32_t* d_ci) {
    if (rows < 0 || cols < 0) invalid("negative matrix dimension");
    if (nnz > 0 && !d_ci) invalid("csr: null column indices");
    unsigned long long* err = reinterpret_cast<unsigned long long*>(ctx.dscal(6));
    ADA_CUDA(cudaMemsetAsync(err, 0xff, sizeof(unsigned long long), ctx.stream));
    const int64_t g = std::min<int64_t>((rows + 255) / 256 + 1, static_cast<int64_t>(ctx.sm_count) * 16);
    csr_validate_kernel<<<static_cast<unsigned>(g), 256, 0, ctx.stream>>>(rows, cols, nnz, d_ro, d_ci, err);
    ADA_LAUNCHED(ctx);
    const unsigned long long e = static_cast<unsigned long long>(ctx.fetch_scalar(ctx.dscal(6)));
    if (e == ~0ull) return;
    const int kind = static_cast<int>(e >> 56);
    const std::string row = std::to_string(e & ((1ull << 56) - 1));
    if (kind == 0) invalid("csr: row_offsets[0] != 0 or row_offsets[rows] != nnz");
    if (kind == 1) invalid("csr: row_offsets not nondecreasing");
    if (kind == 2) invalid("csr: column index out of range");
    invalid("csr: columns not strictly increasing in row " + row);
}

Matrix* matrix_create_device(Context& ctx, int64_t rows, int64_t cols, int64_t nnz,
                             const int64_t* d_ro, const int32_t* d_ci, const void* d_vals,
                             int dtype, bool pattern) {
    if (rows < 0 || cols < 0) invalid("negative matrix dimension");
    if (rows >= (int64_t(1) << 31) || cols >= (int64_t(1) << 31))
        invalid("matrix dimension exceeds the device int32 index range");
    auto* m = new Matrix();
    try {
        m->ctx = &ctx;
        m->rows = rows;
        m->cols = cols;
        m->nnz = nnz;
        m->dtype = dtype;
        m->pattern = pattern;
        m->id = g_matrix_ids.fetch_add(1);
        const int vb = m->vbytes();
        m->row_off.ensure(sizeof(int64_t) * static_cast<size_t>(rows + 1));
        m->col_idx.ensure(sizeof(int32_t) * static_cast<size_t>(std::max<int64_t>(nnz, 1)));
        m->vals.ensure(static_cast<size_t>(vb) * static_cast<size_t>(std::max<int64_t>(nnz, 1)));
        ADA_CUDA(cudaMemcpyAsync(m->row_off.p, d_ro, sizeof(int64_t) * static_cast<size_t>(rows + 1),
                                 cudaMemcpyDeviceToDevice, ctx.stream));
        if (nnz > 0) {
            ADA_CUDA(cudaMemcpyAsync(m->col_idx.p, d_ci, sizeof(int32_t) * static_cast<size_t>(nnz),
                                     cudaMemcpyDeviceToDevice, ctx.stream));
            if (d_vals) {
                ADA_CUDA(cudaMemcpyAsync(m->vals.p, d_vals, static_cast<size_t>(vb) * static_cast<size_t>(nnz),
                                         cudaMemcpyDeviceToDevice, ctx.stream));
            } else {
                fill_ones_kernel<<<grid_for(ctx, nnz, 256), 256, 0, ctx.stream>>>(m->vals.p, nnz, vb);
                ADA_LAUNCHED(ctx);
            }
        }
        if (dtype == ADASPMV_F64) finish_matrix<double>(ctx, *m);
        else finish_matrix<float>(ctx, *m);
        ctx.sync();
        return m;
    } catch (...) {
        delete m;
        throw;
    }
}

// transpose (sparse.hpp:262-275): the two layouts swap roles.
Matrix* matrix_transpose(Context& ctx, const Matrix& src) {
    auto* m = new Matrix();
    try {
        m->ctx = &ctx;
        m->rows = src.cols;
        m->cols = src.rows;
        m->nnz = src.nnz;
        m->dtype = src.dtype;
        m->pattern = src.pattern;
        m->id = g_matrix_ids.fetch_add(1);
        const size_t vb = static_cast<size_t>(src.vbytes());
        const size_t z = static_cast<size_t>(std::max<int64_t>(src.nnz, 1));
        auto copy = [&](DevBuf& dst, const DevBuf& s, size_t bytes) {
            dst.ensure(bytes);
            ADA_CUDA(cudaMemcpyAsync(dst.p, s.p, bytes, cudaMemcpyDeviceToDevice, ctx.stream));
        };
        copy(m->row_off, src.col_off, sizeof(int64_t) * static_cast<size_t>(src.cols + 1));
        copy(m->col_idx, src.row_idx, sizeof(int32_t) * z);
        copy(m->vals, src.cvals, vb * z);
        copy(m->col_off, src.row_off, sizeof(int64_t) * static_cast<size_t>(src.rows + 1));
        copy(m->row_idx, src.col_idx, sizeof(int32_t) * z);
        copy(m->cvals, src.vals, vb * z);
        build_pairs(ctx, *m);
        build_tiles(ctx, *m);
        compute_features(ctx, *m);
        m->gather_spread = matrix_gather_spread(ctx, *m);
        ctx.sync();
        return m;
    } catch (...) {
        delete m;
        throw;
    }
}

// sum of the k smallest column degrees (k <= cols)
int64_t Matrix::nnz_s_lower(int64_t k) const {
    if (k <= 0 || cdeg.empty()) return 0;
    // first distinct degree i with cdeg_cnt[i+1] >= k
    const auto it = std::lower_bound(cdeg_cnt.begin() + 1, cdeg_cnt.end(), k);
    if (it == cdeg_cnt.end()) return cdeg_sum.back();
    const size_t i = static_cast<size_t>(it - cdeg_cnt.begin()) - 1;
    return cdeg_sum[i] + (k - cdeg_cnt[i]) * cdeg[i];
}
// sum of the k largest column degrees
int64_t Matrix::nnz_s_upper(int64_t k) const {
    if (k <= 0 || cdeg.empty()) return 0;
    const int64_t n = cdeg_cnt.back();
    if (k >= n) return cdeg_sum.back();
    return cdeg_sum.back() - nnz_s_lower(n - k);
}

}  // namespace ada

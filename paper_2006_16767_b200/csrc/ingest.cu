// ingest.cu -- DualMatrix::from_triplets (sparse.hpp:220-258) on the device.
//
// The reference canonicalises triplets on the host: bucket by row in input
// order, std::sort each row by column, then sum runs of equal columns
// sequentially from 0 (`real_t sum = 0; sum += ...`), keeping zero sums.  At
// C2 (64 M triplets) that takes 14.3 s on one core.
// Here the triplets are uploaded once and
//   1. validated (any coordinate out of range -> std::invalid_argument, as
//      sparse.hpp:226-227) and split into int32 row / column arrays;
//   2. stably sorted by (row, column) with two LSD radix sorts of
//      (key, triplet index): by column, then by row -- stable, so equal
//      (row, column) triplets keep their input order, the order in which
//      the reference's per-row sort leaves them (libstdc++ std::sort is an
//      insertion sort below 17 elements; longer rows with duplicates may
//      be summed in another order there);
//   3. one scan over run heads writes each unique entry: column, row, and
//      the run's values summed in order from V(0);
//   4. row offsets by a lower-bound search per row.
// The CSR then enters matrix_create_device (CSC, features) like any other.
#include <algorithm>
#include <cstdint>

#include "device.cuh"
#include "internal.hpp"
#include "prims.cuh"

namespace ada {

namespace {

unsigned grid_of(const Context& ctx, int64_t work, int threads) {
    const int64_t b = std::max<int64_t>((work + threads - 1) / threads, 1);
    return static_cast<unsigned>(std::min<int64_t>(b, static_cast<int64_t>(ctx.sm_count) * 32));
}

__global__ void triplet_split_kernel(int64_t n, int64_t rows, int64_t cols, const int64_t* __restrict__ tr,
                                     const int64_t* __restrict__ tc, int32_t* __restrict__ r32,
                                     int32_t* __restrict__ c32, uint32_t* __restrict__ ckey,
                                     uint32_t* __restrict__ idx, unsigned long long* __restrict__ bad) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride) {
        const int64_t r = tr[i], c = tc[i];
        if (r < 0 || r >= rows || c < 0 || c >= cols) {
            atomicMin(bad, static_cast<unsigned long long>(i));
            continue;
        }
        r32[i] = static_cast<int32_t>(r);
        c32[i] = static_cast<int32_t>(c);
        ckey[i] = static_cast<uint32_t>(c);
        idx[i] = static_cast<uint32_t>(i);
    }
}

__global__ void gather_row_keys_kernel(int64_t n, const uint32_t* __restrict__ perm,
                                       const int32_t* __restrict__ r32, uint32_t* __restrict__ rkey) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride)
        rkey[i] = static_cast<uint32_t>(r32[perm[i]]);
}

struct RunHead {
    const uint32_t* perm;
    const int32_t* r32;
    const int32_t* c32;
    __device__ int64_t operator()(int64_t i) const {
        if (i == 0) return 1;
        const uint32_t a = perm[i - 1], b = perm[i];
        return (r32[a] != r32[b] || c32[a] != c32[b]) ? 1 : 0;
    }
};

template <class V>
struct RunSum {
    int64_t n;
    const uint32_t* perm;
    const int32_t* r32;
    const int32_t* c32;
    const V* tv;
    int32_t* out_row;
    int32_t* out_col;
    V* out_val;
    __device__ void operator()(int64_t i, int64_t p, int64_t head) const {
        if (!head) return;
        const uint32_t t = perm[i];
        const int32_t r = r32[t], c = c32[t];
        V sum = V(0);  // sparse.hpp:250-251: sum from 0, in sorted (input) order
        for (int64_t j = i; j < n; ++j) {
            const uint32_t u = perm[j];
            if (j > i && (r32[u] != r || c32[u] != c)) break;
            sum += tv[u];
        }
        out_row[p] = r;
        out_col[p] = c;
        out_val[p] = sum;
    }
};

// ro[r] = first unique entry with row >= r, r in [0, rows]
__global__ void row_offsets_kernel(int64_t rows, int64_t u, const int32_t* __restrict__ out_row,
                                   int64_t* __restrict__ ro) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r <= rows; r += stride) {
        int64_t lo = 0, hi = u;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (out_row[mid] < r) lo = mid + 1;
            else hi = mid;
        }
        ro[r] = lo;
    }
}

template <class V>
Matrix* build(Context& ctx, int64_t rows, int64_t cols, int64_t n, const int64_t* h_r, const int64_t* h_c,
              const V* h_v, int dtype) {
    const size_t z = static_cast<size_t>(std::max<int64_t>(n, 1));
    DevBuf d_tr, d_tc, d_tv, r32, c32, k0, p0, k1, p1, orow, ocol, oval, ro, counts, tmp;
    int64_t* tr = static_cast<int64_t*>(d_tr.ensure(sizeof(int64_t) * z));
    int64_t* tc = static_cast<int64_t*>(d_tc.ensure(sizeof(int64_t) * z));
    V* tv = static_cast<V*>(d_tv.ensure(sizeof(V) * z));
    ADA_CUDA(cudaMemcpyAsync(tr, h_r, sizeof(int64_t) * static_cast<size_t>(n), cudaMemcpyHostToDevice, ctx.stream));
    ADA_CUDA(cudaMemcpyAsync(tc, h_c, sizeof(int64_t) * static_cast<size_t>(n), cudaMemcpyHostToDevice, ctx.stream));
    ADA_CUDA(cudaMemcpyAsync(tv, h_v, sizeof(V) * static_cast<size_t>(n), cudaMemcpyHostToDevice, ctx.stream));
    int32_t* pr = static_cast<int32_t*>(r32.ensure(sizeof(int32_t) * z));
    int32_t* pc = static_cast<int32_t*>(c32.ensure(sizeof(int32_t) * z));
    uint32_t* key0 = static_cast<uint32_t*>(k0.ensure(sizeof(uint32_t) * z));
    uint32_t* pay0 = static_cast<uint32_t*>(p0.ensure(sizeof(uint32_t) * z));
    uint32_t* key1 = static_cast<uint32_t*>(k1.ensure(sizeof(uint32_t) * z));
    uint32_t* pay1 = static_cast<uint32_t*>(p1.ensure(sizeof(uint32_t) * z));
    unsigned long long* bad = reinterpret_cast<unsigned long long*>(ctx.dscal(8));
    ADA_CUDA(cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), ctx.stream));
    triplet_split_kernel<<<grid_of(ctx, n, 256), 256, 0, ctx.stream>>>(n, rows, cols, tr, tc, pr, pc, key0, pay0, bad);
    ADA_LAUNCHED(ctx);
    if (static_cast<unsigned long long>(ctx.fetch_scalar(ctx.dscal(8))) != ~0ull)
        invalid("triplet coordinate out of range");
    d_tr.release();
    d_tc.release();
    // stable (row, column) order: by column, then stably by row
    int w = radix_sort_pairs<uint32_t>(ctx, key0, pay0, key1, pay1, n, bits_for(cols), counts, tmp);
    uint32_t* perm = w ? pay1 : pay0;
    uint32_t* rk = w ? key1 : key0;  // column keys are no longer needed: row keys go here
    gather_row_keys_kernel<<<grid_of(ctx, n, 256), 256, 0, ctx.stream>>>(n, perm, pr, rk);
    ADA_LAUNCHED(ctx);
    const int w2 = radix_sort_pairs<uint32_t>(ctx, rk, perm, w ? key0 : key1, w ? pay0 : pay1, n, bits_for(rows),
                                              counts, tmp);
    perm = (w2 ? (w ? pay0 : pay1) : perm);
    int32_t* out_row = static_cast<int32_t*>(orow.ensure(sizeof(int32_t) * z));
    int32_t* out_col = static_cast<int32_t*>(ocol.ensure(sizeof(int32_t) * z));
    V* out_val = static_cast<V*>(oval.ensure(sizeof(V) * z));
    scan3(ctx, n, RunHead{perm, pr, pc}, RunSum<V>{n, perm, pr, pc, tv, out_row, out_col, out_val}, ctx.dscal(9),
          tmp);
    const int64_t u = ctx.fetch_scalar(ctx.dscal(9));
    int64_t* d_ro = static_cast<int64_t*>(ro.ensure(sizeof(int64_t) * static_cast<size_t>(rows + 1)));
    row_offsets_kernel<<<grid_of(ctx, rows + 1, 256), 256, 0, ctx.stream>>>(rows, u, out_row, d_ro);
    ADA_LAUNCHED(ctx);
    Matrix* m = matrix_create_device(ctx, rows, cols, u, d_ro, out_col, out_val, dtype, false);
    ctx.sync();  // the staging buffers above are released on return
    return m;
}

}  // namespace

Matrix* matrix_from_triplets_device(Context& ctx, int64_t rows, int64_t cols, int64_t count, const int64_t* h_r,
                                    const int64_t* h_c, const void* h_v, int dtype) {
    if (rows < 0 || cols < 0) invalid("negative matrix dimension");
    if (count < 0) invalid("negative triplet count");
    if (rows >= (int64_t(1) << 31) || cols >= (int64_t(1) << 31))
        invalid("matrix dimension exceeds the device int32 index range");
    if (count >= (int64_t(1) << 32)) invalid("triplet count exceeds the device index range");
    if (count == 0) {
        DevBuf ro;
        int64_t* d_ro = static_cast<int64_t*>(ro.ensure(sizeof(int64_t) * static_cast<size_t>(rows + 1)));
        ADA_CUDA(cudaMemsetAsync(d_ro, 0, sizeof(int64_t) * static_cast<size_t>(rows + 1), ctx.stream));
        Matrix* m = matrix_create_device(ctx, rows, cols, 0, d_ro, nullptr, nullptr, dtype, false);
        ctx.sync();
        return m;
    }
    if (dtype == ADASPMV_F64)
        return build<double>(ctx, rows, cols, count, h_r, h_c, static_cast<const double*>(h_v), dtype);
    return build<float>(ctx, rows, cols, count, h_r, h_c, static_cast<const float*>(h_v), dtype);
}

}  // namespace ada

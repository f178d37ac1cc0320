// kernels_row.cu -- the four row-major kernels (CSR gather over x):
//
//   K0 spmv_direct  kernels.hpp:242-250  whole rows per lane group
//   K1 spmv_lb      kernels.hpp:251-277  equal-nnz tiles (make_partition)
//   K2 row_direct   as K0 + bitmask validation before value/x loads (:233-235)
//   K3 row_lb       as K1 + bitmask validation
//
// Direct: G lanes per row (G from the average row length), each lane keeping
// U independent (col, val, x) loads in flight, then a width-G shuffle tree.
// LB: one CTA per tile of kRowTile = 2048 nonzeros (tile t owns items
// [t*T, (t+1)*T), i.e. make_partition with W = ceil(nnz/T), partition.hpp:
// 37-56).  Column/value words are streamed with 128-bit no-allocate loads,
// each thread owning 4 consecutive items per round; row runs are resolved by
// a binary search (segment_of, partition.hpp:30-33) plus a forward walk, and
// joined across threads by a block-wide segmented scan.  Rows shared between
// tiles leave partials that a deterministic fix-up kernel combines in tile
// order -- the device analogue of the reference's sequential boundary fix-up
// (kernels.hpp:275-276).
#include <algorithm>

#include "device.cuh"
#include "internal.hpp"
#include "kernels.hpp"

namespace ada {

namespace {

constexpr int kNT = 256;
// independent (col, val, x) loads in flight per lane per iteration: a whole
// short row for 1-2 lanes per row, 4 otherwise
template <int G>
constexpr int unroll_for() { return G <= 2 ? 8 : 4; }

template <class V, int G, bool VALIDATE, int SR>
__global__ void __launch_bounds__(kNT) row_direct_kernel(int64_t rows,
                                                         const int64_t* __restrict__ ro,
                                                         const int32_t* __restrict__ ci,
                                                         const V* __restrict__ vals,
                                                         const V* __restrict__ x,
                                                         const uint32_t* __restrict__ mask,
                                                         V* __restrict__ y,
                                                         unsigned long long* __restrict__ ctr) {
    using S = Semiring<SR, V>;
    constexpr int kU = unroll_for<G>();
    unsigned cnt = 0;
    const int64_t gid = static_cast<int64_t>(blockIdx.x) * kNT + threadIdx.x;
    const int64_t row = gid / G;
    const int lg = threadIdx.x & (G - 1);
    const bool valid = row < rows;  // lanes stay alive for the full-warp shuffles
    const int64_t b = valid ? __ldg(ro + row) : 0, e = valid ? __ldg(ro + row + 1) : 0;
    V acc = S::zero();
    for (int64_t k0 = b + lg; k0 < e; k0 += G * kU) {
        int c[kU];
        bool ok[kU];
#pragma unroll
        for (int j = 0; j < kU; ++j) {
            const int64_t k = k0 + j * G;
            ok[j] = k < e;
            c[j] = ok[j] ? __ldg(ci + k) : 0;
        }
        if (VALIDATE) {
#pragma unroll
            for (int j = 0; j < kU; ++j)
                if (ok[j]) ok[j] = (__ldg(mask + (c[j] >> 5)) >> (c[j] & 31)) & 1u;
        }
        V a[kU], xv[kU];
#pragma unroll
        for (int j = 0; j < kU; ++j) {
            if (ok[j]) {
                a[j] = S::kUsesValues ? __ldg(vals + k0 + j * G) : V(1);
                xv[j] = __ldg(x + c[j]);
            }
        }
#pragma unroll
        for (int j = 0; j < kU; ++j)
            if (ok[j]) {
                acc = S::fma(a[j], xv[j], acc);
                ++cnt;
            }
    }
#pragma unroll
    for (int d = G / 2; d > 0; d >>= 1) acc = S::add(acc, __shfl_xor_sync(kFull, acc, d, G));
    if (valid && lg == 0) y[row] = acc;
    count_add(ctr, 0, cnt);
}

// Short-row Direct kernel: one thread per row, the row's U loads issued as
// one unrolled step, registers capped so that 8 CTAs (2048 threads) share an
// SM.  Measured on C1 fp64 (tools/microbench/c1_mb.cu, CUDA-graph replay
// after a clean L2 flush): the lane-group kernel above with G = 1 (U = 8,
// 64 registers, half the warps resident) 17.5 us; this one (U = 5, 32
// registers) 14.4 us = 89 % of HBM; staging the CTA's products in shared
// memory 20.9 us; a warp per 32 rows with a shuffle scan 27.4 us.
template <class V, bool VALIDATE, int SR, int U>
__global__ void __launch_bounds__(kNT, U <= 5 ? 8 : 6) row_thread_kernel(int64_t rows,
                                                            const int64_t* __restrict__ ro,
                                                            const int32_t* __restrict__ ci,
                                                            const V* __restrict__ vals,
                                                            const V* __restrict__ x,
                                                            const uint32_t* __restrict__ mask,
                                                            V* __restrict__ y,
                                                            unsigned long long* __restrict__ ctr) {
    using S = Semiring<SR, V>;
    const int64_t r = static_cast<int64_t>(blockIdx.x) * kNT + threadIdx.x;
    if (r >= rows) return;
    const int64_t b = __ldg(ro + r), e = __ldg(ro + r + 1);
    V acc = S::zero();
    unsigned cnt = 0;
    for (int64_t k0 = b; k0 < e; k0 += U) {
        int c[U];
        bool ok[U];
#pragma unroll
        for (int j = 0; j < U; ++j) {
            ok[j] = k0 + j < e;
            c[j] = ok[j] ? __ldg(ci + k0 + j) : 0;
        }
        if (VALIDATE) {
#pragma unroll
            for (int j = 0; j < U; ++j)
                if (ok[j]) ok[j] = (__ldg(mask + (c[j] >> 5)) >> (c[j] & 31)) & 1u;
        }
        V a[U], xv[U];
#pragma unroll
        for (int j = 0; j < U; ++j) {
            a[j] = ok[j] && S::kUsesValues ? __ldg(vals + k0 + j) : V(1);
            xv[j] = ok[j] ? __ldg(x + c[j]) : S::zero();
        }
#pragma unroll
        for (int j = 0; j < U; ++j)
            if (ok[j]) acc = S::fma(a[j], xv[j], acc);
        if (ctr) {
#pragma unroll
            for (int j = 0; j < U; ++j) cnt += ok[j];
        }
    }
    y[r] = acc;
    count_add(ctr, 0, cnt);
}

// ---------------------------------------------------------------------------
// LB warp-tile kernel.  Warp w of the grid owns items [w*T, (w+1)*T), T =
// kRowTile = 256: two rounds of 128 items, lane l holding the 4 consecutive
// items 4l..4l+3 of each round (one 128-bit load of columns, one/two of
// values: fully coalesced).  All 8 x gathers per lane are issued before any
// is consumed.  The row window of the tile (<= 33 offsets) sits in shared
// memory; lanes find their row by binary search there and walk their 4
// items; runs are joined across lanes by a warp segmented scan (no block
// barriers).  Tiles spanning more than 128 rows (empty / 1-2 nnz rows) take
// the same code path with the offsets read from global memory, the search
// bounded by the next tile's window start.
// ---------------------------------------------------------------------------
constexpr int kIPT = 4;                       // items per lane per round
constexpr int kRound = 32 * kIPT;             // 128
constexpr int kRounds = kRowTile / kRound;    // 2
constexpr int kWin = 129;                     // offsets held per warp window (128 rows)
constexpr int kWarps = kNT / 32;
static_assert(kRounds * kRound == kRowTile, "tile shape");

template <class V>
struct Vec4;
template <>
struct Vec4<float> {
    __device__ static void load(const float* p, float (&o)[4]) {
        float4 v = ld_stream(reinterpret_cast<const float4*>(p));
        o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
    }
};
template <>
struct Vec4<double> {
    __device__ static void load(const double* p, double (&o)[4]) {
        double2 a = ld_stream(reinterpret_cast<const double2*>(p));
        double2 b = ld_stream(reinterpret_cast<const double2*>(p + 2));
        o[0] = a.x; o[1] = a.y; o[2] = b.x; o[3] = b.y;
    }
};

// Row offsets of one warp tile, relative to the tile start tb and clamped to
// [-1, kRowTile + 1] (only comparisons with positions 0..kRowTile matter), and
// row ids relative to the window start ws: all per-item arithmetic is 32-bit.
// SmemWin: the offsets are staged in shared memory (<= kWin rows);
// GlobWin: tiles spanning more rows read them from global memory.
struct SmemWin {
    const int* rel;
    __device__ int off(int i) const { return rel[i]; }
};
struct GlobWin {
    const int64_t* __restrict__ ro;
    int64_t ws, tb;
    __device__ int off(int i) const {
        const int64_t o = __ldg(ro + ws + i) - tb;
        return static_cast<int>(o < -1 ? -1 : (o > kRowTile + 1 ? kRowTile + 1 : o));
    }
};

// largest i in [lo, hi) with off(i) <= p, given off(lo) <= p
// (segment_of, partition.hpp:30-33)
template <class W>
__device__ __forceinline__ int win_row_of(const W& w, int p, int hi, int lo = 0) {
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (w.off(mid) <= p) lo = mid;
        else hi = mid;
    }
    return lo;
}

template <class V, int SR, class W>
__device__ __forceinline__ void lb_tile_body(const W& win, int nrow, int64_t ws, int64_t t, int ten,
                                             int lane, const int (&c)[kRounds][kIPT],
                                             const V (&a)[kRounds][kIPT], const V (&xv)[kRounds][kIPT],
                                             V* __restrict__ y, V* __restrict__ head_part,
                                             V* __restrict__ tail_part, int64_t* __restrict__ tail_row) {
    using S = Semiring<SR, V>;
    // (empty rows are written by the fix-up kernel from the matrix's list)
    V carry = S::zero();  // value of the row open at the start of the round
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
        const int p0 = r * kRound + lane * kIPT;
        const int p1 = min(p0 + kIPT, ten);
        const bool active = p0 < ten;
        int row = 0, first_row = 0;
        bool cont = false, head_closed = false, last_open = false, first = true;
        V head_val = S::zero(), acc = S::zero();
        if (active) {
            row = win_row_of(win, p0, nrow);
            first_row = row;
            cont = win.off(row) < p0;
            int row_end = win.off(row + 1);
#pragma unroll
            for (int j = 0; j < kIPT; ++j) {
                const int p = p0 + j;
                if (p < p1) {
                    if (p >= row_end) {  // close the run of `row` (it holds items of this lane)
                        if (first && cont) {
                            head_closed = true;
                            head_val = acc;
                        } else {
                            y[ws + row] = acc;  // complete inside this lane
                        }
                        first = false;
                        // rows strictly between hold no items (empty): jump to p's row
                        row = win.off(row + 2) > p ? row + 1 : win_row_of(win, p, nrow, row + 1);
                        row_end = win.off(row + 1);
                        acc = S::zero();
                    }
                    if (c[r][j] >= 0) acc = S::fma(a[r][j], xv[r][j], acc);
                }
            }
            last_open = row_end > p1;
            if (!last_open) {  // last run closes exactly at the lane's end
                if (first && cont) {
                    head_closed = true;
                    head_val = acc;
                } else {
                    y[ws + row] = acc;
                }
                acc = S::zero();
                first = false;
            }
        }
        // segmented-scan element: pass-through only inside one open continuing row
        SegPair<V> e;
        e.f = (active && !(first && cont && last_open)) ? 1 : 0;
        e.v = (active && last_open) ? acc : S::zero();
        SegPair<V> inc = warp_seg_inclusive(e, [](V u, V w) { return S::add(u, w); });
        const V incl = inc.f ? inc.v : S::add(carry, inc.v);
        V excl = __shfl_up_sync(kFull, incl, 1);
        if (lane == 0) excl = carry;
        if (active && head_closed) {
            const V total = S::add(excl, head_val);
            if (win.off(first_row) >= 0) y[ws + first_row] = total;  // row began in this tile
            else head_part[t] = total;                                // shared head row
        }
        carry = __shfl_sync(kFull, incl, 31);
    }
    // tile epilogue: the row open at te
    if (lane == 0) {
        const int R = win_row_of(win, ten - 1, nrow);
        int64_t tr = -1;
        if (win.off(R + 1) > ten) {
            if (win.off(R) >= 0) {
                tail_part[t] = carry;
                tr = ws + R;
            } else {
                head_part[t] = carry;  // tile lies entirely inside row R
            }
        }
        tail_row[t] = tr;
    }
}

template <class V, bool VALIDATE, int SR>
__global__ void __launch_bounds__(kNT, sizeof(V) == 8 ? 3 : 4) row_lb_kernel(
    int64_t rows, int64_t nnz, int64_t ntiles, const int64_t* __restrict__ ro,
    const int32_t* __restrict__ ci, const V* __restrict__ vals, const V* __restrict__ x,
    const uint32_t* __restrict__ mask, const int64_t* __restrict__ tile_head, V* __restrict__ y,
    V* __restrict__ head_part, V* __restrict__ tail_part, int64_t* __restrict__ tail_row,
    unsigned long long* __restrict__ ctr) {
    using S = Semiring<SR, V>;
    __shared__ int swin[kWarps][kWin];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t t = static_cast<int64_t>(blockIdx.x) * kWarps + warp;
    if (t >= ntiles) return;  // whole warp; no block barriers below
    const int64_t tb = t * kRowTile;
    const int ten = static_cast<int>(min(static_cast<int64_t>(kRowTile), nnz - tb));

    // ---- stream the tile: all loads of both rounds issued before use -------
    int c[kRounds][kIPT];
    V a[kRounds][kIPT];
    V xv[kRounds][kIPT];
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
        const int p0 = r * kRound + lane * kIPT;
        // K3 consults the bitmask before loading a value (kernels.hpp:229-240):
        // its values are loaded below, only for entries whose x is set
        constexpr bool kStreamVals = S::kUsesValues && !VALIDATE;
        if (p0 + kIPT <= ten) {
            int4 cc = ld_stream(reinterpret_cast<const int4*>(ci + tb + p0));
            c[r][0] = cc.x; c[r][1] = cc.y; c[r][2] = cc.z; c[r][3] = cc.w;
            if (kStreamVals) Vec4<V>::load(vals + tb + p0, a[r]);
        } else {
#pragma unroll
            for (int j = 0; j < kIPT; ++j) {
                const bool in = p0 + j < ten;
                c[r][j] = in ? ld_stream(ci + tb + p0 + j) : 0;
                if (kStreamVals) a[r][j] = in ? ld_stream(vals + tb + p0 + j) : V(0);
            }
        }
        if (!S::kUsesValues) {
#pragma unroll
            for (int j = 0; j < kIPT; ++j) a[r][j] = V(1);
        }
    }
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
        const int p0 = r * kRound + lane * kIPT;
        bool okv[kIPT];
#pragma unroll
        for (int j = 0; j < kIPT; ++j) {
            bool ok = p0 + j < ten;
            if (VALIDATE && ok) ok = (__ldg(mask + (c[r][j] >> 5)) >> (c[r][j] & 31)) & 1u;
            okv[j] = ok;
        }
        if (VALIDATE && S::kUsesValues) {  // value loads of the validated entries only
            if (okv[0] && okv[1] && okv[2] && okv[3]) {
                Vec4<V>::load(vals + tb + p0, a[r]);
            } else {
#pragma unroll
                for (int j = 0; j < kIPT; ++j) a[r][j] = okv[j] ? ld_stream(vals + tb + p0 + j) : V(0);
            }
        }
#pragma unroll
        for (int j = 0; j < kIPT; ++j) {
            xv[r][j] = okv[j] ? __ldg(x + c[r][j]) : V(0);
            if (!okv[j]) c[r][j] = -1;  // marks "no contribution"
            else if (ctr) count_add(ctr, 0, 1);  // values_read: one value load (kernels.hpp:108)
        }
    }

    // ---- row window: rows ws .. row_hi-1 hold this tile's items and the empty
    // rows it owns; row_hi <= next tile's window start + 1 --------------------
    const int64_t ws = __ldg(tile_head + t);
    const int64_t row_hi = min(__ldg(tile_head + t + 1) + 1, rows);
    const int64_t nrow64 = row_hi - ws;
    if (nrow64 + 1 <= kWin) {
        const int nrow = static_cast<int>(nrow64);
        for (int i = lane; i <= nrow; i += 32) {
            const int64_t o = __ldg(ro + ws + i) - tb;
            swin[warp][i] = static_cast<int>(o < -1 ? -1 : (o > kRowTile + 1 ? kRowTile + 1 : o));
        }
        __syncwarp();
        lb_tile_body<V, SR>(SmemWin{&swin[warp][0]}, nrow, ws, t, ten, lane, c, a, xv, y, head_part,
                            tail_part, tail_row);
    } else {
        lb_tile_body<V, SR>(GlobWin{ro, ws, tb}, static_cast<int>(nrow64), ws, t, ten, lane, c, a, xv, y,
                            head_part, tail_part, tail_row);
    }
}

// Combines the partials of rows that span tiles, in tile order, and writes
// the identity into the matrix's empty rows (precomputed list).
template <class V, int SR>
__global__ void row_lb_fixup_kernel(int64_t ntiles, const int64_t* __restrict__ ro,
                                    const V* __restrict__ head_part,
                                    const V* __restrict__ tail_part,
                                    const int64_t* __restrict__ tail_row,
                                    const int32_t* __restrict__ empty_rows, int64_t n_empty,
                                    V* __restrict__ y) {
    using S = Semiring<SR, V>;
    constexpr int64_t kSerial = 32;  // chains longer than this are summed by the whole warp
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    const int64_t nthreads = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = t; i < n_empty; i += nthreads) y[empty_rows[i]] = S::zero();
    const int lane = threadIdx.x & 31;
    const int64_t R = t < ntiles ? tail_row[t] : -1;
    int64_t k = 0;  // continuation tiles t+1 .. t+k hold the rest of row R
    if (R >= 0) {
        const int64_t end = ro[R + 1];
        k = min((end - 1) / kRowTile, ntiles - 1) - t;
    }
    if (R >= 0 && k <= kSerial) {  // short chain: sequential, in tile order
        V s = tail_part[t];
        for (int64_t u = t + 1; u <= t + k; ++u) s = S::add(s, head_part[u]);
        y[R] = s;
    }
    // long chains (hub rows spanning hundreds of tiles): one at a time, every
    // lane summing a strided slice, then a fixed shuffle tree (deterministic)
    unsigned pending = __ballot_sync(kFull, R >= 0 && k > kSerial);
    while (pending) {
        const int src = __ffs(pending) - 1;
        pending &= pending - 1;
        const int64_t ts = __shfl_sync(kFull, t, src);
        const int64_t ks = __shfl_sync(kFull, k, src);
        V s = S::zero();
        for (int64_t u = ts + 1 + lane; u <= ts + ks; u += 32) s = S::add(s, head_part[u]);
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) s = S::add(s, __shfl_xor_sync(kFull, s, d));
        if (lane == src) y[R] = S::add(tail_part[t], s);
    }
}

template <class V, bool VALIDATE, int SR>
void launch_direct(Context& ctx, const Matrix& m, const V* x, const uint32_t* mask, V* y, int G) {
    const int64_t threads = m.rows * G;
    const unsigned blocks = static_cast<unsigned>((threads + kNT - 1) / kNT);
    if (blocks == 0) return;
#define ADA_G(GG)                                                                              \
    case GG:                                                                                   \
        row_direct_kernel<V, GG, VALIDATE, SR><<<blocks, kNT, 0, ctx.stream>>>(                \
            m.rows, m.row_off.as<int64_t>(), m.col_idx.as<int32_t>(), m.vals.as<V>(), x, mask, \
            y, ctx.ctr);                                                                       \
        break;
    if (G == 1 && m.feat[3] <= 8.0) {  // short rows: one unrolled step per row
        if (m.feat[3] <= 5.0)
            row_thread_kernel<V, VALIDATE, SR, 5><<<blocks, kNT, 0, ctx.stream>>>(
                m.rows, m.row_off.as<int64_t>(), m.col_idx.as<int32_t>(), m.vals.as<V>(), x, mask, y, ctx.ctr);
        else
            row_thread_kernel<V, VALIDATE, SR, 8><<<blocks, kNT, 0, ctx.stream>>>(
                m.rows, m.row_off.as<int64_t>(), m.col_idx.as<int32_t>(), m.vals.as<V>(), x, mask, y, ctx.ctr);
        ADA_LAUNCHED(ctx);
        return;
    }
    switch (G) {
        ADA_G(1) ADA_G(2) ADA_G(4) ADA_G(8) ADA_G(16) ADA_G(32)
        default: invalid("lanes_per_row must be a power of two <= 32");
    }
#undef ADA_G
    ADA_LAUNCHED(ctx);
}

template <class V, bool VALIDATE, int SR>
void launch_lb(Context& ctx, const Matrix& m, const V* x, const uint32_t* mask, V* y) {
    if (m.nnz == 0) {
        fill_value<V, SR>(ctx, y, m.rows);
        return;
    }
    const int64_t T = m.n_row_tiles;
    // head partial, tail partial (V) and tail row (int64) per tile
    V* head = static_cast<V*>(ctx.lb_partials.ensure((2 * sizeof(V) + sizeof(int64_t)) * static_cast<size_t>(T)));
    V* tail = head + T;
    int64_t* trow = reinterpret_cast<int64_t*>(tail + T);
    row_lb_kernel<V, VALIDATE, SR><<<static_cast<unsigned>((T + kWarps - 1) / kWarps), kNT, 0, ctx.stream>>>(
        m.rows, m.nnz, T, m.row_off.as<int64_t>(), m.col_idx.as<int32_t>(), m.vals.as<V>(), x, mask,
        m.tile_head.as<int64_t>(), y, head, tail, trow, ctx.ctr);
    ADA_LAUNCHED(ctx);
    if (T > 1 || m.n_empty > 0) {
        const int64_t work = std::max<int64_t>(T, std::min<int64_t>(m.n_empty, 256LL * ctx.sm_count * 8));
        row_lb_fixup_kernel<V, SR><<<static_cast<unsigned>((work + 255) / 256), 256, 0, ctx.stream>>>(
            T, m.row_off.as<int64_t>(), head, tail, trow, m.empty_rows.as<int32_t>(), m.n_empty, y);
        ADA_LAUNCHED(ctx);
    }
}

}  // namespace

// ~4 items per lane (one unrolled iteration of independent loads); measured
// on B200 (tools/kernel_sweep.py): C1 (avg 5) 1 lane 27.7 us vs 4 lanes 48 us;
// C2 (avg 16) 1/2/4/8 lanes 354/313/305/332 us.
int default_lanes_per_row(double avg) {
    int g = 1;
    while (g < 32 && g * 6 <= avg) g <<= 1;
    return g;
}

template <class V, int SR>
void run_row_major(Context& ctx, const Matrix& m, const V* x, const uint32_t* mask, bool lb,
                   int lanes, V* y) {
    const bool validate = mask != nullptr;
    if (!lb) {
        const int G = lanes > 0 ? lanes : default_lanes_per_row(m.feat[5]);
        if (validate) launch_direct<V, true, SR>(ctx, m, x, mask, y, G);
        else launch_direct<V, false, SR>(ctx, m, x, mask, y, G);
    } else {
        if (validate) launch_lb<V, true, SR>(ctx, m, x, mask, y);
        else launch_lb<V, false, SR>(ctx, m, x, mask, y);
    }
}

#define ADA_INST(V, SR) \
    template void run_row_major<V, SR>(Context&, const Matrix&, const V*, const uint32_t*, bool, int, V*);
ADA_INST(float, SR_PLUS_TIMES)
ADA_INST(double, SR_PLUS_TIMES)
ADA_INST(float, SR_OR_AND)
ADA_INST(double, SR_OR_AND)
ADA_INST(float, SR_MIN_PLUS)
ADA_INST(double, SR_MIN_PLUS)
#undef ADA_INST

}  // namespace ada

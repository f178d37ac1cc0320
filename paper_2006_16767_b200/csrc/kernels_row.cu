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
constexpr int kU = 4;

template <class V, int G, bool VALIDATE, int SR>
__global__ void __launch_bounds__(kNT) row_direct_kernel(int64_t rows,
                                                         const int64_t* __restrict__ ro,
                                                         const int32_t* __restrict__ ci,
                                                         const V* __restrict__ vals,
                                                         const V* __restrict__ x,
                                                         const uint32_t* __restrict__ mask,
                                                         V* __restrict__ y) {
    using S = Semiring<SR, V>;
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
            if (ok[j]) acc = S::fma(a[j], xv[j], acc);
    }
#pragma unroll
    for (int d = G / 2; d > 0; d >>= 1) acc = S::add(acc, __shfl_xor_sync(kFull, acc, d, G));
    if (valid && lg == 0) y[row] = acc;
}

// ---------------------------------------------------------------------------
// LB warp-tile kernel.  Warp w of the grid owns items [w*T, (w+1)*T), T =
// kRowTile = 256: two rounds of 128 items, lane l holding the 4 consecutive
// items 4l..4l+3 of each round (one 128-bit load of columns, one/two of
// values: fully coalesced).  All 8 x gathers per lane are issued before any
// is consumed.  The row window of the tile (<= 33 offsets) sits in shared
// memory; lanes find their row by binary search there and walk their 4
// items; runs are joined across lanes by a warp segmented scan (no block
// barriers).  Tiles whose window exceeds 33 rows take the same code path
// with the offsets read from global memory.
// ---------------------------------------------------------------------------
constexpr int kIPT = 4;                       // items per lane per round
constexpr int kRound = 32 * kIPT;             // 128
constexpr int kRounds = kRowTile / kRound;    // 2
constexpr int kWin = 33;                      // offsets held per warp window
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

// Row offsets as seen by one warp tile: a shared-memory window [ws, ws+33)
// when it covers the tile, else global memory.
struct RowWindow {
    const int64_t* __restrict__ ro;
    const int64_t* win;  // smem, valid when fast
    int64_t ws, rows;
    bool fast;
    __device__ int64_t off(int64_t r) const { return fast ? win[r - ws] : __ldg(ro + r); }
    // segment_of (partition.hpp:30-33) for a position inside the tile
    __device__ int64_t row_of(int64_t pos, int64_t hi) const {
        int64_t lo = ws;  // off(ws) <= pos
        while (hi - lo > 1) {
            const int64_t mid = (lo + hi) >> 1;
            if (off(mid) <= pos) lo = mid;
            else hi = mid;
        }
        return lo;
    }
};

template <class V, bool VALIDATE, int SR>
__global__ void __launch_bounds__(kNT) row_lb_kernel(
    int64_t rows, int64_t nnz, int64_t ntiles, const int64_t* __restrict__ ro,
    const int32_t* __restrict__ ci, const V* __restrict__ vals, const V* __restrict__ x,
    const uint32_t* __restrict__ mask, const int64_t* __restrict__ tile_head, V* __restrict__ y,
    V* __restrict__ head_part, V* __restrict__ tail_part, int64_t* __restrict__ tail_row) {
    using S = Semiring<SR, V>;
    __shared__ int64_t swin[kWarps][kWin];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t t = static_cast<int64_t>(blockIdx.x) * kWarps + warp;
    if (t >= ntiles) return;  // whole warp; no block barriers below
    const int64_t tb = t * kRowTile;
    const int64_t te = min(tb + static_cast<int64_t>(kRowTile), nnz);

    // ---- stream the tile: all loads of both rounds issued before use -------
    int c[kRounds][kIPT];
    V a[kRounds][kIPT];
    V xv[kRounds][kIPT];
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
        const int64_t p0 = tb + r * kRound + lane * kIPT;
        if (p0 + kIPT <= te) {
            int4 cc = ld_stream(reinterpret_cast<const int4*>(ci + p0));
            c[r][0] = cc.x; c[r][1] = cc.y; c[r][2] = cc.z; c[r][3] = cc.w;
            if (S::kUsesValues) Vec4<V>::load(vals + p0, a[r]);
        } else {
#pragma unroll
            for (int j = 0; j < kIPT; ++j) {
                const bool in = p0 + j < te;
                c[r][j] = in ? ld_stream(ci + p0 + j) : 0;
                if (S::kUsesValues) a[r][j] = in ? ld_stream(vals + p0 + j) : V(0);
            }
        }
        if (!S::kUsesValues) {
#pragma unroll
            for (int j = 0; j < kIPT; ++j) a[r][j] = V(1);
        }
    }
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
        const int64_t p0 = tb + r * kRound + lane * kIPT;
#pragma unroll
        for (int j = 0; j < kIPT; ++j) {
            bool ok = p0 + j < te;
            if (VALIDATE && ok) ok = (__ldg(mask + (c[r][j] >> 5)) >> (c[r][j] & 31)) & 1u;
            xv[r][j] = ok ? __ldg(x + c[r][j]) : V(0);
            if (!ok) c[r][j] = -1;  // marks "no contribution"
        }
    }

    // ---- row window ----------------------------------------------------------
    const int64_t ws = __ldg(tile_head + t);
    const int64_t wlast = min(ws + kWin - 1, rows);  // last offset index held
    {
        const int64_t r = ws + lane;
        swin[warp][lane] = r <= rows ? __ldg(ro + r) : nnz;
        if (lane == 0) swin[warp][32] = ws + 32 <= rows ? __ldg(ro + ws + 32) : nnz;
    }
    __syncwarp();
    // fast iff every item's row and row end lies in the window
    const bool fast = swin[warp][wlast - ws] >= te || wlast == rows;
    RowWindow W{ro, &swin[warp][0], ws, rows, fast};
    const int64_t hi = fast ? wlast : rows;  // exclusive bound of row_of results (< rows)
    const int64_t row_hi = min(hi, rows);

    // ---- empty rows starting in [tb, te) belong to this tile ----------------
    if (fast) {
        const int64_t r = ws + lane;
        if (r < rows && lane < kWin - 1) {
            const int64_t o0 = swin[warp][lane], o1 = swin[warp][lane + 1];
            if (o0 == o1 && o0 >= tb && o0 < te) y[r] = S::zero();
        }
    } else {
        for (int64_t r = ws + lane; r < rows; r += 32) {
            const int64_t o0 = __ldg(ro + r);
            if (o0 >= te) break;
            if (o0 >= tb && o0 == __ldg(ro + r + 1)) y[r] = S::zero();
        }
    }

    V carry = S::zero();  // value of the row open at the start of the round
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
        const int64_t p0 = tb + r * kRound + lane * kIPT;
        const int64_t p1 = min(p0 + kIPT, te);
        const bool active = p0 < te;
        int64_t row = 0, first_row = 0;
        bool cont = false, head_closed = false, last_open = false, first = true;
        V head_val = S::zero(), acc = S::zero();
        if (active) {
            row = W.row_of(p0, row_hi);
            first_row = row;
            cont = W.off(row) < p0;
            int64_t row_end = W.off(row + 1);
#pragma unroll
            for (int j = 0; j < kIPT; ++j) {
                const int64_t p = p0 + j;
                if (p < p1) {
                    while (p >= row_end) {  // close the run of `row`
                        if (first && cont) {
                            head_closed = true;
                            head_val = acc;
                        } else if (W.off(row) < row_end) {
                            y[row] = acc;  // complete inside this lane
                        }
                        first = false;
                        ++row;
                        row_end = W.off(row + 1);
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
                    y[row] = acc;
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
            if (W.off(first_row) >= tb) y[first_row] = total;  // row began in this tile
            else head_part[t] = total;                           // shared head row
        }
        carry = __shfl_sync(kFull, incl, 31);
    }

    // ---- tile epilogue: the row open at te ----------------------------------
    if (lane == 0) {
        const int64_t R = W.row_of(te - 1, row_hi);
        int64_t tr = -1;
        if (W.off(R + 1) > te) {
            if (W.off(R) >= tb) {
                tail_part[t] = carry;
                tr = R;
            } else {
                head_part[t] = carry;  // tile lies entirely inside row R
            }
        }
        tail_row[t] = tr;
    }
}

// Combines the partials of rows that span tiles, in tile order.
template <class V, int SR>
__global__ void row_lb_fixup_kernel(int64_t ntiles, const int64_t* __restrict__ ro,
                                    const V* __restrict__ head_part,
                                    const V* __restrict__ tail_part,
                                    const int64_t* __restrict__ tail_row, V* __restrict__ y) {
    using S = Semiring<SR, V>;
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (t >= ntiles) return;
    const int64_t R = tail_row[t];
    if (R < 0) return;
    V s = tail_part[t];
    const int64_t end = ro[R + 1];
    for (int64_t u = t + 1; u < ntiles && u * kRowTile < end; ++u) s = S::add(s, head_part[u]);
    y[R] = s;
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
            y);                                                                                \
        break;
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
    V* head = reinterpret_cast<V*>(m.tile_partials.p);
    V* tail = head + T;
    int64_t* trow = reinterpret_cast<int64_t*>(tail + T);
    row_lb_kernel<V, VALIDATE, SR><<<static_cast<unsigned>((T + kWarps - 1) / kWarps), kNT, 0, ctx.stream>>>(
        m.rows, m.nnz, T, m.row_off.as<int64_t>(), m.col_idx.as<int32_t>(), m.vals.as<V>(), x, mask,
        m.tile_head.as<int64_t>(), y, head, tail, trow);
    ADA_LAUNCHED(ctx);
    if (T > 1) {
        row_lb_fixup_kernel<V, SR><<<static_cast<unsigned>((T + 255) / 256), 256, 0, ctx.stream>>>(
            T, m.row_off.as<int64_t>(), head, tail, trow, y);
        ADA_LAUNCHED(ctx);
    }
    if (m.trail_start < m.rows) fill_value<V, SR>(ctx, y + m.trail_start, m.rows - m.trail_start);
}

}  // namespace

int default_lanes_per_row(double avg) {
    int g = 1;
    while (g < 32 && g * 2 <= avg) g <<= 1;  // ~2 items per lane
    return g < 2 ? 2 : g;
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

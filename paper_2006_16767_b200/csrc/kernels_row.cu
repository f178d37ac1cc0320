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
// LB tile kernel
// ---------------------------------------------------------------------------
constexpr int kIPT = 4;                     // items per thread per round
constexpr int kRound = kNT * kIPT;          // 1024
constexpr int kRounds = kRowTile / kRound;  // 2
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

template <class V, bool VALIDATE, int SR>
__global__ void __launch_bounds__(kNT) row_lb_kernel(
    int64_t rows, int64_t nnz, const int64_t* __restrict__ ro, const int32_t* __restrict__ ci,
    const V* __restrict__ vals, const V* __restrict__ x, const uint32_t* __restrict__ mask,
    const int64_t* __restrict__ tile_head, const int64_t* __restrict__ tile_rs, V* __restrict__ y,
    V* __restrict__ head_part, V* __restrict__ tail_part, int64_t* __restrict__ tail_row) {
    using S = Semiring<SR, V>;
    __shared__ int sf[kNT / 32];
    __shared__ V sv[kNT / 32];
    __shared__ V sp[kNT / 32 + 1];

    const int64_t t = blockIdx.x;
    const int64_t tb = t * kRowTile;
    const int64_t te = min(tb + static_cast<int64_t>(kRowTile), nnz);
    const int64_t h = tile_head[t];
    const int64_t hi = min(tile_head[t + 1] + 1, rows);  // search bound (exclusive)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

    // ---- stream the tile: all loads of both rounds issued before use -------
    int c[kRounds][kIPT];
    V a[kRounds][kIPT];
    V xv[kRounds][kIPT];
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
        const int64_t p0 = tb + r * kRound + threadIdx.x * kIPT;
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
        const int64_t p0 = tb + r * kRound + threadIdx.x * kIPT;
#pragma unroll
        for (int j = 0; j < kIPT; ++j) {
            bool ok = p0 + j < te;
            if (VALIDATE && ok) ok = (__ldg(mask + (c[r][j] >> 5)) >> (c[r][j] & 31)) & 1u;
            xv[r][j] = ok ? __ldg(x + c[r][j]) : V(0);
            if (!ok) c[r][j] = -1;  // marks "no contribution"
        }
    }

    // ---- rows owned by this tile that are empty: y = zero (SR identity) ----
    {
        const int64_t rs = tile_rs[t], re = tile_rs[t + 1];
        for (int64_t r = rs + threadIdx.x; r < re; r += kNT)
            if (__ldg(ro + r) == __ldg(ro + r + 1)) y[r] = S::zero();
    }

    V carry = S::zero();  // value of the row open at the start of the round
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
        const int64_t p0 = tb + r * kRound + threadIdx.x * kIPT;
        const int64_t p1 = min(p0 + kIPT, te);
        const bool active = p0 < te;
        int64_t row = 0;
        bool cont = false, head_closed = false, last_open = false;
        V head_val = S::zero(), acc = S::zero();
        bool first = true;
        int64_t first_row = 0;
        if (active) {
            row = segment_search(ro, h, hi, p0);
            first_row = row;
            cont = __ldg(ro + row) < p0;
            int64_t row_end = __ldg(ro + row + 1);
#pragma unroll
            for (int j = 0; j < kIPT; ++j) {
                const int64_t p = p0 + j;
                if (p < p1) {
                    while (p >= row_end) {  // close the run of `row`
                        if (first && cont) {
                            head_closed = true;
                            head_val = acc;
                        } else if (__ldg(ro + row) < row_end) {
                            y[row] = acc;  // complete inside this thread
                        }
                        first = false;
                        ++row;
                        row_end = __ldg(ro + row + 1);
                        acc = S::zero();
                    }
                    if (c[r][j] >= 0) acc = S::fma(a[r][j], xv[r][j], acc);
                }
            }
            last_open = row_end > p1;
            if (!last_open) {  // last run closes exactly at the thread end
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
        // segmented-scan element: pass-through only if the thread is inside
        // one continuing row that stays open.
        SegPair<V> e;
        e.f = (active && first && cont && last_open) ? 0 : 1;
        e.v = (active && last_open) ? acc : S::zero();
        if (!active) e.f = 0, e.v = S::zero();  // neutral
        SegPair<V> inc = warp_seg_inclusive(e, [](V u, V w) { return S::add(u, w); });
        if (lane == 31) {
            sf[warp] = inc.f;
            sv[warp] = inc.v;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            V pcur = carry;
            sp[0] = pcur;
#pragma unroll
            for (int w = 0; w < kNT / 32; ++w) {
                pcur = sf[w] ? sv[w] : S::add(pcur, sv[w]);
                sp[w + 1] = pcur;
            }
        }
        __syncthreads();
        const V wpre = sp[warp];
        const V incl = inc.f ? inc.v : S::add(wpre, inc.v);
        V excl = __shfl_up_sync(kFull, incl, 1);
        if (lane == 0) excl = wpre;
        const V round_carry = sp[kNT / 32];
        if (active && head_closed) {
            const V total = S::add(excl, head_val);
            if (__ldg(ro + first_row) >= tb) y[first_row] = total;  // row began in this tile
            else head_part[t] = total;                               // shared head row
        }
        carry = round_carry;
        __syncthreads();  // sf/sv/sp reuse
    }

    // ---- tile epilogue: the row open at te ----------------------------------
    if (threadIdx.x == 0) {
        const int64_t R = segment_search(ro, h, hi, te - 1);
        const int64_t rend = __ldg(ro + R + 1);
        int64_t tr = -1;
        if (rend > te) {
            if (__ldg(ro + R) >= tb) {
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
    row_lb_kernel<V, VALIDATE, SR><<<static_cast<unsigned>(T), kNT, 0, ctx.stream>>>(
        m.rows, m.nnz, m.row_off.as<int64_t>(), m.col_idx.as<int32_t>(), m.vals.as<V>(), x, mask,
        m.tile_head.as<int64_t>(), m.tile_rs.as<int64_t>(), y, head, tail, trow);
    ADA_LAUNCHED(ctx);
    if (T > 1) {
        row_lb_fixup_kernel<V, SR><<<static_cast<unsigned>((T + 255) / 256), 256, 0, ctx.stream>>>(
            T, m.row_off.as<int64_t>(), head, tail, trow, y);
        ADA_LAUNCHED(ctx);
    }
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

// kernels_col.cu -- the four column-major kernels (CSC scatter driven by the
// nonzeros of x; spmspv_col, kernels.hpp:377-514).  Only the effective
// nonzeros (sparse.hpp:346-359) are read.
//
//   K4 col_direct_atomic  whole support columns per lane group (:394-398),
//                         atomic write-back into a dense y (:436-451)
//   K5 col_direct_sort    same distribution, sort write-back (:489-513)
//   K6 col_lb_atomic      equal effective-nnz tiles over eff_offsets
//                         (:399-432), atomic write-back
//   K7 col_lb_sort        LB distribution, sort write-back
//
// Sort write-back (emit pairs, sort, reduce-by-key):
// (row, a_rj * x_j) pairs are emitted at position eff_offsets[s] + (k -
// col_offsets[j]) -- a deterministic order -- then stably radix-sorted by row
// and reduced by key in order, exact-zero sums dropped (kernels.hpp:331), so
// the sparse y is bitwise reproducible run to run (kernels.hpp:374-376).
// Inputs whose pair count fits one CTA (kSmallPairs) run emit + sort + reduce
// + compaction in a single launch with no host synchronisation: the
// latency-bound sparse end of the sweep.
#include <type_traits>
#include <algorithm>

#include "device.cuh"
#include "internal.hpp"
#include "kernels.hpp"
#include "prims.cuh"

namespace ada {

namespace {

constexpr int kNT = 256;
constexpr int kU = 4;
constexpr int kColTile = 256;            // effective entries per LB warp tile
constexpr int kSmallPairs = 4096;        // single-CTA sort path capacity
constexpr int kSmallNT = 1024;

int blocks_for(int64_t work, int t) {
    return static_cast<int>(std::max<int64_t>(1, (work + t - 1) / t));
}

// ---------------------------------------------------------------------------
// K4: G lanes per support column, atomic scatter
// ---------------------------------------------------------------------------
template <class V, int G, int SR>
__global__ void __launch_bounds__(kNT) col_direct_atomic_kernel(
    int64_t nnz_x, const int32_t* __restrict__ xi, const V* __restrict__ xv,
    const int64_t* __restrict__ co, const int32_t* __restrict__ ri, const V* __restrict__ cv,
    const uint2* __restrict__ cp, V* __restrict__ y, unsigned long long* __restrict__ ctr, float amin) {
    using S = Semiring<SR, V>;
    const int64_t gid = static_cast<int64_t>(blockIdx.x) * kNT + threadIdx.x;
    const int64_t s = gid / G;
    const int lg = threadIdx.x & (G - 1);
    if (s >= nnz_x) return;  // no cross-lane communication below
    const int32_t col = __ldg(xi + s);
    const V xval = __ldg(xv + s);
    const bool safe = addends_normal<SR>(xval, amin);  // once per column (device.cuh combine_batch)
    const int64_t b = __ldg(co + col), e = __ldg(co + col + 1);
    if (ctr && lg == 0) count_add(ctr, 0, static_cast<unsigned long long>(e - b));  // the column's entries
    for (int64_t k0 = b + lg; k0 < e; k0 += G * kU) {
        int r[kU];
        V a[kU];
#pragma unroll
        for (int j = 0; j < kU; ++j) {
            const int64_t k = k0 + j * G;
            if (k < e) {
                if (sizeof(V) == 4 && cp) {  // interleaved (row, value) pair: one 8-B load
                    const uint2 pr = __ldg(cp + k);
                    r[j] = static_cast<int>(pr.x);
                    a[j] = S::kUsesValues ? static_cast<V>(__uint_as_float(pr.y)) : V(1);
                } else {
                    r[j] = __ldg(ri + k);
                    a[j] = S::kUsesValues ? __ldg(cv + k) : V(1);
                }
            } else {
                r[j] = -1;
            }
        }
        V pv[kU];
        bool ok[kU];
#pragma unroll
        for (int j = 0; j < kU; ++j) {
            ok[j] = r[j] >= 0;
            pv[j] = S::mul(a[j], xval);
        }
        combine_batch<SR>(y, r, pv, ok, safe);
    }
}

// ---------------------------------------------------------------------------
// K6 (and K7's emission): equal effective-nnz tiles -- make_partition over
// eff_offsets (kernels.hpp:399-432) with W = ceil(nnz_s / kColTile).  One warp
// per tile of kColTile = 256 effective entries; lane l takes entries 32j + l,
// so a warp instruction reads 32 consecutive entries of one column
// (coalesced).  The tile's support span (found by a warp-cooperative 32-ary
// search over eff_offsets, segment_of, partition.hpp:30-33) is staged in
// shared memory: per support position the CSC start rebased to the effective
// stream (entry_range clipping, kernels.hpp:422-432), the x value and the
// tile-relative end.  Lanes walk it forward; all loads of the 8 entries are
// issued before the write-back.  Spans wider than kColWin positions (many
// empty support columns) read the same data from global memory.
// ---------------------------------------------------------------------------
constexpr int kColWin = 128;

// largest s in [lo, hi) with eff[s] <= pos (warp-cooperative, all lanes)
__device__ __forceinline__ int64_t warp_segment_of(const int64_t* __restrict__ eff, int64_t lo, int64_t hi,
                                                   int64_t pos, int lane) {
    while (hi - lo > 32) {
        const int64_t step = (hi - lo + 31) / 32;
        const int64_t probe = lo + lane * step;
        const unsigned b = __ballot_sync(kFull, probe < hi && __ldg(eff + probe) <= pos);
        const int last = 31 - __clz(b);  // bit 0 is always set (eff[lo] <= pos)
        lo += last * step;
        hi = min(lo + step, hi);
    }
    const int64_t probe = lo + lane;
    const unsigned b = __ballot_sync(kFull, probe < hi && __ldg(eff + probe) <= pos);
    return lo + (31 - __clz(b));
}

// MODE 0: atomic write-back into y (K6); 1: pair emission (K7); 2: the BFS
// push -- each row not yet visited (lv < 0) is claimed once (atomicCAS on
// its level) and appended to the next frontier (keys/pvals = its indices and
// values, bfs_cnt[0] its size, bfs_cnt[1] its effective nnz).
template <class V, int SR, int MODE>
__global__ void __launch_bounds__(kNT) col_lb_kernel(
    int64_t nnz_x, int64_t nnz_s, int64_t ntiles, const int64_t* __restrict__ eff,
    const int32_t* __restrict__ xi, const V* __restrict__ xv, const int64_t* __restrict__ co,
    const int32_t* __restrict__ ri, const V* __restrict__ cv, V* __restrict__ y,
    uint32_t* __restrict__ keys, V* __restrict__ pvals, unsigned long long* __restrict__ ctr,
    int32_t* __restrict__ lv = nullptr, int32_t level = 0, unsigned long long* __restrict__ bfs_cnt = nullptr,
    V bfs_value = V(1), float amin = 3.0e38f) {
    using S = Semiring<SR, V>;
    constexpr bool EMIT = MODE == 1;
    constexpr int kW = kNT / 32;
    constexpr int kJ = kColTile / 32;  // entries per lane
    __shared__ int64_t s_base[kW][kColWin];  // co[xi[s]] - eff[s]
    __shared__ int s_end[kW][kColWin];       // eff[s+1] - tb (clamped)
    __shared__ V s_xv[kW][kColWin];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t t = static_cast<int64_t>(blockIdx.x) * kW + warp;
    if (t >= ntiles) return;
    const int64_t tb = t * kColTile;
    const int ten = static_cast<int>(min(static_cast<int64_t>(kColTile), nnz_s - tb));
    if (lane == 0) {  // the tile's effective entries, each consumed (and emitted) once
        count_add(ctr, 0, static_cast<unsigned long long>(ten));
        if (EMIT) count_add(ctr, 1, static_cast<unsigned long long>(ten));
    }
    const int64_t s_lo = warp_segment_of(eff, 0, nnz_x + 1, tb, lane);
    const int64_t s_hi = warp_segment_of(eff, s_lo, nnz_x + 1, tb + ten - 1, lane);  // inclusive
    const int64_t span = s_hi - s_lo + 1;
    int64_t kidx[kJ];
    V xval[kJ];
    if (span <= kColWin) {
        for (int i = lane; i < span; i += 32) {
            const int64_t s = s_lo + i;
            const int32_t col = __ldg(xi + s);
            const int64_t e0 = __ldg(eff + s), e1 = __ldg(eff + s + 1);
            s_base[warp][i] = __ldg(co + col) - e0;
            const int64_t rel = e1 - tb;
            s_end[warp][i] = static_cast<int>(rel > kColTile + 1 ? kColTile + 1 : rel);
            s_xv[warp][i] = __ldg(xv + s);
        }
        __syncwarp();
        // first support position holding entry `lane`, then walk forward
        int si = 0;
        {
            int hi = static_cast<int>(span);
            while (hi - si > 1) {  // largest si with end[si-1] <= lane, i.e. end[si] > lane
                const int mid = (si + hi) >> 1;
                if (s_end[warp][mid - 1] <= lane) si = mid;
                else hi = mid;
            }
        }
#pragma unroll
        for (int j = 0; j < kJ; ++j) {
            const int i = 32 * j + lane;
            if (i < ten) {
                while (s_end[warp][si] <= i) ++si;
                kidx[j] = s_base[warp][si] + tb + i;
                xval[j] = s_xv[warp][si];
            } else {
                kidx[j] = -1;
            }
        }
    } else {
#pragma unroll
        for (int j = 0; j < kJ; ++j) {
            const int i = 32 * j + lane;
            if (i < ten) {
                const int64_t s = segment_search(eff, s_lo, s_hi + 1, tb + i);
                kidx[j] = __ldg(co + __ldg(xi + s)) - __ldg(eff + s) + tb + i;
                xval[j] = __ldg(xv + s);
            } else {
                kidx[j] = -1;
            }
        }
    }
    int r[kJ];
    V a[kJ];
#pragma unroll
    for (int j = 0; j < kJ; ++j) {
        if (kidx[j] >= 0) {
            r[j] = ld_stream(ri + kidx[j]);
            a[j] = S::kUsesValues ? ld_stream(cv + kidx[j]) : V(1);
        }
    }
    if constexpr (MODE == 2) {
        // claims are appended warp-aggregated: one counter update per warp
        // instruction, slots by the claiming lanes' rank
#pragma unroll
        for (int j = 0; j < kJ; ++j) {
            const int32_t row = kidx[j] >= 0 ? r[j] : 0;
            const bool claim = kidx[j] >= 0 && lv[row] < 0 && atomicCAS(lv + row, -1, level) == -1;
            const unsigned ballot = __ballot_sync(kFull, claim);
            if (ballot == 0u) continue;  // warp-uniform
            const long long deg = warp_sum(claim ? static_cast<long long>(__ldg(co + row + 1) - __ldg(co + row)) : 0ll);
            const int leader = __ffs(ballot) - 1;
            unsigned long long base = 0;
            if (lane == leader) {
                base = atomicAdd(bfs_cnt, static_cast<unsigned long long>(__popc(ballot)));
                atomicAdd(bfs_cnt + 1, static_cast<unsigned long long>(deg));
            }
            base = __shfl_sync(kFull, base, leader);
            if (claim) {
                const unsigned long long slot = base + __popc(ballot & lanemask_lt());
                reinterpret_cast<int32_t*>(keys)[slot] = row;
                pvals[slot] = bfs_value;
            }
        }
        return;
    }
    if (EMIT) {
#pragma unroll
        for (int j = 0; j < kJ; ++j) {
            if (kidx[j] < 0) continue;
            keys[tb + 32 * j + lane] = static_cast<uint32_t>(r[j]);
            pvals[tb + 32 * j + lane] = S::mul(a[j], xval[j]);
        }
    } else {
        V pv[kJ];
        bool ok[kJ];
        bool normal = true;  // the tile's x values rule out subnormal-range products (device.cuh)
#pragma unroll
        for (int j = 0; j < kJ; ++j) {
            ok[j] = kidx[j] >= 0;
            pv[j] = S::mul(a[j], xval[j]);
            normal = normal && (!ok[j] || addends_normal<SR>(xval[j], amin));
        }
        combine_batch<SR>(y, r, pv, ok, __all_sync(kFull, normal));
    }
}

// K5 emission: G lanes per support column write pairs at eff[s] + offset.
template <class V, int G, int SR>
__global__ void __launch_bounds__(kNT) col_direct_emit_kernel(
    int64_t nnz_x, const int64_t* __restrict__ eff, const int32_t* __restrict__ xi,
    const V* __restrict__ xv, const int64_t* __restrict__ co, const int32_t* __restrict__ ri,
    const V* __restrict__ cv, uint32_t* __restrict__ keys, V* __restrict__ pvals,
    unsigned long long* __restrict__ ctr) {
    using S = Semiring<SR, V>;
    const int64_t gid = static_cast<int64_t>(blockIdx.x) * kNT + threadIdx.x;
    const int64_t s = gid / G;
    const int lg = threadIdx.x & (G - 1);
    if (s >= nnz_x) return;
    const int32_t col = __ldg(xi + s);
    const V xval = __ldg(xv + s);
    const int64_t b = __ldg(co + col), e = __ldg(co + col + 1);
    if (ctr && lg == 0) {
        count_add(ctr, 0, static_cast<unsigned long long>(e - b));
        count_add(ctr, 1, static_cast<unsigned long long>(e - b));
    }
    const int64_t out = __ldg(eff + s) - b;
    for (int64_t k = b + lg; k < e; k += G) {
        keys[out + k] = static_cast<uint32_t>(__ldg(ri + k));
        pvals[out + k] = S::mul(S::kUsesValues ? __ldg(cv + k) : V(1), xval);
    }
}

// ---------------------------------------------------------------------------
// Segment sums of the row-sorted pair stream (reduce_sorted_pairs,
// kernels.hpp:323-337) as a parallel segmented scan, so a hub row's long run
// is summed by many threads instead of one: tiles of kSegTile pairs (kSegIPT
// consecutive pairs per thread); pass 1 reduces each tile to (has a run head,
// sum of its last run's part), pass 2 scans those across tiles (one CTA) into
// each tile's carry-in, pass 3 rescans each tile with its carry-in and writes
// the run's sum at the run's LAST pair (keep = sum != zero), where the
// compaction picks it up in row order.  The combine order is a fixed tree:
// deterministic run to run (not the reference's left-to-right order: fp sums
// agree within the 8(c) tolerance).
// ---------------------------------------------------------------------------
constexpr int kSegNT = 256, kSegIPT = 8, kSegTile = kSegNT * kSegIPT;

// Block-wide segmented scan of per-thread aggregates: returns the EXCLUSIVE
// carry of thread t (the combined value of threads < t since the last head,
// identity when none); *tile_inc gets the block's inclusive total.
template <int NT, class V, class Add>
__device__ __forceinline__ SegPair<V> block_seg_exclusive(SegPair<V> p, V ident, Add add, SegPair<V>* smem,
                                                         SegPair<V>* tile_inc) {
    constexpr int NW = NT / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    SegPair<V> inc = warp_seg_inclusive(p, add);
    if (lane == 31) smem[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        SegPair<V> w = lane < NW ? smem[lane] : SegPair<V>{0, ident};
        SegPair<V> wi = warp_seg_inclusive(w, add);
        if (lane < NW) smem[NW + 1 + lane] = wi;  // inclusive over warps
    }
    __syncthreads();
    // exclusive within the warp
    SegPair<V> ex{0, ident};
    {
        const int f = __shfl_up_sync(kFull, inc.f, 1);
        const V v = __shfl_up_sync(kFull, inc.v, 1);
        if (lane > 0) ex = SegPair<V>{f, v};
    }
    if (warp > 0 && !ex.f) {  // nothing in this warp before me resets: add the earlier warps
        const SegPair<V> pw = smem[NW + 1 + warp - 1];
        ex.v = lane > 0 ? add(pw.v, ex.v) : pw.v;
        ex.f = pw.f;
    } else if (warp > 0 && lane == 0) {
        ex = smem[NW + 1 + warp - 1];
    }
    *tile_inc = smem[NW + 1 + NW - 1];
    __syncthreads();
    return ex;
}

template <class V, int SR>
struct SegAdd {
    __device__ V operator()(V a, V b) const { return Semiring<SR, V>::add(a, b); }
};

// The kSegIPT consecutive pairs of one thread (+ the keys just before and
// after): 16-B loads when the group is in range.
template <class V>
__device__ __forceinline__ void seg_load(int64_t n, int64_t i0, const uint32_t* __restrict__ keys,
                                         const V* __restrict__ vals, V ident, uint32_t (&k)[kSegIPT + 2],
                                         V (&v)[kSegIPT]) {
    if (i0 + kSegIPT <= n) {
        const uint4* kp = reinterpret_cast<const uint4*>(keys + i0);
#pragma unroll
        for (int q = 0; q < kSegIPT / 4; ++q) {
            const uint4 w = kp[q];
            k[1 + 4 * q] = w.x;
            k[2 + 4 * q] = w.y;
            k[3 + 4 * q] = w.z;
            k[4 + 4 * q] = w.w;
        }
        constexpr int kVec = 16 / sizeof(V);
        using VV = typename std::conditional<sizeof(V) == 4, float4, double2>::type;
        const VV* vp = reinterpret_cast<const VV*>(vals + i0);
#pragma unroll
        for (int q = 0; q < kSegIPT / kVec; ++q) {
            const VV w = vp[q];
            const V* e = reinterpret_cast<const V*>(&w);
#pragma unroll
            for (int r = 0; r < kVec; ++r) v[q * kVec + r] = e[r];
        }
    } else {
#pragma unroll
        for (int q = 0; q < kSegIPT; ++q) {
            const bool in = i0 + q < n;
            k[1 + q] = in ? keys[i0 + q] : 0u;
            v[q] = in ? vals[i0 + q] : ident;
        }
    }
    k[0] = i0 > 0 && i0 <= n ? keys[i0 - 1] : ~k[1];
    k[kSegIPT + 1] = i0 + kSegIPT < n ? keys[i0 + kSegIPT] : ~k[kSegIPT];
}

// pass 1: per tile (any head in the tile, segmented total = its last run's part)
template <class V, int SR>
__global__ void __launch_bounds__(kSegNT) seg_tile_kernel(int64_t n, const uint32_t* __restrict__ keys,
                                                          const V* __restrict__ vals,
                                                          SegPair<V>* __restrict__ tiles) {
    using S = Semiring<SR, V>;
    __shared__ SegPair<V> sm[2 * (kSegNT / 32) + 2];
    const int64_t i0 = static_cast<int64_t>(blockIdx.x) * kSegTile + threadIdx.x * kSegIPT;
    uint32_t k[kSegIPT + 2];
    V v[kSegIPT];
    seg_load(n, i0, keys, vals, S::zero(), k, v);
    SegPair<V> p{0, S::zero()};
#pragma unroll
    for (int q = 0; q < kSegIPT; ++q) {
        if (i0 + q >= n) break;
        if (k[q + 1] != k[q]) p = SegPair<V>{1, v[q]};  // head (k[0] of pair 0 differs when i0 == 0)
        else p.v = S::add(p.v, v[q]);
    }
    SegPair<V> tot;
    block_seg_exclusive<kSegNT>(p, S::zero(), SegAdd<V, SR>{}, sm, &tot);
    if (threadIdx.x == 0) tiles[blockIdx.x] = tot;
}

// pass 2 (one CTA of 1024): exclusive segmented scan over the tiles -> carry-in
template <class V, int SR>
__global__ void __launch_bounds__(1024) seg_carry_kernel(int64_t ntiles, SegPair<V>* __restrict__ tiles) {
    using S = Semiring<SR, V>;
    __shared__ SegPair<V> sm[2 * 32 + 2];
    const int64_t per = (ntiles + 1023) / 1024;
    const int64_t t0 = threadIdx.x * per, t1 = t0 + per < ntiles ? t0 + per : ntiles;
    SegPair<V> p{0, S::zero()};
    for (int64_t t = t0; t < t1; t += 8) {  // 8 independent loads in flight
        SegPair<V> x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) x[u] = t + u < t1 ? tiles[t + u] : SegPair<V>{0, S::zero()};
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (x[u].f) p = x[u];
            else p.v = S::add(p.v, x[u].v);
        }
    }
    SegPair<V> tot;
    SegPair<V> c = block_seg_exclusive<1024>(p, S::zero(), SegAdd<V, SR>{}, sm, &tot);
    for (int64_t t = t0; t < t1; t += 8) {  // tiles[t] <- carry into tile t (its value before tile t)
        SegPair<V> x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) x[u] = t + u < t1 ? tiles[t + u] : SegPair<V>{0, S::zero()};
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (t + u < t1) tiles[t + u] = c;
            if (x[u].f) c = x[u];
            else c.v = S::add(c.v, x[u].v);
        }
    }
}

// pass 3: rescan each tile from its carry-in; write each run's sum at its last pair
template <class V, int SR>
__global__ void __launch_bounds__(kSegNT) seg_final_kernel(int64_t n, const uint32_t* __restrict__ keys,
                                                           const V* __restrict__ vals,
                                                           const SegPair<V>* __restrict__ carry,
                                                           V* __restrict__ sums, uint8_t* __restrict__ keep) {
    using S = Semiring<SR, V>;
    __shared__ SegPair<V> sm[2 * (kSegNT / 32) + 2];
    const int64_t i0 = static_cast<int64_t>(blockIdx.x) * kSegTile + threadIdx.x * kSegIPT;
    uint32_t k[kSegIPT + 2];
    V v[kSegIPT];
    seg_load(n, i0, keys, vals, S::zero(), k, v);
    SegPair<V> p{0, S::zero()};
#pragma unroll
    for (int q = 0; q < kSegIPT; ++q) {
        if (i0 + q >= n) break;
        if (k[q + 1] != k[q]) p = SegPair<V>{1, v[q]};
        else p.v = S::add(p.v, v[q]);
    }
    SegPair<V> tot;
    SegPair<V> ex = block_seg_exclusive<kSegNT>(p, S::zero(), SegAdd<V, SR>{}, sm, &tot);
    const SegPair<V> cin = carry[blockIdx.x];
    V acc = ex.f ? ex.v : (threadIdx.x > 0 ? S::add(cin.v, ex.v) : cin.v);
    uint8_t kp[kSegIPT];
#pragma unroll
    for (int q = 0; q < kSegIPT; ++q) {
        kp[q] = 0;
        const int64_t i = i0 + q;
        if (i >= n) continue;
        acc = k[q + 1] != k[q] ? v[q] : S::add(acc, v[q]);
        if (i + 1 >= n || k[q + 2] != k[q + 1]) {  // the run's last pair
            sums[i] = acc;
            kp[q] = acc != S::zero() ? 1 : 0;
        }
    }
    if (i0 + kSegIPT <= n) {
        uint2 w;
        w.x = kp[0] | (kp[1] << 8) | (kp[2] << 16) | (static_cast<uint32_t>(kp[3]) << 24);
        w.y = kp[4] | (kp[5] << 8) | (kp[6] << 16) | (static_cast<uint32_t>(kp[7]) << 24);
        *reinterpret_cast<uint2*>(keep + i0) = w;
    } else {
        for (int q = 0; q < kSegIPT && i0 + q < n; ++q) keep[i0 + q] = kp[q];
    }
}

template <class V, int SR>
void seg_reduce(Context& ctx, int64_t n, const uint32_t* keys, const V* vals, V* sums, uint8_t* keep,
                DevBuf& tmp) {
    if (n <= 0) return;
    const int64_t ntiles = (n + kSegTile - 1) / kSegTile;
    SegPair<V>* tiles = static_cast<SegPair<V>*>(tmp.ensure(sizeof(SegPair<V>) * static_cast<size_t>(ntiles)));
    seg_tile_kernel<V, SR><<<static_cast<unsigned>(ntiles), kSegNT, 0, ctx.stream>>>(n, keys, vals, tiles);
    ADA_LAUNCHED(ctx);
    seg_carry_kernel<V, SR><<<1, 1024, 0, ctx.stream>>>(ntiles, tiles);
    ADA_LAUNCHED(ctx);
    seg_final_kernel<V, SR><<<static_cast<unsigned>(ntiles), kSegNT, 0, ctx.stream>>>(n, keys, vals, tiles, sums,
                                                                                     keep);
    ADA_LAUNCHED(ctx);
}

struct KeepIn {
    const uint8_t* keep;
    __device__ int64_t operator()(int64_t i) const { return keep[i]; }
};

template <class V>
struct KeepEpi {
    const uint32_t* keys;
    const V* sums;
    int32_t* out_idx;
    V* out_val;
    __device__ void operator()(int64_t i, int64_t p, int64_t v) const {
        if (v) {
            out_idx[p] = static_cast<int32_t>(keys[i]);
            out_val[p] = sums[i];
        }
    }
};

// ---------------------------------------------------------------------------
// Single-CTA sort write-back for <= kSmallPairs pairs: degrees + scan of the
// support, emission into shared memory, bitonic sort on (row, emission index)
// -- unique keys, hence stable --, reduce-by-key and compaction.
// ---------------------------------------------------------------------------
template <class V, int SR>
__global__ void __launch_bounds__(kSmallNT) col_sort_small_kernel(
    int64_t nnz_x, const int32_t* __restrict__ xi, const V* __restrict__ xv,
    const int64_t* __restrict__ co, const int32_t* __restrict__ ri, const V* __restrict__ cv,
    int32_t* __restrict__ out_idx, V* __restrict__ out_val, int64_t* __restrict__ d_nnz,
    unsigned long long* __restrict__ ctr) {
    using S = Semiring<SR, V>;
    extern __shared__ __align__(16) unsigned char smem[];
    uint64_t* skey = reinterpret_cast<uint64_t*>(smem);                  // kSmallPairs
    V* sval = reinterpret_cast<V*>(skey + kSmallPairs);                  // kSmallPairs
    int* sflag = reinterpret_cast<int*>(sval + kSmallPairs);             // kSmallPairs
    __shared__ int64_t sm_scan[kSmallNT / 32 + 1];
    __shared__ int64_t s_base[kSmallNT];   // col_offsets[col] of the chunk's columns
    __shared__ int s_off[kSmallNT + 1];    // chunk-relative emission offsets
    __shared__ V s_xv[kSmallNT];

    // 1. emit: support processed in chunks of kSmallNT columns.  The chunk's
    //    degrees are scanned, then every thread emits pairs o = tid, tid+NT, ...
    //    (support position by binary search over the offsets), so all matrix
    //    loads of a chunk are independent and in flight together.
    int64_t base = 0;
    for (int64_t c0 = 0; c0 < nnz_x; c0 += kSmallNT) {
        const int64_t s = c0 + threadIdx.x;
        int64_t deg = 0;
        if (s < nnz_x) {
            const int32_t col = xi[s];
            const int64_t b = co[col];
            deg = co[col + 1] - b;
            s_base[threadIdx.x] = b;
            s_xv[threadIdx.x] = xv[s];
        }
        int64_t tot;
        const int64_t off = block_exclusive_sum<kSmallNT>(deg, sm_scan, &tot);
        s_off[threadIdx.x] = static_cast<int>(off);
        if (threadIdx.x == 0) s_off[kSmallNT] = static_cast<int>(tot);
        __syncthreads();
        const int ncols = static_cast<int>(nnz_x - c0 < kSmallNT ? nnz_x - c0 : kSmallNT);
        for (int o = threadIdx.x; o < tot; o += kSmallNT) {
            int lo = 0, hi = ncols;  // largest c with s_off[c] <= o
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (s_off[mid] <= o) lo = mid;
                else hi = mid;
            }
            const int64_t k = s_base[lo] + (o - s_off[lo]);
            const int64_t g = base + o;
            skey[g] = (static_cast<uint64_t>(static_cast<uint32_t>(ri[k])) << 32) |
                      static_cast<uint64_t>(g);
            sval[g] = S::mul(S::kUsesValues ? cv[k] : V(1), s_xv[lo]);
        }
        base += tot;
        __syncthreads();
    }
    const int n = static_cast<int>(base);
    if (threadIdx.x == 0) {  // every emitted pair consumed one matrix entry
        count_add(ctr, 0, static_cast<unsigned long long>(n));
        count_add(ctr, 1, static_cast<unsigned long long>(n));
    }
    int np2 = 1;
    while (np2 < n) np2 <<= 1;
    for (int i = n + threadIdx.x; i < np2; i += kSmallNT) skey[i] = ~0ull;
    __syncthreads();
    // 2. bitonic sort (ascending) of keys with values
    for (int k = 2; k <= np2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < np2; i += kSmallNT) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const bool up = (i & k) == 0;
                    const uint64_t a = skey[i], b = skey[ixj];
                    if ((a > b) == up) {
                        skey[i] = b;
                        skey[ixj] = a;
                        const V t = sval[i];  // padded slots carry garbage values
                        sval[i] = sval[ixj];
                        sval[ixj] = t;
                    }
                }
            }
            __syncthreads();
        }
    }
    // 3. reduce by key: segmented scan, kSmallPairs / kSmallNT consecutive
    //    pairs per thread; a run's sum lands at its LAST pair
    {
        static_assert(kSmallPairs == kSmallNT * 4, "four pairs per thread");
        __shared__ SegPair<V> ssm[2 * (kSmallNT / 32) + 2];
        const int i0 = threadIdx.x * 4;
        uint32_t kk[5];
        V vv[4];
        bool hd[4];
        SegPair<V> p{0, S::zero()};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int i = i0 + q;
            kk[q] = 0;
            vv[q] = S::zero();
            hd[q] = false;
            if (i >= n) continue;
            kk[q] = static_cast<uint32_t>(skey[i] >> 32);
            vv[q] = sval[i];
            hd[q] = i == 0 || static_cast<uint32_t>(skey[i - 1] >> 32) != kk[q];
            if (hd[q]) p = SegPair<V>{1, vv[q]};
            else p.v = S::add(p.v, vv[q]);
        }
        kk[4] = i0 + 4 < n ? static_cast<uint32_t>(skey[i0 + 4] >> 32) : ~kk[3];
        SegPair<V> tot;
        const SegPair<V> ex = block_seg_exclusive<kSmallNT>(p, S::zero(), SegAdd<V, SR>{}, ssm, &tot);
        V acc = ex.v;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int i = i0 + q;
            if (i >= n) break;
            acc = hd[q] ? vv[q] : S::add(acc, vv[q]);
            const bool last = i + 1 >= n || kk[q + 1] != kk[q];
            const int keep = last && acc != S::zero();
            if (keep) sval[i] = acc;  // only kept pairs are read back
            sflag[i] = keep;
        }
    }
    __syncthreads();
    // 4. compaction in row order
    int64_t outbase = 0;
    for (int c0 = 0; c0 < n; c0 += kSmallNT) {
        const int i = c0 + threadIdx.x;
        const int64_t f = i < n ? sflag[i] : 0;
        int64_t tot;
        const int64_t p = block_exclusive_sum<kSmallNT>(f, sm_scan, &tot) + outbase;
        if (f) {
            out_idx[p] = static_cast<int32_t>(skey[i] >> 32);
            out_val[p] = sval[i];
        }
        outbase += tot;
    }
    if (threadIdx.x == 0) *d_nnz = outbase;
}

template <class V, int SR>
size_t small_smem_bytes() {
    return kSmallPairs * (sizeof(uint64_t) + sizeof(V) + sizeof(int));
}

template <class V, int SR>
void launch_small_sort(Context& ctx, const Matrix& m, Vector& x, int32_t* y_idx, V* y_val,
                       int64_t* d_nnz) {
    const size_t smem = small_smem_bytes<V, SR>();
    // per device; a host-side attribute write, no synchronisation
    ADA_CUDA(cudaFuncSetAttribute(col_sort_small_kernel<V, SR>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    col_sort_small_kernel<V, SR><<<1, kSmallNT, smem, ctx.stream>>>(
        x.nnz, x.sp_idx.as<int32_t>(), x.sp_val.as<V>(), m.col_off.as<int64_t>(),
        m.row_idx.as<int32_t>(), m.cvals.as<V>(), y_idx, y_val, d_nnz, ctx.ctr);
    ADA_LAUNCHED(ctx);
}

template <class V, int SR>
void launch_direct_atomic(Context& ctx, const Matrix& m, Vector& x, int G, V* y) {
    const unsigned blocks = static_cast<unsigned>(blocks_for(x.nnz * G, kNT));
#define ADA_G(GG)                                                                            \
    case GG:                                                                                 \
        col_direct_atomic_kernel<V, GG, SR><<<blocks, kNT, 0, ctx.stream>>>(                 \
            x.nnz, x.sp_idx.as<int32_t>(), x.sp_val.as<V>(), m.col_off.as<int64_t>(),        \
            m.row_idx.as<int32_t>(), m.cvals.as<V>(), m.cpairs.as<uint2>(), y, ctx.ctr, m.amin); \
        break;
    switch (G) {
        ADA_G(1) ADA_G(2) ADA_G(4) ADA_G(8) ADA_G(16) ADA_G(32)
        default: invalid("lanes_per_row must be a power of two <= 32");
    }
#undef ADA_G
    ADA_LAUNCHED(ctx);
}

template <class V, int SR>
void launch_direct_emit(Context& ctx, const Matrix& m, Vector& x, int G, uint32_t* keys, V* pv) {
    const unsigned blocks = static_cast<unsigned>(blocks_for(x.nnz * G, kNT));
#define ADA_G(GG)                                                                            \
    case GG:                                                                                 \
        col_direct_emit_kernel<V, GG, SR><<<blocks, kNT, 0, ctx.stream>>>(                   \
            x.nnz, x.eff.as<int64_t>(), x.sp_idx.as<int32_t>(), x.sp_val.as<V>(),            \
            m.col_off.as<int64_t>(), m.row_idx.as<int32_t>(), m.cvals.as<V>(), keys, pv,     \
            ctx.ctr);                                                                        \
        break;
    switch (G) {
        ADA_G(1) ADA_G(2) ADA_G(4) ADA_G(8) ADA_G(16) ADA_G(32)
        default: invalid("lanes_per_row must be a power of two <= 32");
    }
#undef ADA_G
    ADA_LAUNCHED(ctx);
}

// KernelConfig::atomic_private_accumulators (kernels.hpp:152-162, :452-478):
// each CTA accumulates its share into a shared-memory copy of y (all rows fit),
// then flushes the touched rows with one global atomic each.  Shares follow
// the reference: Direct = chunk_range of support positions (parallel.hpp:153),
// LoadBalanced = make_partition of the effective entries with W = #CTAs.
// (On the GPU the flush is atomic, so like the plain atomic path the result is
// deterministic only up to summation order.)
template <class V, int SR, bool LB>
__global__ void __launch_bounds__(kNT) col_private_kernel(
    int64_t nnz_x, int64_t nnz_s, int64_t rows, const int64_t* __restrict__ eff,
    const int32_t* __restrict__ xi, const V* __restrict__ xv, const int64_t* __restrict__ co,
    const int32_t* __restrict__ ri, const V* __restrict__ cv, V* __restrict__ y,
    unsigned long long* __restrict__ ctr) {
    using S = Semiring<SR, V>;
    extern __shared__ __align__(16) unsigned char priv_smem[];
    V* acc = reinterpret_cast<V*>(priv_smem);
    for (int64_t r = threadIdx.x; r < rows; r += kNT) acc[r] = S::zero();
    __syncthreads();
    const int64_t W = gridDim.x, c = blockIdx.x;
    if (LB) {
        const int64_t ib = nnz_s * c / W, ie = nnz_s * (c + 1) / W;
        const int64_t len = ie - ib;
        if (threadIdx.x == 0) count_add(ctr, 0, static_cast<unsigned long long>(len));
        const int64_t p0 = ib + len * threadIdx.x / kNT, p1 = ib + len * (threadIdx.x + 1) / kNT;
        if (p0 < p1) {
            int64_t s = segment_search(eff, 0, nnz_x + 1, p0);
            int64_t s_end = __ldg(eff + s + 1);
            int64_t base = __ldg(co + __ldg(xi + s)) - __ldg(eff + s);
            V xval = __ldg(xv + s);
            for (int64_t p = p0; p < p1; ++p) {
                while (p >= s_end) {
                    ++s;
                    s_end = __ldg(eff + s + 1);
                    base = __ldg(co + __ldg(xi + s)) - __ldg(eff + s);
                    xval = __ldg(xv + s);
                }
                const int64_t k = base + p;
                AtomicCombine<SR>::apply(acc + __ldg(ri + k), S::mul(S::kUsesValues ? __ldg(cv + k) : V(1), xval));
            }
        }
    } else {
        const int64_t sb = nnz_x * c / W, se = nnz_x * (c + 1) / W;
        for (int64_t s = sb + threadIdx.x; s < se; s += kNT) {
            const int32_t col = __ldg(xi + s);
            const V xval = __ldg(xv + s);
            count_add(ctr, 0, static_cast<unsigned long long>(__ldg(co + col + 1) - __ldg(co + col)));
            for (int64_t k = __ldg(co + col); k < __ldg(co + col + 1); ++k)
                AtomicCombine<SR>::apply(acc + __ldg(ri + k), S::mul(S::kUsesValues ? __ldg(cv + k) : V(1), xval));
        }
    }
    __syncthreads();
    for (int64_t r = threadIdx.x; r < rows; r += kNT)
        if (acc[r] != S::zero()) AtomicCombine<SR>::apply(y + r, acc[r]);
}

constexpr size_t kPrivateSmem = 200 * 1024;

template <class V, int SR>
bool launch_private(Context& ctx, const Matrix& m, Vector& x, bool lb, V* y) {
    const size_t smem = sizeof(V) * static_cast<size_t>(m.rows);
    if (smem > kPrivateSmem || m.rows == 0) return false;  // y does not fit: plain atomic path
    const int64_t nnz_s = lb ? vector_nnz_s(ctx, x, m) : 0;
    if (lb) vector_ensure_eff(ctx, x, m, SR);  // nnz_s may be known without the offsets
    const unsigned grid = static_cast<unsigned>(2 * ctx.sm_count);
    if (lb) {
        ADA_CUDA(cudaFuncSetAttribute(col_private_kernel<V, SR, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(kPrivateSmem)));
        col_private_kernel<V, SR, true><<<grid, kNT, smem, ctx.stream>>>(
            x.nnz, nnz_s, m.rows, x.eff.as<int64_t>(), x.sp_idx.as<int32_t>(), x.sp_val.as<V>(),
            m.col_off.as<int64_t>(), m.row_idx.as<int32_t>(), m.cvals.as<V>(), y, ctx.ctr);
    } else {
        ADA_CUDA(cudaFuncSetAttribute(col_private_kernel<V, SR, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(kPrivateSmem)));
        col_private_kernel<V, SR, false><<<grid, kNT, smem, ctx.stream>>>(
            x.nnz, 0, m.rows, nullptr, x.sp_idx.as<int32_t>(), x.sp_val.as<V>(), m.col_off.as<int64_t>(),
            m.row_idx.as<int32_t>(), m.cvals.as<V>(), y, ctx.ctr);
    }
    ADA_LAUNCHED(ctx);
    return true;
}

}  // namespace

// BFS push (OR_AND) over the LB tiles of K6: x needs its eff offsets;
// next_idx / next_val receive the next frontier, cnt[0..1] its size and nnz_s.
template <class V>
void bfs_push_lb(Context& ctx, const Matrix& m, Vector& x, int32_t* lv, int32_t level, int32_t* next_idx,
                 V* next_val, V value, unsigned long long* cnt) {
    const int64_t nnz_s = vector_nnz_s(ctx, x, m);
    if (nnz_s == 0) return;
    vector_ensure_eff(ctx, x, m, SR_OR_AND);
    const int64_t tiles = (nnz_s + kColTile - 1) / kColTile;
    col_lb_kernel<V, SR_OR_AND, 2><<<static_cast<unsigned>((tiles + 7) / 8), kNT, 0, ctx.stream>>>(
        x.nnz, nnz_s, tiles, x.eff.as<int64_t>(), x.sp_idx.as<int32_t>(), x.sp_val.as<V>(), m.col_off.as<int64_t>(),
        m.row_idx.as<int32_t>(), m.cvals.as<V>(), nullptr, reinterpret_cast<uint32_t*>(next_idx), next_val, ctx.ctr,
        lv, level, cnt, value);
    ADA_LAUNCHED(ctx);
}
template void bfs_push_lb<float>(Context&, const Matrix&, Vector&, int32_t*, int32_t, int32_t*, float*, float,
                                 unsigned long long*);
template void bfs_push_lb<double>(Context&, const Matrix&, Vector&, int32_t*, int32_t, int32_t*, double*, double,
                                  unsigned long long*);

template <class V, int SR>
void run_col_major(Context& ctx, const Matrix& m, Vector& x, bool lb, bool sort, bool private_acc,
                   int lanes, V* y_dense, int32_t* y_idx, V* y_val, int64_t* d_nnz,
                   int64_t* h_nnz) {
    vector_ensure_sparse(ctx, x, SR);
    const int G = lanes > 0 ? lanes : default_lanes_per_row(m.avg_col);
    *h_nnz = -1;
    if (!sort) {
        // row-segmented write-back (kernels_colseg.cu: every row stored once,
        // no identity fill), opt-in with ADASPMV_COLSEG=1 -- measured at par
        // with the L2-atomic path on C4 and slower on C2, so not the default
        if (x.nnz > 0 && m.nnz > 0 && !private_acc && colseg_mode() == 1 &&
            run_col_segmented<V, SR>(ctx, m, x, y_dense))
            return;
        // atomic write-back into a dense y initialised to the identity
        fill_value<V, SR>(ctx, y_dense, m.rows);
        if (x.nnz == 0 || m.nnz == 0) return;
        if (private_acc && launch_private<V, SR>(ctx, m, x, lb, y_dense)) return;
        if (!lb) {
            launch_direct_atomic<V, SR>(ctx, m, x, G, y_dense);
            return;
        }
        const int64_t nnz_s = vector_nnz_s(ctx, x, m);
        if (nnz_s == 0) return;
        vector_ensure_eff(ctx, x, m, SR);  // nnz_s may be known without the offsets
        const int64_t tiles = (nnz_s + kColTile - 1) / kColTile;
        col_lb_kernel<V, SR, 0><<<static_cast<unsigned>((tiles + 7) / 8), kNT, 0, ctx.stream>>>(
            x.nnz, nnz_s, tiles, x.eff.as<int64_t>(), x.sp_idx.as<int32_t>(), x.sp_val.as<V>(),
            m.col_off.as<int64_t>(), m.row_idx.as<int32_t>(), m.cvals.as<V>(), y_dense, nullptr,
            nullptr, ctx.ctr, nullptr, 0, nullptr, V(1), m.amin);
        ADA_LAUNCHED(ctx);
        return;
    }
    // ---- sort write-back -> sparse y ---------------------------------------
    if (x.nnz == 0 || m.nnz == 0) {
        ADA_CUDA(cudaMemsetAsync(d_nnz, 0, sizeof(int64_t), ctx.stream));
        *h_nnz = 0;
        return;
    }
    // pair-count bound without a device round trip when possible
    int64_t bound = m.max_col_deg > 0 && x.nnz <= kSmallPairs ? x.nnz * m.max_col_deg : INT64_MAX;
    if (x.nnz_s >= 0 && x.nnz_s_matrix == m.id) bound = x.nnz_s;
    if (bound > kSmallPairs) bound = vector_nnz_s(ctx, x, m);
    if (bound <= kSmallPairs && x.nnz <= kSmallPairs) {
        launch_small_sort<V, SR>(ctx, m, x, y_idx, y_val, d_nnz);
        return;
    }
    const int64_t nnz_s = vector_nnz_s(ctx, x, m);
    if (nnz_s == 0) {  // every support column is empty: no pairs, empty y
        ADA_CUDA(cudaMemsetAsync(d_nnz, 0, sizeof(int64_t), ctx.stream));
        *h_nnz = 0;
        return;
    }
    vector_ensure_eff(ctx, x, m, SR);  // nnz_s may be known without the offsets
    DevBuf& kb0 = ctx.scratch[0];
    DevBuf& kb1 = ctx.scratch[1];
    DevBuf& vb0 = ctx.scratch[2];
    DevBuf& vb1 = ctx.scratch[3];
    const size_t z = static_cast<size_t>(nnz_s);
    uint32_t* k0 = static_cast<uint32_t*>(kb0.ensure(sizeof(uint32_t) * z));
    uint32_t* k1 = static_cast<uint32_t*>(kb1.ensure(sizeof(uint32_t) * z));
    V* v0 = static_cast<V*>(vb0.ensure(sizeof(V) * z));
    V* v1 = static_cast<V*>(vb1.ensure(sizeof(V) * z));
    if (!lb) {
        launch_direct_emit<V, SR>(ctx, m, x, G, k0, v0);
    } else {
        const int64_t tiles = (nnz_s + kColTile - 1) / kColTile;
        col_lb_kernel<V, SR, 1><<<static_cast<unsigned>((tiles + 7) / 8), kNT, 0, ctx.stream>>>(
            x.nnz, nnz_s, tiles, x.eff.as<int64_t>(), x.sp_idx.as<int32_t>(), x.sp_val.as<V>(),
            m.col_off.as<int64_t>(), m.row_idx.as<int32_t>(), m.cvals.as<V>(), nullptr, k0, v0, ctx.ctr);
        ADA_LAUNCHED(ctx);
    }
    DevBuf& counts = ctx.scratch[6];
    DevBuf& scan_tmp = ctx.scratch[7];
    DevBuf& sums = ctx.scratch[8];
    DevBuf& keep = ctx.scratch[9];
    const int which = radix_sort_pairs<V>(ctx, k0, v0, k1, v1, nnz_s, bits_for(m.rows), counts,
                                          scan_tmp);
    const uint32_t* sk = which ? k1 : k0;
    const V* sv = which ? v1 : v0;
    V* ssum = static_cast<V*>(sums.ensure(sizeof(V) * z));
    uint8_t* kp = static_cast<uint8_t*>(keep.ensure(z));
    seg_reduce<V, SR>(ctx, nnz_s, sk, sv, ssum, kp, ctx.scratch[4]);
    scan3(ctx, nnz_s, KeepIn{kp}, KeepEpi<V>{sk, ssum, y_idx, y_val}, d_nnz, scan_tmp);
}

namespace {
__global__ void rows_to_keys_kernel(int64_t n, const int32_t* __restrict__ rows,
                                    uint32_t* __restrict__ keys) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < n) keys[i] = static_cast<uint32_t>(rows[i]);
}

template <class V>
int64_t sort_reduce_t(Context& ctx, int64_t n, const int32_t* d_rows, const void* d_vals,
                      int64_t nrows, int32_t* out_idx, V* out_val) {
    if (n == 0) return 0;
    const size_t z = static_cast<size_t>(n);
    DevBuf k0, k1, v0, v1, counts, scan_tmp, sums, keep;
    uint32_t* pk0 = static_cast<uint32_t*>(k0.ensure(sizeof(uint32_t) * z));
    uint32_t* pk1 = static_cast<uint32_t*>(k1.ensure(sizeof(uint32_t) * z));
    V* pv0 = static_cast<V*>(v0.ensure(sizeof(V) * z));
    V* pv1 = static_cast<V*>(v1.ensure(sizeof(V) * z));
    rows_to_keys_kernel<<<blocks_for(n, 256), 256, 0, ctx.stream>>>(n, d_rows, pk0);
    ADA_LAUNCHED(ctx);
    ADA_CUDA(cudaMemcpyAsync(pv0, d_vals, sizeof(V) * z, cudaMemcpyDeviceToDevice, ctx.stream));
    const int which = radix_sort_pairs<V>(ctx, pk0, pv0, pk1, pv1, n, bits_for(nrows), counts, scan_tmp);
    const uint32_t* sk = which ? pk1 : pk0;
    const V* sv = which ? pv1 : pv0;
    V* ssum = static_cast<V*>(sums.ensure(sizeof(V) * z));
    uint8_t* kp = static_cast<uint8_t*>(keep.ensure(z));
    DevBuf seg_tmp;
    seg_reduce<V, SR_PLUS_TIMES>(ctx, n, sk, sv, ssum, kp, seg_tmp);
    scan3(ctx, n, KeepIn{kp}, KeepEpi<V>{sk, ssum, out_idx, out_val}, ctx.dscal(1), scan_tmp);
    const int64_t r = ctx.fetch_scalar(ctx.dscal(1));
    return r;
}
}  // namespace

int64_t sort_reduce_pairs_device(Context& ctx, int64_t npairs, const int32_t* d_rows,
                                 const void* d_vals, int dtype, int64_t nrows, int32_t* d_out_idx,
                                 void* d_out_val) {
    if (dtype == ADASPMV_F64)
        return sort_reduce_t<double>(ctx, npairs, d_rows, d_vals, nrows, d_out_idx,
                                     static_cast<double*>(d_out_val));
    return sort_reduce_t<float>(ctx, npairs, d_rows, d_vals, nrows, d_out_idx,
                                static_cast<float*>(d_out_val));
}

#define ADA_INST(V, SR)                                                                       \
    template void run_col_major<V, SR>(Context&, const Matrix&, Vector&, bool, bool, bool, int, \
                                       V*, int32_t*, V*, int64_t*, int64_t*);
ADA_INST(float, SR_PLUS_TIMES)
ADA_INST(double, SR_PLUS_TIMES)
ADA_INST(float, SR_OR_AND)
ADA_INST(double, SR_OR_AND)
ADA_INST(float, SR_MIN_PLUS)
ADA_INST(double, SR_MIN_PLUS)
#undef ADA_INST

}  // namespace ada

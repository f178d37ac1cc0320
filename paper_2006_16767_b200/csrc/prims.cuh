// prims.cuh -- device-wide primitives written for this library (no CUB /
// Thrust on the product path): a deterministic 3-phase exclusive scan with a
// user epilogue (used for effective-nnz offsets, stream compaction and radix
// digit offsets) and a stable LSD radix sort of (key, payload) pairs.
//
// These replace the reference's CPU-side parallel primitives
// (parallel_reduce parallel.hpp:165-180, the 3-pass count/scan/scatter of
// dense_to_sparse sparse.hpp:298-319, std::sort kernels.hpp:503-504).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "device.cuh"
#include "internal.hpp"

namespace ada {

// ---------------------------------------------------------------------------
// scan3: out = exclusive prefix of in(i) over i in [0, n), delivered to
// epi(i, prefix, value) for every i; *d_total (device int64) = total.
// `In`  : __device__ int64_t operator()(int64_t i) const  (i < n)
// `Epi` : __device__ void operator()(int64_t i, int64_t prefix, int64_t v) const
// Deterministic: block-local sequential order, fixed tile grid.
// ---------------------------------------------------------------------------
constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

// Items of a tile are read STRIPED (item base + j*kScanThreads + t to thread
// t, j < kScanItems), so each warp load covers 32 consecutive items.
template <class In>
__global__ void __launch_bounds__(kScanThreads) scan_tile_sums_kernel(int64_t n, In in,
                                                                       int64_t* tile_sums) {
    __shared__ int64_t sm[kScanThreads / 32 + 1];
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile + threadIdx.x;
    int64_t s = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j)
        if (base + j * kScanThreads < n) s += in(base + j * kScanThreads);
    int64_t total;
    (void)block_exclusive_sum<kScanThreads>(s, sm, &total);
    if (threadIdx.x == 0) tile_sums[blockIdx.x] = total;
}

// Single CTA: exclusive scan of tile_sums[0..nt) in place; total -> *d_total.
__global__ void __launch_bounds__(1024) scan_spine_kernel(int64_t nt, int64_t* tile_sums,
                                                          int64_t* d_total);

template <class In, class Epi>
__global__ void __launch_bounds__(kScanThreads) scan_apply_kernel(int64_t n, In in, Epi epi,
                                                                  const int64_t* tile_offsets,
                                                                  int64_t* d_total,
                                                                  int single) {
    // striped items: row j of the tile = items [j*256, (j+1)*256), warp w
    // holds its 32-item slice; prefixes: warp scan within the slice, then
    // the slices' totals in (row, warp) order
    constexpr int NW = kScanThreads / 32;
    __shared__ int64_t wt[kScanItems * NW];
    __shared__ int64_t woff[kScanItems * NW + 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile + threadIdx.x;
    int64_t v[kScanItems], inc[kScanItems];
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        const int64_t i = base + j * kScanThreads;
        v[j] = i < n ? in(i) : 0;
        inc[j] = warp_inclusive_sum(v[j]);
        if (lane == 31) wt[j * NW + warp] = inc[j];
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // exclusive scan of the kScanItems * NW slice totals (64 <= 2 per lane)
        static_assert(kScanItems * NW == 64, "two slice totals per lane");
        const int64_t a = wt[2 * lane], b = wt[2 * lane + 1];
        const int64_t pair = a + b;
        const int64_t pinc = warp_inclusive_sum(pair);
        const int64_t pex = pinc - pair;
        woff[2 * lane] = pex;
        woff[2 * lane + 1] = pex + a;
        if (lane == 31) woff[kScanItems * NW] = pinc;
    }
    __syncthreads();
    const int64_t off = single ? 0 : tile_offsets[blockIdx.x];
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        const int64_t i = base + j * kScanThreads;
        if (i < n) epi(i, off + woff[j * NW + warp] + inc[j] - v[j], v[j]);
    }
    if (single && threadIdx.x == 0 && d_total) *d_total = woff[kScanItems * NW];
}

__global__ void scan_zero_kernel(int64_t* p);

// Host driver.  `tmp` must hold max(1, ceil(n/kScanTile)) int64.  d_total
// (device int64, or the device alias of mapped host memory) gets the total.
template <class In, class Epi>
void scan3(Context& ctx, int64_t n, In in, Epi epi, int64_t* d_total, DevBuf& tmp) {
    if (n <= 0) {  // d_total may be mapped host memory: a store, not a memset
        if (d_total) {
            scan_zero_kernel<<<1, 1, 0, ctx.stream>>>(d_total);
            ADA_LAUNCHED(ctx);
        }
        return;
    }
    const int64_t nt = (n + kScanTile - 1) / kScanTile;
    if (nt == 1) {
        scan_apply_kernel<<<1, kScanThreads, 0, ctx.stream>>>(n, in, epi, nullptr, d_total, 1);
        ADA_LAUNCHED(ctx);
        return;
    }
    int64_t* ts = static_cast<int64_t*>(tmp.ensure(sizeof(int64_t) * static_cast<size_t>(nt)));
    scan_tile_sums_kernel<<<static_cast<unsigned>(nt), kScanThreads, 0, ctx.stream>>>(n, in, ts);
    ADA_LAUNCHED(ctx);
    scan_spine_kernel<<<1, 1024, 0, ctx.stream>>>(nt, ts, d_total);
    ADA_LAUNCHED(ctx);
    scan_apply_kernel<<<static_cast<unsigned>(nt), kScanThreads, 0, ctx.stream>>>(n, in, epi, ts,
                                                                                   nullptr, 0);
    ADA_LAUNCHED(ctx);
}

// Common functors --------------------------------------------------------------
struct WriteExclusive {  // out[i] = prefix; out[n] = total written via d_total alias
    int64_t* out;
    __device__ void operator()(int64_t i, int64_t p, int64_t) const { out[i] = p; }
};

// ---------------------------------------------------------------------------
// Stable LSD radix sort of (uint32 key, P payload), 8-bit digits.
// Tile = 8 warps x 16 rounds x 32 lanes; item i of a tile is handled by warp
// i/512, round (i%512)/32, lane i%32, so warp-match ranks + per-warp running
// digit counts + a digit-major (digit, tile) offset scan give a stable order.
// ---------------------------------------------------------------------------
constexpr int kRsThreads = 256;
constexpr int kRsRounds = 16;
constexpr int kRsTile = kRsThreads * kRsRounds;  // 4096
constexpr int kRsRadix = 256;

__global__ void __launch_bounds__(kRsThreads) radix_upsweep_kernel(const uint32_t* __restrict__ keys,
                                                                   int64_t n, int shift,
                                                                   int64_t ntiles,
                                                                   int64_t* __restrict__ counts);

template <class P>
__global__ void __launch_bounds__(kRsThreads) radix_downsweep_kernel(
    const uint32_t* __restrict__ kin, const P* __restrict__ pin, uint32_t* __restrict__ kout,
    P* __restrict__ pout, int64_t n, int shift, int64_t ntiles, const int64_t* __restrict__ offs) {
    __shared__ int wh[kRsThreads / 32][kRsRadix];
    __shared__ int64_t sbase[kRsRadix];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t tile = blockIdx.x;
    for (int i = threadIdx.x; i < (kRsThreads / 32) * kRsRadix; i += kRsThreads) (&wh[0][0])[i] = 0;
    sbase[threadIdx.x] = offs[static_cast<int64_t>(threadIdx.x) * ntiles + tile];
    __syncthreads();
    const int64_t wbase = tile * kRsTile + static_cast<int64_t>(warp) * (kRsRounds * 32);
    uint32_t key[kRsRounds];
    P pay[kRsRounds];
    int pos[kRsRounds];
#pragma unroll
    for (int r = 0; r < kRsRounds; ++r) {
        const int64_t i = wbase + r * 32 + lane;
        if (i < n) {
            key[r] = kin[i];
            pay[r] = pin[i];
        } else {
            key[r] = 0;
        }
    }
#pragma unroll
    for (int r = 0; r < kRsRounds; ++r) {
        const int64_t i = wbase + r * 32 + lane;
        const bool valid = i < n;
        const unsigned act = __ballot_sync(kFull, valid);
        const int d = (key[r] >> shift) & (kRsRadix - 1);
        if (valid) {
            const unsigned peers = __match_any_sync(act, d);
            const int rank = __popc(peers & lanemask_lt());
            pos[r] = wh[warp][d] + rank;
            __syncwarp(act);
            if (rank == 0) wh[warp][d] += __popc(peers);
        }
        __syncwarp();
    }
    __syncthreads();
    __shared__ int toff[kRsRadix];
    __shared__ int sm_scan[kRsThreads / 32 + 1];
    {   // per-digit exclusive prefix over warps (thread = digit), then over digits
        const int d = threadIdx.x;
        int run = 0;
#pragma unroll
        for (int w = 0; w < kRsThreads / 32; ++w) {
            const int t = wh[w][d];
            wh[w][d] = run;
            run += t;
        }
        int total;
        toff[d] = block_exclusive_sum<kRsThreads>(run, sm_scan, &total);
    }
    __syncthreads();
    // stage the tile in digit order in shared memory, then write each digit's
    // run contiguously (coalesced) instead of scattering item by item
    extern __shared__ __align__(16) unsigned char rs_smem[];
    uint32_t* skey = reinterpret_cast<uint32_t*>(rs_smem);
    P* spay = reinterpret_cast<P*>(rs_smem + kRsTile * sizeof(uint32_t));
#pragma unroll
    for (int r = 0; r < kRsRounds; ++r) {
        const int64_t i = wbase + r * 32 + lane;
        if (i < n) {
            const int d = (key[r] >> shift) & (kRsRadix - 1);
            const int p = toff[d] + wh[warp][d] + pos[r];
            skey[p] = key[r];
            spay[p] = pay[r];
        }
    }
    __syncthreads();
    const int tile_n = static_cast<int>(min(static_cast<int64_t>(kRsTile), n - tile * kRsTile));
    for (int i = threadIdx.x; i < tile_n; i += kRsThreads) {
        const uint32_t k = skey[i];
        const int d = (k >> shift) & (kRsRadix - 1);
        const int64_t o = sbase[d] + (i - toff[d]);
        kout[o] = k;
        pout[o] = spay[i];
    }
}

struct CountsIn {
    const int64_t* c;
    __device__ int64_t operator()(int64_t i) const { return c[i]; }
};

// Sorts n pairs on the low `bits` bits of the keys.  Buffers (k0,p0) hold the
// input; (k1,p1) are scratch of the same size.  Returns 0 if the result ended
// in (k0,p0), 1 if in (k1,p1).
template <class P>
int radix_sort_pairs(Context& ctx, uint32_t* k0, P* p0, uint32_t* k1, P* p1, int64_t n, int bits,
                     DevBuf& counts_buf, DevBuf& scan_tmp) {
    if (n <= 1 || bits <= 0) return 0;
    const int64_t ntiles = (n + kRsTile - 1) / kRsTile;
    int64_t* counts = static_cast<int64_t*>(
        counts_buf.ensure(sizeof(int64_t) * static_cast<size_t>(kRsRadix * ntiles)));
    const size_t smem = kRsTile * (sizeof(uint32_t) + sizeof(P));
    ADA_CUDA(cudaFuncSetAttribute(radix_downsweep_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    int cur = 0;
    for (int shift = 0; shift < bits; shift += 8) {
        uint32_t* kin = cur ? k1 : k0;
        P* pin = cur ? p1 : p0;
        uint32_t* kout = cur ? k0 : k1;
        P* pout = cur ? p0 : p1;
        radix_upsweep_kernel<<<static_cast<unsigned>(ntiles), kRsThreads, 0, ctx.stream>>>(
            kin, n, shift, ntiles, counts);
        ADA_LAUNCHED(ctx);
        scan3(ctx, kRsRadix * ntiles, CountsIn{counts}, WriteExclusive{counts}, nullptr, scan_tmp);
        radix_downsweep_kernel<P><<<static_cast<unsigned>(ntiles), kRsThreads, smem, ctx.stream>>>(
            kin, pin, kout, pout, n, shift, ntiles, counts);
        ADA_LAUNCHED(ctx);
        cur ^= 1;
    }
    return cur;
}

inline int bits_for(int64_t max_key_exclusive) {
    int b = 0;
    while (b < 32 && (int64_t(1) << b) < max_key_exclusive) ++b;
    return b;
}

}  // namespace ada

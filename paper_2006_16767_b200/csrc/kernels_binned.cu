// kernels_binned.cu -- row-block ("binned") execution of the row-major
// kernels K0 spmv_direct / K2 row_direct for matrices whose x gathers are
// scattered.
//
// Why: in CSR order every nonzero gathers x[col] on its own; for a matrix
// whose columns are spread (uniform random, R-MAT) each gather is a separate
// 128-B L1TEX wavefront and L2 request, and the SM's ~1 wavefront/cycle
// bounds the multiply at ~35 % of HBM.  Here the rows
// are cut into bins of R rows (R*V bytes fit one CTA's shared memory); the
// entries of a bin are stored in COLUMN order, so the 32 gathers of a warp
// instruction fall on a few consecutive lines of x (~9 instead of 32 at C2),
// and each product is accumulated into the bin's y segment held in shared
// memory.  One CTA owns a bin (the reference's Direct distribution: every
// worker a contiguous block of rows, kernels.hpp:242-250); bins heavier than
// the tile cap are split into column-contiguous tiles whose partial segments
// are combined with global atomics (y pre-filled with the identity).
//
// Layout (Matrix::BinLayout, built once on the device from the CSC): the CSC
// order (columns ascending, rows ascending within a column: csr_to_csc,
// sparse.hpp:157-178) stably partitioned by bin.  Entry word =
// (col & (2^cw - 1)) << rbits | slot; columns are split in chunks of 2^cw
// (cw = 32 - rbits) whose offsets per bin are stored, so an entry is 4 B of
// index + V of value -- the same bytes per nonzero as the CSR.  Every
// (bin, chunk) run is padded to 128-entry groups stored interleaved (lane l
// loads entries {l, l+32, l+64, l+96} of a group with one 16-B load).
// Light bins are contiguous row ranges (slot = row - bin_row0); rows of high
// degree (power-law hubs) go to heavy bins holding only heavy rows (slot ->
// row through a map), where a row rarely recurs inside a warp's window.
//
// Summation order inside a row is not the reference's (shared-memory atomics
// in column order), so results match within the floating-point tolerance of
// SURVEY.md 8(c) and are not run-to-run bitwise reproducible, like the
// atomic column kernels.  OR_AND and MIN_PLUS are exact.
#include <cooperative_groups.h>

#include <algorithm>
#include <array>
#include <functional>
#include <numeric>
#include <vector>

#include <type_traits>

#include "device.cuh"
#include "internal.hpp"
#include "kernels.hpp"
#include "prims.cuh"

namespace ada {

namespace {

constexpr uint32_t kBinSmemBytes = 229376;  // <= 224 KiB of y segment per CTA (1 CTA / SM)
constexpr int kBinClusterAuto = 1;          // bin_cluster = 0 resolves to this

template <class V>
struct PkVal {
    uint32_t pk;
    V val;
};

// Rows of the bins: light bins are contiguous row ranges [r0[b], r0[b+1]);
// heavy bins (b >= nlight) hold up to rh heavy rows each, listed in hrows
// (ascending), slot s of heavy bin h = row hrows[h*rh + s].  hbits marks the
// heavy rows (they lie inside light bins' ranges but are written by their
// heavy bin).
struct BinRows {
    const int64_t* r0;
    int64_t nlight;
    const int32_t* hrows;
    int64_t nheavy;
    int rh;
    const uint32_t* hbits;
};

// One warp per column of the CSC: key = bin of the row, payload = packed
// entry; counts per (bin, chunk) for the chunk offsets.  A heavy row
// (hpos[row] >= 0) goes to heavy bin nlight + hpos / rh, slot hpos % rh.
template <class V>
__global__ void bin_expand_kernel(const int64_t* __restrict__ co, const int32_t* __restrict__ ri,
                                  const V* __restrict__ cv, int64_t cols, const int64_t* __restrict__ r0s,
                                  int rbits, int cw, int64_t nchunks, const int32_t* __restrict__ hpos, int rh,
                                  int64_t nlight, uint32_t* __restrict__ keys, PkVal<V>* __restrict__ pay,
                                  unsigned long long* __restrict__ counts) {
    const int64_t warp = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    const uint32_t cmask = cw >= 32 ? 0xffffffffu : ((1u << cw) - 1u);
    for (int64_t j = warp; j < cols; j += nwarps) {
        const int64_t b = co[j], e = co[j + 1];
        const int64_t chunk = j >> cw;
        int64_t prev_bin = -1;
        int run = 0;
        for (int64_t k = b + lane; k < e; k += 32) {
            const int64_t row = ri[k];
            const int32_t hp = hpos ? __ldg(hpos + row) : -1;
            int64_t bin;
            uint32_t rl;
            if (hp >= 0) {
                bin = nlight + hp / rh;
                rl = static_cast<uint32_t>(hp % rh);
            } else {
                int64_t lo = 0, hi = nlight;  // bin: largest b with r0s[b] <= row
                while (hi - lo > 1) {
                    const int64_t mid = (lo + hi) >> 1;
                    if (__ldg(r0s + mid) <= row) lo = mid;
                    else hi = mid;
                }
                bin = lo;
                rl = static_cast<uint32_t>(row - __ldg(r0s + bin));
            }
            keys[k] = static_cast<uint32_t>(bin);
            pay[k] = PkVal<V>{((static_cast<uint32_t>(j) & cmask) << rbits) | rl, cv[k]};
            // runs of equal bins per lane (rows ascend within the column)
            if (bin != prev_bin) {
                if (run) atomicAdd(counts + prev_bin * nchunks + chunk, static_cast<unsigned long long>(run));
                prev_bin = bin;
                run = 0;
            }
            ++run;
        }
        if (run) atomicAdd(counts + prev_bin * nchunks + chunk, static_cast<unsigned long long>(run));
    }
}

// Sorted position k (bins ascending, CSC order inside a bin) -> padded,
// interleaved position: every (bin, chunk) run starts at a multiple of 128
// entries (poff); inside a run, entry r of 128-group q lands at word
// q*128 + (r % 32)*4 + r / 32 of that group, so lane l of a warp loads
// entries {l, l+32, l+64, l+96} of the group as one 16-B word.
template <class V>
__global__ void bin_scatter_kernel(const PkVal<V>* __restrict__ pay, const uint32_t* __restrict__ keys,
                                   int64_t nlight, int64_t nchunks, const int64_t* __restrict__ uoff,
                                   const int64_t* __restrict__ poff, uint32_t* __restrict__ pk,
                                   V* __restrict__ bv) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < nlight; k += stride) {
        const int64_t b = keys[k];
        const int64_t* u = uoff + b * nchunks;
        int64_t lo = 0, hi = nchunks;  // chunk: largest c with u[c] <= k
        while (hi - lo > 1) {
            const int64_t mid = (lo + hi) >> 1;
            if (u[mid] <= k) lo = mid;
            else hi = mid;
        }
        const int64_t r = k - u[lo];
        const int64_t dst = poff[b * nchunks + lo] + (r & ~int64_t(127)) + ((r & 31) << 2) + ((r >> 5) & 3);
        const PkVal<V> v = pay[k];
        pk[dst] = v.pk;
        bv[dst] = v.val;
    }
}

template <class V>
__global__ void bin_pad_fill_kernel(int64_t n, uint32_t pad, uint32_t* __restrict__ pk, V* __restrict__ bv) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n; k += stride) {
        pk[k] = pad;
        bv[k] = V(0);
    }
}

struct PaddedCounts {
    const unsigned long long* c;
    __device__ int64_t operator()(int64_t i) const { return (static_cast<int64_t>(c[i]) + 127) & ~int64_t(127); }
};

struct U64Counts {
    const unsigned long long* c;
    __device__ int64_t operator()(int64_t i) const { return static_cast<int64_t>(c[i]); }
};

// mean |col - row * n/m| over the nonzeros (x-gather spread, in columns),
// accumulated as double per block.
__global__ void gather_spread_kernel(const int64_t* __restrict__ ro, const int32_t* __restrict__ ci,
                                     int64_t rows, double slope, double* __restrict__ out) {
    double s = 0;
    const int64_t warp = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int64_t r = warp; r < rows; r += nwarps) {
        const double d = static_cast<double>(r) * slope;
        for (int64_t k = ro[r] + lane; k < ro[r + 1]; k += 32) s += fabs(static_cast<double>(ci[k]) - d);
    }
    s = warp_sum(s);
    if (lane == 0) atomicAdd(out, s);
}

// ---------------------------------------------------------------------------
// The multiply.  CTA = one tile (bin, entry range [e0, e1)).  Thread t of the
// CTA handles entries e0 + i*NT*U + j*NT + t: each warp instruction covers 32
// consecutive (column-sorted) entries.  Each thread walks the bin's chunk
// offsets monotonically to know the chunk (high column bits) of its entries.
// ---------------------------------------------------------------------------
// 1024 threads x 8 entries in flight per thread: measured best on C2 (B200):
// 1024x8 170 us, 1024x6 174, 1024x4 197, 512x16 217, 512x12 227, 256x32 363.
//
// CL = 2: the tiles come in pairs (2p, 2p+1) covering the two halves of one
// bin tile; the pair is a thread-block cluster, each CTA accumulates its
// half into its own shared-memory y segment, and after a cluster barrier CTA
// r combines rows [r*nr/2, (r+1)*nr/2) of both segments (the peer's over
// DSMEM) and writes them.  Bins twice as tall halve the number of times x is
// streamed through L2 and double the entries per x line (fewer L1
// wavefronts per gather instruction).
template <class V, int SR, bool MASKED, int CL = 1, int kBinUnroll = 8, bool NOALLOC = false,
          int kBinThreads = 1024, bool PIPE = false, bool FUSE = false>
__global__ void __launch_bounds__(kBinThreads, 1) binned_row_kernel(
    int64_t tile0, BinRows br, int rbits, int cw, int64_t nchunks,
    const int64_t* __restrict__ tiles, const int32_t* __restrict__ tile_bin,
    const int32_t* __restrict__ tile_multi, const int64_t* __restrict__ chunk_off,
    const uint32_t* __restrict__ pk, const V* __restrict__ bv, const V* __restrict__ x,
    const uint32_t* __restrict__ mask, V* __restrict__ y, unsigned long long* __restrict__ ctr,
    char* const* __restrict__ peers, int npeers, int64_t peer_row0) {
    using S = Semiring<SR, V>;
    extern __shared__ __align__(16) unsigned char bin_smem[];
    V* ys = reinterpret_cast<V*>(bin_smem);
    const int64_t t = tile0 + blockIdx.x;
    const int64_t bin = tile_bin[t];
    const int64_t e0 = tiles[2 * t], e1 = tiles[2 * t + 1];
    int64_t r0 = 0;
    int nr;
    const int32_t* __restrict__ rmap = nullptr;  // heavy bin: slot -> row
    if (bin < br.nlight) {
        r0 = br.r0[bin];
        nr = static_cast<int>(br.r0[bin + 1] - r0);
    } else {
        const int64_t hb = (bin - br.nlight) * br.rh;
        nr = static_cast<int>(min(static_cast<int64_t>(br.rh), br.nheavy - hb));
        rmap = br.hrows + hb;
    }
    for (int i = threadIdx.x; i < nr; i += kBinThreads) ys[i] = S::zero();
    __syncthreads();

    const int64_t* __restrict__ co = chunk_off + bin * nchunks;
    const uint32_t rmask = (1u << rbits) - 1u;  // row slot rmask marks a padding entry
    unsigned n_used = 0;                        // entries consumed (KernelCounters)
    if (e0 < e1) {
        // 128-entry groups: warp w takes groups g0 + w, g0 + w + NW, ...;
        // lane l holds entries {l, l+32, l+64, l+96} of its group as one 16-B
        // word, so warp instruction j of a group still gathers x for 32
        // consecutive (column-sorted) entries.  Groups never straddle a chunk,
        // so the chunk (high column bits) is walked once per group, warp-uniform.
        constexpr int NW = kBinThreads / 32;
        constexpr int GU = kBinUnroll / 4;  // groups per warp in flight
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        const int64_t g0 = e0 >> 7, g1 = e1 >> 7;
        int lo = 0, hi = static_cast<int>(nchunks);  // chunk of the warp's first group
        const int64_t efirst = (g0 + warp) << 7;
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (__ldg(co + mid) <= efirst) lo = mid;
            else hi = mid;
        }
        int c = lo;
        int64_t nb = __ldg(co + c + 1);
        auto load_groups = [&](int64_t g, uint32_t (&p)[GU][4], V (&a)[GU][4], bool (&has)[GU]) {
#pragma unroll
            for (int u = 0; u < GU; ++u) {
                const int64_t gg = g + u * NW;
                has[u] = gg < g1;
                const int4 w = has[u] ? ld_stream(reinterpret_cast<const int4*>(pk + (gg << 7)) + lane)
                                      : make_int4(static_cast<int>(rmask), static_cast<int>(rmask),
                                                  static_cast<int>(rmask), static_cast<int>(rmask));
                p[u][0] = static_cast<uint32_t>(w.x);
                p[u][1] = static_cast<uint32_t>(w.y);
                p[u][2] = static_cast<uint32_t>(w.z);
                p[u][3] = static_cast<uint32_t>(w.w);
                if (S::kUsesValues && !MASKED) {
                    if (has[u]) ld_stream4(bv + (gg << 7) + 4 * lane, a[u]);
                    else a[u][0] = a[u][1] = a[u][2] = a[u][3] = V(0);
                } else {
                    a[u][0] = a[u][1] = a[u][2] = a[u][3] = V(1);
                }
            }
        };
        constexpr int64_t step = static_cast<int64_t>(NW) * GU;
        uint32_t p[GU][4];
        V a[GU][4];
        bool has[GU];
        if (PIPE) load_groups(g0 + warp, p, a, has);
        for (int64_t g = g0 + warp; g < g1; g += step) {
            if (!PIPE) load_groups(g, p, a, has);
            uint32_t cb[GU];
#pragma unroll
            for (int u = 0; u < GU; ++u) {
                const int64_t e = (g + u * NW) << 7;
                if (has[u] && e >= nb) {  // warp-uniform
                    do {
                        ++c;
                        nb = __ldg(co + c + 1);
                    } while (e >= nb);
                }
                cb[u] = static_cast<uint32_t>(c) << cw;
            }
            bool ok[GU][4];
            uint32_t col[GU][4];
#pragma unroll
            for (int u = 0; u < GU; ++u)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    ok[u][j] = (p[u][j] & rmask) != rmask;
                    col[u][j] = cb[u] + (p[u][j] >> rbits);
                    if (MASKED && ok[u][j]) ok[u][j] = (__ldg(mask + (col[u][j] >> 5)) >> (col[u][j] & 31)) & 1u;
                    n_used += ok[u][j];
                }
            if (MASKED && S::kUsesValues) {  // K2 loads a value only after its mask test (kernels.hpp:229-240)
#pragma unroll
                for (int u = 0; u < GU; ++u)
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        if (ok[u][j]) a[u][j] = __ldg(bv + ((g + u * NW) << 7) + 4 * lane + j);
            }
            V xv[GU][4];
#pragma unroll
            for (int u = 0; u < GU; ++u)
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    xv[u][j] = ok[u][j] ? (NOALLOC ? ld_stream(x + col[u][j]) : __ldg(x + col[u][j])) : S::zero();
            uint32_t rw[GU][4];
            V av[GU][4];
#pragma unroll
            for (int u = 0; u < GU; ++u)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    rw[u][j] = p[u][j] & rmask;
                    av[u][j] = a[u][j];
                }
            // the next groups' entries stream in while this batch updates y
            if (PIPE) load_groups(g + step, p, a, has);
#pragma unroll
            for (int u = 0; u < GU; ++u)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if (!ok[u][j]) continue;
                    V* slot = ys + rw[u][j];
                    if (SR == SR_PLUS_TIMES) {
                        const V prod = av[u][j] * xv[u][j];
                        // adding +-0 never changes a sum that starts at +0
                        if (prod != V(0)) atomicAdd(slot, prod);
                    } else if (SR == SR_OR_AND) {
                        if (xv[u][j] != V(0)) *reinterpret_cast<volatile V*>(slot) = V(1);
                    } else {
                        const V v = av[u][j] + xv[u][j];
                        if (v < *slot) AtomicCombine<SR_MIN_PLUS>::apply(slot, v);
                    }
                }
        }
    }
    if (ctr) {  // values_read (kernels.hpp:108): entries consumed; under K2, value loads after the mask test
        const unsigned n = warp_sum(n_used);
        if ((threadIdx.x & 31) == 0) count_add(ctr, 0, n);
    }
    int lo = 0, hi = nr;
    const V* peer = nullptr;
    if constexpr (CL == 2) {
        namespace cg = cooperative_groups;
        cg::cluster_group cl = cg::this_cluster();
        cl.sync();  // both halves accumulated
        const unsigned rank = cl.block_rank();
        peer = cl.map_shared_rank(ys, rank ^ 1u);
        const int half = (nr + 1) >> 1;
        lo = rank ? half : 0;
        hi = rank ? nr : half;
    } else {
        __syncthreads();
    }
    const int mode = tile_multi[t];
    for (int i = lo + static_cast<int>(threadIdx.x); i < hi; i += kBinThreads) {
        const V v = CL == 2 ? S::add(ys[i], peer[i]) : ys[i];
        int64_t row;
        if (rmap) {
            row = rmap[i];
        } else {
            row = r0 + i;
            // a heavy row inside this range is written by its heavy bin
            if (br.hbits && ((br.hbits[row >> 5] >> (row & 31)) & 1u)) continue;
        }
        if (mode == 0) {  // the tile owns its bin's rows: plain stores
            y[row] = v;
            // fused y all-gather (peer.cu): the same row into every rank's
            // full y over NVLink, at this rank's block offset
            if constexpr (FUSE)
                for (int p = 0; p < npeers; ++p) reinterpret_cast<V*>(peers[p])[peer_row0 + row] = v;
        } else if (mode == 2) {  // owns the rows in a later column panel: y += segment
            if (v != S::zero()) y[row] = S::add(y[row], v);
        } else if (v != S::zero()) {  // partial segment: combine into the identity-filled y
            AtomicCombine<SR>::apply(y + row, v);
        }
    }
    if constexpr (CL == 2) cooperative_groups::this_cluster().sync();  // peer reads done before exit
}

constexpr int64_t kHeavySeg = 8192;  // heavy-row threshold scale (rows of degree > kHeavySeg / 2)

__global__ void heavy_rows_kernel(const int64_t* __restrict__ ro, int64_t rows, int64_t heavy_min,
                                  int64_t* __restrict__ list, unsigned long long* __restrict__ count) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < rows; r += stride) {
        const int64_t b = ro[r], e = ro[r + 1];
        if (e - b > heavy_min) {
            const unsigned long long i = atomicAdd(count, 1ull);
            list[3 * i] = r;
            list[3 * i + 1] = b;
            list[3 * i + 2] = e;
        }
    }
}

__global__ void heavy_pos_kernel(const int32_t* __restrict__ hrows, int64_t nh, int32_t* __restrict__ hpos,
                                 uint32_t* __restrict__ hbits) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < nh) {
        const int32_t r = hrows[i];
        hpos[r] = static_cast<int32_t>(i);
        atomicOr(hbits + (r >> 5), 1u << (r & 31));
    }
}

// Heavy rows (degree > heavy_min), ascending, and their position map (for the
// expansion) and bitmap (for the light bins' write-back).
void plan_heavy(Context& ctx, const Matrix& m, BinLayout& L, DevBuf& hpos) {
    L.nheavy = 0;
    if (L.heavy_min <= 0 || m.rows == 0) return;
    DevBuf list, cnt;
    unsigned long long* dcount = static_cast<unsigned long long*>(cnt.ensure(sizeof(unsigned long long)));
    ADA_CUDA(cudaMemsetAsync(dcount, 0, sizeof(unsigned long long), ctx.stream));
    const int64_t cap = std::max<int64_t>(m.nnz / (L.heavy_min + 1) + 1, 1);
    list.ensure(sizeof(int64_t) * 3 * static_cast<size_t>(cap));
    const int64_t g = std::min<int64_t>((m.rows + 255) / 256, static_cast<int64_t>(ctx.sm_count) * 16);
    heavy_rows_kernel<<<static_cast<unsigned>(g), 256, 0, ctx.stream>>>(m.row_off.as<int64_t>(), m.rows,
                                                                         L.heavy_min, list.as<int64_t>(), dcount);
    ADA_LAUNCHED(ctx);
    unsigned long long n = 0;
    ADA_CUDA(cudaMemcpyAsync(&n, dcount, sizeof(n), cudaMemcpyDeviceToHost, ctx.stream));
    ctx.sync();
    if (n == 0) return;
    std::vector<int64_t> h(3 * static_cast<size_t>(n));
    ADA_CUDA(cudaMemcpyAsync(h.data(), list.p, sizeof(int64_t) * h.size(), cudaMemcpyDeviceToHost, ctx.stream));
    ctx.sync();
    std::vector<int32_t> rows(static_cast<size_t>(n));
    for (size_t i = 0; i < rows.size(); ++i) rows[i] = static_cast<int32_t>(h[3 * i]);
    std::sort(rows.begin(), rows.end());
    L.nheavy = static_cast<int64_t>(n);
    L.hrows.ensure(sizeof(int32_t) * rows.size());
    ADA_CUDA(cudaMemcpyAsync(L.hrows.p, rows.data(), sizeof(int32_t) * rows.size(), cudaMemcpyHostToDevice,
                             ctx.stream));
    int32_t* hp = static_cast<int32_t*>(hpos.ensure(sizeof(int32_t) * static_cast<size_t>(m.rows)));
    ADA_CUDA(cudaMemsetAsync(hp, 0xff, sizeof(int32_t) * static_cast<size_t>(m.rows), ctx.stream));
    const size_t nw = static_cast<size_t>((m.rows + 31) / 32);
    uint32_t* hb = static_cast<uint32_t*>(L.hbits.ensure(sizeof(uint32_t) * nw));
    ADA_CUDA(cudaMemsetAsync(hb, 0, sizeof(uint32_t) * nw, ctx.stream));
    heavy_pos_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, ctx.stream>>>(L.hrows.as<int32_t>(),
                                                                                     L.nheavy, hp, hb);
    ADA_LAUNCHED(ctx);
    ctx.sync();  // host rows go out of scope
}

struct LightDegIn {
    const int64_t* ro;
    int64_t heavy_min;  // 0: every row is light
    __device__ int64_t operator()(int64_t r) const {
        const int64_t d = ro[r + 1] - ro[r];
        return heavy_min > 0 && d > heavy_min ? 0 : d;
    }
};

// cut[k] = first row r with prefix(r) >= k * total / nb (prefix = light
// entries of rows < r), k = 1 .. nb-1
__global__ void work_cuts_kernel(const int64_t* __restrict__ pre, int64_t rows, int64_t nb, int64_t* __restrict__ cut) {
    const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x + 1;
    if (k >= nb) return;
    const int64_t total = pre[rows];
    const int64_t t = static_cast<int64_t>(static_cast<double>(total) * static_cast<double>(k) / static_cast<double>(nb));
    int64_t lo = 0, hi = rows;  // first r in [0, rows] with pre[r] >= t
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (pre[mid] < t) lo = mid + 1;
        else hi = mid;
    }
    cut[k - 1] = lo;
}

struct WritePrefix {
    int64_t* out;
    __device__ void operator()(int64_t i, int64_t p, int64_t) const { out[i] = p; }
};

// Row cuts of `nb` bins holding equal shares of the light entries (sorted,
// deduplicated, starting at row 0).
std::vector<int64_t> equal_work_cuts(Context& ctx, const Matrix& m, int64_t nb, int64_t heavy_min) {
    std::vector<int64_t> cuts{0};
    if (nb <= 1 || m.rows == 0) return cuts;
    DevBuf pre, cut;
    int64_t* p = static_cast<int64_t*>(pre.ensure(sizeof(int64_t) * static_cast<size_t>(m.rows + 1)));
    scan3(ctx, m.rows, LightDegIn{m.row_off.as<int64_t>(), heavy_min}, WritePrefix{p}, p + m.rows, ctx.scratch[5]);
    int64_t* c = static_cast<int64_t*>(cut.ensure(sizeof(int64_t) * static_cast<size_t>(nb)));
    work_cuts_kernel<<<static_cast<unsigned>((nb + 255) / 256), 256, 0, ctx.stream>>>(p, m.rows, nb, c);
    ADA_LAUNCHED(ctx);
    std::vector<int64_t> h(static_cast<size_t>(nb - 1));
    ADA_CUDA(cudaMemcpyAsync(h.data(), c, sizeof(int64_t) * h.size(), cudaMemcpyDeviceToHost, ctx.stream));
    ctx.sync();
    for (int64_t v : h)
        if (v > cuts.back() && v < m.rows) cuts.push_back(v);
    return cuts;
}

template <class V>
void build_layout(Context& ctx, const Matrix& m, BinLayout& L) {
    const int vb = sizeof(V);
    const int64_t rmax = kBinSmemBytes / vb;
    int rbits = 0;
    while ((int64_t(1) << rbits) < rmax) ++rbits;
    int64_t nbins;
    L.cluster = 1;
    if (L.force_rows > 0) {
        nbins = (m.rows + L.force_rows - 1) / L.force_rows;
        L.cluster = L.cluster_req == 2 ? 2 : 1;
    } else {
        nbins = (m.rows + rmax - 1) / rmax;
        // at least one bin per SM when rows allow bins of >= 1024 rows
        nbins = std::max<int64_t>(nbins, std::min<int64_t>(ctx.sm_count, (m.rows + 1023) / 1024));
        // cluster pairs: one bin per SM pair, twice as tall, when it still fits
        const int64_t r1 = (m.rows + nbins - 1) / nbins;
        if (L.cluster_req == 2 && nbins >= 2 && 2 * r1 <= rmax) {
            nbins = (nbins + 1) / 2;
            L.cluster = 2;
        }
    }
    nbins = std::max<int64_t>(nbins, 1);
    // heavy rows: a row whose entries would put several lanes of one warp
    // instruction on the same shared-memory slot (degree well above the
    // column-sorted window a warp covers) leaves the light bins for the heavy
    // bins (heavy rows only: their column-sorted window is narrow enough
    // that a row rarely recurs in it)
    const int64_t per_bin = m.nnz / nbins + 1;
    L.heavy_min = m.feat[3] > static_cast<double>(kHeavySeg / 2)
                      ? std::max<int64_t>(kHeavySeg / 2, per_bin / 512) : 0;
    // Skewed (power-law) matrices: hub rows meet hub columns, so in the low
    // columns of a bin the same rows recur inside one warp's 32-entry window
    // and serialise on their shared-memory slots even at modest degree.
    // With the heavy rows in heavy bins (not CSR segments) a low cut pays;
    // K0 on B200, x = 100 %, cut 128 / 256 / 512 / 1024 / 2048:
    //   R-MAT 22  409 / 402 / 413 / 509 / 519 us
    //   R-MAT 26  8.31 / 8.61 / 8.63 / 9.14 / 9.74 ms   (spmv_lb 0.65 / 11.4 ms)
    if (m.feat[8] > 0.5 && m.feat[3] > 256.0) L.heavy_min = 256;
    if (L.cluster == 2) L.heavy_min = 0;  // cluster pairs: light bins only
    std::vector<int64_t> cuts;
    if (L.force_rows > 0 || L.cluster == 2 || m.nnz == 0) {  // equal-height bins
        const int64_t R0 = std::max<int64_t>((m.rows + nbins - 1) / nbins, 1);
        if (R0 > rmax) invalid("binned layout: rows per bin exceed the shared-memory segment");
        for (int64_t r = 0; r < m.rows; r += R0) cuts.push_back(r);
    } else {  // equal-work bins (light entries), no taller than the segment
        cuts = equal_work_cuts(ctx, m, nbins, L.heavy_min);
        std::vector<int64_t> split;
        for (size_t i = 0; i < cuts.size(); ++i) {
            const int64_t a = cuts[i], b = i + 1 < cuts.size() ? cuts[i + 1] : m.rows;
            const int64_t parts = std::max<int64_t>((b - a + rmax - 1) / rmax, 1);
            for (int64_t p = 0; p < parts; ++p) split.push_back(a + (b - a) * p / parts);
        }
        cuts.swap(split);
    }
    if (cuts.empty()) cuts.push_back(0);
    cuts.push_back(m.rows);
    nbins = static_cast<int64_t>(cuts.size()) - 1;
    if (nbins >= (int64_t(1) << 31)) invalid("binned layout: too many bins");
    int64_t R = 1;
    for (int64_t b = 0; b < nbins; ++b) R = std::max<int64_t>(R, cuts[static_cast<size_t>(b + 1)] - cuts[static_cast<size_t>(b)]);
    if (R > rmax) invalid("binned layout: rows per bin exceed the shared-memory segment");
    L.bin_r0.ensure(sizeof(int64_t) * cuts.size());
    ADA_CUDA(cudaMemcpyAsync(L.bin_r0.p, cuts.data(), sizeof(int64_t) * cuts.size(), cudaMemcpyHostToDevice,
                             ctx.stream));
    ctx.sync();  // host cuts go out of scope
    const int cw = 32 - rbits;
    const int64_t nchunks = std::max<int64_t>((m.cols + (int64_t(1) << cw) - 1) >> cw, 1);
    L.R = R;
    L.rbits = rbits;
    L.cw = cw;
    L.nchunks = nchunks;
    DevBuf hpos;
    plan_heavy(ctx, m, L, hpos);
    L.nlight = nbins;
    L.rh = static_cast<int>(R);
    if (L.nheavy > 0) nbins += (L.nheavy + R - 1) / R;  // heavy bins after the light ones
    L.nbins = nbins;
    const int64_t nnz = m.nnz;
    const size_t z = static_cast<size_t>(std::max<int64_t>(nnz, 1));
    const int64_t nkeys = nbins * nchunks;
    L.chunk_off.ensure(sizeof(int64_t) * static_cast<size_t>(nkeys + 1));
    DevBuf counts, uoff;
    counts.ensure(sizeof(unsigned long long) * static_cast<size_t>(nkeys));
    uoff.ensure(sizeof(int64_t) * static_cast<size_t>(nkeys + 1));
    ADA_CUDA(cudaMemsetAsync(counts.p, 0, sizeof(unsigned long long) * static_cast<size_t>(nkeys), ctx.stream));
    DevBuf k0, k1, p0, p1, cnt;
    int which = 0;
    if (nnz > 0) {
        k0.ensure(sizeof(uint32_t) * z);
        k1.ensure(sizeof(uint32_t) * z);
        p0.ensure(sizeof(PkVal<V>) * z);
        p1.ensure(sizeof(PkVal<V>) * z);
        const int64_t warps = std::min<int64_t>(m.cols, static_cast<int64_t>(ctx.sm_count) * 64);
        bin_expand_kernel<V><<<static_cast<unsigned>(std::max<int64_t>((warps * 32 + 255) / 256, 1)), 256, 0,
                               ctx.stream>>>(m.col_off.as<int64_t>(), m.row_idx.as<int32_t>(),
                                             m.cvals.as<V>(), m.cols, L.bin_r0.as<int64_t>(), rbits, cw, nchunks,
                                             L.nheavy ? hpos.as<int32_t>() : nullptr, L.rh, L.nlight,
                                             k0.as<uint32_t>(), p0.as<PkVal<V>>(),
                                             counts.as<unsigned long long>());
        ADA_LAUNCHED(ctx);
        which = radix_sort_pairs<PkVal<V>>(ctx, k0.as<uint32_t>(), p0.as<PkVal<V>>(), k1.as<uint32_t>(),
                                           p1.as<PkVal<V>>(), nnz, bits_for(nbins + 1), cnt, ctx.scratch[5]);
    }
    // unpadded run offsets (sorted positions) and padded ones (the layout)
    int64_t* uo = uoff.as<int64_t>();
    int64_t* off = L.chunk_off.as<int64_t>();
    scan3(ctx, nkeys, U64Counts{counts.as<unsigned long long>()}, WriteExclusive{uo}, uo + nkeys, ctx.scratch[5]);
    scan3(ctx, nkeys, PaddedCounts{counts.as<unsigned long long>()}, WriteExclusive{off}, off + nkeys,
          ctx.scratch[5]);
    int64_t tot[2] = {0, 0};
    ADA_CUDA(cudaMemcpyAsync(&tot[0], uo + nkeys, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx.stream));
    ADA_CUDA(cudaMemcpyAsync(&tot[1], off + nkeys, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx.stream));
    ctx.sync();
    const int64_t nlight = tot[0], npad = tot[1];
    L.n_binned = nlight;
    L.n_padded = npad;
    // + 4 entries so an empty layout still has a valid allocation
    L.pk.ensure(sizeof(uint32_t) * static_cast<size_t>(npad + 4));
    L.bv.ensure(sizeof(V) * static_cast<size_t>(npad + 4));
    if (npad > 0) {
        const int64_t g = std::min<int64_t>((npad + 255) / 256, static_cast<int64_t>(ctx.sm_count) * 32);
        bin_pad_fill_kernel<V><<<static_cast<unsigned>(g), 256, 0, ctx.stream>>>(
            npad, (1u << rbits) - 1u, L.pk.as<uint32_t>(), L.bv.as<V>());
        ADA_LAUNCHED(ctx);
    }
    if (nlight > 0) {
        const PkVal<V>* sorted = which ? p1.as<PkVal<V>>() : p0.as<PkVal<V>>();
        const uint32_t* skeys = which ? k1.as<uint32_t>() : k0.as<uint32_t>();
        const int64_t g = std::min<int64_t>((nlight + 255) / 256, static_cast<int64_t>(ctx.sm_count) * 32);
        bin_scatter_kernel<V><<<static_cast<unsigned>(g), 256, 0, ctx.stream>>>(
            sorted, skeys, nlight, nchunks, uo, off, L.pk.as<uint32_t>(), L.bv.as<V>());
        ADA_LAUNCHED(ctx);
    }
    ctx.sync();  // the sort buffers are released on return
    // per-bin entry counts on the host (tile planning)
    std::vector<int64_t> all(static_cast<size_t>(nkeys + 1));
    ADA_CUDA(cudaMemcpyAsync(all.data(), off, sizeof(int64_t) * all.size(), cudaMemcpyDeviceToHost, ctx.stream));
    ctx.sync();
    L.bin_start.resize(static_cast<size_t>(nbins + 1));
    for (int64_t b = 0; b <= nbins; ++b) L.bin_start[static_cast<size_t>(b)] = all[static_cast<size_t>(b * nchunks)];
    L.h_chunk_off.swap(all);
    L.tile_cap = -1;
    L.built = true;
}

// Tiles: every bin gets ceil(count / cap) equal column-contiguous tiles (at
// least one, so its rows are written); heaviest first (longest-processing-
// time order for the hardware block scheduler).
// Tile cap (entries per CTA) for the single-panel plan: the one-wave
// makespan of heaviest-first list scheduling of the bins' tiles over the SMs
// (the order the tiles are launched in), over caps of 0.5-1.5x the fair share.
// A tile costs its entries plus its y segment: zeroing and a coalesced store
// for a whole bin, an atomic combine (~4x) for a split one.  Uniform matrices
// keep one tile per bin; skewed ones (R-MAT) trade splits against the second
// partial wave that a 1.25x cap leaves.
int64_t choose_cap(const BinLayout& L, int sms, int64_t nnz) {
    const double fair = static_cast<double>(nnz) / static_cast<double>(sms);
    const double seg = static_cast<double>(L.R);
    int64_t best_cap = std::max<int64_t>(static_cast<int64_t>(fair * 1.25), 16384);
    double best = 1e300;
    std::vector<double> cost;
    for (int f = 50; f <= 150; f += 5) {
        const int64_t cap = std::max<int64_t>(static_cast<int64_t>(fair * f / 100.0), 16384);
        cost.clear();
        for (int64_t b = 0; b < L.nbins; ++b) {
            const int64_t n = L.bin_start[static_cast<size_t>(b + 1)] - L.bin_start[static_cast<size_t>(b)];
            const int64_t k = std::max<int64_t>((n + cap - 1) / cap, 1);
            for (int64_t i = 0; i < k; ++i)
                cost.push_back(static_cast<double>(n) / static_cast<double>(k) + (k > 1 ? 4.0 : 1.0) * seg);
        }
        std::sort(cost.begin(), cost.end(), std::greater<double>());
        std::vector<double> sm(static_cast<size_t>(sms), 0.0);  // min-heap of SM finish times
        std::make_heap(sm.begin(), sm.end(), std::greater<double>());
        double span = 0;
        for (double c : cost) {
            std::pop_heap(sm.begin(), sm.end(), std::greater<double>());
            sm.back() += c;
            span = std::max(span, sm.back());
            std::push_heap(sm.begin(), sm.end(), std::greater<double>());
        }
        if (span < best * 0.999) {
            best = span;
            best_cap = cap;
        }
    }
    return best_cap;
}

void plan_tiles(Context& ctx, const Matrix& m, BinLayout& L, int64_t cap_req, int64_t panel_chunks) {
    panel_chunks = std::min<int64_t>(std::max<int64_t>(panel_chunks, 1), L.nchunks);
    if (L.cluster == 2) panel_chunks = L.nchunks;  // pairs: one panel
    if (L.tile_cap_req == cap_req && L.panel_chunks == panel_chunks && L.tile_cap >= 0) return;
    int64_t cap = cap_req;
    if (cap <= 0) {
        const double fair = static_cast<double>(m.nnz) / static_cast<double>(ctx.sm_count);
        cap = L.cluster == 1 && panel_chunks == L.nchunks
                  ? choose_cap(L, ctx.sm_count, m.nnz)
                  : std::max<int64_t>(static_cast<int64_t>(fair * 1.25), 16384);
    }
    L.tile_cap_req = cap_req;
    // Column panels of `panel_chunks` chunks are launched one after another;
    // within a panel a work unit is one CTA (cluster 1) or a CTA pair
    // (cluster 2) of <= `cap` entries per CTA, a bin's units being equal
    // column-contiguous splits.  mode: 0 store the bin's rows, 1 atomic
    // combine (bin split in this panel), 2 load-add-store (later panel).
    struct T { int64_t e0, e1; int32_t bin, mode; };
    std::vector<T> ts;
    std::vector<int64_t> p0;
    bool multi = false;
    const int cl = L.cluster;
    const int64_t nc = L.nchunks;
    for (int64_t c0 = 0; c0 < nc; c0 += panel_chunks) {
        const int64_t c1 = std::min(c0 + panel_chunks, nc);
        const size_t first = ts.size();
        p0.push_back(static_cast<int64_t>(first));
        for (int64_t b = 0; b < L.nbins; ++b) {
            const int64_t s = L.h_chunk_off[static_cast<size_t>(b * nc + c0)];
            const int64_t e = L.h_chunk_off[static_cast<size_t>(b * nc + c1)];
            if (c0 > 0 && e == s) continue;  // nothing to add in a later panel
            const int64_t k = std::max<int64_t>((e - s + cl * cap - 1) / (cl * cap), 1);
            const int32_t mode = k > 1 ? 1 : (c0 > 0 ? 2 : 0);
            for (int64_t i = 0; i < k * cl; ++i)
                ts.push_back(T{s + (((e - s) * i / (k * cl)) & ~int64_t(127)),
                                 i + 1 == k * cl ? e : s + (((e - s) * (i + 1) / (k * cl)) & ~int64_t(127)),
                                 static_cast<int32_t>(b), mode});
            multi = multi || k > 1;
        }
        if (cl == 1) {
            std::stable_sort(ts.begin() + static_cast<std::ptrdiff_t>(first), ts.end(),
                             [](const T& a, const T& b) { return a.e1 - a.e0 > b.e1 - b.e0; });
        } else {  // heaviest pair first, pairs kept adjacent (cluster = CTAs 2p, 2p+1)
            std::vector<size_t> pr((ts.size() - first) / 2);
            std::iota(pr.begin(), pr.end(), size_t(0));
            auto at = [&](size_t i) -> const T& { return ts[first + i]; };
            std::stable_sort(pr.begin(), pr.end(), [&](size_t a, size_t b) {
                return at(2 * a + 1).e1 - at(2 * a).e0 > at(2 * b + 1).e1 - at(2 * b).e0;
            });
            std::vector<T> o;
            o.reserve(ts.size() - first);
            for (size_t q : pr) {
                o.push_back(at(2 * q));
                o.push_back(at(2 * q + 1));
            }
            std::copy(o.begin(), o.end(), ts.begin() + static_cast<std::ptrdiff_t>(first));
        }
    }
    p0.push_back(static_cast<int64_t>(ts.size()));
    L.panel_tile0.swap(p0);
    L.panel_chunks = panel_chunks;
    const size_t nt = ts.size();
    std::vector<int64_t> h_t(2 * nt);
    std::vector<int32_t> h_b(nt), h_m(nt);
    for (size_t i = 0; i < nt; ++i) {
        h_t[2 * i] = ts[i].e0;
        h_t[2 * i + 1] = ts[i].e1;
        h_b[i] = ts[i].bin;
        h_m[i] = ts[i].mode;
    }
    L.tiles.ensure(sizeof(int64_t) * h_t.size());
    L.tile_bin.ensure(sizeof(int32_t) * nt);
    L.tile_multi.ensure(sizeof(int32_t) * nt);
    ADA_CUDA(cudaMemcpyAsync(L.tiles.p, h_t.data(), sizeof(int64_t) * h_t.size(), cudaMemcpyHostToDevice, ctx.stream));
    ADA_CUDA(cudaMemcpyAsync(L.tile_bin.p, h_b.data(), sizeof(int32_t) * nt, cudaMemcpyHostToDevice, ctx.stream));
    ADA_CUDA(cudaMemcpyAsync(L.tile_multi.p, h_m.data(), sizeof(int32_t) * nt, cudaMemcpyHostToDevice, ctx.stream));
    ctx.sync();  // host vectors go out of scope
    L.ntiles = static_cast<int64_t>(nt);
    L.multi = multi;
    L.tile_cap = cap;
}

}  // namespace

double matrix_gather_spread(Context& ctx, const Matrix& m) {
    if (m.nnz == 0 || m.rows == 0) return 0.0;
    DevBuf acc;
    acc.ensure(sizeof(double));
    ADA_CUDA(cudaMemsetAsync(acc.p, 0, sizeof(double), ctx.stream));
    const double slope = static_cast<double>(m.cols) / static_cast<double>(m.rows);
    const int64_t warps = std::min<int64_t>(m.rows, static_cast<int64_t>(ctx.sm_count) * 64);
    gather_spread_kernel<<<static_cast<unsigned>((warps * 32 + 255) / 256), 256, 0, ctx.stream>>>(
        m.row_off.as<int64_t>(), m.col_idx.as<int32_t>(), m.rows, slope, acc.as<double>());
    ADA_LAUNCHED(ctx);
    double h = 0;
    ADA_CUDA(cudaMemcpyAsync(&h, acc.p, sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
    ctx.sync();
    return h / static_cast<double>(m.nnz);
}

bool binned_preferred(const Matrix& m) {
    // scattered gathers (mean distance from the diagonal > 64 KiB of x) on a
    // matrix large enough to fill the GPU with 1024-thread CTAs
    return m.nnz >= (int64_t(1) << 20) && m.gather_spread * m.vbytes() > 65536.0;
}

template <class V, int SR>
void run_row_binned(Context& ctx, const Matrix& m, const V* x, const uint32_t* mask, V* y,
                    int64_t force_rows, int64_t tile_cap, int cluster, int panel_kib) {
    if (cluster < 0 || cluster > 2) invalid("bin_cluster must be 0, 1 or 2");
    const int creq = cluster == 0 ? kBinClusterAuto : cluster;
    // the layout and tile plan are built once, under the matrix's lock, and
    // completed on this stream before another context may launch from them
    std::unique_lock<std::mutex> lk(m.lazy);
    bool built_now = false;
    if (!m.bins->built || m.bins->force_rows != force_rows || m.bins->dtype != m.dtype ||
        m.bins->cluster_req != creq) {
        m.bins.reset(new BinLayout());
        m.bins->force_rows = force_rows;
        m.bins->cluster_req = creq;
        m.bins->dtype = m.dtype;
        build_layout<V>(ctx, m, *m.bins);
        built_now = true;
    }
    BinLayout& L = *m.bins;
    // column panels (opt-in): x streamed in pieces of panel_kib.  Off by
    // default: on R-MAT 26 (x = 268 MB > L2) 16-96 MiB panels measured 3-25 %
    // slower than one pass (the gathers concentrate on hub columns that stay
    // in L2; the bound is the L1 data pipe)
    const int64_t chunk_bytes = (int64_t(1) << L.cw) * static_cast<int64_t>(sizeof(V));
    const int64_t pbytes = panel_kib > 0 ? int64_t(panel_kib) * 1024 : INT64_MAX / 2;
    const int64_t plan0[2] = {L.ntiles, L.panel_chunks};
    plan_tiles(ctx, m, L, tile_cap, std::max<int64_t>(pbytes / chunk_bytes, 1));
    if (built_now || plan0[0] != L.ntiles || plan0[1] != L.panel_chunks) ctx.sync();
    lk.unlock();
    if (m.rows == 0) return;
    if (L.multi) fill_value<V, SR>(ctx, y, m.rows);
    // the distributed y all-gather rides on the store epilogue when every
    // tile owns its rows (plain stores, one pass over the panels)
    const bool fuse = ctx.peer_dst && !L.multi && L.panel_tile0.size() == 2 && L.cluster == 1;
    char* const* peers = fuse ? ctx.peer_dst : nullptr;
    const int npeers = fuse ? ctx.peer_world : 0;
    if (fuse) ctx.peer_fused = true;
    const size_t smem = sizeof(V) * static_cast<size_t>(L.R);
    const int nt = 1024;
    auto launch = [&](auto kern, int cl, int64_t t0, int64_t nt_) {
        ADA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        cudaLaunchConfig_t lc{};
        lc.gridDim = dim3(static_cast<unsigned>(nt_));
        lc.blockDim = dim3(nt);
        lc.dynamicSmemBytes = smem;
        lc.stream = ctx.stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = static_cast<unsigned>(cl);
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        const BinRows br{L.bin_r0.as<int64_t>(), L.nlight, L.hrows.as<int32_t>(), L.nheavy, L.rh,
                         L.nheavy ? L.hbits.as<uint32_t>() : nullptr};
        ADA_CUDA(cudaLaunchKernelEx(&lc, kern, t0, br, L.rbits,
                                    L.cw, L.nchunks, L.tiles.as<int64_t>(),
                                    L.tile_bin.as<int32_t>(), L.tile_multi.as<int32_t>(),
                                    L.chunk_off.as<int64_t>(), L.pk.as<uint32_t>(), L.bv.as<V>(), x, mask, y,
                                    ctx.ctr, peers, npeers, ctx.peer_row0));
        ADA_LAUNCHED(ctx);
    };
    for (size_t p = 0; p + 1 < L.panel_tile0.size(); ++p) {  // panels in column order, same stream
        const int64_t t0 = L.panel_tile0[p], t1 = L.panel_tile0[p + 1];
        if (t1 <= t0) continue;
        if (L.cluster == 2) {
            if (mask) launch(binned_row_kernel<V, SR, true, 2>, 2, t0, t1 - t0);
            else launch(binned_row_kernel<V, SR, false, 2>, 2, t0, t1 - t0);
        } else {
            // fp32 K0: the next groups' entries stream in during the y updates
            // (C2 x = 0.5: 145 vs 156 us); x gathers skip L1 allocation on
            // matrices without hub columns (C2: 160 vs 162 us; R-MAT 22, whose
            // hub columns reuse L1 lines: 564 vs 525 us, so skewed ones keep
            // it); fp64 keeps the plain loop (the pipelined one spills at 64
            // registers)
#define ADA_BIN_LAUNCH(F)                                                                                     \
    if (mask) {                                                                                               \
        launch(binned_row_kernel<V, SR, true, 1, 8, false, 1024, false, F>, 1, t0, t1 - t0);                  \
    } else if constexpr (sizeof(V) == 4) {                                                                    \
        if (m.feat[8] > 0.5)                                                                                  \
            launch(binned_row_kernel<V, SR, false, 1, 8, false, 1024, true, F>, 1, t0, t1 - t0);              \
        else                                                                                                  \
            launch(binned_row_kernel<V, SR, false, 1, 8, true, 1024, true, F>, 1, t0, t1 - t0);               \
    } else {                                                                                                  \
        launch(binned_row_kernel<V, SR, false, 1, 8, false, 1024, false, F>, 1, t0, t1 - t0);                 \
    }
            // F: the fused all-gather epilogue (only when requested)
            if (fuse) {
                ADA_BIN_LAUNCH(true)
            } else {
                ADA_BIN_LAUNCH(false)
            }
#undef ADA_BIN_LAUNCH
        }
    }
}

#define ADA_INST(V, SR)                                                                                \
    template void run_row_binned<V, SR>(Context&, const Matrix&, const V*, const uint32_t*, V*, int64_t, \
                                        int64_t, int, int);
ADA_INST(float, SR_PLUS_TIMES)
ADA_INST(double, SR_PLUS_TIMES)
ADA_INST(float, SR_OR_AND)
ADA_INST(double, SR_OR_AND)
ADA_INST(float, SR_MIN_PLUS)
ADA_INST(double, SR_MIN_PLUS)
#undef ADA_INST

}  // namespace ada

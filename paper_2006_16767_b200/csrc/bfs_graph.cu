// bfs_graph.cu -- the device-resident BFS level loop (SPEC.md:489-497 driver,
// "levels 3-5 are <= 5 MB each, so they are launch- and
// latency-dominated: keep the BFS loop device-side or graph-captured").
//
// When the next frontier's membership does not depend on values (the
// boolean semiring, or a pattern matrix under plus-times / min-plus, where
// y_i != identity iff row i has a frontier neighbour) every level is one of
//
//   push  (column choices K4-K7): K6's load-balanced tiles over the
//         frontier's effective entries (eff offsets = scan of the frontier's
//         column degrees); each unvisited row is claimed once (atomicCAS on
//         its level) and appended to the next frontier (warp-aggregated);
//   pull  (row choices K0-K3): the output-masked row pull (K2/K3 with the
//         visited rows skipped); a frontier neighbour is a column whose level
//         is the previous level, and a row stops at its first one;
//
// and the choice -- the built-in bytes model, or the trained selector's
// three trees walked ON THE DEVICE over the same 13 features the host
// selector reads (matrix features + nnz_x / x_sparsity / nnz_s / m_sparsity
// from the frontier counters) -- is made by a one-warp kernel at the start
// of the level.  The whole traversal is ONE CUDA graph built once per
// (matrix, context, policy): a WHILE conditional node repeats a two-level
// body; in each level the decision kernel sets IF(push) / IF(pull)
// conditional handles so only the chosen branch's kernels run, every kernel
// reading its sizes from device memory.  One graph launch and one host
// synchronisation per traversal.  Per-level reports (kernel, frontier size,
// effective nnz, device time from %globaltimer) are logged on the device.
#include <algorithm>
#include <functional>
#include <cstring>
#include <vector>

#include "device.cuh"
#include "internal.hpp"
#include "kernels.hpp"
#include "prims.cuh"

namespace ada {

namespace {

constexpr int kMaxLog = 1 << 16;    // per-level log capacity
constexpr int kScanBlocks = 256;    // fixed grid of the eff-offset scan
constexpr int kTile = 256;          // effective entries per push warp tile
constexpr int kWin = 128;           // support positions staged per warp tile
enum { kModeDone = 0, kModePush = 1, kModePull = 2 };
// bodies of a level's SWITCH node (any other value: no body runs)
enum { kBranchEffPush = 0, kBranchPush = 1, kBranchPull = 2, kBranchPushSmall = 3, kBranchCompactPush = 4,
       kBranchNone = 5 };
constexpr int kSpread = 256;  // a pull level's (count, degree) counters, spread against contention
constexpr unsigned long long kSmallPush = 4096;  // effective entries of a frontier pushed without offsets

// Device-side loop state (one per plan).
struct alignas(8) BfsState {
    unsigned long long nf[2];   // frontier size, by parity
    unsigned long long ns[2];   // its effective nnz (sum of column degrees)
    long long visited;          // vertices with a level
    int level;                  // level of the vertices the current step discovers
    int mode;                   // kMode*
    int kernel;                 // KernelId::index() selected for this level
    int done;
    int nlog;                   // levels logged
    int eff_ok;                 // the current frontier's eff offsets are valid (compaction / init wrote them)
    long long tot;              // packed (count << kCntShift | nnz_s) of a pull level's compaction scan
    int pending;                // a level ran since the last decision (its results not yet accounted)
    int list_ok;                // the current frontier exists as a list (a pull only marks levels)
};
static_assert(sizeof(BfsState) == 80, "BfsState is copied as 10 int64 words");
constexpr int kCntShift = 36;  // pull compaction packing: nnz_s < 2^36, frontier < 2^27

struct LogEntry {               // one row of adaspmv_iteration_report
    long long nnz_x, nnz_s;
    int kernel, exec_mode;
    unsigned long long t0;      // %globaltimer at the level's decision (ns)
};

// Flattened decision trees for the device walk.
struct DevTrees {
    const int32_t* feature;
    const int32_t* left;
    const int32_t* right;
    const int32_t* leaf;
    const double* threshold;
    int root[4];  // [3] = -1 without a workload_col tree (schema 1)
};

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ int tree_walk(const DevTrees& t, int which, const double* f) {
    int i = t.root[which];
    for (int guard = 0; guard < 4096; ++guard) {
        const int32_t feat = t.feature[i];
        if (feat < 0) return t.leaf[i];
        i = f[feat] <= t.threshold[i] ? t.left[i] : t.right[i];  // <= goes left
    }
    return 0;
}

// Start of a level: decide push / pull for the frontier of parity p.
// The level's branch is selected by setting the graph's conditional
// handles: IF(push) and IF(pull) bodies (only the chosen one runs), and the
// WHILE handle that repeats the two-level body until the frontier is empty.
__global__ void bfs_decide_kernel(BfsState* st, LogEntry* log, int p, DevTrees trees, int use_trees,
                                  const double* mfeat, int64_t n, int64_t nnz, int vbytes,
                                  unsigned long long* pcnt, cudaGraphConditionalHandle hbranch,
                                  cudaGraphConditionalHandle hwhile) {
    // a pull level left its frontier as marks + spread (count, degree) counters:
    // the warp sums and clears them
    unsigned long long pc = 0, pd = 0;
    const bool pulled = st->pending && st->mode == kModePull;
    if (pulled) {
        for (int i = threadIdx.x; i < kSpread; i += 32) {
            pc += pcnt[2 * i];
            pd += pcnt[2 * i + 1];
            pcnt[2 * i] = pcnt[2 * i + 1] = 0;
        }
        pc = warp_sum(pc);
        pd = warp_sum(pd);
    }
    if (threadIdx.x != 0) return;
    cudaGraphSetConditional(hbranch, kBranchNone);
    if (st->pending) {  // account for the level that produced this frontier
        if (pulled) {
            st->nf[p] = pc;
            st->ns[p] = pd;
            st->list_ok = 0;
            st->eff_ok = 0;
        } else {  // a push appended it (counters already set), unordered: offsets to be scanned
            st->list_ok = 1;
            st->eff_ok = 0;
        }
        st->visited += static_cast<long long>(st->nf[p]);
        st->pending = 0;
    }
    if (st->done) {
        st->mode = kModeDone;
        cudaGraphSetConditional(hwhile, 0);
        return;
    }
    const unsigned long long nf = st->nf[p], ns = st->ns[p];
    const unsigned long long now = globaltimer();
    if (nf == 0) {
        st->done = 1;
        st->mode = kModeDone;
        cudaGraphSetConditional(hwhile, 0);
        if (st->nlog < kMaxLog) log[st->nlog].t0 = now;  // end stamp of the last level
        return;
    }
    int k;
    if (use_trees) {
        // the 13 features in frozen order, as selector.cpp reads them
        double f[ADASPMV_NUM_FEATURES];
        for (int i = 0; i < 9; ++i) f[i] = mfeat[i];
        f[9] = static_cast<double>(nf);
        f[10] = n > 0 ? static_cast<double>(nf) / static_cast<double>(n) : 0.0;
        f[11] = static_cast<double>(ns);
        f[12] = nnz > 0 ? static_cast<double>(ns) / static_cast<double>(nnz) : 0.0;
        const int pattern = tree_walk(trees, 0, f);
        const int lb = tree_walk(trees, pattern == 0 && trees.root[3] >= 0 ? 3 : 1, f) == 1 ? 1 : 0;
        if (pattern == 2) k = lb;
        else if (pattern == 1) k = 2 + lb;
        else k = 4 + 2 * lb + (tree_walk(trees, 2, f) == 1 ? 1 : 0);
    } else {
        // bfs.cu heuristic_kernel: SURVEY.md 8(d) push / masked-pull bytes
        const double unvisited = n > 0 ? 1.0 - static_cast<double>(st->visited) / static_cast<double>(n) : 0.0;
        const double push = static_cast<double>(nf) * 20.0 + static_cast<double>(ns) * (4.0 + vbytes) +
                            (ns <= 4096 ? 0.0 : static_cast<double>(n) * vbytes);
        const double pull = static_cast<double>(n + 1) * 8.0 + static_cast<double>(nnz) * 4.0 * unvisited +
                            static_cast<double>(n) / 8.0 + static_cast<double>(n) * vbytes * unvisited;
        k = push <= pull ? (ns <= 4096 ? 7 : 6) : 2;
    }
    st->kernel = k;
    st->mode = k >= 4 ? kModePush : kModePull;
    cudaGraphSetConditional(hbranch, k < 4              ? kBranchPull
                                     : !st->list_ok     ? kBranchCompactPush
                                     : st->eff_ok       ? kBranchPush
                                     : ns <= kSmallPush ? kBranchPushSmall
                                                        : kBranchEffPush);
    st->level += 1;
    st->nf[p ^ 1] = 0;
    st->ns[p ^ 1] = 0;
    st->tot = 0;
    st->pending = 1;
    if (st->nlog < kMaxLog) {
        LogEntry& e = log[st->nlog];
        e.nnz_x = static_cast<long long>(nf);
        e.nnz_s = static_cast<long long>(ns);
        e.kernel = k;
        e.exec_mode = k >= 4 ? ADASPMV_EXEC_FUSED_PUSH_LB : ADASPMV_EXEC_MASKED_PULL;
        e.t0 = now;
    }
    st->nlog += 1;
}

// ---- eff offsets of the frontier (push only): fixed-grid reduce-then-scan
__global__ void __launch_bounds__(256) bfs_eff_partial_kernel(const BfsState* st, int p, const int32_t* __restrict__ f,
                                                              const int64_t* __restrict__ co,
                                                              long long* __restrict__ part) {
    if (st->mode != kModePush) return;
    const long long n = static_cast<long long>(st->nf[p]);
    const long long chunk = (n + gridDim.x - 1) / gridDim.x;
    const long long b0 = blockIdx.x * chunk, b1 = min(n, b0 + chunk);
    long long s = 0;
    for (long long i = b0 + threadIdx.x; i < b1; i += 256) {
        const int32_t c = f[i];
        s += co[c + 1] - co[c];
    }
    __shared__ long long red[8];
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long t = 0;
        for (int w = 0; w < 8; ++w) t += red[w];
        part[blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(kScanBlocks) bfs_eff_top_kernel(const BfsState* st, long long* __restrict__ part) {
    if (st->mode != kModePush) return;
    __shared__ long long sm[kScanBlocks / 32 + 1];
    const long long v = part[threadIdx.x];
    long long tot;
    const long long ex = block_exclusive_sum<kScanBlocks>(v, sm, &tot);
    part[threadIdx.x] = ex;
}

__global__ void __launch_bounds__(256) bfs_eff_write_kernel(const BfsState* st, int p, const int32_t* __restrict__ f,
                                                            const int64_t* __restrict__ co,
                                                            const long long* __restrict__ part,
                                                            int64_t* __restrict__ eff) {
    if (st->mode != kModePush) return;
    const long long n = static_cast<long long>(st->nf[p]);
    const long long chunk = (n + gridDim.x - 1) / gridDim.x;
    const long long b0 = blockIdx.x * chunk, b1 = min(n, b0 + chunk);
    if (b0 >= b1) return;  // block-uniform
    __shared__ long long sm[256 / 32 + 1];
    long long run = part[blockIdx.x];
    for (long long i0 = b0; i0 < b1; i0 += 256) {
        const long long i = i0 + threadIdx.x;
        long long d = 0;
        if (i < b1) {
            const int32_t c = f[i];
            d = co[c + 1] - co[c];
        }
        long long tot;
        const long long ex = block_exclusive_sum<256>(d, sm, &tot);
        if (i < b1) eff[i] = run + ex;
        run += tot;
    }
    if (b1 == n && threadIdx.x == 0) eff[n] = run;
}

// largest s in [lo, hi) with eff[s] <= pos (warp-cooperative; eff[lo] <= pos)
__device__ __forceinline__ long long warp_seg(const int64_t* __restrict__ eff, long long lo, long long hi,
                                              long long pos, int lane) {
    while (hi - lo > 32) {
        const long long step = (hi - lo + 31) / 32;
        const long long probe = lo + lane * step;
        const unsigned b = __ballot_sync(kFull, probe < hi && __ldg(eff + probe) <= pos);
        lo += static_cast<long long>(31 - __clz(b)) * step;
        hi = min(lo + step, hi);
    }
    const long long probe = lo + lane;
    const unsigned b = __ballot_sync(kFull, probe < hi && __ldg(eff + probe) <= pos);
    return lo + (31 - __clz(b));
}

// Appends `row` (when `claim`) to the next frontier: one counter update per
// warp instruction, slots by rank among the claiming lanes.
__device__ __forceinline__ void append_claimed(bool claim, int32_t row, const int64_t* __restrict__ co,
                                               BfsState* st, int q, int32_t* __restrict__ nf_out, int lane) {
    const unsigned ballot = __ballot_sync(kFull, claim);
    if (ballot == 0u) return;
    const long long deg = warp_sum(claim ? static_cast<long long>(__ldg(co + row + 1) - __ldg(co + row)) : 0ll);
    const int leader = __ffs(ballot) - 1;
    unsigned long long base = 0;
    if (lane == leader) {
        base = atomicAdd(&st->nf[q], static_cast<unsigned long long>(__popc(ballot)));
        atomicAdd(&st->ns[q], static_cast<unsigned long long>(deg));
    }
    base = __shfl_sync(kFull, base, leader);
    if (claim) nf_out[base + __popc(ballot & lanemask_lt())] = row;
}

// Push over K6's load-balanced tiles (kernels_col.cu col_lb_kernel MODE 2),
// grid-stride over the tiles of the frontier's effective entries.
__global__ void __launch_bounds__(256) bfs_push_kernel(BfsState* st, int p, const int32_t* __restrict__ f,
                                                       const int64_t* __restrict__ eff,
                                                       const int64_t* __restrict__ co,
                                                       const int32_t* __restrict__ ri, int32_t* __restrict__ lv,
                                                       int32_t* __restrict__ nf_out) {
    if (st->mode != kModePush) return;
    constexpr int kW = 8, kJ = kTile / 32;
    __shared__ long long s_base[kW][kWin];
    __shared__ int s_end[kW][kWin];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long nx = static_cast<long long>(st->nf[p]);
    const long long nnz_s = static_cast<long long>(st->ns[p]);
    const int level = st->level;
    const int q = p ^ 1;
    const long long ntiles = (nnz_s + kTile - 1) / kTile;
    for (long long t = static_cast<long long>(blockIdx.x) * kW + warp; t < ntiles;
         t += static_cast<long long>(gridDim.x) * kW) {
        const long long tb = t * kTile;
        const int ten = static_cast<int>(min(static_cast<long long>(kTile), nnz_s - tb));
        const long long s_lo = warp_seg(eff, 0, nx + 1, tb, lane);
        const long long s_hi = warp_seg(eff, s_lo, nx + 1, tb + ten - 1, lane);
        const long long span = s_hi - s_lo + 1;
        long long kidx[kJ];
        if (span <= kWin) {
            for (int i = lane; i < span; i += 32) {
                const long long s = s_lo + i;
                const long long e0 = __ldg(eff + s), e1 = __ldg(eff + s + 1);
                s_base[warp][i] = __ldg(co + __ldg(f + s)) - e0;
                const long long rel = e1 - tb;
                s_end[warp][i] = static_cast<int>(rel > kTile + 1 ? kTile + 1 : rel);
            }
            __syncwarp();
            int si = 0;
            {
                int hi = static_cast<int>(span);
                while (hi - si > 1) {
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
                } else {
                    kidx[j] = -1;
                }
            }
            __syncwarp();
        } else {
#pragma unroll
            for (int j = 0; j < kJ; ++j) {
                const int i = 32 * j + lane;
                if (i < ten) {
                    const long long s = segment_search(eff, s_lo, s_hi + 1, tb + i);
                    kidx[j] = __ldg(co + __ldg(f + s)) - __ldg(eff + s) + tb + i;
                } else {
                    kidx[j] = -1;
                }
            }
        }
        int r[kJ];
#pragma unroll
        for (int j = 0; j < kJ; ++j) r[j] = kidx[j] >= 0 ? ld_stream(ri + kidx[j]) : 0;
#pragma unroll
        for (int j = 0; j < kJ; ++j) {
            const bool claim = kidx[j] >= 0 && lv[r[j]] < 0 && atomicCAS(lv + r[j], -1, level) == -1;
            append_claimed(claim, r[j], co, st, q, nf_out, lane);
        }
    }
}

// Output-masked pull with early exit (bfs.cu bfs_pull_kernel), G lanes per
// row, one group per row (full grid: the block scheduler balances rows that
// run long); a row with a frontier neighbour (a column of the previous
// level, read from the level array: no frontier bitmap to build and clear)
// gets its level.
// The next frontier is then compacted by a scan over the levels (no shared
// append counter: the fat pull levels would serialise on it).
template <int G>
__global__ void __launch_bounds__(256) bfs_pull_mark_kernel(const BfsState* st, int64_t rows,
                                                            const int64_t* __restrict__ ro,
                                                            const int32_t* __restrict__ ci,
                                                            const int64_t* __restrict__ co,
                                                            int32_t* __restrict__ lv,
                                                            unsigned long long* __restrict__ pcnt) {
    const int level = st->level;  // frontier = the vertices of level - 1
    const int lane = threadIdx.x & 31;
    const int lg = threadIdx.x & (G - 1);
    const long long row = (static_cast<long long>(blockIdx.x) * 256 + threadIdx.x) / G;
    const bool live = row < rows && lv[row] < 0;
    bool hit = false;
    if (live) {
        const long long b = __ldg(ro + row), e = __ldg(ro + row + 1);
        for (long long k0 = b + lg; k0 < e && !hit; k0 += G * 4) {
            int c[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) c[j] = k0 + j * G < e ? __ldg(ci + k0 + j * G) : -1;
#pragma unroll
            for (int j = 0; j < 4; ++j) hit = hit || (c[j] >= 0 && lv[c[j]] == level - 1);
        }
    }
    const unsigned grp = G == 32 ? kFull : (((1u << G) - 1u) << (lane & ~(G - 1)));
    const bool any = (__ballot_sync(kFull, hit) & grp) != 0u;
    const bool join = live && any && lg == 0;
    if (join) lv[row] = level;
    // the level's size and effective nnz, one spread counter update per warp
    const unsigned long long c = __popc(__ballot_sync(kFull, join));
    if (c) {
        const unsigned long long d = warp_sum(join ? static_cast<unsigned long long>(__ldg(co + row + 1) - __ldg(co + row)) : 0ull);
        if (lane == 0) {
            const int slot = static_cast<int>((blockIdx.x * 8u + (threadIdx.x >> 5)) % kSpread);
            atomicAdd(pcnt + 2 * slot, c);
            atomicAdd(pcnt + 2 * slot + 1, d);
        }
    }
}

// compaction items: (row joined at this level) << kCntShift | its column degree
struct LevelIn {  // rows of level *level + off
    const int32_t* lv;
    const int* level;
    int off;
    const int64_t* co;
    __device__ int64_t operator()(int64_t r) const {
        return lv[r] == *level + off ? (int64_t(1) << kCntShift) | (co[r + 1] - co[r]) : 0;
    }
};
struct LevelEpi {  // the next frontier and its eff offsets (degree prefix)
    int32_t* out;
    int64_t* eff;
    __device__ void operator()(int64_t r, int64_t p, int64_t v) const {
        if (!v) return;
        const int64_t slot = p >> kCntShift;
        out[slot] = static_cast<int32_t>(r);
        eff[slot] = p & ((int64_t(1) << kCntShift) - 1);
    }
};

// Push of a small frontier (<= kSmallPush effective entries) that a push
// appended (no eff offsets): one block per frontier vertex, its column walked
// by the block's warps -- one launch instead of the offset scan + LB push.
__global__ void __launch_bounds__(256) bfs_push_small_kernel(BfsState* st, int p, const int32_t* __restrict__ f,
                                                             const int64_t* __restrict__ co,
                                                             const int32_t* __restrict__ ri,
                                                             int32_t* __restrict__ lv, int32_t* __restrict__ nf_out) {
    const long long nx = static_cast<long long>(st->nf[p]);
    const int level = st->level;
    const int lane = threadIdx.x & 31;
    for (long long s = blockIdx.x; s < nx; s += gridDim.x) {
        const int32_t v = f[s];
        const long long b = __ldg(co + v), e = __ldg(co + v + 1);
        for (long long k0 = b + (threadIdx.x & ~31); k0 < e; k0 += 256) {  // warp-uniform trip count
            const long long k = k0 + lane;
            const int32_t r = k < e ? __ldg(ri + k) : 0;
            const bool claim = k < e && lv[r] < 0 && atomicCAS(lv + r, -1, level) == -1;
            append_claimed(claim, r, co, st, p ^ 1, nf_out, lane);
        }
    }
}

// eff[nnz_x] = nnz_s after a compaction (the scan's epilogue writes the
// offsets of the entries only)
__global__ void bfs_eff_tail_kernel(const BfsState* st, int p, int64_t* __restrict__ eff) {
    if (threadIdx.x == 0) eff[st->nf[p]] = static_cast<int64_t>(st->ns[p]);
}

__global__ void bfs_init_kernel(BfsState* st, int32_t* lv, int64_t n, int64_t source, int32_t* f0,
                                const int64_t* __restrict__ co, int64_t* __restrict__ eff) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride)
        lv[i] = i == source ? 0 : -1;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        f0[0] = static_cast<int32_t>(source);
        st->nf[0] = 1;
        st->ns[0] = static_cast<unsigned long long>(co[source + 1] - co[source]);
        st->nf[1] = st->ns[1] = 0;
        st->visited = 1;
        st->level = 0;
        st->mode = kModeDone;
        st->kernel = -1;
        st->done = 0;
        st->nlog = 0;
        st->tot = 0;
        st->pending = 0;
        st->eff_ok = 1;
        st->list_ok = 1;
        eff[0] = 0;
        eff[1] = static_cast<int64_t>(st->ns[0]);
    }
}

}  // namespace

// One captured traversal plan: buffers, flattened trees and the graph.
struct BfsPlan {
    cudaStream_t stream = nullptr;
    uint64_t bundle_id = 0;  // 0 = heuristic
    DevBuf state, log, f[2], eff, part, lv, trees_i, trees_d, mfeat;
    DevTrees dt{};
    DevBuf scan_tmp;  // the compaction's tile sums (sized before capture)
    DevBuf pcnt;      // a pull level's spread (count, degree) counters
    cudaGraphExec_t exec = nullptr;
    ~BfsPlan() {
        if (exec) cudaGraphExecDestroy(exec);
    }
};

void BfsPlanDeleter::operator()(BfsPlan* p) const { delete p; }

bool bfs_graph_applicable(const Matrix& m, int semiring, int forced) {
    // membership-only levels (see the header), policy = heuristic or selector
    return forced < 0 && (semiring == ADASPMV_OR_AND || m.pattern) && m.rows == m.cols && m.rows > 0 &&
           m.rows < (int64_t(1) << 31) - 1;
}

namespace {

void upload_trees(Context& ctx, const Bundle& b, BfsPlan& P) {
    std::vector<int32_t> feat, left, right, leaf;
    std::vector<double> thr;
    P.dt.root[3] = -1;
    for (int t = 0; t < (b.has_col ? 4 : 3); ++t) {
        const Tree& tr = b.trees[t];
        const int32_t base = static_cast<int32_t>(feat.size());
        P.dt.root[t] = base;
        for (size_t i = 0; i < tr.feature.size(); ++i) {
            feat.push_back(tr.feature[i]);
            left.push_back(tr.feature[i] < 0 ? 0 : base + tr.left[i]);
            right.push_back(tr.feature[i] < 0 ? 0 : base + tr.right[i]);
            leaf.push_back(tr.leaf[i]);
            thr.push_back(tr.threshold[i]);
        }
    }
    const size_t nn = std::max<size_t>(feat.size(), 1);
    int32_t* di = static_cast<int32_t*>(P.trees_i.ensure(sizeof(int32_t) * 4 * nn));
    double* dd = static_cast<double*>(P.trees_d.ensure(sizeof(double) * nn));
    std::vector<int32_t> packed(4 * nn, 0);
    std::copy(feat.begin(), feat.end(), packed.begin());
    std::copy(left.begin(), left.end(), packed.begin() + static_cast<std::ptrdiff_t>(nn));
    std::copy(right.begin(), right.end(), packed.begin() + static_cast<std::ptrdiff_t>(2 * nn));
    std::copy(leaf.begin(), leaf.end(), packed.begin() + static_cast<std::ptrdiff_t>(3 * nn));
    ADA_CUDA(cudaMemcpyAsync(di, packed.data(), sizeof(int32_t) * packed.size(), cudaMemcpyHostToDevice, ctx.stream));
    if (!thr.empty())
        ADA_CUDA(cudaMemcpyAsync(dd, thr.data(), sizeof(double) * thr.size(), cudaMemcpyHostToDevice, ctx.stream));
    P.dt.feature = di;
    P.dt.left = di + nn;
    P.dt.right = di + 2 * nn;
    P.dt.leaf = di + 3 * nn;
    P.dt.threshold = dd;
    ctx.sync();  // host vectors go out of scope
}

template <int G>
void launch_pull_mark(cudaStream_t s, unsigned grid, BfsState* st, const Matrix& m, int32_t* lv,
                      unsigned long long* pcnt) {
    bfs_pull_mark_kernel<G><<<grid, 256, 0, s>>>(st, m.rows, m.row_off.as<int64_t>(), m.col_idx.as<int32_t>(),
                                                 m.col_off.as<int64_t>(), lv, pcnt);
}

// Appends SWITCH(handle) with one body per element of `bodies` to the graph
// being captured on `s`; body i is captured from bodies[i] on the side stream
// `s2` (the library's kernels take the context's stream, so it is swapped for
// the duration).
template <class F>
void capture_switch(Context& ctx, cudaStream_t s, cudaStream_t s2, cudaGraphConditionalHandle h,
                    const std::vector<F>& bodies) {
    cudaStreamCaptureStatus cs;
    cudaGraph_t g = nullptr;
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    ADA_CUDA(cudaStreamGetCaptureInfo(s, &cs, nullptr, &g, &deps, &nd));
    cudaGraphNodeParams ip{};
    ip.type = cudaGraphNodeTypeConditional;
    ip.conditional.handle = h;
    ip.conditional.type = cudaGraphCondTypeSwitch;
    ip.conditional.size = static_cast<unsigned>(bodies.size());
    cudaGraphNode_t node;
    ADA_CUDA(cudaGraphAddNode(&node, g, deps, nd, &ip));
    ADA_CUDA(cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies));
    const cudaStream_t keep = ctx.stream;
    for (size_t i = 0; i < bodies.size(); ++i) {
        cudaGraph_t bg = ip.conditional.phGraph_out[i];
        ADA_CUDA(cudaStreamBeginCaptureToGraph(s2, bg, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
        ctx.stream = s2;
        try {
            bodies[i](s2);
        } catch (...) {
            ctx.stream = keep;
            cudaStreamEndCapture(s2, &bg);
            throw;
        }
        ctx.stream = keep;
        ADA_CUDA(cudaStreamEndCapture(s2, &bg));
    }
}

// The whole traversal as ONE graph: WHILE(frontier) { level p = 0; level
// p = 1 }, a level being decide -> IF(push) {eff offsets, push} -> IF(pull)
// {frontier bitmap, pull, compaction scan, bitmap clear} -> account.  Only
// the chosen branch's kernels run; sizes live on the device.
void build_plan(Context& ctx, const Matrix& m, const Bundle* b, BfsPlan& P) {
    const int64_t n = m.rows;
    P.stream = ctx.stream;
    P.bundle_id = b ? b->id : 0;
    P.state.ensure(sizeof(BfsState));
    P.log.ensure(sizeof(LogEntry) * kMaxLog);
    for (auto& f : P.f) f.ensure(sizeof(int32_t) * static_cast<size_t>(n));
    P.eff.ensure(sizeof(int64_t) * static_cast<size_t>(n + 1));
    P.part.ensure(sizeof(long long) * kScanBlocks);
    P.lv.ensure(sizeof(int32_t) * static_cast<size_t>(n));
    P.scan_tmp.ensure(sizeof(int64_t) * static_cast<size_t>((n + kScanTile - 1) / kScanTile + 1));
    P.pcnt.ensure(sizeof(unsigned long long) * 2 * kSpread);
    ADA_CUDA(cudaMemsetAsync(P.pcnt.p, 0, sizeof(unsigned long long) * 2 * kSpread, ctx.stream));

    double* mf = static_cast<double*>(P.mfeat.ensure(sizeof(double) * 9));
    ADA_CUDA(cudaMemcpyAsync(mf, m.feat, sizeof(double) * 9, cudaMemcpyHostToDevice, ctx.stream));
    if (b) upload_trees(ctx, *b, P);
    ctx.sync();
    BfsState* st = P.state.as<BfsState>();
    LogEntry* lg = P.log.as<LogEntry>();
    int32_t* lv = P.lv.as<int32_t>();
    const int64_t* co = m.col_off.as<int64_t>();
    const unsigned push_grid = static_cast<unsigned>(ctx.sm_count) * 8;
    const int G = std::max(1, default_lanes_per_row(m.feat[5]) / 8);
    const unsigned pull_grid = static_cast<unsigned>(std::max<int64_t>((n * G + 255) / 256, 1));
    cudaGraph_t graph = nullptr;
    ADA_CUDA(cudaGraphCreate(&graph, 0));
    cudaStream_t s2 = nullptr;
    ADA_CUDA(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
    struct Cleanup {
        cudaGraph_t* g;
        cudaStream_t s;
        ~Cleanup() {
            if (*g) cudaGraphDestroy(*g);
            cudaStreamDestroy(s);
        }
    } cleanup{&graph, s2};
    cudaGraphConditionalHandle hw, hbranch[2];
    ADA_CUDA(cudaGraphConditionalHandleCreate(&hw, graph, 1, cudaGraphCondAssignDefault));
    for (int q = 0; q < 2; ++q)
        ADA_CUDA(cudaGraphConditionalHandleCreate(&hbranch[q], graph, kBranchNone, cudaGraphCondAssignDefault));
    cudaGraphNodeParams wp{};
    wp.type = cudaGraphNodeTypeConditional;
    wp.conditional.handle = hw;
    wp.conditional.type = cudaGraphCondTypeWhile;
    wp.conditional.size = 1;
    cudaGraphNode_t wnode;
    ADA_CUDA(cudaGraphAddNode(&wnode, graph, nullptr, 0, &wp));
    cudaGraph_t body = wp.conditional.phGraph_out[0];
    cudaStream_t s = ctx.stream;
    ADA_CUDA(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    try {
        for (int p = 0; p < 2; ++p) {
            bfs_decide_kernel<<<1, 32, 0, s>>>(st, lg, p, P.dt, b ? 1 : 0, mf, n, m.nnz, m.vbytes(),
                                               P.pcnt.as<unsigned long long>(), hbranch[p], hw);
            auto eff_scan = [&, p](cudaStream_t cs) {  // offsets of a frontier a push appended
                bfs_eff_partial_kernel<<<kScanBlocks, 256, 0, cs>>>(st, p, P.f[p].as<int32_t>(), co,
                                                                    P.part.as<long long>());
                bfs_eff_top_kernel<<<1, kScanBlocks, 0, cs>>>(st, P.part.as<long long>());
                bfs_eff_write_kernel<<<kScanBlocks, 256, 0, cs>>>(st, p, P.f[p].as<int32_t>(), co,
                                                                  P.part.as<long long>(), P.eff.as<int64_t>());
            };
            auto push = [&, p](cudaStream_t cs) {
                bfs_push_kernel<<<push_grid, 256, 0, cs>>>(st, p, P.f[p].as<int32_t>(), P.eff.as<int64_t>(), co,
                                                           m.row_idx.as<int32_t>(), lv, P.f[p ^ 1].as<int32_t>());
            };
            auto pull = [&, p](cudaStream_t cs) {  // marks only; the list is compacted if a push needs it
                unsigned long long* pc = P.pcnt.as<unsigned long long>();
                switch (G) {
                    case 1: launch_pull_mark<1>(cs, pull_grid, st, m, lv, pc); break;
                    case 2: launch_pull_mark<2>(cs, pull_grid, st, m, lv, pc); break;
                    case 4: launch_pull_mark<4>(cs, pull_grid, st, m, lv, pc); break;
                    default: launch_pull_mark<8>(cs, pull_grid, st, m, lv, pc); break;
                }
            };
            auto compact = [&, p](cudaStream_t) {  // the frontier (rows of level - 1) as a list + eff
                scan3(ctx, n, LevelIn{lv, &st->level, -1, co},
                      LevelEpi{P.f[p].as<int32_t>(), P.eff.as<int64_t>()}, reinterpret_cast<int64_t*>(&st->tot),
                      P.scan_tmp);
                bfs_eff_tail_kernel<<<1, 32, 0, ctx.stream>>>(st, p, P.eff.as<int64_t>());
            };
            std::vector<std::function<void(cudaStream_t)>> bodies(5);
            bodies[kBranchCompactPush] = [&](cudaStream_t cs) {
                compact(cs);
                push(cs);
            };
            bodies[kBranchEffPush] = [&](cudaStream_t cs) {
                eff_scan(cs);
                push(cs);
            };
            bodies[kBranchPush] = push;
            bodies[kBranchPull] = pull;
            bodies[kBranchPushSmall] = [&, p](cudaStream_t cs) {
                bfs_push_small_kernel<<<static_cast<unsigned>(ctx.sm_count) * 2, 256, 0, cs>>>(
                    st, p, P.f[p].as<int32_t>(), co, m.row_idx.as<int32_t>(), lv, P.f[p ^ 1].as<int32_t>());
            };
            capture_switch(ctx, s, s2, hbranch[p], bodies);
        }
        ADA_CUDA(cudaGetLastError());
    } catch (...) {
        cudaStreamEndCapture(s, &body);
        throw;
    }
    ADA_CUDA(cudaStreamEndCapture(s, &body));
    ADA_CUDA(cudaGraphInstantiate(&P.exec, graph, 0));
}

}  // namespace

void bfs_graph(Context& ctx, const Matrix& m, int64_t source, const Bundle* b, int64_t* levels, int64_t* n_levels,
               adaspmv_iteration_report* reports, int64_t max_reports) {
    const int64_t n = m.rows;
    if (source < 0 || source >= n) out_of_range("bfs: source out of range");
    std::unique_lock<std::mutex> lk(m.lazy);  // one traversal per matrix at a time (plan buffers)
    auto& plan = m.bfs_plan;
    if (!plan || plan->stream != ctx.stream || plan->bundle_id != (b ? b->id : 0)) {
        plan.reset(new BfsPlan());
        build_plan(ctx, m, b, *plan);
    }
    BfsPlan& P = *plan;
    BfsState* st = P.state.as<BfsState>();
    const unsigned ig = static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, static_cast<int64_t>(ctx.sm_count) * 16));
    bfs_init_kernel<<<ig, 256, 0, ctx.stream>>>(st, P.lv.as<int32_t>(), n, source, P.f[0].as<int32_t>(),
                                                m.col_off.as<int64_t>(), P.eff.as<int64_t>());
    ADA_LAUNCHED(ctx);
    // the whole traversal: one graph launch, one synchronisation (the state
    // comes back through the mapped host scalars)
    ADA_CUDA(cudaGraphLaunch(P.exec, ctx.stream));
    ++ctx.launches;
    copy_scalars_kernel_launch(ctx, reinterpret_cast<const int64_t*>(st), ctx.h_scalars_dev,
                               static_cast<int>(sizeof(BfsState) / sizeof(int64_t)));
    ctx.sync();
    if (!reinterpret_cast<const BfsState*>(ctx.h_scalars)->done)
        throw Error(ADASPMV_ERR_INTERNAL, "bfs: device level loop ended without an empty frontier");
    const BfsState* hs = reinterpret_cast<const BfsState*>(ctx.h_scalars);
    const int nlog = hs->nlog;
    *n_levels = nlog;
    if (reports && max_reports > 0) {
        const int nr = static_cast<int>(std::min<int64_t>(std::min<int64_t>(nlog, max_reports), kMaxLog - 1));
        std::vector<LogEntry> h(static_cast<size_t>(nr + 1));
        ADA_CUDA(cudaMemcpyAsync(h.data(), P.log.p, sizeof(LogEntry) * h.size(), cudaMemcpyDeviceToHost, ctx.stream));
        ctx.sync();
        for (int i = 0; i < nr; ++i) {
            adaspmv_iteration_report& r = reports[i];
            r.iteration = i;
            r.nnz_x = h[static_cast<size_t>(i)].nnz_x;
            r.kernel = h[static_cast<size_t>(i)].kernel;
            r.exec_mode = h[static_cast<size_t>(i)].exec_mode;
            r.feature_s = 0;
            r.predict_s = 0;  // decided on the device, inside the level's time
            r.convert_s = 0;  // no format conversion: the frontier is produced in the form the level reads
            const unsigned long long t1 = h[static_cast<size_t>(i + 1)].t0, t0 = h[static_cast<size_t>(i)].t0;
            r.kernel_s = t1 > t0 ? static_cast<double>(t1 - t0) * 1e-9 : 0.0;
        }
    }
    if (!levels) return;
    DevBuf l64;
    int64_t* d64 = static_cast<int64_t*>(l64.ensure(sizeof(int64_t) * static_cast<size_t>(n)));
    widen_levels(ctx, P.lv.as<int32_t>(), n, d64);
    ADA_CUDA(cudaMemcpyAsync(levels, d64, sizeof(int64_t) * static_cast<size_t>(n), cudaMemcpyDeviceToHost,
                             ctx.stream));
    ctx.sync();
}

}  // namespace ada

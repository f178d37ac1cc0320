// bfs_graph.cu -- the device-resident BFS level loop (SPEC.md:489-497 driver,
// "levels 3-5 are <= 5 MB each, so they are launch- and
// latency-dominated: keep the BFS loop device-side or graph-captured").
//
// When the next frontier's membership does not depend on values (the
// boolean semiring, or a pattern matrix under plus-times / min-plus, where
// y_i != identity iff row i has a frontier neighbour) every level is one of
//
//   push  (column choices K4-K7): each unvisited row reached from the
//         frontier is claimed once (atomicCAS on its level) and appended to
//         the next frontier list (one counter update per warp and batch);
//   pull  (row choices K0-K3): the output-masked row pull (K2/K3 with the
//         visited rows skipped); a frontier neighbour is a column whose level
//         is the previous level, and a row stops at its first one.  A pull
//         only marks levels and counts the new frontier (size, effective
//         nnz) in spread counters: no list is built.
//
// and the choice -- the built-in bytes model, or the trained selector's
// trees walked ON THE DEVICE over the same 13 features the host selector
// reads (matrix features + nnz_x / x_sparsity / nnz_s / m_sparsity from the
// frontier counters; the splits on matrix features folded on the host, so
// the walk is a few shared-memory nodes) -- is made by a one-warp kernel at
// the start of the level.  The whole traversal is ONE CUDA graph built once
// per (matrix, context, policy): a WHILE conditional node repeats a
// two-level body; in each level the decision kernel sets a SWITCH handle so
// only the chosen branch runs, every kernel reading its sizes from device
// memory:
//
//   Push      the source's push over K6's load-balanced tiles (eff offsets
//             written by the init kernel);
//   Pull      the masked pull, 4 rows per thread;
//   MarkPush  a push from the previous (pull) level's marks, one pass over
//             the level array; vertices of high degree become chunk tasks
//             for a second, grid-wide kernel;
//   ListPush  the same over the list a push appended;
//   Tail      small frontiers pushed level after level by one block, with
//             the per-level decision made in the kernel (one node for the
//             whole tail of the traversal).
//
// Kernel nodes inside conditional bodies cost ~5 us each and a
// WHILE/SWITCH level ~6 us on B200 (tools/microbench/graph_cond_mb.cu), so
// every branch is at most two kernels and none needs a scan.  One graph
// launch and one host synchronisation per traversal.  Per-level reports
// (kernel, frontier size, effective nnz, device time from %globaltimer) are
// logged on the device.
#include <algorithm>
#include <functional>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "device.cuh"
#include "internal.hpp"
#include "kernels.hpp"
#include "prims.cuh"

namespace ada {

namespace {

constexpr int kMaxLog = 1 << 16;    // per-level log capacity
constexpr int kTile = 256;          // effective entries per push warp tile
constexpr int kWin = 128;           // support positions staged per warp tile
enum { kModeDone = 0, kModePush = 1, kModePull = 2 };
// bodies of a level's SWITCH node (any other value: no body runs)
enum { kBranchPush = 0, kBranchPull = 1, kBranchTail = 2, kBranchMarkPush = 3, kBranchListPush = 4, kBranchNone = 5 };
constexpr int kSpread = 256;  // a pull level's (count, degree) counters, spread against contention
constexpr unsigned long long kTailMax = 4096;    // frontier size the one-block tail loop takes
constexpr unsigned long long kTailEdges = 8192;  // and its effective entries

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
    int eff_ok;                 // the current frontier's eff offsets are valid (init wrote them)
    int pending;                // a level ran since the last decision (its results not yet accounted)
    int list_ok;                // the current frontier exists as a list (a pull only marks levels)
};
static_assert(sizeof(BfsState) % 8 == 0, "BfsState is copied as int64 words");

struct LogEntry {               // one row of adaspmv_iteration_report
    long long nnz_x, nnz_s;
    int kernel, exec_mode;
    unsigned long long t0;      // %globaltimer at the level's decision (ns)
#ifdef ADA_BFS_TRACE
    unsigned long long tk0, tk1;  // first block start / last block end of the level's kernels
#endif
};

// Flattened decision trees for the device walk.
struct DevTrees {
    const int32_t* feature;
    const int32_t* left;
    const int32_t* right;
    const int32_t* leaf;
    const double* threshold;
    int root[4];  // [3] = -1 without a workload_col tree (schema 1)
    // The same trees specialised to the matrix: every split on a matrix
    // feature (0-8, fixed for the traversal) folded on the host, leaving only
    // splits on the frontier features 9-12 -- a few nodes, staged in shared
    // memory by the deciding kernel (a walk through global memory is a chain
    // of dependent loads per node, ~10 us per decision).  nsmall = 0: use
    // the full trees.
    const struct SmallNode* small;
    int nsmall;
    int sroot[4];
};
struct SmallNode {
    double thr;
    int16_t feat, left, right, leaf;
};
constexpr int kSmallNodes = 256;

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Diagnostic build (-DADA_BFS_TRACE): the level's kernels record their
// first-block start / last-block end in its log entry.
#ifdef ADA_BFS_TRACE
__device__ LogEntry* g_bfs_log;
#define BFS_TRACE_BEGIN(st) \
    if (threadIdx.x == 0 && (st)->nlog > 0) atomicMin(&g_bfs_log[(st)->nlog - 1].tk0, globaltimer())
#define BFS_TRACE_END(st)                                                                          \
    do {                                                                                           \
        __syncthreads();                                                                           \
        if (threadIdx.x == 0 && (st)->nlog > 0) atomicMax(&g_bfs_log[(st)->nlog - 1].tk1, globaltimer()); \
    } while (0)
#else
#define BFS_TRACE_BEGIN(st)
#define BFS_TRACE_END(st)
#endif

__device__ int tree_walk(const DevTrees& t, const SmallNode* sn, int which, const double* f) {
    if (sn) {
        int i = t.sroot[which];
        for (int guard = 0; guard < kSmallNodes; ++guard) {
            const SmallNode& nd = sn[i];
            if (nd.feat < 0) return nd.leaf;
            i = f[nd.feat] <= nd.thr ? nd.left : nd.right;  // <= goes left
        }
        return 0;
    }
    int i = t.root[which];
    for (int guard = 0; guard < 4096; ++guard) {
        const int32_t feat = t.feature[i];
        if (feat < 0) return t.leaf[i];
        i = f[feat] <= t.threshold[i] ? t.left[i] : t.right[i];  // <= goes left
    }
    return 0;
}

// Stages the specialised trees in shared memory (all threads of the calling
// group take part; returns nullptr when they are not available).
__device__ __forceinline__ const SmallNode* stage_trees(const DevTrees& t, int use_trees, SmallNode* buf, int tid,
                                                        int nthreads) {
    if (!use_trees || t.nsmall <= 0) return nullptr;
    for (int i = tid; i < t.nsmall; i += nthreads) buf[i] = t.small[i];
    return buf;
}

// The kernel for a frontier of nf vertices / ns effective entries: the
// trained selector's trees (SPEC.md:226 feature order, as selector.cpp reads
// them) or the built-in bytes model (bfs.cu heuristic_kernel).  `visited`
// counts the frontier.
__device__ int bfs_choose(const DevTrees& trees, const SmallNode* sn, int use_trees, const double* mfeat, int64_t n,
                          int64_t nnz, int vbytes, long long visited, unsigned long long nf, unsigned long long ns) {
    if (use_trees) {
        double f[ADASPMV_NUM_FEATURES];
        for (int i = 0; i < 9; ++i) f[i] = sn ? 0.0 : mfeat[i];  // folded into the specialised trees
        f[9] = static_cast<double>(nf);
        f[10] = n > 0 ? static_cast<double>(nf) / static_cast<double>(n) : 0.0;
        f[11] = static_cast<double>(ns);
        f[12] = nnz > 0 ? static_cast<double>(ns) / static_cast<double>(nnz) : 0.0;
        const int pattern = tree_walk(trees, sn, 0, f);
        const int lb = tree_walk(trees, sn, pattern == 0 && trees.root[3] >= 0 ? 3 : 1, f) == 1 ? 1 : 0;
        if (pattern == 2) return lb;
        if (pattern == 1) return 2 + lb;
        return 4 + 2 * lb + (tree_walk(trees, sn, 2, f) == 1 ? 1 : 0);
    }
    // SURVEY.md 8(d) push / masked-pull bytes
    const double unvisited = n > 0 ? 1.0 - static_cast<double>(visited) / static_cast<double>(n) : 0.0;
    const double push = static_cast<double>(nf) * 20.0 + static_cast<double>(ns) * (4.0 + vbytes) +
                        (ns <= 4096 ? 0.0 : static_cast<double>(n) * vbytes);
    const double pull = static_cast<double>(n + 1) * 8.0 + static_cast<double>(nnz) * 4.0 * unvisited +
                        static_cast<double>(n) / 8.0 + static_cast<double>(n) * vbytes * unvisited;
    return push <= pull ? (ns <= 4096 ? 7 : 6) : 2;
}

// Start of a level: decide push / pull for the frontier of parity p.
// The level's branch is selected by setting the graph's conditional
// handles: IF(push) and IF(pull) bodies (only the chosen one runs), and the
// WHILE handle that repeats the two-level body until the frontier is empty.
__global__ void bfs_decide_kernel(BfsState* st, LogEntry* log, int p, DevTrees trees, int use_trees,
                                  const double* mfeat, int64_t n, int64_t nnz, int vbytes,
                                  unsigned long long* pcnt, unsigned long long* bigc,
                                  cudaGraphConditionalHandle hbranch, cudaGraphConditionalHandle hwhile) {
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
    __shared__ SmallNode s_tree[kSmallNodes];
    const SmallNode* sn = stage_trees(trees, use_trees, s_tree, threadIdx.x, 32);
    __syncwarp();
    if (threadIdx.x != 0) return;
    cudaGraphSetConditional(hbranch, kBranchNone);
    *bigc = 0;  // the scan push's big-vertex tasks of this level
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
    const int k = bfs_choose(trees, sn, use_trees, mfeat, n, nnz, vbytes, st->visited, nf, ns);
    st->kernel = k;
    st->mode = k >= 4 ? kModePush : kModePull;
    cudaGraphSetConditional(hbranch, k < 4                                ? kBranchPull
                                     : !st->list_ok                       ? kBranchMarkPush
                                     : st->eff_ok                         ? kBranchPush
                                     : ns <= kTailEdges && nf <= kTailMax ? kBranchTail
                                                                          : kBranchListPush);
    st->level += 1;
    st->nf[p ^ 1] = 0;
    st->ns[p ^ 1] = 0;
    st->pending = 1;
    if (st->nlog < kMaxLog) {
        LogEntry& e = log[st->nlog];
        e.nnz_x = static_cast<long long>(nf);
        e.nnz_s = static_cast<long long>(ns);
        e.kernel = k;
        e.exec_mode = k >= 4 ? ADASPMV_EXEC_FUSED_PUSH_LB : ADASPMV_EXEC_MASKED_PULL;
        e.t0 = now;
#ifdef ADA_BFS_TRACE
        e.tk0 = ~0ull;
        e.tk1 = 0;
#endif
    }
    st->nlog += 1;
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

// Push over K6's load-balanced tiles (kernels_col.cu col_lb_kernel MODE 2),
// grid-stride over the tiles of the frontier's effective entries.
__global__ void __launch_bounds__(256) bfs_push_kernel(BfsState* st, int p, const int32_t* __restrict__ f,
                                                       const int64_t* __restrict__ eff,
                                                       const int64_t* __restrict__ co,
                                                       const int32_t* __restrict__ ri, int32_t* __restrict__ lv,
                                                       int32_t* __restrict__ nf_out) {
    BFS_TRACE_BEGIN(st);
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
        // claims of the whole tile, appended with one counter update per warp
        // and tile (per instruction, the fat levels serialise on the counters)
        unsigned bal[kJ];
        long long deg = 0;
        int cnt = 0;
        // all the tile's level reads, then all its claims, in flight together
        int lr[kJ];
#pragma unroll
        for (int j = 0; j < kJ; ++j) lr[j] = kidx[j] >= 0 ? lv[r[j]] : 0;
        bool claim[kJ];
#pragma unroll
        for (int j = 0; j < kJ; ++j) claim[j] = lr[j] < 0 && atomicCAS(lv + r[j], -1, level) == -1;
#pragma unroll
        for (int j = 0; j < kJ; ++j) {
            bal[j] = __ballot_sync(kFull, claim[j]);
            cnt += __popc(bal[j]);
            if (claim[j]) deg += __ldg(co + r[j] + 1) - __ldg(co + r[j]);
        }
        if (cnt == 0) continue;  // warp-uniform
        deg = warp_sum(deg);
        unsigned long long base = 0;
        if (lane == 0) {
            base = atomicAdd(&st->nf[q], static_cast<unsigned long long>(cnt));
            atomicAdd(&st->ns[q], static_cast<unsigned long long>(deg));
        }
        base = __shfl_sync(kFull, base, 0);
#pragma unroll
        for (int j = 0; j < kJ; ++j) {
            if ((bal[j] >> lane) & 1u) nf_out[base + __popc(bal[j] & lanemask_lt())] = r[j];
            base += __popc(bal[j]);
        }
    }
    BFS_TRACE_END(st);
}

// Output-masked pull with early exit (bfs.cu bfs_pull_kernel), G lanes per
// row; a row with a frontier neighbour (a column of the previous level, read
// from the level array: no frontier bitmap to build and clear) gets its
// level.  A resident grid strides over 256-thread row windows: a full grid
// (one block per window, 16 K blocks on C3) pays ~10 us of block launches
// per level on B200 (tools/microbench/graph_cond_mb.cu), and the fine
// interleave of windows keeps rows that run long spread over the SMs.
// A push after a pull reads the marks (MarkPush): no list is compacted.
template <int G>
__device__ __forceinline__ void pull_body(long long bid, long long nblk, int level, int64_t rows,
                                          const int64_t* __restrict__ ro, const int32_t* __restrict__ ci,
                                          const int64_t* __restrict__ co, int32_t* __restrict__ lv,
                                          unsigned long long* __restrict__ pcnt) {
    // level: of the rows this step discovers (frontier = the vertices of level - 1)
    const int lane = threadIdx.x & 31;
    const int lg = threadIdx.x & (G - 1);
    const unsigned grp = G == 32 ? kFull : (((1u << G) - 1u) << (lane & ~(G - 1)));
    unsigned long long c = 0, d = 0;  // this lane's joins and their column degrees (lane 0 sums the warp)
    const long long total = rows * G;
    for (long long base = bid * 256; base < total; base += nblk * 256) {  // block-uniform trip count
        const long long row = (base + threadIdx.x) / G;
        const bool live = row < rows && lv[row] < 0;
        bool hit = false;
        if (live) {
            const long long b = __ldg(ro + row), e = __ldg(ro + row + 1);
            for (long long k0 = b + lg; k0 < e && !hit; k0 += G * 4) {
                // 4 neighbours' levels in flight at once (a short-circuit
                // chain would serialise the 4 dependent loads)
                int cc[4], lc[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) cc[j] = k0 + j * G < e ? __ldg(ci + k0 + j * G) : -1;
#pragma unroll
                for (int j = 0; j < 4; ++j) lc[j] = cc[j] >= 0 ? lv[cc[j]] : -2;
#pragma unroll
                for (int j = 0; j < 4; ++j) hit |= lc[j] == level - 1;
            }
        }
        const bool any = (__ballot_sync(kFull, hit) & grp) != 0u;
        const bool join = live && any && lg == 0;
        if (join) {
            lv[row] = level;
            c += 1;
            d += static_cast<unsigned long long>(__ldg(co + row + 1) - __ldg(co + row));
        }
    }
    // the level's size and effective nnz, one spread counter update per warp
    c = warp_sum(c);
    if (c) {
        d = warp_sum(d);
        if (lane == 0) {
            const int slot = static_cast<int>((bid * 8 + (threadIdx.x >> 5)) % kSpread);
            atomicAdd(pcnt + 2 * slot, c);
            atomicAdd(pcnt + 2 * slot + 1, d);
        }
    }
}

template <int G>
__global__ void __launch_bounds__(256) bfs_pull_mark_kernel(const BfsState* st, int64_t rows,
                                                            const int64_t* __restrict__ ro,
                                                            const int32_t* __restrict__ ci,
                                                            const int64_t* __restrict__ co,
                                                            int32_t* __restrict__ lv,
                                                            unsigned long long* __restrict__ pcnt) {
    pull_body<G>(blockIdx.x, gridDim.x, st->level, rows, ro, ci, co, lv, pcnt);
}

// The pull with one lane per row, 4 rows per thread (consecutive: one 16-B
// level load) and their first kProbe neighbours' levels in flight together:
// a thread holding one row waits ~4 dependent round trips (level, offsets,
// neighbour, its level) per row, and with ~14 rows per thread per level on
// C3 those chains, not bandwidth, set the level's time.  Rows not settled
// by the probe continue 4 neighbours at a time.
constexpr int kProbe = 2;

__device__ __forceinline__ void pull4_body(long long bid, long long nblk, int level, int64_t rows,
                                           const int64_t* __restrict__ ro, const int32_t* __restrict__ ci,
                                           const int64_t* __restrict__ co, int32_t* __restrict__ lv,
                                           unsigned long long* __restrict__ pcnt) {
    const int lane = threadIdx.x & 31;
    unsigned long long c = 0, d = 0;
    for (long long w = bid; w * 1024 < rows; w += nblk) {
        const long long r0 = w * 1024 + threadIdx.x * 4;
        if (r0 >= rows) continue;
        int l4[4];
        if (r0 + 3 < rows) {
            const int4 t = *reinterpret_cast<const int4*>(lv + r0);
            l4[0] = t.x;
            l4[1] = t.y;
            l4[2] = t.z;
            l4[3] = t.w;
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) l4[j] = r0 + j < rows ? lv[r0 + j] : 0;
        }
        bool live[4];
        bool any_live = false;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            live[j] = l4[j] < 0;
            any_live |= live[j];
        }
        if (!any_live) continue;
        long long off[5];
#pragma unroll
        for (int j = 0; j < 5; ++j) off[j] = r0 + j <= rows ? __ldg(ro + r0 + j) : 0;
        int cc[4][kProbe];
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int t = 0; t < kProbe; ++t)
                cc[j][t] = live[j] && off[j] + t < off[j + 1] ? __ldg(ci + off[j] + t) : -1;
        int lc[4][kProbe];
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int t = 0; t < kProbe; ++t) lc[j][t] = cc[j][t] >= 0 ? lv[cc[j][t]] : -2;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (!live[j]) continue;
            bool hit = false;
#pragma unroll
            for (int t = 0; t < kProbe; ++t) hit |= lc[j][t] == level - 1;
            const long long e = off[j + 1];
            for (long long k0 = off[j] + kProbe; k0 < e && !hit; k0 += 4) {
                int c4[4], l4n[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) c4[u] = k0 + u < e ? __ldg(ci + k0 + u) : -1;
#pragma unroll
                for (int u = 0; u < 4; ++u) l4n[u] = c4[u] >= 0 ? lv[c4[u]] : -2;
#pragma unroll
                for (int u = 0; u < 4; ++u) hit |= l4n[u] == level - 1;
            }
            if (hit) {
                lv[r0 + j] = level;
                c += 1;
                d += static_cast<unsigned long long>(__ldg(co + r0 + j + 1) - __ldg(co + r0 + j));
            }
        }
    }
    c = warp_sum(c);
    if (c) {
        d = warp_sum(d);
        if (lane == 0) {
            const int slot = static_cast<int>((bid * 8 + (threadIdx.x >> 5)) % kSpread);
            atomicAdd(pcnt + 2 * slot, c);
            atomicAdd(pcnt + 2 * slot + 1, d);
        }
    }
}

__global__ void __launch_bounds__(256) bfs_pull_mark4_kernel(const BfsState* st, int64_t rows,
                                                             const int64_t* __restrict__ ro,
                                                             const int32_t* __restrict__ ci,
                                                             const int64_t* __restrict__ co,
                                                             int32_t* __restrict__ lv,
                                                             unsigned long long* __restrict__ pcnt) {
    BFS_TRACE_BEGIN(st);
    pull4_body(blockIdx.x, gridDim.x, st->level, rows, ro, ci, co, lv, pcnt);
    BFS_TRACE_END(st);
}

// Push without offsets: the frontier is read either from the previous
// level's marks (a pull left no list: every vertex with lv == level - 1) or
// from the list a push appended, in one pass -- no compaction or offset scan
// (3-5 kernel nodes per level through the graph machinery).  A resident grid
// strides over 256-vertex windows; each warp flattens the effective entries
// of its 32 vertices (degree prefix in registers, the owning lane found by a
// 5-step shuffle search) and moves them 4 per lane at a time with all loads,
// level reads and claims in flight together.  Vertices of degree >
// kBigDeg become (vertex, chunk) tasks of kBigChunk entries, appended with
// ONE 64-bit atomic (count << 40 | tasks) so the list's task starts ascend,
// and bfs_big_push_kernel spreads them over the whole grid.
constexpr int kBigDeg = 256;
constexpr int kBigChunk = 1024;
constexpr int kBigShift = 40;

__device__ __forceinline__ void claim_and_append(const int32_t (&r)[4], int32_t* __restrict__ lv, int level,
                                                 const int64_t* __restrict__ co, unsigned long long* out_nf,
                                                 unsigned long long* out_ns, int32_t* __restrict__ nf_out, int lane) {
    int lr[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) lr[j] = r[j] >= 0 ? lv[r[j]] : 0;
    bool claim[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) claim[j] = lr[j] < 0 && atomicCAS(lv + r[j], -1, level) == -1;
    unsigned bal[4];
    int cnt = 0;
    long long deg = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        bal[j] = __ballot_sync(kFull, claim[j]);
        cnt += __popc(bal[j]);
        if (claim[j]) deg += __ldg(co + r[j] + 1) - __ldg(co + r[j]);
    }
    if (cnt == 0) return;  // warp-uniform
    deg = warp_sum(deg);
    unsigned long long base = 0;
    if (lane == 0) {
        base = atomicAdd(out_nf, static_cast<unsigned long long>(cnt));
        atomicAdd(out_ns, static_cast<unsigned long long>(deg));
    }
    base = __shfl_sync(kFull, base, 0);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        if (claim[j]) nf_out[base + __popc(bal[j] & lanemask_lt())] = r[j];
        base += __popc(bal[j]);
    }
}

// One warp pushes the frontier vertices its lanes hold (v < 0: none).
__device__ __forceinline__ void push_members(int32_t v, int level, const int64_t* __restrict__ co,
                                             const int32_t* __restrict__ ri, int32_t* __restrict__ lv,
                                             unsigned long long* out_nf, unsigned long long* out_ns,
                                             int32_t* __restrict__ nf_out, unsigned long long* __restrict__ bigc,
                                             uint2* __restrict__ bigl, int lane) {
    long long b = 0, deg = 0;
    if (v >= 0) {
        b = __ldg(co + v);
        deg = __ldg(co + v + 1) - b;
    }
    if (deg > kBigDeg) {
        const unsigned long long nch = static_cast<unsigned long long>((deg + kBigChunk - 1) / kBigChunk);
        const unsigned long long old = atomicAdd(bigc, (1ull << kBigShift) + nch);
        bigl[old >> kBigShift] =
            make_uint2(static_cast<unsigned>(v), static_cast<unsigned>(old & ((1ull << kBigShift) - 1)));
        deg = 0;
    }
    const long long incl = warp_inclusive_sum(deg);
    const long long wtot = __shfl_sync(kFull, incl, 31);
    const long long excl = incl - deg;
    for (long long e0 = 0; e0 < wtot; e0 += 128) {  // warp-uniform trip count
        int32_t r[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const long long e = e0 + j * 32 + lane;
            int lo = 0;  // largest lane whose exclusive prefix <= e (every lane shuffles)
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                const int cand = lo + step;
                const long long ev = __shfl_sync(kFull, excl, cand & 31);
                if (cand < 32 && ev <= e) lo = cand;
            }
            const long long ob = __shfl_sync(kFull, b, lo), oe = __shfl_sync(kFull, excl, lo);
            r[j] = e < wtot ? __ldg(ri + ob + (e - oe)) : -1;
        }
        claim_and_append(r, lv, level, co, out_nf, out_ns, nf_out, lane);
    }
}

// Warp-granular grid stride.  List mode: 32 list entries per warp window.
// Mark mode: 128 vertices per warp window (one 16-B level load per lane),
// the members gathered through shared memory and pushed 32 at a time -- a
// frontier of a few % of the vertices costs ~4 dependent round trips per
// 128 vertices, not per 32.
template <bool kList>
__device__ __forceinline__ void scan_push_body(long long bid, long long nblk, int level, const int32_t* __restrict__ fl,
                                               long long cnt, int64_t n, const int64_t* __restrict__ co,
                                               const int32_t* __restrict__ ri, int32_t* __restrict__ lv,
                                               unsigned long long* out_nf, unsigned long long* out_ns,
                                               int32_t* __restrict__ nf_out, unsigned long long* __restrict__ bigc,
                                               uint2* __restrict__ bigl, int32_t (*s_mem)[128]) {
    // level: of the vertices this step discovers; cnt: list length (list mode)
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const long long gw = bid * 8 + wib;
    const long long nw = nblk * 8;
    if (kList) {
        for (long long w = gw; w * 32 < cnt; w += nw) {
            const long long i = w * 32 + lane;
            push_members(i < cnt ? fl[i] : -1, level, co, ri, lv, out_nf, out_ns, nf_out, bigc, bigl, lane);
        }
    } else {
        for (long long w = gw; w * 128 < n; w += nw) {
            const long long v0 = w * 128 + lane * 4;
            int l4[4];
            if (v0 + 3 < n) {
                const int4 t = *reinterpret_cast<const int4*>(lv + v0);
                l4[0] = t.x;
                l4[1] = t.y;
                l4[2] = t.z;
                l4[3] = t.w;
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j) l4[j] = v0 + j < n ? lv[v0 + j] : 0;
            }
            int mine = 0;
#pragma unroll
            for (int j = 0; j < 4; ++j) mine += l4[j] == level - 1;
            const int incl = warp_inclusive_sum(mine);
            const int tot = __shfl_sync(kFull, incl, 31);
            if (tot == 0) continue;  // warp-uniform
            int o = incl - mine;
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (l4[j] == level - 1) s_mem[wib][o++] = static_cast<int32_t>(v0 + j);
            __syncwarp();
            for (int k = 0; k < tot; k += 32)
                push_members(k + lane < tot ? s_mem[wib][k + lane] : -1, level, co, ri, lv, out_nf, out_ns, nf_out,
                             bigc, bigl, lane);
            __syncwarp();
        }
    }
}

template <bool kList>
__global__ void __launch_bounds__(256) bfs_scan_push_kernel(BfsState* st, int p, const int32_t* __restrict__ fl,
                                                            int64_t n, const int64_t* __restrict__ co,
                                                            const int32_t* __restrict__ ri, int32_t* __restrict__ lv,
                                                            int32_t* __restrict__ nf_out,
                                                            unsigned long long* __restrict__ bigc,
                                                            uint2* __restrict__ bigl) {
    __shared__ int32_t s_mem[8][128];
    BFS_TRACE_BEGIN(st);
    const int q = p ^ 1;
    scan_push_body<kList>(blockIdx.x, gridDim.x, st->level, fl, kList ? static_cast<long long>(st->nf[p]) : 0, n, co,
                          ri, lv, &st->nf[q], &st->ns[q], nf_out, bigc, bigl, s_mem);
    BFS_TRACE_END(st);
}

// The big vertices' chunks: task t -> (vertex, chunk) by a search over the
// ascending task starts; 256 threads x 4 entries per task.
__device__ __forceinline__ void big_push_body(long long bid, long long nblk, int level,
                                              const int64_t* __restrict__ co, const int32_t* __restrict__ ri,
                                              int32_t* __restrict__ lv, unsigned long long* out_nf,
                                              unsigned long long* out_ns, int32_t* __restrict__ nf_out,
                                              unsigned long long c, const uint2* __restrict__ bigl) {
    const long long nb = static_cast<long long>(c >> kBigShift);
    const long long ntask = static_cast<long long>(c & ((1ull << kBigShift) - 1));
    const int lane = threadIdx.x & 31;
    for (long long t = bid; t < ntask; t += nblk) {
        long long lo = 0, hi = nb;  // largest entry with start <= t
        while (hi - lo > 1) {
            const long long mid = (lo + hi) >> 1;
            if (static_cast<long long>(bigl[mid].y) <= t) lo = mid;
            else hi = mid;
        }
        const uint2 ent = bigl[lo];
        const long long b = __ldg(co + ent.x), e = __ldg(co + ent.x + 1);
        const long long c0 = b + (t - static_cast<long long>(ent.y)) * kBigChunk;
        const long long c1 = min(e, c0 + kBigChunk);
        for (long long k0 = c0 + (threadIdx.x & ~31) * 4; k0 < c1; k0 += 256 * 4) {  // warp-uniform
            int32_t r[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const long long k = k0 + j * 32 + lane;
                r[j] = k < c1 ? __ldg(ri + k) : -1;
            }
            claim_and_append(r, lv, level, co, out_nf, out_ns, nf_out, lane);
        }
    }
}

__global__ void __launch_bounds__(256) bfs_big_push_kernel(BfsState* st, int p, const int64_t* __restrict__ co,
                                                           const int32_t* __restrict__ ri, int32_t* __restrict__ lv,
                                                           int32_t* __restrict__ nf_out,
                                                           const unsigned long long* __restrict__ bigc,
                                                           const uint2* __restrict__ bigl) {
    const unsigned long long c = *bigc;
    if ((c & ((1ull << kBigShift) - 1)) == 0) return;
    BFS_TRACE_BEGIN(st);
    const int q = p ^ 1;
    big_push_body(blockIdx.x, gridDim.x, st->level, co, ri, lv, &st->nf[q], &st->ns[q], nf_out, c, bigl);
    BFS_TRACE_END(st);
}

// The tail of a traversal: a small frontier (<= kTailMax vertices, <=
// kTailEdges effective entries) that a push appended is pushed by ONE block,
// and so are the following levels while the decision for them is again a
// small push -- one kernel node for the whole tail instead of a decision, a
// SWITCH and a push per level (~11 us each through the graph machinery:
// tools/microbench/graph_cond_mb.cu).  Each continued level is decided and
// logged exactly as bfs_decide_kernel would (same bfs_choose, same
// accounting); on exit the last frontier is left, pending, at parity p ^ 1
// for the graph's next decision.
__global__ void __launch_bounds__(1024) bfs_tail_kernel(BfsState* st, LogEntry* log, int p, int32_t* __restrict__ f0,
                                                        int32_t* __restrict__ f1, const int64_t* __restrict__ co,
                                                        const int32_t* __restrict__ ri, int32_t* __restrict__ lv,
                                                        DevTrees trees, int use_trees, const double* mfeat, int64_t n,
                                                        int64_t nnz, int vbytes) {
    __shared__ unsigned long long s_nf, s_ns;
    __shared__ int s_go;
    __shared__ int s_eff[kTailMax + 1];  // the frontier's degree prefix
    __shared__ int32_t s_v[kTailMax];    // and its vertices
    __shared__ int s_scan[1024 / 32 + 1];
    __shared__ SmallNode s_tree[kSmallNodes];
    const SmallNode* sn = stage_trees(trees, use_trees, s_tree, threadIdx.x, 1024);  // the loop syncs first
    const int lane = threadIdx.x & 31;
    int cp = p;  // parity of the frontier being pushed
    for (;;) {
        const int32_t* fin = cp ? f1 : f0;
        int32_t* fout = cp ? f0 : f1;
        const int nx = static_cast<int>(st->nf[cp]);
        const int level = st->level;
        // the frontier's effective entries flattened over the block (<= 4 per
        // thread): every edge's loads are independent, not a per-vertex walk
        int d[kTailMax / 1024], loc = 0;
#pragma unroll
        for (int j = 0; j < kTailMax / 1024; ++j) {
            const int i = threadIdx.x * (kTailMax / 1024) + j;
            d[j] = 0;
            if (i < nx) {
                const int32_t v = fin[i];
                s_v[i] = v;
                d[j] = static_cast<int>(__ldg(co + v + 1) - __ldg(co + v));
            }
            loc += d[j];
        }
        int tot;
        int ex = block_exclusive_sum<1024>(loc, s_scan, &tot);
#pragma unroll
        for (int j = 0; j < kTailMax / 1024; ++j) {
            const int i = threadIdx.x * (kTailMax / 1024) + j;
            if (i < nx) s_eff[i] = ex;
            ex += d[j];
        }
        if (threadIdx.x == 0) s_nf = s_ns = 0;
        __syncthreads();
        constexpr int kE = kTailEdges / 1024;
        int32_t r[kE];
#pragma unroll
        for (int j = 0; j < kE; ++j) {
            const int e = threadIdx.x + j * 1024;
            r[j] = -1;
            if (e < tot) {
                int lo = 0, hi = nx;  // largest i with s_eff[i] <= e
                while (hi - lo > 1) {
                    const int mid = (lo + hi) >> 1;
                    if (s_eff[mid] <= e) lo = mid;
                    else hi = mid;
                }
                r[j] = __ldg(ri + __ldg(co + s_v[lo]) + (e - s_eff[lo]));
            }
        }
        int lr[kE];
#pragma unroll
        for (int j = 0; j < kE; ++j) lr[j] = r[j] >= 0 ? lv[r[j]] : 0;
        bool claim[kE];
#pragma unroll
        for (int j = 0; j < kE; ++j) claim[j] = lr[j] < 0 && atomicCAS(lv + r[j], -1, level) == -1;
#pragma unroll
        for (int j = 0; j < kE; ++j) {
            const unsigned bal = __ballot_sync(kFull, claim[j]);
            if (bal == 0u) continue;
            const unsigned long long dg =
                warp_sum(claim[j] ? static_cast<unsigned long long>(__ldg(co + r[j] + 1) - __ldg(co + r[j])) : 0ull);
            unsigned long long base = 0;
            if (lane == 0) {
                base = atomicAdd(&s_nf, static_cast<unsigned long long>(__popc(bal)));
                atomicAdd(&s_ns, dg);
            }
            base = __shfl_sync(kFull, base, 0);
            if (claim[j]) fout[base + __popc(bal & lanemask_lt())] = r[j];
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned long long nf = s_nf, ns = s_ns;
            st->nf[cp ^ 1] = nf;
            st->ns[cp ^ 1] = ns;
            int go = 0;
            if (nf > 0 && nf <= kTailMax && ns <= kTailEdges) {
                const long long visited = st->visited + static_cast<long long>(nf);
                const int k = bfs_choose(trees, sn, use_trees, mfeat, n, nnz, vbytes, visited, nf, ns);
                if (k >= 4) {  // the next level is a small push again: account and continue
                    go = 1;
                    st->visited = visited;
                    st->level = level + 1;
                    st->kernel = k;
                    st->nf[cp] = 0;
                    st->ns[cp] = 0;
                    if (st->nlog < kMaxLog) {
                        LogEntry& le = log[st->nlog];
                        le.nnz_x = static_cast<long long>(nf);
                        le.nnz_s = static_cast<long long>(ns);
                        le.kernel = k;
                        le.exec_mode = ADASPMV_EXEC_FUSED_PUSH_LB;
                        le.t0 = globaltimer();
                    }
                    st->nlog += 1;
                }
            }
            s_go = go;
        }
        __syncthreads();
        if (!s_go) break;
        cp ^= 1;
    }
    // the last frontier sits at parity cp ^ 1; the next decision reads p ^ 1
    if (cp != p) {
        const long long nx = static_cast<long long>(st->nf[p]);
        int32_t* dst = p ? f0 : f1;
        const int32_t* src = p ? f1 : f0;
        for (long long i = threadIdx.x; i < nx; i += 1024) dst[i] = src[i];
        if (threadIdx.x == 0) {
            st->nf[p ^ 1] = st->nf[p];
            st->ns[p ^ 1] = st->ns[p];
        }
    }
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
            st->pending = 0;
        st->eff_ok = 1;
        st->list_ok = 1;
        eff[0] = 0;
        eff[1] = static_cast<int64_t>(st->ns[0]);
    }
}

// ---------------------------------------------------------------------------
// The whole traversal as ONE cooperative persistent kernel (the default when
// the device supports cooperative launch): the level bodies above run
// grid-strided over exactly the co-resident blocks, separated by grid
// barriers -- one per pull level, one or two per push level -- instead of
// the graph's per-level decision node, SWITCH and kernel nodes (~15 us per
// level through the graph machinery).  Every block makes the same decision
// from the same counters (no broadcast needed); block 0 alone logs and keeps
// the bookkeeping.  Per-level counters rotate over 3 slots: slot (L+1) % 3
// is written by step L, read by every block after the barrier that ends it,
// and block 0 zeroes slot (L+2) % 3 during step L (its last readers passed
// the barrier ending step L-1, its next writers start after the one ending
// step L).
struct PSlot {
    unsigned long long nf, ns, bigc, pulled;
    unsigned long long pc[2 * kSpread];
};

struct PArgs {
    BfsState* st;
    LogEntry* log;
    int32_t* lv;
    const int64_t* ro;
    const int32_t* ci;
    const int64_t* co;
    const int32_t* ri;
    int32_t* f[2];
    PSlot* slots;
    unsigned* bar;  // [0] root arrivals, [1] generation, then the group counters
    uint2* bigl;
    DevTrees trees;
    int use_trees;
    const double* mfeat;
    int64_t n, nnz;
    int vbytes;
    int64_t source;
    int64_t* host_state;  // mapped host copy of the final BfsState (Context::h_scalars)
};

// Visibility: every block reads what the others wrote in earlier steps
// (levels, lists, counters, tasks) with plain loads.  The barrier's
// gpu-scope fences after the generation flips (release by the last
// arrival, acquire by each waiter, then bar.sync) order those writes before
// the loads and drop the SM's stale L1 lines, as grid.sync() does.
// Grid barrier over co-resident blocks (cooperative launch), two-level:
// a block arrives on one of kBarGroups group counters (own 128-B lines) and
// the last arrival of a group on the root; the last root arrival resets and
// bumps the generation the others wait on.  One flat counter serialises all
// ~740 same-address atomics (~10 us per barrier on B200, measured).
constexpr int kBarGroups = 32;
constexpr int kBarStride = 32;  // unsigned words per counter (128 B)

__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned nblk) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned* gen = bar + 1;
        const unsigned g = *gen;
        const unsigned ng = nblk < kBarGroups ? nblk : kBarGroups;
        const unsigned grp = blockIdx.x % ng;
        const unsigned gsize = nblk / ng + (grp < nblk % ng ? 1u : 0u);
        unsigned* gc = bar + kBarStride * (1 + grp);
        __threadfence();
        bool last = false;
        if (atomicAdd(gc, 1u) == gsize - 1) {
            atomicExch(gc, 0u);
            last = atomicAdd(bar, 1u) == ng - 1;
        }
        if (last) {
            atomicExch(bar, 0u);
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (*gen == g) __nanosleep(64);
        }
        __threadfence();
    }
    __syncthreads();
}

template <int G>
__global__ void __launch_bounds__(256) bfs_persist_kernel(PArgs a) {
    __shared__ int32_t s_mem[8][128];
    __shared__ SmallNode s_tree[kSmallNodes];
    __shared__ unsigned long long s_red[2][8];
    __shared__ int s_k;
    const SmallNode* sn = stage_trees(a.trees, a.use_trees, s_tree, threadIdx.x, 256);
    const long long bid = blockIdx.x, nblk = gridDim.x;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    long long visited = 0;
    int nlog = 0;
    bool list = true;  // the frontier exists as a list (a pull leaves marks)
    // prologue (no separate init launches): levels, the first frontier, the
    // counter slots; the barrier's own words return to 0 after every barrier
    for (long long i = bid * 256 + threadIdx.x; i < a.n; i += nblk * 256) a.lv[i] = i == a.source ? 0 : -1;
    if (bid == 0) {
        for (int s3 = 0; s3 < 3; ++s3) {
            for (int i = threadIdx.x; i < 2 * kSpread; i += 256) a.slots[s3].pc[i] = 0;
            if (threadIdx.x == 0) a.slots[s3].nf = a.slots[s3].ns = a.slots[s3].bigc = a.slots[s3].pulled = 0;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            a.f[0][0] = static_cast<int32_t>(a.source);
            a.slots[0].nf = 1;
            a.slots[0].ns = static_cast<unsigned long long>(a.co[a.source + 1] - a.co[a.source]);
        }
    }
    grid_barrier(a.bar, static_cast<unsigned>(nblk));
    for (int L = 0;; ++L) {
        PSlot* cur = a.slots + L % 3;
        PSlot* nxt = a.slots + (L + 1) % 3;
        // the frontier F_L: a push's counters, or the pull's spread counters
        unsigned long long nf, ns;
        if (__ldcg(&cur->pulled)) {
            unsigned long long c = 0, d = 0;
            for (int i = threadIdx.x; i < kSpread; i += 256) {
                c += __ldcg(cur->pc + 2 * i);
                d += __ldcg(cur->pc + 2 * i + 1);
            }
            c = warp_sum(c);
            d = warp_sum(d);
            if (lane == 0) {
                s_red[0][wib] = c;
                s_red[1][wib] = d;
            }
            __syncthreads();
            nf = ns = 0;
            for (int w = 0; w < 8; ++w) {
                nf += s_red[0][w];
                ns += s_red[1][w];
            }
            __syncthreads();
        } else {
            nf = __ldcg(&cur->nf);
            ns = __ldcg(&cur->ns);
        }
        const unsigned long long now = globaltimer();
        if (nf == 0) {  // every block leaves here, on the same step
            if (bid == 0 && threadIdx.x == 0) {
                if (nlog < kMaxLog) a.log[nlog].t0 = now;  // end stamp of the last level
                BfsState fin{};
                fin.nlog = nlog;
                fin.visited = visited;
                fin.level = L;
                fin.done = 1;
                fin.mode = kModeDone;
                *a.st = fin;
                // straight into the mapped host scalars: no copy launch after the traversal
                const int64_t* w = reinterpret_cast<const int64_t*>(&fin);
                volatile int64_t* h = a.host_state;
                for (size_t i = 0; i < sizeof(BfsState) / sizeof(int64_t); ++i) h[i] = w[i];
                __threadfence_system();
            }
            return;
        }
        visited += static_cast<long long>(nf);
        if (threadIdx.x == 0)
            s_k = bfs_choose(a.trees, sn, a.use_trees, a.mfeat, a.n, a.nnz, a.vbytes, visited, nf, ns);
        __syncthreads();
        const int k = s_k;
        if (bid == 0) {
            if (threadIdx.x == 0 && nlog < kMaxLog) {
                LogEntry& e = a.log[nlog];
                e.nnz_x = static_cast<long long>(nf);
                e.nnz_s = static_cast<long long>(ns);
                e.kernel = k;
                e.exec_mode = k >= 4 ? ADASPMV_EXEC_FUSED_PUSH_LB : ADASPMV_EXEC_MASKED_PULL;
                e.t0 = now;
            }
            PSlot* z = a.slots + (L + 2) % 3;
            for (int i = threadIdx.x; i < 2 * kSpread; i += 256) z->pc[i] = 0;
            if (threadIdx.x == 0) z->nf = z->ns = z->bigc = z->pulled = 0;
        }
        ++nlog;
        const int level = L + 1;  // of the vertices this step discovers
        if (k < 4) {
            if (G == 1) pull4_body(bid, nblk, level, a.n, a.ro, a.ci, a.co, a.lv, nxt->pc);
            else pull_body<G>(bid, nblk, level, a.n, a.ro, a.ci, a.co, a.lv, nxt->pc);
            if (bid == 0 && threadIdx.x == 0) nxt->pulled = 1;
            list = false;
#ifdef ADA_BFS_TRACE
            __syncthreads();
            if (bid == 0 && threadIdx.x == 0 && nlog - 1 < kMaxLog) a.log[nlog - 1].tk0 = globaltimer();
#endif
            grid_barrier(a.bar, static_cast<unsigned>(nblk));
#ifdef ADA_BFS_TRACE
            if (bid == 0 && threadIdx.x == 0 && nlog - 1 < kMaxLog) a.log[nlog - 1].tk1 = globaltimer();
#endif
        } else {
            int32_t* fin = a.f[L & 1];
            int32_t* fout = a.f[(L + 1) & 1];
            if (list)
                scan_push_body<true>(bid, nblk, level, fin, static_cast<long long>(nf), a.n, a.co, a.ri, a.lv,
                                     &nxt->nf, &nxt->ns, fout, &nxt->bigc, a.bigl, s_mem);
            else
                scan_push_body<false>(bid, nblk, level, nullptr, 0, a.n, a.co, a.ri, a.lv, &nxt->nf, &nxt->ns, fout,
                                      &nxt->bigc, a.bigl, s_mem);
            list = true;
#ifdef ADA_BFS_TRACE
            __syncthreads();
            if (bid == 0 && threadIdx.x == 0 && nlog - 1 < kMaxLog) a.log[nlog - 1].tk0 = globaltimer();
#endif
            grid_barrier(a.bar, static_cast<unsigned>(nblk));
#ifdef ADA_BFS_TRACE
            if (bid == 0 && threadIdx.x == 0 && nlog - 1 < kMaxLog) a.log[nlog - 1].tk1 = globaltimer();
#endif
            const unsigned long long c = *reinterpret_cast<volatile unsigned long long*>(&nxt->bigc);
            if (c & ((1ull << kBigShift) - 1)) {
                big_push_body(bid, nblk, level, a.co, a.ri, a.lv, &nxt->nf, &nxt->ns, fout, c, a.bigl);
                grid_barrier(a.bar, static_cast<unsigned>(nblk));
            }
        }
    }
}

}  // namespace

// One captured traversal plan: buffers, flattened trees and the graph.
struct BfsPlan {
    cudaStream_t stream = nullptr;
    uint64_t bundle_id = 0;  // 0 = heuristic
    DevBuf state, log, f[2], eff, lv, trees_i, trees_d, trees_small, mfeat;
    DevTrees dt{};
    DevBuf pcnt;      // a pull level's spread (count, degree) counters
    DevBuf bigc, bigl;  // the scan push's big-vertex tasks (counter, list)
    DevBuf slots, bar;  // the persistent kernel's rotating counters and grid barrier
    // the per-level log in mapped pinned host memory: the reports are read
    // after the traversal's one synchronisation, no copy (the diagnostic
    // trace build keeps it on the device: it updates entries atomically)
    LogEntry* hlog = nullptr;
    LogEntry* dlog = nullptr;
    int persist_G = 0;  // > 0: one cooperative persistent kernel (pull lanes G) instead of the graph
    unsigned persist_grid = 0;
    cudaGraphExec_t exec = nullptr;
    ~BfsPlan() {
        if (exec) cudaGraphExecDestroy(exec);
        if (hlog) cudaFreeHost(hlog);
    }
};

void BfsPlanDeleter::operator()(BfsPlan* p) const { delete p; }

bool bfs_graph_applicable(const Matrix& m, int semiring, int forced) {
    // membership-only levels (see the header), policy = heuristic or selector
    return forced < 0 && (semiring == ADASPMV_OR_AND || m.pattern) && m.rows == m.cols && m.rows > 0 &&
           m.rows < (int64_t(1) << 31) - 1;
}

namespace {

void upload_trees(Context& ctx, const Bundle& b, const double* m_feat, BfsPlan& P) {
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
    // specialised copy: fold the splits on matrix features (the comparison
    // the device walk would make, on the same doubles)
    std::vector<SmallNode> sm;
    bool fits = true;
    std::function<int(const Tree&, int)> add = [&](const Tree& tr, int i) -> int {
        while (tr.feature[static_cast<size_t>(i)] >= 0 && tr.feature[static_cast<size_t>(i)] < 9) {
            const size_t u = static_cast<size_t>(i);
            i = m_feat[tr.feature[u]] <= tr.threshold[u] ? tr.left[u] : tr.right[u];
        }
        const size_t u = static_cast<size_t>(i);
        const int me = static_cast<int>(sm.size());
        if (me >= kSmallNodes) {
            fits = false;
            return 0;
        }
        sm.push_back(SmallNode{0.0, -1, 0, 0, 0});
        if (tr.feature[u] < 0) {
            sm[static_cast<size_t>(me)].leaf = static_cast<int16_t>(tr.leaf[u]);
            return me;
        }
        const int l = add(tr, tr.left[u]);
        const int r = add(tr, tr.right[u]);
        if (!fits) return 0;
        SmallNode& nd = sm[static_cast<size_t>(me)];
        nd.thr = tr.threshold[u];
        nd.feat = static_cast<int16_t>(tr.feature[u]);
        nd.left = static_cast<int16_t>(l);
        nd.right = static_cast<int16_t>(r);
        return me;
    };
    P.dt.sroot[3] = -1;
    for (int t = 0; t < (b.has_col ? 4 : 3) && fits; ++t) P.dt.sroot[t] = add(b.trees[t], 0);
    P.dt.nsmall = 0;
    P.dt.small = nullptr;
    if (fits && !sm.empty()) {
        SmallNode* ds = static_cast<SmallNode*>(P.trees_small.ensure(sizeof(SmallNode) * sm.size()));
        ADA_CUDA(cudaMemcpyAsync(ds, sm.data(), sizeof(SmallNode) * sm.size(), cudaMemcpyHostToDevice, ctx.stream));
        P.dt.small = ds;
        P.dt.nsmall = static_cast<int>(sm.size());
    }
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
// p = 1 }, a level being decide -> SWITCH(branch).  Only the chosen
// branch's kernels run; sizes live on the device.
void build_graph(Context& ctx, const Matrix& m, const Bundle* b, BfsPlan& P);

void build_plan(Context& ctx, const Matrix& m, const Bundle* b, BfsPlan& P) {
    const int64_t n = m.rows;
    P.stream = ctx.stream;
    P.bundle_id = b ? b->id : 0;
    P.state.ensure(sizeof(BfsState));
#ifdef ADA_BFS_TRACE
    P.dlog = static_cast<LogEntry*>(P.log.ensure(sizeof(LogEntry) * kMaxLog));
#else
    ADA_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&P.hlog), sizeof(LogEntry) * kMaxLog, cudaHostAllocMapped));
    ADA_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&P.dlog), P.hlog, 0));
#endif
    for (auto& f : P.f) f.ensure(sizeof(int32_t) * static_cast<size_t>(n));
    P.eff.ensure(sizeof(int64_t) * static_cast<size_t>(n + 1));
    P.lv.ensure(sizeof(int32_t) * static_cast<size_t>(n));
    P.pcnt.ensure(sizeof(unsigned long long) * 2 * kSpread);
    P.bigc.ensure(sizeof(unsigned long long));
    P.bigl.ensure(sizeof(uint2) * static_cast<size_t>(std::min<int64_t>(n, m.nnz / (kBigDeg + 1) + 1)));
    ADA_CUDA(cudaMemsetAsync(P.pcnt.p, 0, sizeof(unsigned long long) * 2 * kSpread, ctx.stream));

    double* mf = static_cast<double*>(P.mfeat.ensure(sizeof(double) * 9));
    ADA_CUDA(cudaMemcpyAsync(mf, m.feat, sizeof(double) * 9, cudaMemcpyHostToDevice, ctx.stream));
    if (b) upload_trees(ctx, *b, m.feat, P);
#ifdef ADA_BFS_TRACE
    {
        LogEntry* lp = P.dlog;
        ADA_CUDA(cudaMemcpyToSymbolAsync(g_bfs_log, &lp, sizeof(lp), 0, cudaMemcpyHostToDevice, ctx.stream));
    }
#endif
    ctx.sync();
    {  // the persistent kernel when the device can co-schedule it (ADASPMV_BFS_PERSIST=0: the graph)
        const char* env = std::getenv("ADASPMV_BFS_PERSIST");
        int coop = 0;
        ADA_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, ctx.device));
        const int G = std::max(1, default_lanes_per_row(m.feat[5]) / 8);
        const void* fn = G == 1   ? reinterpret_cast<const void*>(&bfs_persist_kernel<1>)
                         : G == 2 ? reinterpret_cast<const void*>(&bfs_persist_kernel<2>)
                         : G == 4 ? reinterpret_cast<const void*>(&bfs_persist_kernel<4>)
                                  : reinterpret_cast<const void*>(&bfs_persist_kernel<8>);
        int nb = 0;
        ADA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, 256, 0));
        if (coop && nb > 0 && !(env && std::atoi(env) == 0)) {
            P.persist_G = G == 1 || G == 2 || G == 4 ? G : 8;
            P.persist_grid = static_cast<unsigned>(nb * ctx.sm_count);
            if (env && std::atoi(env) == 2) P.persist_grid *= 4;  // test hook: a grid that cannot be co-scheduled
            P.slots.ensure(sizeof(PSlot) * 3);
            P.bar.ensure(sizeof(unsigned) * kBarStride * (1 + kBarGroups));
            ADA_CUDA(cudaMemsetAsync(P.bar.p, 0, sizeof(unsigned) * kBarStride * (1 + kBarGroups), ctx.stream));
            ctx.sync();
            return;
        }
    }
    build_graph(ctx, m, b, P);
}

// The CUDA-graph form of the traversal (see the header).
void build_graph(Context& ctx, const Matrix& m, const Bundle* b, BfsPlan& P) {
    const int64_t n = m.rows;
    double* mf = P.mfeat.as<double>();
    BfsState* st = P.state.as<BfsState>();
    LogEntry* lg = P.dlog;
    int32_t* lv = P.lv.as<int32_t>();
    const int64_t* co = m.col_off.as<int64_t>();
    const unsigned push_grid = static_cast<unsigned>(ctx.sm_count) * 8;
    const int G = std::max(1, default_lanes_per_row(m.feat[5]) / 8);
    // grid-stride kernels: exactly the resident blocks (a second wave of a
    // grid-stride grid would start late and finish its full share late)
    auto resident = [&](const void* fn) {
        int nb = 0;
        ADA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, 256, 0));
        return static_cast<unsigned>(std::max(1, nb) * ctx.sm_count);
    };
    const unsigned pull4_grid = std::min<unsigned>(
        resident(reinterpret_cast<const void*>(&bfs_pull_mark4_kernel)),
        static_cast<unsigned>(std::max<int64_t>((n + 1023) / 1024, 1)));
    const unsigned scan_grid = resident(reinterpret_cast<const void*>(&bfs_scan_push_kernel<false>));
    const unsigned big_grid = resident(reinterpret_cast<const void*>(&bfs_big_push_kernel));
    const unsigned pull_grid = static_cast<unsigned>(
        std::max<int64_t>(std::min<int64_t>((n * G + 255) / 256, static_cast<int64_t>(ctx.sm_count) * 8), 1));
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
                                               P.pcnt.as<unsigned long long>(), P.bigc.as<unsigned long long>(),
                                               hbranch[p], hw);
            auto push = [&, p](cudaStream_t cs) {
                bfs_push_kernel<<<push_grid, 256, 0, cs>>>(st, p, P.f[p].as<int32_t>(), P.eff.as<int64_t>(), co,
                                                           m.row_idx.as<int32_t>(), lv, P.f[p ^ 1].as<int32_t>());
            };
            auto pull = [&, p](cudaStream_t cs) {  // marks only: a push after it reads the marks
                unsigned long long* pc = P.pcnt.as<unsigned long long>();
                switch (G) {
                    case 1:
                        bfs_pull_mark4_kernel<<<pull4_grid, 256, 0, cs>>>(st, m.rows, m.row_off.as<int64_t>(),
                                                                          m.col_idx.as<int32_t>(),
                                                                          m.col_off.as<int64_t>(), lv, pc);
                        break;
                    case 2: launch_pull_mark<2>(cs, pull_grid, st, m, lv, pc); break;
                    case 4: launch_pull_mark<4>(cs, pull_grid, st, m, lv, pc); break;
                    default: launch_pull_mark<8>(cs, pull_grid, st, m, lv, pc); break;
                }
            };
            auto scan_push = [&, p](cudaStream_t cs, bool list) {  // one pass + the big vertices' tasks
                unsigned long long* bc = P.bigc.as<unsigned long long>();
                uint2* bl = P.bigl.as<uint2>();
                if (list)
                    bfs_scan_push_kernel<true><<<scan_grid, 256, 0, cs>>>(st, p, P.f[p].as<int32_t>(), n, co,
                                                                          m.row_idx.as<int32_t>(), lv,
                                                                          P.f[p ^ 1].as<int32_t>(), bc, bl);
                else
                    bfs_scan_push_kernel<false><<<scan_grid, 256, 0, cs>>>(st, p, nullptr, n, co,
                                                                           m.row_idx.as<int32_t>(), lv,
                                                                           P.f[p ^ 1].as<int32_t>(), bc, bl);
                bfs_big_push_kernel<<<big_grid, 256, 0, cs>>>(st, p, co, m.row_idx.as<int32_t>(), lv,
                                                               P.f[p ^ 1].as<int32_t>(), bc, bl);
            };
            std::vector<std::function<void(cudaStream_t)>> bodies(5);
            bodies[kBranchPush] = push;
            bodies[kBranchPull] = pull;
            bodies[kBranchMarkPush] = [&](cudaStream_t cs) { scan_push(cs, false); };
            bodies[kBranchListPush] = [&](cudaStream_t cs) { scan_push(cs, true); };
            bodies[kBranchTail] = [&, p](cudaStream_t cs) {
                bfs_tail_kernel<<<1, 1024, 0, cs>>>(st, lg, p, P.f[0].as<int32_t>(), P.f[1].as<int32_t>(), co,
                                                    m.row_idx.as<int32_t>(), lv, P.dt, b ? 1 : 0, mf, n, m.nnz,
                                                    m.vbytes());
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
    // the whole traversal: one persistent kernel (or init + one graph launch
    // + a copy), one synchronisation (the state comes back through the
    // mapped host scalars)
    if (P.persist_G > 0) {
        PSlot* slots = P.slots.as<PSlot>();
        unsigned* bar = P.bar.as<unsigned>();
        PArgs a{};
        a.st = st;
        a.log = P.dlog;
        a.lv = P.lv.as<int32_t>();
        a.ro = m.row_off.as<int64_t>();
        a.ci = m.col_idx.as<int32_t>();
        a.co = m.col_off.as<int64_t>();
        a.ri = m.row_idx.as<int32_t>();
        a.f[0] = P.f[0].as<int32_t>();
        a.f[1] = P.f[1].as<int32_t>();
        a.slots = slots;
        a.bar = bar;
        a.bigl = P.bigl.as<uint2>();
        a.trees = P.dt;
        a.use_trees = b ? 1 : 0;
        a.mfeat = P.mfeat.as<double>();
        a.n = n;
        a.nnz = m.nnz;
        a.vbytes = m.vbytes();
        a.source = source;
        a.host_state = ctx.h_scalars_dev;
        void* args[] = {&a};
        const void* fn = P.persist_G == 1   ? reinterpret_cast<const void*>(&bfs_persist_kernel<1>)
                         : P.persist_G == 2 ? reinterpret_cast<const void*>(&bfs_persist_kernel<2>)
                         : P.persist_G == 4 ? reinterpret_cast<const void*>(&bfs_persist_kernel<4>)
                                            : reinterpret_cast<const void*>(&bfs_persist_kernel<8>);
        reinterpret_cast<BfsState*>(ctx.h_scalars)->done = 0;
        const cudaError_t le = cudaLaunchCooperativeKernel(fn, dim3(P.persist_grid), dim3(256), args, 0, ctx.stream);
        if (le == cudaErrorCooperativeLaunchTooLarge || le == cudaErrorNotSupported) {
            // the grid cannot be co-scheduled here (e.g. SMs held by MPS
            // clients): this plan falls back to the graph form for good
            (void)cudaGetLastError();
            P.persist_G = 0;
            build_graph(ctx, m, b, P);
        } else {
            ADA_CUDA(le);
            ++ctx.launches;
        }
    }
    if (P.persist_G == 0) {
        const unsigned ig =
            static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, static_cast<int64_t>(ctx.sm_count) * 16));
        bfs_init_kernel<<<ig, 256, 0, ctx.stream>>>(st, P.lv.as<int32_t>(), n, source, P.f[0].as<int32_t>(),
                                                    m.col_off.as<int64_t>(), P.eff.as<int64_t>());
        ADA_LAUNCHED(ctx);
        ADA_CUDA(cudaGraphLaunch(P.exec, ctx.stream));
        ++ctx.launches;
        copy_scalars_kernel_launch(ctx, reinterpret_cast<const int64_t*>(st), ctx.h_scalars_dev,
                                   static_cast<int>(sizeof(BfsState) / sizeof(int64_t)));
    }
    ctx.sync();
    if (!reinterpret_cast<const BfsState*>(ctx.h_scalars)->done)
        throw Error(ADASPMV_ERR_INTERNAL, "bfs: device level loop ended without an empty frontier");
    const BfsState* hs = reinterpret_cast<const BfsState*>(ctx.h_scalars);
    const int nlog = hs->nlog;
    *n_levels = nlog;
    if (reports && max_reports > 0) {
        const int nr = static_cast<int>(std::min<int64_t>(std::min<int64_t>(nlog, max_reports), kMaxLog - 1));
        std::vector<LogEntry> h(static_cast<size_t>(nr + 1));
        if (P.hlog) {
            std::memcpy(h.data(), P.hlog, sizeof(LogEntry) * h.size());
        } else {
            ADA_CUDA(cudaMemcpyAsync(h.data(), P.dlog, sizeof(LogEntry) * h.size(), cudaMemcpyDeviceToHost,
                                     ctx.stream));
            ctx.sync();
        }
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
#ifdef ADA_BFS_TRACE
            const LogEntry& le = h[static_cast<size_t>(i)];
            if (P.persist_G > 0)
                std::fprintf(stderr, "bfs trace level %d: block 0 body %.1f us, first barrier %.1f us\n", i,
                             (le.tk0 - t0) * 1e-3, (le.tk1 - le.tk0) * 1e-3);
            else
                std::fprintf(stderr, "bfs trace level %d: kernels %.1f us (start +%.1f us after the decision)\n", i,
                             le.tk1 > le.tk0 ? (le.tk1 - le.tk0) * 1e-3 : 0.0,
                             le.tk0 != ~0ull && le.tk0 > t0 ? (le.tk0 - t0) * 1e-3 : 0.0);
#endif
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

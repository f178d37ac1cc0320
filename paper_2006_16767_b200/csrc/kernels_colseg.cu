// kernels_colseg.cu -- row-segmented accumulation for the atomic column
// kernels (K6 col_lb_atomic, and K4 when asked): the reference's private
// accumulators (KernelConfig::atomic_private_accumulators, kernels.hpp:152-162,
// :452-478) generalised to a y that does not fit one CTA's shared memory.
//
// The row space is cut into segments of R rows (R * sizeof(V) <= 112 KiB).
// Heavy columns -- at least one entry per segment on average -- carry a
// table, built once per matrix, of where each segment starts inside the
// column (absolute CSC positions, [nseg + 1][nheavy] int64).  A multiply
// splits the support of x into its heavy and light columns; one CTA per
// segment accumulates the slices of every heavy support column into a
// shared-memory y segment (load-balanced over the flattened slices, 256
// entries per warp step, the next step's loads in flight during the updates) and stores the segment with plain coalesced stores
// -- every row of y is written exactly once, so no identity fill and no
// global atomics; the light columns (few entries each) follow with the
// ordinary atomic write-back (combine_batch).  Sums follow the atomic
// kernels' contract: correct up to summation order (kernels.hpp:436-451).
//
// Opt-in (ADASPMV_COLSEG=1): on C4 it measured 0.75-1.0x the L2-atomic K6
// (profiles/r02_colseg_experiment.txt) -- the slices of a segment are short
// (~10 entries), so the entry stream is latency-bound at 32 warps per SM.
#include <algorithm>
#include <cstdlib>

#include "device.cuh"
#include "internal.hpp"
#include "kernels.hpp"

namespace ada {

namespace {

constexpr int kSegNT = 1024;
constexpr int kSegBatch = 4096;       // heavy support columns staged per pass
constexpr size_t kSegYBytes = 112 * 1024;
constexpr size_t kSegTableBudget = size_t(1) << 30;  // table bytes cap (raises the heavy threshold)

__global__ void cs_classify_kernel(int64_t cols, const int64_t* __restrict__ co, int64_t lmin,
                                   int32_t* __restrict__ hid, int32_t* __restrict__ hcols,
                                   unsigned long long* __restrict__ cnt) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; c < cols; c += stride) {
        const int64_t len = co[c + 1] - co[c];
        int32_t id = -1;
        if (len >= lmin) {
            id = static_cast<int32_t>(atomicAdd(cnt, 1ull));
            atomicAdd(cnt + 1, static_cast<unsigned long long>(len));
            hcols[id] = static_cast<int32_t>(c);
        }
        hid[c] = id;
    }
}

// tab[b * nheavy + h] = first position of column hcols[h] with row >= b * R
__global__ void cs_table_kernel(int64_t nheavy, int64_t nseg, int64_t R, int64_t rows,
                                const int32_t* __restrict__ hcols, const int64_t* __restrict__ co,
                                const int32_t* __restrict__ ri, int64_t* __restrict__ tab) {
    const int64_t n = nheavy * (nseg + 1);
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n; t += stride) {
        const int64_t b = t / nheavy, h = t - b * nheavy;
        const int32_t c = hcols[h];
        int64_t lo = co[c], hi = co[c + 1];
        const int64_t key = min(b * R, rows);
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (ri[mid] < key) lo = mid + 1;
            else hi = mid;
        }
        tab[t] = lo;
    }
}

// split the support of x: heavy columns -> (heavy id, x), light -> (column, x)
template <class V>
__global__ void cs_split_kernel(int64_t nnz_x, const int32_t* __restrict__ xi, const V* __restrict__ xv,
                                const int32_t* __restrict__ hid, int32_t* __restrict__ hs, V* __restrict__ hx,
                                int32_t* __restrict__ ls, V* __restrict__ lx, unsigned long long* __restrict__ cnt) {
    const int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    const bool in = s < nnz_x;
    const int32_t col = in ? xi[s] : 0;
    const int32_t h = in ? hid[col] : -1;
    const bool heavy = in && h >= 0, light = in && h < 0;
    const int lane = threadIdx.x & 31;
    // warp-aggregated appends (one atomic per warp and list)
    const unsigned bh = __ballot_sync(kFull, heavy), bl = __ballot_sync(kFull, light);
    unsigned long long base_h = 0, base_l = 0;
    if (lane == 0) {
        if (bh) base_h = atomicAdd(cnt, static_cast<unsigned long long>(__popc(bh)));
        if (bl) base_l = atomicAdd(cnt + 1, static_cast<unsigned long long>(__popc(bl)));
    }
    base_h = __shfl_sync(kFull, base_h, 0);
    base_l = __shfl_sync(kFull, base_l, 0);
    const unsigned below = (1u << lane) - 1u;
    if (heavy) {
        const unsigned long long p = base_h + __popc(bh & below);
        hs[p] = h;
        hx[p] = xv[s];
    } else if (light) {
        const unsigned long long p = base_l + __popc(bl & below);
        ls[p] = col;
        lx[p] = xv[s];
    }
}

// One CTA per row segment: the heavy support columns' slices into a
// shared-memory y segment, then one plain store per row.
template <class V, int SR>
__global__ void __launch_bounds__(kSegNT, 1) cs_segment_kernel(
    int64_t rows, int64_t R, int64_t nheavy, const unsigned long long* __restrict__ cnt,
    const int32_t* __restrict__ hs, const V* __restrict__ hx, const int64_t* __restrict__ tab,
    const int32_t* __restrict__ ri, const V* __restrict__ cv, const uint2* __restrict__ cp, V* __restrict__ y,
    unsigned long long* __restrict__ ctr) {
    using S = Semiring<SR, V>;
    extern __shared__ __align__(16) unsigned char cs_smem[];
    V* ys = reinterpret_cast<V*>(cs_smem);
    int64_t* base = reinterpret_cast<int64_t*>(cs_smem + ((R * sizeof(V) + 15) & ~size_t(15)));
    V* xs = reinterpret_cast<V*>(base + kSegBatch);
    int32_t* pre = reinterpret_cast<int32_t*>(xs + kSegBatch);  // kSegBatch + 1 (+ scan scratch)
    unsigned long long* scan_tmp =                              // kSegNT / 32 + 1
        reinterpret_cast<unsigned long long*>(cs_smem + ((R * sizeof(V) + 15) & ~size_t(15)) +
                                              kSegBatch * (8 + sizeof(V)) + ((kSegBatch + 1) * 4 + 7) / 8 * 8);

    const int64_t seg = blockIdx.x;
    const int64_t r0 = seg * R;
    const int nr = static_cast<int>(min(R, rows - r0));
    for (int i = threadIdx.x; i < nr; i += kSegNT) ys[i] = S::zero();
    const int64_t nh = static_cast<int64_t>(*cnt);
    const int64_t* __restrict__ t0 = tab + seg * nheavy;
    const int64_t* __restrict__ t1 = t0 + nheavy;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned long long used = 0;
    constexpr int PT = kSegBatch / kSegNT;  // staged slices per thread
    for (int64_t bs = 0; bs < nh; bs += kSegBatch) {
        const int nbat = static_cast<int>(min(static_cast<int64_t>(kSegBatch), nh - bs));
        // stage this batch: slice start, x value and length of each heavy
        // support column; empty slices are dropped so that every slice
        // boundary is a distinct flattened position (the lane arithmetic below)
        int64_t b[PT];
        int32_t len[PT];
        V xq[PT];
        unsigned long long packed = 0;  // (nonempty count << 32) | entries
#pragma unroll
        for (int u = 0; u < PT; ++u) {
            const int i = PT * threadIdx.x + u;
            len[u] = 0;
            b[u] = 0;
            if (i < nbat) {
                const int32_t h = __ldg(hs + bs + i);
                b[u] = __ldg(t0 + h);
                len[u] = static_cast<int32_t>(__ldg(t1 + h) - b[u]);
                xq[u] = __ldg(hx + bs + i);
            }
            packed += (static_cast<unsigned long long>(len[u] > 0) << 32) | static_cast<unsigned>(len[u]);
        }
        unsigned long long ptotal;
        unsigned long long ex = block_exclusive_sum<kSegNT>(packed, scan_tmp, &ptotal);
#pragma unroll
        for (int u = 0; u < PT; ++u) {
            if (len[u] > 0) {
                const int o = static_cast<int>(ex >> 32);
                base[o] = b[u];
                xs[o] = xq[u];
                pre[o] = static_cast<int32_t>(ex & 0xffffffffull);
                ex += (1ull << 32) | static_cast<unsigned>(len[u]);
            }
        }
        const int nb = static_cast<int>(ptotal >> 32);
        const int32_t total = static_cast<int32_t>(ptotal & 0xffffffffull);
        if (threadIdx.x == 0) pre[nb] = total;
        __syncthreads();
        used += static_cast<unsigned long long>(total);
        // flattened entries per warp step (8 per lane; 4 for fp64), software
        // pipelined: the next step's loads are in flight during this step's
        // shared-memory updates
        constexpr int U = sizeof(V) == 4 ? 8 : 4;
        constexpr int kSegStep = 32 * U;
        constexpr int32_t kStride = (kSegNT / 32) * kSegStep;
        struct Step {
            uint32_t rr[U];  // row (absolute), or ~0u: no entry
            V a[U], xv[U];
        };
        auto fetch = [&](int32_t q0, Step& st) {
            // sb = slice holding q0 - 1 (largest s with pre[s] <= q0 - 1; -1 at q0 = 0)
            int sb = -1;
            if (q0 > 0) {
                int lo = 0, hi = nb;
                while (hi - lo > 1) {
                    const int step = (hi - lo + 31) / 32;
                    const int probe = lo + lane * step;
                    const unsigned bal = __ballot_sync(kFull, probe < hi && pre[probe] <= q0 - 1);
                    lo += (31 - __clz(bal)) * step;
                    hi = min(lo + step, hi);
                }
                sb = lo;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                // lane j reads boundary sb + 1 + j; a boundary at row offset t
                // moves lanes t..31 one slice on (boundaries are distinct)
                const int32_t row0 = q0 + u * 32;
                const int jb = sb + 1 + lane;
                const int32_t t = jb <= nb ? pre[jb] - row0 : 32;
                const unsigned bit = t < 32 ? (1u << t) : 0u;
                const unsigned B = __reduce_or_sync(kFull, bit);
                const int sl = sb + __popc(B & (0xffffffffu >> (31 - lane)));
                sb += __popc(B);
                const int32_t q = row0 + lane;
                st.rr[u] = ~0u;
                st.a[u] = V(1);
                st.xv[u] = S::zero();
                if (q < total) {
                    const int64_t k = base[sl] + (q - pre[sl]);
                    st.xv[u] = xs[sl];
                    if (sizeof(V) == 4 && cp) {
                        const uint2 pr = __ldg(cp + k);
                        st.rr[u] = pr.x;
                        if (S::kUsesValues) st.a[u] = static_cast<V>(__uint_as_float(pr.y));
                    } else {
                        st.rr[u] = static_cast<uint32_t>(__ldg(ri + k));
                        if (S::kUsesValues) st.a[u] = __ldg(cv + k);
                    }
                }
            }
        };
        auto update = [&](const Step& st) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (st.rr[u] == ~0u) continue;
                V* slot = ys + (st.rr[u] - static_cast<uint32_t>(r0));
                if (SR == SR_PLUS_TIMES) {
                    const V prod = st.a[u] * st.xv[u];
                    if (prod != V(0)) atomicAdd(slot, prod);  // shared CAS loop: keeps subnormals
                } else if (SR == SR_OR_AND) {
                    if (st.xv[u] != V(0)) *reinterpret_cast<volatile V*>(slot) = V(1);
                } else {
                    const V v = st.a[u] + st.xv[u];
                    if (v < *slot) AtomicCombine<SR_MIN_PLUS>::apply(slot, v);
                }
            }
        };
        int32_t q0 = warp * kSegStep;
        if (q0 < total) {
            Step cur, nxt;
            fetch(q0, cur);
            for (; q0 < total; q0 += kStride) {
                if (q0 + kStride < total) fetch(q0 + kStride, nxt);
                update(cur);
                cur = nxt;
            }
        }
        __syncthreads();  // the batch arrays are rewritten next pass
    }
    if (ctr && threadIdx.x == 0) count_add(ctr, 0, used);
    __syncthreads();
    for (int i = threadIdx.x; i < nr; i += kSegNT) y[r0 + i] = ys[i];
}

// light columns: a warp per column, ordinary atomic write-back
template <class V, int SR>
__global__ void __launch_bounds__(256) cs_light_kernel(
    const unsigned long long* __restrict__ cnt, const int32_t* __restrict__ ls, const V* __restrict__ lx,
    const int64_t* __restrict__ co, const int32_t* __restrict__ ri, const V* __restrict__ cv,
    const uint2* __restrict__ cp, V* __restrict__ y, unsigned long long* __restrict__ ctr, float amin) {
    using S = Semiring<SR, V>;
    const int64_t nl = static_cast<int64_t>(cnt[1]);
    const int lane = threadIdx.x & 31;
    const int64_t wstride = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    unsigned long long used = 0;
    for (int64_t s = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; s < nl; s += wstride) {
        const int32_t col = __ldg(ls + s);
        const V xval = __ldg(lx + s);
        const bool safe = addends_normal<SR>(xval, amin);
        const int64_t b = __ldg(co + col), e = __ldg(co + col + 1);
        used += static_cast<unsigned long long>(e - b);
        for (int64_t k0 = b + lane; k0 < e; k0 += 64) {
            int r[2];
            V pv[2];
            bool ok[2];
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int64_t k = k0 + 32 * j;
                ok[j] = k < e;
                r[j] = 0;
                pv[j] = S::zero();
                if (ok[j]) {
                    V a;
                    if (sizeof(V) == 4 && cp) {
                        const uint2 pr = __ldg(cp + k);
                        r[j] = static_cast<int>(pr.x);
                        a = S::kUsesValues ? static_cast<V>(__uint_as_float(pr.y)) : V(1);
                    } else {
                        r[j] = __ldg(ri + k);
                        a = S::kUsesValues ? __ldg(cv + k) : V(1);
                    }
                    pv[j] = S::mul(a, xval);
                }
            }
            combine_batch<SR>(y, r, pv, ok, safe);
        }
    }
    if (ctr && lane == 0 && used) count_add(ctr, 0, used);
}

size_t segment_smem(int64_t R, int vbytes) {
    return ((static_cast<size_t>(R) * vbytes + 15) & ~size_t(15)) + kSegBatch * (8 + vbytes) +
           ((kSegBatch + 1) * 4 + 7) / 8 * 8 + (kSegNT / 32 + 1) * 8;
}

// builds (once per matrix and dtype) the heavy-column segment table
void ensure_colsegs(Context& ctx, const Matrix& m) {
    ColSegs& cs = *m.csegs;
    if (cs.built) return;
    const int vb = m.vbytes();
    const int64_t rmax = static_cast<int64_t>(kSegYBytes) / vb;
    int64_t nseg = (m.rows + rmax - 1) / rmax;
    if (nseg > ctx.sm_count) nseg = (nseg + ctx.sm_count - 1) / ctx.sm_count * ctx.sm_count;  // whole waves
    nseg = std::max<int64_t>(nseg, 1);
    int64_t R = (m.rows + nseg - 1) / nseg;
    if (const char* e = std::getenv("ADASPMV_COLSEG_ROWS")) {  // test hook: small segments
        const int64_t r = std::atoll(e);
        if (r > 0 && r <= rmax) {
            R = r;
            nseg = (m.rows + R - 1) / R;
        }
    }
    int32_t* hid = static_cast<int32_t*>(cs.hid.ensure(sizeof(int32_t) * std::max<int64_t>(m.cols, 1)));
    int32_t* hcols = static_cast<int32_t*>(cs.hcols.ensure(sizeof(int32_t) * std::max<int64_t>(m.cols, 1)));
    unsigned long long* d_cnt = static_cast<unsigned long long*>(cs.cnt.ensure(sizeof(unsigned long long) * 2));
    int64_t lmin = std::max<int64_t>(nseg, 2);
    unsigned long long nheavy = 0, h_cnt[2] = {0, 0};
    for (;;) {
        ADA_CUDA(cudaMemsetAsync(d_cnt, 0, 2 * sizeof(unsigned long long), ctx.stream));
        const int blocks = static_cast<int>(std::min<int64_t>((m.cols + 255) / 256, 4 * 1024));
        if (m.cols > 0) {
            cs_classify_kernel<<<std::max(blocks, 1), 256, 0, ctx.stream>>>(m.cols, m.col_off.as<int64_t>(), lmin,
                                                                              hid, hcols, d_cnt);
            ADA_LAUNCHED(ctx);
        }
        ADA_CUDA(cudaMemcpyAsync(h_cnt, d_cnt, sizeof(h_cnt), cudaMemcpyDeviceToHost, ctx.stream));
        ADA_CUDA(cudaStreamSynchronize(ctx.stream));
        nheavy = h_cnt[0];
        if (static_cast<size_t>(nheavy) * (nseg + 1) * 8 <= kSegTableBudget) break;
        lmin *= 2;
    }
    int64_t* tab = static_cast<int64_t*>(cs.tab.ensure(sizeof(int64_t) * std::max<int64_t>(1, nheavy * (nseg + 1))));
    if (nheavy > 0) {
        const int64_t n = static_cast<int64_t>(nheavy) * (nseg + 1);
        cs_table_kernel<<<static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 16 * 1024)), 256, 0,
                          ctx.stream>>>(static_cast<int64_t>(nheavy), nseg, R, m.rows, hcols,
                                        m.col_off.as<int64_t>(), m.row_idx.as<int32_t>(), tab);
        ADA_LAUNCHED(ctx);
    }
    cs.R = R;
    cs.nseg = nseg;
    cs.lmin = lmin;
    cs.nheavy = static_cast<int64_t>(nheavy);
    cs.heavy_nnz = static_cast<int64_t>(h_cnt[1]);
    cs.built = true;
}

}  // namespace

int colseg_mode() {
    const char* e = std::getenv("ADASPMV_COLSEG");
    if (!e || !*e) return -1;
    return std::atoi(e) != 0 ? 1 : 0;
}

template <class V, int SR>
bool run_col_segmented(Context& ctx, const Matrix& m, Vector& x, V* y) {
    if (m.rows == 0 || x.nnz <= 0) return false;
    {
        std::lock_guard<std::mutex> g(m.lazy);
        ensure_colsegs(ctx, m);
    }
    const ColSegs& cs = *m.csegs;
    const size_t smem = segment_smem(cs.R, sizeof(V));
    const size_t z = static_cast<size_t>(x.nnz);
    int32_t* hs = static_cast<int32_t*>(ctx.scratch[0].ensure(sizeof(int32_t) * z));
    V* hx = static_cast<V*>(ctx.scratch[2].ensure(sizeof(V) * z));
    int32_t* ls = static_cast<int32_t*>(ctx.scratch[1].ensure(sizeof(int32_t) * z));
    V* lx = static_cast<V*>(ctx.scratch[3].ensure(sizeof(V) * z));
    unsigned long long* cnt = static_cast<unsigned long long*>(ctx.scratch[5].ensure(2 * sizeof(unsigned long long)));
    ADA_CUDA(cudaMemsetAsync(cnt, 0, 2 * sizeof(unsigned long long), ctx.stream));
    cs_split_kernel<V><<<static_cast<unsigned>((x.nnz + 255) / 256), 256, 0, ctx.stream>>>(
        x.nnz, x.sp_idx.as<int32_t>(), x.sp_val.as<V>(), cs.hid.as<int32_t>(), hs, hx, ls, lx, cnt);
    ADA_LAUNCHED(ctx);
    ADA_CUDA(cudaFuncSetAttribute(cs_segment_kernel<V, SR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    const uint2* cp = sizeof(V) == 4 ? m.cpairs.as<uint2>() : nullptr;
    cs_segment_kernel<V, SR><<<static_cast<unsigned>(cs.nseg), kSegNT, smem, ctx.stream>>>(
        m.rows, cs.R, cs.nheavy, cnt, hs, hx, cs.tab.as<int64_t>(), m.row_idx.as<int32_t>(), m.cvals.as<V>(), cp,
        y, ctx.ctr);
    ADA_LAUNCHED(ctx);
    const int64_t warps = std::min<int64_t>(x.nnz, static_cast<int64_t>(ctx.sm_count) * 64);
    cs_light_kernel<V, SR><<<static_cast<unsigned>((warps + 7) / 8), 256, 0, ctx.stream>>>(
        cnt, ls, lx, m.col_off.as<int64_t>(), m.row_idx.as<int32_t>(), m.cvals.as<V>(), cp, y, ctx.ctr, m.amin);
    ADA_LAUNCHED(ctx);
    return true;
}

#define ADA_INST(V, SR) template bool run_col_segmented<V, SR>(Context&, const Matrix&, Vector&, V*);
ADA_INST(float, SR_PLUS_TIMES)
ADA_INST(float, SR_OR_AND)
ADA_INST(float, SR_MIN_PLUS)
ADA_INST(double, SR_PLUS_TIMES)
ADA_INST(double, SR_OR_AND)
ADA_INST(double, SR_MIN_PLUS)
#undef ADA_INST

}  // namespace ada

// Microbenchmark (design exploration, not product): row bins in column order,
// cut into ROUNDS of NT*U entries in which every row appears at most once, so
// the shared-memory y update is a plain load-add-store (no ATOMS CAS loop),
// with one CTA barrier per round.  Compared with the same layout updated by
// float atomicAdd and with no update at all.  C2-like input: 2^22 x 2^22,
// 2^26 uniform draws, fp32.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o rounds_mb rounds_mb.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <deque>
#include <random>
#include <vector>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); exit(1); } } while (0)

// MODE 0 plain RMW + barrier per round, 1 atomicAdd (no barrier), 2 no update,
// 3 plain RMW, no barrier (racy), 4 plain + barrier, next round's stream
// loaded before this round's gathers (software pipeline)
template <int MODE, int NT, int U>
__global__ void __launch_bounds__(NT, 1) rounds_kernel(int R, int rbits, const int64_t* __restrict__ bin_round0,
                                                      const int32_t* __restrict__ rbase, const uint32_t* __restrict__ pk,
                                                      const float* __restrict__ v, const float* __restrict__ x,
                                                      float* __restrict__ y, int rows) {
    extern __shared__ float ys[];
    const int b = blockIdx.x;
    for (int i = threadIdx.x; i <= R; i += NT) ys[i] = 0.f;
    __syncthreads();
    const uint32_t rmask = (1u << rbits) - 1u;
    constexpr int C = NT * U;
    const int64_t q0 = bin_round0[b], q1 = bin_round0[b + 1];
    float sink = 0.f;
    uint32_t p[U];
    float a[U];
    auto load = [&](int64_t q) {
        const uint32_t* pq = pk + q * C + threadIdx.x;
        const float* vq = v + q * C + threadIdx.x;
#pragma unroll
        for (int j = 0; j < U; ++j) {
            p[j] = __ldcs(pq + j * NT);
            a[j] = __ldcs(vq + j * NT);
        }
    };
    if (MODE == 4 && q0 < q1) load(q0);
    for (int64_t q = q0; q < q1; ++q) {
        if (MODE != 4) load(q);
        const float* xb = x + rbase[q];
        uint32_t pp[U];
        float aa[U], xv[U];
#pragma unroll
        for (int j = 0; j < U; ++j) {
            pp[j] = p[j];
            aa[j] = a[j];
        }
        if (MODE == 4 && q + 1 < q1) load(q + 1);
#pragma unroll
        for (int j = 0; j < U; ++j) xv[j] = __ldg(xb + (pp[j] >> rbits));
#pragma unroll
        for (int j = 0; j < U; ++j) {
            const float pr = aa[j] * xv[j];
            float* s = ys + (pp[j] & rmask);
            if (MODE == 0 || MODE == 3 || MODE == 4) *s += pr;
            else if (MODE == 1) atomicAdd(s, pr);
            else sink += pr;
        }
        if (MODE == 0 || MODE == 4) __syncthreads();
    }
    if (MODE == 2) ys[R] = sink;
    __syncthreads();
    const int r0 = b * R;
    for (int i = threadIdx.x; i < R && r0 + i < rows; i += NT) y[r0 + i] = ys[i];
}

__global__ void csr_kernel(int rows, const int64_t* ro, const int* ci, const float* v, const float* x, float* y) {
    const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int row = (int)(gid / 4), lg = threadIdx.x & 3;
    float acc = 0;
    if (row < rows)
        for (int64_t k = ro[row] + lg; k < ro[row + 1]; k += 4) acc = fmaf(v[k], x[ci[k]], acc);
    acc += __shfl_xor_sync(0xffffffff, acc, 1, 4);
    acc += __shfl_xor_sync(0xffffffff, acc, 2, 4);
    if (row < rows && lg == 0) y[row] = acc;
}

int main(int argc, char** argv) {
    const int n = 1 << 22, rows = 1 << 22;
    const int64_t nnz_t = (int64_t)1 << 26;
    std::mt19937_64 g(1);
    std::uniform_int_distribution<int> uc(0, n - 1);
    std::uniform_real_distribution<float> uv(-1, 1);
    std::vector<int64_t> ro(rows + 1, 0);
    std::vector<int> rowof(nnz_t);
    for (int64_t k = 0; k < nnz_t; k++) { rowof[k] = uc(g); ro[rowof[k] + 1]++; }
    for (int i = 0; i < rows; i++) ro[i + 1] += ro[i];
    std::vector<int> ci(nnz_t);
    std::vector<float> vals(nnz_t);
    {
        std::vector<int64_t> pos(ro.begin(), ro.end() - 1);
        for (int64_t k = 0; k < nnz_t; k++) { int64_t p = pos[rowof[k]]++; ci[p] = uc(g); vals[p] = uv(g); }
    }
    std::vector<int> rk(nnz_t);
    for (int i = 0; i < rows; i++) for (int64_t k = ro[i]; k < ro[i + 1]; k++) rk[k] = i;
    std::vector<float> xh(n);
    for (auto& t : xh) t = uv(g);
    int64_t* d_ro; int* d_ci; float *d_v, *d_x, *d_y; char* d_flush;
    CK(cudaMalloc(&d_ro, 8 * (rows + 1))); CK(cudaMalloc(&d_ci, 4 * nnz_t)); CK(cudaMalloc(&d_v, 4 * nnz_t));
    CK(cudaMalloc(&d_x, 4 * n)); CK(cudaMalloc(&d_y, 4 * rows)); CK(cudaMalloc(&d_flush, 256 << 20));
    CK(cudaMemcpy(d_ro, ro.data(), 8 * (rows + 1), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_ci, ci.data(), 4 * nnz_t, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_v, vals.data(), 4 * nnz_t, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_x, xh.data(), 4 * n, cudaMemcpyHostToDevice));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto timeit = [&](auto f) {
        std::vector<float> ts;
        for (int it = 0; it < 9; it++) {
            CK(cudaMemset(d_flush, it, 256 << 20));
            cudaEventRecord(e0); f(); cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            if (it >= 2) ts.push_back(ms);
        }
        std::sort(ts.begin(), ts.end());
        return ts[ts.size() / 2] * 1000;
    };
    csr_kernel<<<(rows * 4 + 255) / 256, 256>>>(rows, d_ro, d_ci, d_v, d_x, d_y);
    CK(cudaDeviceSynchronize());
    std::vector<float> yref(rows);
    CK(cudaMemcpy(yref.data(), d_y, 4 * rows, cudaMemcpyDeviceToHost));
    const double B_spmv = 8.0 * (rows + 1) + 8.0 * nnz_t + 4.0 * n + 4.0 * rows;

    const int B = 148;
    const int R = (rows + B - 1) / B;
    int rbits = 0;
    while ((1 << rbits) < R + 1) rbits++;
    const int cw = 32 - rbits;
    for (int U : {4, 8}) {
        const int NT = 1024, C = NT * U;
        std::vector<uint32_t> pk;
        std::vector<float> bv;
        std::vector<int32_t> rbase;
        std::vector<int64_t> bin_round0(B + 1, 0);
        int64_t deferred = 0, pads = 0, early = 0;
        for (int b = 0; b < B; b++) {
            const int r0 = b * R, r1 = std::min(rows, r0 + R);
            std::vector<std::pair<int, int64_t>> es;
            for (int64_t k = ro[r0]; k < ro[r1]; k++) es.push_back({ci[k], k});
            std::sort(es.begin(), es.end());
            std::vector<int> stamp(R, -1);
            std::deque<std::pair<int, int64_t>> pend;
            size_t i = 0;
            int q = 0;
            while (i < es.size() || !pend.empty()) {
                std::vector<std::pair<int, int64_t>> cur;
                int lo = INT32_MAX;
                auto fits = [&](int col) { return std::max(lo, col) - std::min(lo == INT32_MAX ? col : lo, col) < (1 << cw) - 1; };
                std::deque<std::pair<int, int64_t>> still;
                while (!pend.empty()) {
                    auto e = pend.front(); pend.pop_front();
                    const int rl = rk[e.second] - r0;
                    if ((int)cur.size() < C && stamp[rl] != q) { stamp[rl] = q; cur.push_back(e); lo = std::min(lo, e.first); }
                    else still.push_back(e);
                }
                pend.swap(still);
                while ((int)cur.size() < C && i < es.size()) {
                    auto e = es[i];
                    if (lo != INT32_MAX && e.first - lo >= (1 << cw) - 1) { early++; break; }
                    const int rl = rk[e.second] - r0;
                    if (stamp[rl] == q) { pend.push_back(e); deferred++; }
                    else { stamp[rl] = q; cur.push_back(e); lo = std::min(lo, e.first); }
                    i++;
                }
                std::sort(cur.begin(), cur.end());
                const int base = cur.empty() ? 0 : cur.front().first;
                rbase.push_back(base);
                // entry e of the round at position j*NT + t: natural order
                for (int t = 0; t < C; t++) {
                    if (t < (int)cur.size()) {
                        const int col = cur[t].first; const int64_t k = cur[t].second;
                        pk.push_back(((uint32_t)(col - base) << rbits) | (uint32_t)(rk[k] - r0));
                        bv.push_back(vals[k]);
                    } else { pk.push_back((uint32_t)R); bv.push_back(0.f); pads++; }
                }
                q++;
            }
            bin_round0[b + 1] = bin_round0[b] + q;
        }
        const int64_t ne = pk.size();
        printf("U=%d rounds=%lld entries=%lld (pad %.2f%%, deferred %.2f%%, early cuts %lld)\n", U,
               (long long)bin_round0[B], (long long)ne, 100.0 * pads / ne, 100.0 * deferred / nnz_t, (long long)early);
        int64_t* d_br; int32_t* d_rb; uint32_t* d_pk; float* d_bv;
        CK(cudaMalloc(&d_br, 8 * (B + 1))); CK(cudaMalloc(&d_rb, 4 * rbase.size()));
        CK(cudaMalloc(&d_pk, 4 * ne)); CK(cudaMalloc(&d_bv, 4 * ne));
        CK(cudaMemcpy(d_br, bin_round0.data(), 8 * (B + 1), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(d_rb, rbase.data(), 4 * rbase.size(), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(d_pk, pk.data(), 4 * ne, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(d_bv, bv.data(), 4 * ne, cudaMemcpyHostToDevice));
        const size_t sm = 4 * (size_t)(R + 1);
        auto run = [&](auto kern, const char* name) {
            CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            const float us = timeit([&] { kern<<<B, NT, sm>>>(R, rbits, d_br, d_rb, d_pk, d_bv, d_x, d_y, rows); });
            CK(cudaGetLastError());
            std::vector<float> yy(rows);
            CK(cudaMemcpy(yy.data(), d_y, 4 * rows, cudaMemcpyDeviceToHost));
            double md = 0;
            for (int r = 0; r < rows; r++) md = std::max(md, (double)fabsf(yy[r] - yref[r]));
            printf("  %-28s %7.1f us  %5.1f%% of 6554 GB/s  max|dy| %.2e\n", name, us, 100.0 * B_spmv / (us * 1e-6) / 6554e9, md);
        };
        if (U == 4) {
            run(rounds_kernel<0, 1024, 4>, "plain+barrier");
            run(rounds_kernel<1, 1024, 4>, "atomicAdd");
            run(rounds_kernel<2, 1024, 4>, "no update");
            run(rounds_kernel<3, 1024, 4>, "plain no barrier (racy)");
            run(rounds_kernel<4, 1024, 4>, "plain+barrier, prefetch");
        } else {
            run(rounds_kernel<0, 1024, 8>, "plain+barrier");
            run(rounds_kernel<1, 1024, 8>, "atomicAdd");
            run(rounds_kernel<2, 1024, 8>, "no update");
            run(rounds_kernel<3, 1024, 8>, "plain no barrier (racy)");
            run(rounds_kernel<4, 1024, 8>, "plain+barrier, prefetch");
        }
        cudaFree(d_br); cudaFree(d_rb); cudaFree(d_pk); cudaFree(d_bv);
    }
    return 0;
}

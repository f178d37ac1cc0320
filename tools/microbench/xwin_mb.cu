// Microbenchmark (design exploration, not product): cost of the binned K0
// inner loop when the x gather is served from shared memory (an x window
// staged per column panel) instead of L2, on the C2 shape (148 bins of 2^22/148
// rows, 2^26 uniform entries, fp32, entries of a bin in column order).
// Proxy layout: pk = (col & 0x1ffff) << 15 | row_local (the gathers keep the
// column-sorted locality of the real layout; the window index is ignored).
//   G  : x from global (L2) + shared float atomicAdd  (the production loop)
//   S  : x from a 16 KB shared window + shared atomicAdd
//   G0 : x from global, no update;  S0 : x from shared, no update
//   N  : stream only
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o xwin_mb xwin_mb.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); exit(1); } } while (0)

template <int MODE, int NT, int U>
__global__ void __launch_bounds__(NT, 1) xwin_kernel(int R, const int64_t* __restrict__ boff, const uint32_t* __restrict__ pk,
                                                    const float* __restrict__ v, const float* __restrict__ x,
                                                    float* __restrict__ y, int rows) {
    extern __shared__ float sm[];
    float* ys = sm;
    float* xs = sm + R + 1;
    const int b = blockIdx.x;
    for (int i = threadIdx.x; i <= R; i += NT) ys[i] = 0.f;
    for (int i = threadIdx.x; i < 4096; i += NT) xs[i] = x[i];
    __syncthreads();
    unsigned peer = 0;
    if (MODE == 5 || MODE == 6) {
        unsigned rank;
        asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(peer) : "r"((unsigned)__cvta_generic_to_shared(ys)), "r"(rank ^ 1u));
        asm volatile("barrier.cluster.arrive.release; barrier.cluster.wait.acquire;" ::: "memory");
    }
    const int64_t e0 = boff[b], e1 = boff[b + 1];
    const uint32_t n = (uint32_t)(e1 - e0);
    const uint32_t* pkt = pk + e0;
    const float* vt = v + e0;
    float sink = 0.f;
    for (uint32_t base = threadIdx.x; base < n; base += NT * U) {
        uint32_t p[U];
        float a[U], xv[U];
        bool ok[U];
#pragma unroll
        for (int j = 0; j < U; ++j) {
            const uint32_t e = base + j * NT;
            ok[j] = e < n;
            p[j] = ok[j] ? __ldcs(pkt + e) : 0u;
            a[j] = ok[j] ? __ldcs(vt + e) : 0.f;
        }
#pragma unroll
        for (int j = 0; j < U; ++j) {
            if (MODE == 0 || MODE == 2 || MODE == 5) xv[j] = ok[j] ? __ldg(x + (p[j] >> 15)) : 0.f;
            else if (MODE == 1 || MODE == 3 || MODE == 6) xv[j] = xs[(p[j] >> 15) & 4095];
            else xv[j] = 1.f;
        }
#pragma unroll
        for (int j = 0; j < U; ++j) {
            if (!ok[j]) continue;
            const float pr = a[j] * xv[j];
            if (MODE <= 1) atomicAdd(ys + (p[j] & 0x7fff), pr);
            else if (MODE == 5 || MODE == 6) {  // the peer CTA's segment (cluster of 2): native remote f32 red
                asm volatile("red.shared::cluster.add.f32 [%0], %1;" ::"r"(peer + 4u * (p[j] & 0x7fff)), "f"(pr) : "memory");
            } else sink += pr;
        }
    }
    if (MODE >= 2 && MODE <= 4) ys[R] = sink;
    if (MODE == 5 || MODE == 6) asm volatile("barrier.cluster.arrive.release; barrier.cluster.wait.acquire;" ::: "memory");
    __syncthreads();
    const int r0 = b * R;
    for (int i = threadIdx.x; i < R && r0 + i < rows; i += NT) y[r0 + i] = ys[i];
}

int main() {
    const int n = 1 << 22, rows = 1 << 22;
    const int64_t nnz_t = (int64_t)1 << 26;
    const int B = 148, R = (rows + B - 1) / B;
    std::mt19937_64 g(1);
    std::uniform_int_distribution<int> uc(0, n - 1);
    std::uniform_real_distribution<float> uv(-1, 1);
    // per bin: entries with random row in the bin and random column, column-sorted
    std::vector<int64_t> boff(B + 1, 0);
    std::vector<uint64_t> keys(nnz_t);
    for (int64_t k = 0; k < nnz_t; k++) {
        const int r = uc(g), c = uc(g);
        const int b = r / R;
        keys[k] = ((uint64_t)b << 48) | ((uint64_t)c << 16) | (uint64_t)(r - b * R);
    }
    std::sort(keys.begin(), keys.end());
    std::vector<uint32_t> pk(nnz_t);
    std::vector<float> vals(nnz_t);
    for (int64_t k = 0; k < nnz_t; k++) {
        const int b = (int)(keys[k] >> 48), c = (int)((keys[k] >> 16) & 0xffffffff), rl = (int)(keys[k] & 0xffff);
        boff[b + 1]++;
        pk[k] = ((uint32_t)(c & 0x1ffff) << 15) | (uint32_t)rl;
        vals[k] = uv(g);
    }
    for (int b = 0; b < B; b++) boff[b + 1] += boff[b];
    std::vector<float> xh(n);
    for (auto& t : xh) t = uv(g);
    int64_t* d_bo; uint32_t* d_pk; float *d_v, *d_x, *d_y; char* d_flush;
    CK(cudaMalloc(&d_bo, 8 * (B + 1))); CK(cudaMalloc(&d_pk, 4 * nnz_t)); CK(cudaMalloc(&d_v, 4 * nnz_t));
    CK(cudaMalloc(&d_x, 4 * n)); CK(cudaMalloc(&d_y, 4 * rows)); CK(cudaMalloc(&d_flush, 256 << 20));
    CK(cudaMemcpy(d_bo, boff.data(), 8 * (B + 1), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_pk, pk.data(), 4 * nnz_t, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_v, vals.data(), 4 * nnz_t, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_x, xh.data(), 4 * n, cudaMemcpyHostToDevice));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const double B_spmv = 8.0 * (rows + 1) + 8.0 * nnz_t + 4.0 * n + 4.0 * rows;
    auto run = [&](auto kern, int NT, const char* name, int extra_kib, int cl = 1) {
        const size_t sm = 4 * (size_t)(R + 1) + 4 * 4096 + (size_t)extra_kib * 1024;
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        std::vector<float> ts;
        for (int it = 0; it < 9; it++) {
            CK(cudaMemset(d_flush, it, 256 << 20));
            cudaEventRecord(e0);
            cudaLaunchConfig_t lc{};
            lc.gridDim = dim3(B); lc.blockDim = dim3(NT); lc.dynamicSmemBytes = sm;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = cl; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
            lc.attrs = at; lc.numAttrs = 1;
            CK(cudaLaunchKernelEx(&lc, kern, R, (const int64_t*)d_bo, (const uint32_t*)d_pk, (const float*)d_v, (const float*)d_x, d_y, rows));
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            if (it >= 2) ts.push_back(ms);
        }
        CK(cudaGetLastError());
        std::sort(ts.begin(), ts.end());
        const float us = ts[ts.size() / 2] * 1000;
        printf("  %-44s %7.1f us  %5.1f%% of 6554 GB/s\n", name, us, 100.0 * B_spmv / (us * 1e-6) / 6554e9);
    };
    run(xwin_kernel<0, 1024, 8>, 1024, "G  x global + atomic   (1024x8)", 0);
    run(xwin_kernel<1, 1024, 8>, 1024, "S  x smem + atomic     (1024x8)", 0);
    run(xwin_kernel<2, 1024, 8>, 1024, "G0 x global, no update (1024x8)", 0);
    run(xwin_kernel<3, 1024, 8>, 1024, "S0 x smem, no update   (1024x8)", 0);
    run(xwin_kernel<4, 1024, 8>, 1024, "N  stream only         (1024x8)", 0);
    run(xwin_kernel<1, 1024, 8>, 1024, "S  x smem + atomic, +64 KiB smem (1024x8)", 64);
    run(xwin_kernel<1, 1024, 8>, 1024, "S  x smem + atomic, +96 KiB smem (1024x8)", 96);
    run(xwin_kernel<4, 1024, 8>, 1024, "N  stream only, +96 KiB smem (1024x8)", 96);
    run(xwin_kernel<1, 1024, 4>, 1024, "S  x smem + atomic     (1024x4)", 0);
    run(xwin_kernel<1, 512, 16>, 512, "S  x smem + atomic     (512x16)", 0);
    run(xwin_kernel<5, 1024, 8>, 1024, "R  x global + peer red.shared::cluster (1024x8)", 0, 2);
    run(xwin_kernel<6, 1024, 8>, 1024, "RS x smem + peer red.shared::cluster (1024x8)", 0, 2);
    run(xwin_kernel<0, 1024, 8>, 1024, "G  x global + atomic, cluster 2 (1024x8)", 0, 2);
    return 0;
}

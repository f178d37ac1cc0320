// Microbenchmark (design exploration, not product): ceiling of random 4-B
// gathers from an L2-resident vector (16 MB fp32, the C2 x) on B200, the
// per-entry x gather of the binned K0.  Each warp instruction gathers 32
// lanes from WIN consecutive sorted random columns (WIN = 300 models a C2 bin
// of 28K rows: ~9 lines per instruction; WIN = 4M: fully random).
//   mode 0: __ldg (L1 allocate)  1: ld.global.nc.L1::no_allocate
// plus a streaming read of 604 MB alongside (the matrix) when STREAM = 1.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2gather_mb l2gather_mb.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <algorithm>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); exit(1); } } while (0)

__device__ __forceinline__ float ld_na(const float* p) { float r; asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(r) : "l"(p)); return r; }
__device__ __forceinline__ int4 ld_s4(const int4* p) { int4 r; asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p)); return r; }

template <int MODE, int U, bool STREAM>
__global__ void __launch_bounds__(1024, 1) gather_kernel(const uint32_t* __restrict__ idx, int64_t n_per_cta, const float* __restrict__ x, const int4* __restrict__ st, float* out) {
    extern __shared__ float dummy_smem[];
    if (n_per_cta < 0) dummy_smem[threadIdx.x] = 0.f;
    const uint32_t* id = idx + blockIdx.x * n_per_cta;
    const int4* sp = st + blockIdx.x * (n_per_cta / 2);
    float acc = 0.f; int sacc = 0;
    for (int64_t b = threadIdx.x; b < n_per_cta; b += 1024 * U) {
        uint32_t c[U]; float v[U];
#pragma unroll
        for (int j = 0; j < U; ++j) { int64_t e = b + j * 1024; c[j] = e < n_per_cta ? __ldg(id + e) : 0u; }
        if (STREAM) {
#pragma unroll
            for (int j = 0; j < U / 2; ++j) { int64_t e = (b - threadIdx.x) / 2 + j * 1024 + threadIdx.x; if (e < n_per_cta / 2) { int4 w = ld_s4(sp + e); sacc += w.x ^ w.y ^ w.z ^ w.w; } }
        }
#pragma unroll
        for (int j = 0; j < U; ++j) v[j] = MODE == 0 ? __ldg(x + c[j]) : ld_na(x + c[j]);
#pragma unroll
        for (int j = 0; j < U; ++j) acc += v[j];
    }
    if (acc == 123.f || sacc == 0x7fffffff) out[0] = acc + sacc;
}

int main() {
    const int ctas = 148; const int64_t n = int64_t(1) << 26; const int64_t per = n / ctas / 1024 * 1024;
    const int64_t ncols = 1 << 22;
    std::mt19937_64 rng(1);
    float *x, *out; uint32_t* idx; int4* st; char* flush;
    CK(cudaMalloc(&x, ncols * 4)); CK(cudaMalloc(&out, 4)); CK(cudaMalloc(&flush, 256 << 20));
    CK(cudaMemset(x, 0, ncols * 4));
    CK(cudaMalloc(&st, (int64_t)ctas * per / 2 * 16)); CK(cudaMemset(st, 1, (int64_t)ctas * per / 2 * 16));
    CK(cudaMalloc(&idx, ctas * per * 4));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int64_t win : {int64_t(300), int64_t(150), int64_t(75), int64_t(4194304)}) {
        // per CTA: per sorted columns; instruction = 32 consecutive entries spanning ~win columns
        std::vector<uint32_t> h(ctas * per);
        for (int b = 0; b < ctas; ++b) {
            std::vector<uint32_t> v(per);
            if (win >= ncols) { for (auto& c : v) c = rng() % ncols; }
            else { double step = double(win) / 32.0; for (int64_t i = 0; i < per; ++i) { double base = i * step; v[i] = uint32_t(std::min<double>(ncols - 1, base + (rng() % 1000) * step / 1000.0)) % ncols; } }
            // reorder so entries b + j*1024 + t ... keep sorted order (thread t handles e = t + k*1024)
            std::copy(v.begin(), v.end(), h.begin() + b * per);
        }
        CK(cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
        auto run = [&](auto kern, const char* name, int smem = 0) {
            CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448));
            float best = 1e9;
            for (int r = 0; r < 5; ++r) {
                CK(cudaMemset(flush, r, 256 << 20));
                cudaEventRecord(e0); kern<<<ctas, 1024, smem>>>(idx, per, x, st, out); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
                float ms; cudaEventElapsedTime(&ms, e0, e1); best = std::min(best, ms);
            }
            printf("win=%8lld %-28s smem %6d %8.1f us  gathers/ns %.1f\n", (long long)win, name, smem, best * 1e3, ctas * per / (best * 1e6));
        };
        for (int sm : {116000, 160000, 200000, 228000}) {
            run(gather_kernel<0, 8, false>, "ldg U8", sm);
            run(gather_kernel<1, 8, false>, "no_allocate U8", sm);
            run(gather_kernel<0, 4, false>, "ldg U4", sm);
        }
        run(gather_kernel<0, 8, false>, "ldg U8");
        run(gather_kernel<1, 8, false>, "no_allocate U8");
        run(gather_kernel<0, 16, false>, "ldg U16");
        run(gather_kernel<0, 8, true>, "ldg U8 + stream");
        run(gather_kernel<1, 8, true>, "no_allocate U8 + stream");
    }
    return 0;
}

// prims.cu -- non-template parts of prims.cuh.
#include "prims.cuh"

namespace ada {

__global__ void __launch_bounds__(1024) scan_spine_kernel(int64_t nt, int64_t* tile_sums,
                                                          int64_t* d_total) {
    __shared__ int64_t sm[1024 / 32 + 1];
    constexpr int kPer = 4;
    int64_t carry = 0;
    for (int64_t base = 0; base < nt; base += 1024 * kPer) {
        const int64_t b = base + threadIdx.x * kPer;
        int64_t v[kPer];
        int64_t s = 0;
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
            v[j] = b + j < nt ? tile_sums[b + j] : 0;
            s += v[j];
        }
        int64_t total;
        int64_t p = block_exclusive_sum<1024>(s, sm, &total) + carry;
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
            if (b + j < nt) tile_sums[b + j] = p;
            p += v[j];
        }
        carry += total;
    }
    if (threadIdx.x == 0 && d_total) *d_total = carry;
}

__global__ void __launch_bounds__(kRsThreads) radix_upsweep_kernel(const uint32_t* __restrict__ keys,
                                                                   int64_t n, int shift,
                                                                   int64_t ntiles,
                                                                   int64_t* __restrict__ counts) {
    __shared__ int hist[kRsRadix];
    hist[threadIdx.x] = 0;
    __syncthreads();
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kRsTile;
#pragma unroll 4
    for (int r = 0; r < kRsRounds; ++r) {
        const int64_t i = base + r * kRsThreads + threadIdx.x;
        if (i < n) atomicAdd(&hist[(keys[i] >> shift) & (kRsRadix - 1)], 1);
    }
    __syncthreads();
    counts[static_cast<int64_t>(threadIdx.x) * ntiles + blockIdx.x] = hist[threadIdx.x];
}

__global__ void scan_zero_kernel(int64_t* p) { *reinterpret_cast<volatile int64_t*>(p) = 0; }

__global__ void copy_scalars_kernel(const int64_t* __restrict__ src, volatile int64_t* dst, int n) {
    if (static_cast<int>(threadIdx.x) < n) dst[threadIdx.x] = src[threadIdx.x];
}

void copy_scalars_kernel_launch(Context& ctx, const int64_t* src, int64_t* dst, int n) {
    copy_scalars_kernel<<<1, 64, 0, ctx.stream>>>(src, dst, n);
    ADA_LAUNCHED(ctx);
}

}  // namespace ada

// device.cuh -- device-side building blocks shared by the sm_100a kernels:
// streaming loads, warp/block scans, value traits, semiring algebra.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace ada {

constexpr unsigned kFull = 0xffffffffu;

// ---- streaming / read-only loads -------------------------------------------
// Matrix arrays are read exactly once per multiply: stream them past L1
// (ld.global.nc.L1::no_allocate); x / offsets go through the default path.
__device__ __forceinline__ int4 ld_stream(const int4* p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ float4 ld_stream(const float4* p) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ double2 ld_stream(const double2* p) {
    double2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];"
                 : "=d"(r.x), "=d"(r.y)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ int ld_stream(const int* p) {
    int r;
    asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}
__device__ __forceinline__ float ld_stream(const float* p) {
    float r;
    asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(r) : "l"(p));
    return r;
}
__device__ __forceinline__ double ld_stream(const double* p) {
    double r;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(r) : "l"(p));
    return r;
}

// four consecutive values (16-B aligned) in one or two 128-bit loads
__device__ __forceinline__ void ld_stream4(const float* p, float (&a)[4]) {
    const float4 v = ld_stream(reinterpret_cast<const float4*>(p));
    a[0] = v.x;
    a[1] = v.y;
    a[2] = v.z;
    a[3] = v.w;
}
__device__ __forceinline__ void ld_stream4(const double* p, double (&a)[4]) {
    const double2 v0 = ld_stream(reinterpret_cast<const double2*>(p));
    const double2 v1 = ld_stream(reinterpret_cast<const double2*>(p) + 1);
    a[0] = v0.x;
    a[1] = v0.y;
    a[2] = v1.x;
    a[3] = v1.y;
}

// KernelCounters (kernels.hpp:106-111) on the device, when the context asks
// for them (adaspmv_ctx_set_counters): ctr[0] values_read = loads from the
// matrix value array (kernels.hpp:108; every kernel loads a value exactly
// when it forms a product -- the row SpMSpV kernels test the mask first,
// kernels.hpp:229-240; under OR_AND, which loads no values, the entries
// consumed), ctr[1] pairs_emitted on the sort write-back.  cas_retries stays
// 0: the atomic write-backs use hardware atomics, not a counted CAS loop.
__device__ __forceinline__ void count_add(unsigned long long* ctr, int slot, unsigned long long v) {
    if (ctr && v) atomicAdd(ctr + slot, v);
}

// ---- semirings ---------------------------------------------------------------
// PlusTimes: the reference algebra (kernels.hpp:236).  MinPlus: y_i =
// min_j (a_ij + x_j), identity +inf.  OrAnd: y_i = OR_j (a_ij != 0 && x_j != 0)
// encoded as 1.0 / 0.0 of the value type; pattern only (no value loads).
enum { SR_PLUS_TIMES = 0, SR_OR_AND = 1, SR_MIN_PLUS = 2 };

template <int SR, class V>
struct Semiring;

template <class V>
struct Semiring<SR_PLUS_TIMES, V> {
    static constexpr bool kUsesValues = true;
    __device__ static V zero() { return V(0); }
    __device__ static V mul(V a, V x) { return a * x; }
    __device__ static V add(V s, V t) { return s + t; }
    __device__ static V fma(V a, V x, V s) { return fma_(a, x, s); }
    __device__ static float fma_(float a, float x, float s) { return __fmaf_rn(a, x, s); }
    __device__ static double fma_(double a, double x, double s) { return __fma_rn(a, x, s); }
};

template <class V>
struct Semiring<SR_MIN_PLUS, V> {
    static constexpr bool kUsesValues = true;
    __device__ static V zero() { return V(INFINITY); }
    __device__ static V mul(V a, V x) { return a + x; }
    __device__ static V add(V s, V t) { return s < t ? s : t; }
    __device__ static V fma(V a, V x, V s) { return add(s, a + x); }
};

template <class V>
struct Semiring<SR_OR_AND, V> {
    static constexpr bool kUsesValues = false;
    __device__ static V zero() { return V(0); }
    __device__ static V mul(V, V x) { return x != V(0) ? V(1) : V(0); }
    __device__ static V add(V s, V t) { return (s != V(0) || t != V(0)) ? V(1) : V(0); }
    __device__ static V fma(V a, V x, V s) { return add(s, mul(a, x)); }
};

// ---- atomics for the semirings' write-back ----------------------------------
template <int SR>
struct AtomicCombine;

// IEEE (subnormal-keeping) float add by compare-and-swap.
__device__ __forceinline__ void atomic_add_f32_exact(float* p, float v) {
    unsigned* a = reinterpret_cast<unsigned*>(p);
    unsigned old = 0u, assumed;  // first guess +0: the first CAS returns the current value
    do {
        assumed = old;
        old = atomicCAS(a, assumed, __float_as_uint(__uint_as_float(assumed) + v));
    } while (old != assumed);
}

template <>
struct AtomicCombine<SR_PLUS_TIMES> {
    // The hardware float reduction (REDG.E.ADD.F32.FTZ) flushes subnormal
    // operands and results to zero; the reference's float sums keep them.
    // An addend below 2^-100 takes an IEEE compare-and-swap add instead
    // (FADD keeps subnormals), so a row whose terms are all tiny is summed
    // exactly like the reference; for a larger addend the flush of a
    // subnormal operand or result is <= 2^-126 absolute, far inside the fp32
    // tolerance of a row bound >= 2^-100.
    __device__ static void apply(float* p, float v) {
        const bool tiny = fabsf(v) < 0x1p-100f;  // NaN: not tiny
        if (!tiny) atomicAdd(p, v);               // predicated RED, no branch
        else if (v != 0.f) atomic_add_f32_exact(p, v);  // adding +-0 never changes a sum that starts at +0
    }
    __device__ static void apply(double* p, double v) { atomicAdd(p, v); }
    // the addend is known to be outside the subnormal range
    __device__ static void apply_fast(float* p, float v) { atomicAdd(p, v); }
    __device__ static void apply_fast(double* p, double v) { atomicAdd(p, v); }
};

template <>
struct AtomicCombine<SR_OR_AND> {
    __device__ static void apply(float* p, float v) {
        if (v != 0.f) *reinterpret_cast<volatile float*>(p) = 1.f;  // idempotent store
    }
    __device__ static void apply(double* p, double v) {
        if (v != 0.0) *reinterpret_cast<volatile double*>(p) = 1.0;
    }
    template <class V>
    __device__ static void apply_fast(V* p, V v) { apply(p, v); }
};
template <>
struct AtomicCombine<SR_MIN_PLUS> {
    // Order-preserving integer image of IEEE floats (handles negatives).
    __device__ static void apply(float* p, float v) {
        int iv = __float_as_int(v);
        if (iv >= 0) atomicMin(reinterpret_cast<int*>(p), iv);
        else atomicMax(reinterpret_cast<unsigned*>(p), static_cast<unsigned>(iv));
    }
    __device__ static void apply(double* p, double v) {
        long long iv = __double_as_longlong(v);
        if (iv >= 0) atomicMin(reinterpret_cast<long long*>(p), iv);
        else atomicMax(reinterpret_cast<unsigned long long*>(p), static_cast<unsigned long long>(iv));
    }
    template <class V>
    __device__ static void apply_fast(V* p, V v) { apply(p, v); }
};

// A batch of N write-backs y[r[j]] (+)= v[j] (ok[j]).  `safe`: the caller
// knows no addend can be below 2^-100 in magnitude (|x| * min|a| >= 2^-100,
// decided once per support column or warp tile, ahead of the products), so
// the hardware reductions issue exactly as plain atomicAdd; otherwise each
// addend is checked and the subnormal-range ones take the IEEE CAS add.  A
// per-entry branch on the product's magnitude in the common path would stall
// every write-back on its product (C4 K6: +15-20 %, measured).
template <int SR, class V, int N>
__device__ __forceinline__ void combine_batch(V* y, const int (&r)[N], const V (&v)[N], const bool (&ok)[N],
                                              bool safe) {
    if (SR != SR_PLUS_TIMES || sizeof(V) != 4 || safe) {
#pragma unroll
        for (int j = 0; j < N; ++j)
            if (ok[j]) AtomicCombine<SR>::apply_fast(y + r[j], v[j]);
    } else {
#pragma unroll
        for (int j = 0; j < N; ++j)
            if (ok[j]) AtomicCombine<SR>::apply(y + r[j], v[j]);
    }
}

// the per-column / per-tile test behind `safe` (fp32 plus-times only)
template <int SR, class V>
__device__ __forceinline__ bool addends_normal(V x, float amin) {
    if constexpr (SR != SR_PLUS_TIMES || sizeof(V) != 4) return true;
    else return fabsf(static_cast<float>(x)) * amin >= 0x1p-100f;  // NaN: not safe
}

// ---- warp / block scans ---------------------------------------------------------
template <class T>
__device__ __forceinline__ T warp_inclusive_sum(T v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        T t = __shfl_up_sync(kFull, v, d);
        if (lane >= d) v += t;
    }
    return v;
}

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(kFull, v, d);
    return v;
}

// Block-wide exclusive sum over NT threads (NT multiple of 32, <= 1024).
// `smem` must hold NT/32 + 1 elements.  Returns the exclusive prefix; *total
// gets the block total.  Contains __syncthreads().
template <int NT, class T>
__device__ __forceinline__ T block_exclusive_sum(T v, T* smem, T* total) {
    constexpr int NW = NT / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T inc = warp_inclusive_sum(v);
    if (lane == 31) smem[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        T w = lane < NW ? smem[lane] : T(0);
        T wi = warp_inclusive_sum(w);
        if (lane < NW) smem[lane] = wi - w;
        if (lane == NW - 1) smem[NW] = wi;
    }
    __syncthreads();
    T r = smem[warp] + inc - v;
    *total = smem[NW];
    __syncthreads();
    return r;
}

// Segmented scan element: flag = "reset here", value.  Inclusive combine:
// (f1,x1) (+) (f2,x2) = (f1|f2, f2 ? x2 : x1+x2).
template <class V>
struct SegPair {
    int f;
    V v;
};

template <class V, class Add>
__device__ __forceinline__ SegPair<V> warp_seg_inclusive(SegPair<V> p, Add add) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        int f = __shfl_up_sync(kFull, p.f, d);
        V v = __shfl_up_sync(kFull, p.v, d);
        if (lane >= d) {
            if (!p.f) p.v = add(v, p.v);
            p.f |= f;
        }
    }
    return p;
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned r;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}

// largest s in [lo, hi) with off[s] <= pos (segment_of, partition.hpp:30-33),
// given off[lo] <= pos.
__device__ __forceinline__ int64_t segment_search(const int64_t* __restrict__ off, int64_t lo,
                                                  int64_t hi, int64_t pos) {
    // invariant: off[lo] <= pos; answer in [lo, hi)
    while (hi - lo > 1) {
        int64_t mid = (lo + hi) >> 1;
        if (__ldg(off + mid) <= pos) lo = mid;
        else hi = mid;
    }
    return lo;
}

}  // namespace ada

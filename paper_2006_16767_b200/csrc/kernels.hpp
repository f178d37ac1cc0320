// kernels.hpp -- internal declarations shared by the kernel translation units.
#pragma once

#include <cuda_runtime.h>

#include "device.cuh"
#include "internal.hpp"

namespace ada {

template <class V, int SR>
__global__ void fill_value_kernel(V* y, int64_t n) {
    const int64_t i0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = i0; i < n; i += stride) y[i] = Semiring<SR, V>::zero();
}

// y[0..n) = the semiring's additive identity (0 for plus-times / or-and,
// +inf for min-plus).
template <class V, int SR>
inline void fill_value(Context& ctx, V* y, int64_t n) {
    if (n <= 0) return;
    if (SR != SR_MIN_PLUS) {
        ADA_CUDA(cudaMemsetAsync(y, 0, sizeof(V) * static_cast<size_t>(n), ctx.stream));
        return;
    }
    int64_t blocks = (n + 255) / 256;
    if (blocks > ctx.sm_count * 16) blocks = ctx.sm_count * 16;
    fill_value_kernel<V, SR><<<static_cast<unsigned>(blocks), 256, 0, ctx.stream>>>(y, n);
    ADA_LAUNCHED(ctx);
}

int default_lanes_per_row(double avg);

// K0-K3 (kernels_row.cu).  mask == nullptr -> SpMV, else RowSpMSpV.
template <class V, int SR>
void run_row_major(Context& ctx, const Matrix& m, const V* x, const uint32_t* mask, bool lb,
                   int lanes, V* y);

// K0/K2 on the row-bin layout (kernels_binned.cu); builds the layout on
// first use.  mask == nullptr -> SpMV.
template <class V, int SR>
void run_row_binned(Context& ctx, const Matrix& m, const V* x, const uint32_t* mask, V* y,
                    int64_t force_rows, int64_t tile_cap, int cluster = 0, int panel_kib = 0);

// K4-K7 (kernels_col.cu).  Atomic -> dense y (y_dense); sort -> sparse y
// (y_idx, y_val, *d_nnz on device).  x is the sparse operand.
// row-segmented atomic column write-back (kernels_colseg.cu), used by K4/K6
// when ADASPMV_COLSEG=1 (colseg_mode() == 1; 0 or unset: off)
int colseg_mode();
template <class V, int SR>
bool run_col_segmented(Context& ctx, const Matrix& m, Vector& x, V* y);

template <class V, int SR>
void run_col_major(Context& ctx, const Matrix& m, Vector& x, bool lb, bool sort, bool private_acc,
                   int lanes, V* y_dense, int32_t* y_idx, V* y_val, int64_t* d_nnz,
                   int64_t* h_nnz);

}  // namespace ada

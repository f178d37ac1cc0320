// multi.cpp -- the row-partitioned multi-GPU mode behind one C-ABI handle
// (SURVEY.md 8(b) `adaspmv_multi_create`, 8(e)): one process drives G devices.
//
// The matrix is cut into G contiguous row blocks of ~nnz/G nonzeros
// (shard_cuts: the segment_of search of partition.hpp:30-33 snapped to row
// starts, so no row is split); shard g holds rows [cut[g], cut[g+1]) as its
// own device DualMatrix (CSR + CSC of the block over all n columns) on its
// own device and stream, and runs its own selector decision -- nnz_s differs
// per shard.  A multiply sends x to every shard (each device copies it from
// the caller's host buffer over its own link, concurrently), every shard
// multiplies its block, and the y blocks land at their row offsets of the
// caller's dense y.  Rows are independent, so there is no other exchange.
// (The torch.distributed flavour, one process per GPU with NCCL, is
// paper_2006_16767_b200/multigpu.py.)
#include <cuda_runtime.h>

#include <algorithm>
#include <exception>
#include <mutex>
#include <thread>
#include <vector>

#include "internal.hpp"

namespace ada {

void shard_cuts(const int64_t* ro, int64_t rows, int g, int64_t* cuts) {
    const int64_t nnz = ro[rows];
    cuts[0] = 0;
    for (int i = 1; i < g; ++i) {
        const int64_t pos = nnz * i / g;
        // first row starting at or after pos: rows are never split
        int64_t r = static_cast<int64_t>(std::lower_bound(ro, ro + rows + 1, pos) - ro);
        if (r > rows) r = rows;
        cuts[i] = std::max(r, cuts[i - 1]);
    }
    cuts[g] = rows;
}

namespace {

// Runs f(g) for every shard on its own host thread (device and allocation
// stream bound); the first failure is rethrown on the caller.
template <class F>
void for_shards(Multi& mm, F&& f) {
    std::mutex mu;
    std::exception_ptr first;
    std::vector<std::thread> th;
    for (size_t g = 0; g < mm.shards.size(); ++g)
        th.emplace_back([&, g] {
            try {
                MultiShard& s = *mm.shards[g];
                ADA_CUDA(cudaSetDevice(s.ctx.device));
                g_alloc_stream = s.ctx.stream;
                f(static_cast<int>(g), s);
            } catch (...) {
                std::lock_guard<std::mutex> lk(mu);
                if (!first) first = std::current_exception();
            }
        });
    for (auto& t : th) t.join();
    if (first) std::rethrow_exception(first);
}

}  // namespace

MultiShard::~MultiShard() {
    cudaSetDevice(ctx.device);
    g_alloc_stream = ctx.stream;
    cudaStreamSynchronize(ctx.stream);
    delete m;
    v.dense.release();
    v.sp_idx.release();
    v.sp_val.release();
    v.mask.release();
    v.eff.release();
    v.stage_idx.release();
    y.dense.release();
    y.sp_idx.release();
    y.sp_val.release();
    y.d_nnz.release();
    context_release(ctx);
}

Multi* multi_create(int ngpu, const int* devices, int64_t rows, int64_t cols, const int64_t* ro,
                    const int64_t* ci, const void* vals, int dtype) {
    if (ngpu <= 0) invalid("multi: ngpu must be positive");
    auto mm = std::make_unique<Multi>();
    mm->rows = rows;
    mm->cols = cols;
    mm->dtype = dtype;
    mm->cuts.resize(static_cast<size_t>(ngpu) + 1);
    shard_cuts(ro, rows, ngpu, mm->cuts.data());
    for (int g = 0; g < ngpu; ++g) {
        auto s = std::make_unique<MultiShard>();
        context_init(s->ctx, devices ? devices[g] : g, nullptr);
        mm->shards.push_back(std::move(s));
    }
    const size_t vb = static_cast<size_t>(value_bytes(dtype));
    for_shards(*mm, [&](int g, MultiShard& s) {
        const int64_t r0 = mm->cuts[static_cast<size_t>(g)], r1 = mm->cuts[static_cast<size_t>(g) + 1];
        const int64_t b = ro[r0], e = ro[r1], nnz = e - b;
        // the block's CSR: offsets rebased, column indices narrowed to int32
        std::vector<int64_t> bro(static_cast<size_t>(r1 - r0) + 1);
        for (int64_t r = r0; r <= r1; ++r) bro[static_cast<size_t>(r - r0)] = ro[r] - b;
        std::vector<int32_t> bci(static_cast<size_t>(std::max<int64_t>(nnz, 1)));
        for (int64_t k = 0; k < nnz; ++k) bci[static_cast<size_t>(k)] = static_cast<int32_t>(ci[b + k]);
        DevBuf d_ro, d_ci, d_v;
        d_ro.ensure(sizeof(int64_t) * bro.size());
        d_ci.ensure(sizeof(int32_t) * bci.size());
        d_v.ensure(vb * static_cast<size_t>(std::max<int64_t>(nnz, 1)));
        ADA_CUDA(cudaMemcpyAsync(d_ro.p, bro.data(), sizeof(int64_t) * bro.size(), cudaMemcpyHostToDevice,
                                 s.ctx.stream));
        if (nnz > 0) {
            ADA_CUDA(cudaMemcpyAsync(d_ci.p, bci.data(), sizeof(int32_t) * static_cast<size_t>(nnz),
                                     cudaMemcpyHostToDevice, s.ctx.stream));
            if (vals)
                ADA_CUDA(cudaMemcpyAsync(d_v.p, static_cast<const char*>(vals) + vb * static_cast<size_t>(b),
                                         vb * static_cast<size_t>(nnz), cudaMemcpyHostToDevice, s.ctx.stream));
        }
        s.m = matrix_create_device(s.ctx, r1 - r0, cols, nnz, d_ro.as<int64_t>(), d_ci.as<int32_t>(),
                                   vals ? d_v.p : nullptr, dtype, vals == nullptr);
        s.ctx.sync();  // the staging above is released on return
        s.v.ctx = &s.ctx;
        s.v.n = cols;
        s.v.dtype = dtype;
        s.y.ctx = &s.ctx;
    });
    return mm.release();
}

void multi_run(Multi& mm, const Bundle* b, int forced, const adaspmv_config& cfg, int64_t nnz_x,
               const int64_t* idx, const void* vals, void* y_host, int* kernels) {
    const size_t vb = static_cast<size_t>(value_bytes(mm.dtype));
    for_shards(mm, [&](int g, MultiShard& s) {
        // x: every shard copies the caller's operand over its own link
        if (nnz_x < 0) {
            s.v.invalidate();
            const size_t bytes = vb * static_cast<size_t>(mm.cols);
            s.v.dense.ensure(std::max<size_t>(bytes, 1));
            if (bytes) ADA_CUDA(cudaMemcpyAsync(s.v.dense.p, vals, bytes, cudaMemcpyHostToDevice, s.ctx.stream));
            s.v.has_dense = true;
        } else {
            vector_set_sparse_host(s.ctx, s.v, nnz_x, idx, vals);
        }
        const int k = forced >= 0 ? forced : predict(s.ctx, *s.m, s.v, *b, nullptr, nullptr);
        run_kernel(s.ctx, *s.m, s.v, k, cfg, s.y);
        output_ensure_dense(s.ctx, s.y);
        const int64_t r0 = mm.cuts[static_cast<size_t>(g)], nr = s.m->rows;
        if (nr > 0 && y_host)
            ADA_CUDA(cudaMemcpyAsync(static_cast<char*>(y_host) + vb * static_cast<size_t>(r0), s.y.dense.p,
                                     vb * static_cast<size_t>(nr), cudaMemcpyDeviceToHost, s.ctx.stream));
        s.ctx.sync();
        if (kernels) kernels[g] = k;
    });
}

}  // namespace ada

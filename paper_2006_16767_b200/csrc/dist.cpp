// dist.cpp -- the exchange steps of the row-partitioned multi-GPU mode, one
// process per GPU (BASELINE.json north_star), inside the
// library: rank g holds the row block [cut[g], cut[g+1]) of the matrix as its
// own DualMatrix (adaspmv_shard_rows: the segment_of cut of
// partition.hpp:30-33 snapped to row starts) and the library moves
//   * x from the root rank into every rank's operand (broadcast: dense
//     values, or count + int32 indices + values),
//   * the y blocks / BFS frontier lists of every rank into every rank
//     (all-gatherv in rank order = ascending global row order),
//   * the per-rank counts the level loop needs (all-gather of one int64),
// on the context's stream, device to device.
//
// Transports:
//   NCCL (the product): a communicator built from an ncclUniqueId the caller
//     distributes (adaspmv_dist_unique_id on rank 0, any bootstrap channel),
//     collectives over NVLink / NVSwitch.  libnccl is loaded at run time
//     (dlopen "libnccl.so.2": in a process that already loaded torch's NCCL
//     the same library is shared), so the library itself has no link-time
//     NCCL dependency and a missing NCCL is a clean ADASPMV_ERR_CUDA error.
//     All-gatherv = one grouped ncclBroadcast per root rank (NCCL has no
//     variable-size all-gather).
//   host (tests, and ranks sharing one GPU, where NCCL refuses a duplicate
//     device): the caller's all-gather callback over host memory, e.g.
//     torch.distributed over gloo.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

#include "internal.hpp"

namespace ada {

namespace {

// ---- run-time NCCL --------------------------------------------------------
struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            const char* e = dlerror();
            api.why = std::string("libnccl.so.2 not loadable: ") + (e ? e : "?");
            return;
        }
        bool all = true;
        auto sym = [&](auto& f, const char* name) {
            f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(h, name));
            if (!f) all = false;
        };
        sym(api.GetUniqueId, "ncclGetUniqueId");
        sym(api.CommInitRank, "ncclCommInitRank");
        sym(api.CommDestroy, "ncclCommDestroy");
        sym(api.Broadcast, "ncclBroadcast");
        sym(api.AllGather, "ncclAllGather");
        sym(api.GroupStart, "ncclGroupStart");
        sym(api.GroupEnd, "ncclGroupEnd");
        sym(api.GetErrorString, "ncclGetErrorString");
        api.ok = all;
        if (!all) api.why = "libnccl.so.2 lacks an expected symbol";
    });
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) {
        const NcclApi& a = nccl();
        throw Error(ADASPMV_ERR_CUDA, std::string(what) + ": " + (a.GetErrorString ? a.GetErrorString(r) : "nccl error"));
    }
}

const NcclApi& nccl_required() {
    const NcclApi& a = nccl();
    if (!a.ok) throw Error(ADASPMV_ERR_CUDA, "dist: NCCL transport unavailable (" + a.why + ")");
    return a;
}

}  // namespace

void dist_unique_id(void* out128) {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    const NcclApi& a = nccl_required();
    ncclUniqueId id;
    nccl_check(a.GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out128, &id, sizeof(id));
}

Dist* dist_create_nccl(Context& ctx, int rank, int world, const void* id128) {
    if (world <= 0 || rank < 0 || rank >= world) invalid("dist: rank / world out of range");
    const NcclApi& a = nccl_required();
    auto d = std::make_unique<Dist>();
    d->ctx = &ctx;
    d->rank = rank;
    d->world = world;
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    ncclComm_t comm = nullptr;
    nccl_check(a.CommInitRank(&comm, world, id, rank), "ncclCommInitRank");
    d->comm = comm;
    return d.release();
}

Dist* dist_create_host(Context& ctx, int rank, int world, adaspmv_allgather_fn fn, void* user) {
    if (world <= 0 || rank < 0 || rank >= world) invalid("dist: rank / world out of range");
    if (!fn) invalid("dist: all-gather callback is NULL");
    auto d = std::make_unique<Dist>();
    d->ctx = &ctx;
    d->rank = rank;
    d->world = world;
    d->host_fn = fn;
    d->host_user = user;
    return d.release();
}

Dist::~Dist() {
    dist_release_peers(*this);
    if (comm) {
        const NcclApi& a = nccl();
        if (a.ok) a.CommDestroy(static_cast<ncclComm_t>(comm));
    }
}

void Dist::host_allgather(const void* send, size_t bytes, void* recv) {
    if (host_fn(host_user, send, static_cast<int64_t>(bytes), recv) != 0)
        throw Error(ADASPMV_ERR_INTERNAL, "dist: the all-gather callback failed");
}

void Dist::allgather_bytes(const void* send, size_t bytes, void* recv) {
    if (!comm) {
        host_allgather(send, bytes, recv);
        return;
    }
    const NcclApi& a = nccl();
    Context& c = *ctx;
    char* d = static_cast<char*>(d_bytes.ensure(bytes * static_cast<size_t>(world + 1)));
    ADA_CUDA(cudaMemcpyAsync(d + bytes * world, send, bytes, cudaMemcpyHostToDevice, c.stream));
    nccl_check(a.AllGather(d + bytes * world, d, bytes, ncclUint8, static_cast<ncclComm_t>(comm), c.stream),
               "ncclAllGather");
    ADA_CUDA(cudaMemcpyAsync(recv, d, bytes * world, cudaMemcpyDeviceToHost, c.stream));
    c.sync();
}

void Dist::allgather_count(int64_t mine, std::vector<int64_t>& all) {
    all.assign(static_cast<size_t>(world), 0);
    Context& c = *ctx;
    if (comm) {
        const NcclApi& a = nccl();
        int64_t* d = static_cast<int64_t*>(d_cnt.ensure(sizeof(int64_t) * static_cast<size_t>(world + 1)));
        ADA_CUDA(cudaMemcpyAsync(d + world, &mine, sizeof(int64_t), cudaMemcpyHostToDevice, c.stream));
        nccl_check(a.AllGather(d + world, d, 1, ncclInt64, static_cast<ncclComm_t>(comm), c.stream), "ncclAllGather");
        ADA_CUDA(cudaMemcpyAsync(all.data(), d, sizeof(int64_t) * static_cast<size_t>(world), cudaMemcpyDeviceToHost,
                                 c.stream));
        c.sync();
    } else {
        host_allgather(&mine, sizeof(int64_t), all.data());
    }
}

int64_t Dist::allgatherv(const void* send, int64_t count, size_t elem, void* recv) {
    if (peer_buf && recv == peer_buf) return dist_peer_allgatherv(*this, send, count, elem);  // NVLink puts (peer.cu)
    allgather_count(count, counts);
    int64_t total = 0, maxc = 0;
    for (int64_t v : counts) {
        total += v;
        maxc = std::max(maxc, v);
    }
    if (total == 0) return 0;
    Context& c = *ctx;
    if (comm) {
        const NcclApi& a = nccl();
        nccl_check(a.GroupStart(), "ncclGroupStart");
        int64_t off = 0;
        for (int g = 0; g < world; ++g) {
            const int64_t n = counts[static_cast<size_t>(g)];
            if (n > 0) {
                char* dst = static_cast<char*>(recv) + off * static_cast<int64_t>(elem);
                nccl_check(a.Broadcast(g == rank ? send : dst, dst, static_cast<size_t>(n) * elem, ncclUint8, g,
                                       static_cast<ncclComm_t>(comm), c.stream),
                           "ncclBroadcast");
            }
            off += n;
        }
        nccl_check(a.GroupEnd(), "ncclGroupEnd");
        return total;
    }
    // host transport: pad every block to the longest one
    const size_t blk = static_cast<size_t>(maxc) * elem;
    h_send.assign(std::max<size_t>(blk, 1), 0);
    h_recv.assign(std::max<size_t>(blk * static_cast<size_t>(world), 1), 0);
    if (count > 0)
        ADA_CUDA(cudaMemcpyAsync(h_send.data(), send, static_cast<size_t>(count) * elem, cudaMemcpyDeviceToHost,
                                 c.stream));
    c.sync();
    host_allgather(h_send.data(), blk, h_recv.data());
    int64_t off = 0;
    for (int g = 0; g < world; ++g) {
        const int64_t n = counts[static_cast<size_t>(g)];
        if (n > 0)
            ADA_CUDA(cudaMemcpyAsync(static_cast<char*>(recv) + off * static_cast<int64_t>(elem),
                                     h_recv.data() + blk * static_cast<size_t>(g), static_cast<size_t>(n) * elem,
                                     cudaMemcpyHostToDevice, c.stream));
        off += n;
    }
    c.sync();  // the host staging is reused by the next call
    return total;
}

void Dist::broadcast(void* buf, int64_t bytes, int root) {
    if (root < 0 || root >= world) invalid("dist: root out of range");
    if (bytes <= 0) return;
    Context& c = *ctx;
    if (comm) {
        const NcclApi& a = nccl();
        nccl_check(a.Broadcast(buf, buf, static_cast<size_t>(bytes), ncclUint8, root, static_cast<ncclComm_t>(comm),
                               c.stream),
                   "ncclBroadcast");
        return;
    }
    const size_t b = static_cast<size_t>(bytes);
    h_send.assign(b, 0);
    h_recv.assign(b * static_cast<size_t>(world), 0);
    if (rank == root) {
        ADA_CUDA(cudaMemcpyAsync(h_send.data(), buf, b, cudaMemcpyDeviceToHost, c.stream));
        c.sync();
    }
    host_allgather(h_send.data(), b, h_recv.data());
    if (rank != root) {
        ADA_CUDA(cudaMemcpyAsync(buf, h_recv.data() + b * static_cast<size_t>(root), b, cudaMemcpyHostToDevice,
                                 c.stream));
        c.sync();
    }
}

// x of the root rank into every rank's operand, in the root's representation
// (sparse when it has one, else dense).  The broadcast is the only exchange
// an SpMV needs: rows are independent.
void dist_bcast_vector(Dist& d, Vector& x, int root) {
    Context& c = *d.ctx;
    int64_t hdr[3] = {0, 0, 0};  // sparse?, nnz, n
    if (d.rank == root) {
        if (!x.has_sparse && !x.has_dense) invalid("dist_bcast_vector: the root's vector is not set");
        hdr[0] = x.has_sparse ? 1 : 0;
        hdr[1] = x.has_sparse ? x.nnz : x.n;
        hdr[2] = x.n;
    }
    {
        int64_t* dh = static_cast<int64_t*>(d.d_cnt.ensure(sizeof(int64_t) * static_cast<size_t>(d.world + 3)));
        ADA_CUDA(cudaMemcpyAsync(dh, hdr, sizeof(hdr), cudaMemcpyHostToDevice, c.stream));
        d.broadcast(dh, sizeof(hdr), root);
        ADA_CUDA(cudaMemcpyAsync(hdr, dh, sizeof(hdr), cudaMemcpyDeviceToHost, c.stream));
        c.sync();
    }
    if (hdr[2] != x.n) invalid("dist_bcast_vector: vector lengths differ across ranks");
    const size_t vb = static_cast<size_t>(value_bytes(x.dtype));
    if (hdr[0]) {
        const int64_t nnz = hdr[1];
        if (d.rank != root) {
            x.invalidate();
            x.sp_idx.ensure(sizeof(int32_t) * static_cast<size_t>(std::max<int64_t>(nnz, 1)));
            x.sp_val.ensure(vb * static_cast<size_t>(std::max<int64_t>(nnz, 1)));
        }
        d.broadcast(x.sp_idx.p, static_cast<int64_t>(sizeof(int32_t)) * nnz, root);
        d.broadcast(x.sp_val.p, static_cast<int64_t>(vb) * nnz, root);
        if (d.rank != root) {
            x.nnz = nnz;
            x.has_sparse = true;
        }
    } else {
        if (d.rank != root) {
            x.invalidate();
            x.dense.ensure(vb * static_cast<size_t>(std::max<int64_t>(x.n, 1)));
        }
        d.broadcast(x.dense.p, static_cast<int64_t>(vb) * x.n, root);
        if (d.rank != root) x.has_dense = true;
    }
}

// Every rank's dense y block, in rank order, into the device buffer y_full
// (the full y on every rank: the exchange an iterative use needs).
int64_t dist_allgather_output(Dist& d, Output& y, void* y_full) {
    output_ensure_dense(*d.ctx, y);
    return d.allgatherv(y.dense.p, y.n, static_cast<size_t>(value_bytes(y.dtype)), y_full);
}

}  // namespace ada

// peer.cu -- the y all-gather of the row-partitioned mode as direct peer
// stores over NVLink / NVSwitch (CUDA IPC), replacing the NCCL broadcasts of
// Dist::allgatherv for a full-y buffer the library allocated
// (adaspmv_dist_alloc_peer_output).  The reference's row partition
// (partition.hpp:30-56) gives each rank a contiguous block of y; every rank
// writes its block straight into every rank's full y (one kernel, each source
// word read once and stored to all peers), between two rank barriers:
//   entry: every rank's earlier stream work (which may read its full y) done;
//   exit : every rank's stores done, so the full y is complete everywhere.
// Peers in the same process (ranks as threads, the one-GPU tests) use the raw
// pointer; other processes open the allocation's IPC handle.
#include <unistd.h>

#include <cstring>

#include "internal.hpp"

namespace ada {

namespace {

struct PeerInfo {
    int64_t pid;
    uint64_t ptr;
    cudaIpcMemHandle_t handle;
};

// dst[p] + off <- src for every peer p; 16-B words when every address allows
__global__ void peer_put_kernel(const char* __restrict__ src, int64_t bytes, char* const* __restrict__ dst,
                                int world, int64_t off) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int64_t t0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    bool vec = (reinterpret_cast<uintptr_t>(src) & 15) == 0 && (off & 15) == 0;
    for (int p = 0; p < world; ++p) vec = vec && (reinterpret_cast<uintptr_t>(dst[p]) & 15) == 0;
    int64_t done = 0;
    if (vec) {
        const int64_t n16 = bytes >> 4;
        for (int64_t i = t0; i < n16; i += stride) {
            const int4 v = __ldg(reinterpret_cast<const int4*>(src) + i);
            for (int p = 0; p < world; ++p) reinterpret_cast<int4*>(dst[p] + off)[i] = v;
        }
        done = n16 << 4;
    }
    for (int64_t i = done + t0; i < bytes; i += stride) {  // tail (or unaligned) bytes
        const char v = src[i];
        for (int p = 0; p < world; ++p) dst[p][off + i] = v;
    }
    __threadfence_system();
}

}  // namespace

void* dist_alloc_peer_output(Dist& d, int64_t bytes) {
    if (bytes <= 0) invalid("dist: peer output size must be positive");
    if (d.peer_buf) invalid("dist: a peer output is already attached");
    void* buf = nullptr;
    ADA_CUDA(cudaMalloc(&buf, static_cast<size_t>(bytes)));  // a base allocation: IPC-exportable
    PeerInfo mine{};
    mine.pid = static_cast<int64_t>(getpid());
    mine.ptr = reinterpret_cast<uint64_t>(buf);
    ADA_CUDA(cudaIpcGetMemHandle(&mine.handle, buf));
    std::vector<PeerInfo> all(static_cast<size_t>(d.world));
    d.allgather_bytes(&mine, sizeof(mine), all.data());
    d.peer_ptrs.assign(static_cast<size_t>(d.world), nullptr);
    d.peer_opened.assign(static_cast<size_t>(d.world), 0);
    for (int r = 0; r < d.world; ++r) {
        const PeerInfo& pi = all[static_cast<size_t>(r)];
        if (pi.pid == mine.pid) {
            d.peer_ptrs[static_cast<size_t>(r)] = reinterpret_cast<void*>(pi.ptr);
        } else {
            void* p = nullptr;
            ADA_CUDA(cudaIpcOpenMemHandle(&p, pi.handle, cudaIpcMemLazyEnablePeerAccess));
            d.peer_ptrs[static_cast<size_t>(r)] = p;
            d.peer_opened[static_cast<size_t>(r)] = 1;
        }
    }
    char** dp = static_cast<char**>(d.d_peers.ensure(sizeof(char*) * static_cast<size_t>(d.world)));
    ADA_CUDA(cudaMemcpyAsync(dp, d.peer_ptrs.data(), sizeof(char*) * static_cast<size_t>(d.world),
                             cudaMemcpyHostToDevice, d.ctx->stream));
    d.ctx->sync();
    d.peer_buf = buf;
    d.peer_bytes = bytes;
    return buf;
}

void dist_release_peers(Dist& d) {
    for (size_t r = 0; r < d.peer_ptrs.size(); ++r)
        if (d.peer_opened[r]) cudaIpcCloseMemHandle(d.peer_ptrs[r]);
    if (d.peer_buf) cudaFree(d.peer_buf);
    d.peer_ptrs.clear();
    d.peer_opened.clear();
    d.peer_buf = nullptr;
    d.peer_bytes = 0;
}

int64_t dist_peer_allgatherv(Dist& d, const void* send, int64_t count, size_t elem) {
    Context& c = *d.ctx;
    c.sync();  // this rank's earlier work on its full y is done ...
    d.allgather_count(count, d.counts);  // ... everywhere (entry barrier), and the block offsets
    int64_t total = 0, off = 0;
    for (int g = 0; g < d.world; ++g) {
        if (g < d.rank) off += d.counts[static_cast<size_t>(g)];
        total += d.counts[static_cast<size_t>(g)];
    }
    if (static_cast<int64_t>(total * elem) > d.peer_bytes) invalid("dist: the peer output is too small");
    const int64_t bytes = count * static_cast<int64_t>(elem);
    if (bytes > 0) {
        const int64_t blocks = std::min<int64_t>((bytes / 16 + 255) / 256 + 1, static_cast<int64_t>(c.sm_count) * 8);
        peer_put_kernel<<<static_cast<unsigned>(blocks), 256, 0, c.stream>>>(
            static_cast<const char*>(send), bytes, d.d_peers.as<char*>(), d.world, off * static_cast<int64_t>(elem));
        ADA_LAUNCHED(c);
    }
    c.sync();
    std::vector<int64_t> done;
    d.allgather_count(0, done);  // exit barrier: every rank's stores are complete
    return total;
}

int64_t dist_run_allgather(Dist& d, const Matrix& m, Vector& x, int k, const adaspmv_config& cfg, Output& y,
                           void* y_full, int* fused) {
    if (!d.peer_buf || y_full != d.peer_buf) invalid("dist: y_full must be the peer output (adaspmv_dist_alloc_peer_output)");
    Context& c = *d.ctx;
    c.sync();  // this rank's earlier work on its full y is done ...
    d.allgather_count(m.rows, d.counts);  // ... everywhere (entry barrier), and the block offsets
    int64_t total = 0, off = 0;
    for (int g = 0; g < d.world; ++g) {
        if (g < d.rank) off += d.counts[static_cast<size_t>(g)];
        total += d.counts[static_cast<size_t>(g)];
    }
    const size_t elem = static_cast<size_t>(m.vbytes());
    if (static_cast<int64_t>(total * elem) > d.peer_bytes) invalid("dist: the peer output is too small");
    c.peer_dst = d.d_peers.as<char*>();
    c.peer_world = d.world;
    c.peer_row0 = off;
    c.peer_fused = false;
    try {
        run_kernel(c, m, x, k, cfg, y);
    } catch (...) {
        c.peer_dst = nullptr;
        c.peer_world = 0;
        throw;
    }
    const bool f = c.peer_fused;
    c.peer_dst = nullptr;
    c.peer_world = 0;
    c.peer_fused = false;
    if (!f && m.rows > 0) {  // the put kernel after the multiply
        output_ensure_dense(c, y);
        const int64_t bytes = m.rows * static_cast<int64_t>(elem);
        const int64_t blocks = std::min<int64_t>((bytes / 16 + 255) / 256 + 1, static_cast<int64_t>(c.sm_count) * 8);
        peer_put_kernel<<<static_cast<unsigned>(blocks), 256, 0, c.stream>>>(
            static_cast<const char*>(y.dense.p), bytes, d.d_peers.as<char*>(), d.world, off * static_cast<int64_t>(elem));
        ADA_LAUNCHED(c);
    }
    if (fused) *fused = f ? 1 : 0;
    c.sync();
    std::vector<int64_t> done;
    d.allgather_count(0, done);  // exit barrier: every rank's stores are complete
    return total;
}

}  // namespace ada

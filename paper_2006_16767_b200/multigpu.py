"""Row-partitioned multi-GPU mode, one process per GPU (BASELINE.json
north_star).

The matrix is cut into G contiguous row blocks with ~nnz/G nonzeros each
(`adaspmv_shard_rows`: the segment_of search of partition.hpp:30-33, snapped
to row starts so no row is split).  Rank g holds rows [cut[g], cut[g+1]) as
its own device DualMatrix (CSR + CSC of the block over all n columns) and runs
its own selector hook, since nnz_s differs per block.

The exchanges run inside the library (`adaspmv_dist_*`, csrc/dist.cpp) on the
rank's stream, device to device:
  1. x is broadcast from the root rank into every rank's operand (dense
     values, or count + int32 indices + values) -- the only exchange an SpMV
     needs, rows being independent;
  2. every rank computes y_block = A_block x with its locally selected kernel;
  3. y blocks are all-gathered only when the caller needs the full vector;
     the BFS level loop (adaspmv_dist_bfs) all-gathers only the new frontier
     index lists, in rank order (= ascending vertex order).
Transport: NCCL when torch.distributed runs the nccl backend (rank 0 makes
the ncclUniqueId, torch.distributed hands it to every rank; NVLink /
NVSwitch between B200s); otherwise the library calls back into a host
all-gather over the process group (gloo: tests, ranks sharing a GPU).
torch.distributed is plumbing here -- the id hand-over and the host
transport -- never the data path of the NCCL transport.
"""
from __future__ import annotations

from typing import Optional

import numpy as np
import torch
import torch.distributed as dist

from . import adaspmv as A


def shard_rows(row_offsets, world: int) -> np.ndarray:
    return A.shard_rows(row_offsets, world)


def block(ro, ci, vals, r0, r1):
    """CSR rows [r0, r1) as a standalone CSR (all columns kept)."""
    b, e = int(ro[r0]), int(ro[r1])
    return ro[r0:r1 + 1] - b, ci[b:e], (None if vals is None else vals[b:e])


def host_allgather(data: bytes) -> list:
    """The host transport's all-gather (adaspmv_allgather_fn contract): every
    rank's bytes, in rank order, over the default process group."""
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, data)
    return out


def make_dist(ctx: A.Context, transport: str = "auto") -> A.Dist:
    """The library exchange for this rank: NCCL (uid from rank 0 through the
    process group) or the host all-gather."""
    rank, world = dist.get_rank(), dist.get_world_size()
    if transport == "auto":
        transport = "nccl" if dist.get_backend() == "nccl" else "host"
    if transport == "nccl":
        uid = [A.dist_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        return A.Dist.nccl(ctx, rank, world, uid[0])
    if transport == "host":
        return A.Dist.host(ctx, rank, world, host_allgather)
    raise ValueError(f"unknown transport {transport!r}")


class RowBlockMatrix:
    """This rank's row block of a row-partitioned matrix, with the library's
    exchange.  Every rank passes the same row_offsets (and at least its own
    block's column indices / values)."""

    def __init__(self, rows, cols, ro, ci, vals, device: int, bundle: Optional[A.SelectorBundle] = None,
                 transport: str = "auto", dtype=None, stream=None):
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.rows, self.cols = int(rows), int(cols)
        self.cuts = shard_rows(ro, self.world)
        self.r0, self.r1 = int(self.cuts[self.rank]), int(self.cuts[self.rank + 1])
        ro_b, ci_b, v_b = block(ro, ci, vals, self.r0, self.r1)
        self.dtype = np.dtype(dtype if dtype is not None else (np.float64 if vals is None else vals.dtype))
        self.device = torch.device("cuda", device)
        self.ctx = A.Context(device, stream=stream)
        self.m = A.DualMatrix.from_csr(self.r1 - self.r0, cols, ro_b, ci_b, v_b, dtype=self.dtype, ctx=self.ctx)
        self.dist = make_dist(self.ctx, transport)
        self.x = A.DeviceVector(cols, self.dtype, self.ctx)
        self.out = A.MultiplyOutput(self.ctx)
        self.bundle = bundle
        self.last_kernel = None

    def multiply(self, x_dense=None, x_sparse=None, root: int = 0, gather: bool = False, kernel: Optional[int] = None,
                 semiring: int = A.PLUS_TIMES) -> torch.Tensor:
        """y = A x with x given on `root` (dense values, or (indices, values)).
        Returns the local y block, or the full y when gather=True (device
        tensors)."""
        if self.rank == root:
            if x_dense is not None:
                self.x.set_dense(np.asarray(x_dense, dtype=self.dtype))
            else:
                self.x.set_sparse(x_sparse[0], np.asarray(x_sparse[1], dtype=self.dtype))
        self.dist.bcast_vector(self.x, root)
        cfg = A.KernelConfig(semiring=semiring)
        if kernel is not None or self.bundle is None:
            k = 1 if kernel is None else int(kernel)
            A.run_kernel(self.m, k, self.x, cfg, out=self.out)
            self.last_kernel = k
        else:
            _, kid = A.run_adaptive(self.m, self.x, self.bundle, cfg, out=self.out)
            self.last_kernel = kid.index()
        tdt = {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64}[self.dtype]
        if gather:
            y = torch.empty(self.rows, dtype=tdt, device=self.device)
            self.dist.allgather_output(self.out, y.data_ptr())
        else:
            y = torch.empty(self.r1 - self.r0, dtype=tdt, device=self.device)
            if y.numel():
                ptr = self.out.device_dense()  # densified on the device if the kernel produced sparse y
                self.ctx.synchronize()
                y.copy_(_device_view(ptr, y.numel(), tdt, self.device))
        self.ctx.synchronize()
        return y

    def bfs(self, source: int, semiring: int = A.OR_AND, kernel: int = -1, gather_levels: bool = True):
        """Level-synchronous BFS over the row blocks
        (adaspmv_dist_bfs).  Returns (levels: full array when gather_levels,
        else this rank's rows; number of levels; this rank's reports)."""
        lv, reps = self.dist.bfs(self.m, self.r0, source, semiring, self.bundle if kernel < 0 else None, kernel)
        nl = len(reps)
        if not gather_levels:
            return lv, nl, reps
        parts = [None] * self.world
        dist.all_gather_object(parts, lv.tobytes())
        return np.concatenate([np.frombuffer(p, dtype=np.int64) for p in parts]), nl, reps

    def close(self):
        self.dist.close()


def _device_view(ptr: int, n: int, dtype, device) -> torch.Tensor:
    """A torch tensor aliasing n elements of device memory at ptr."""
    class _Cuda:
        __cuda_array_interface__ = {"shape": (n,), "typestr": torch.empty(0, dtype=dtype).numpy().dtype.str,
                                    "data": (ptr, False), "version": 2}
    return torch.as_tensor(_Cuda(), device=device)

"""Row-partitioned multi-GPU mode (BASELINE.json north_star).

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch).  The
matrix is cut into G contiguous row blocks with ~nnz/G nonzeros each
(`adaspmv_shard_rows`: the segment_of search of partition.hpp:30-33, snapped
to row starts so no row is split).  Rank g holds rows [cut[g], cut[g+1]) as
its own device DualMatrix (CSR + CSC of the block, all n columns) and runs its
own selector hook, since nnz_s differs per shard.

Per multiply:
  1. x is broadcast from the root rank straight into device buffers: dense
     (n values) or sparse (count, then int32 indices + values) -- the only
     exchange an SpMV needs;
  2. every rank computes y_block = A_block x with its locally selected kernel
     (the vector is handed to the library by device pointer, no host copy);
  3. y is all-gathered only when the caller needs the full vector; for BFS
     only the new frontier index lists are all-gathered (all_gatherv by
     padding to the longest block).

The local compute is a pluggable backend: `CudaShard` (the product: the CUDA
library through its C-ABI) or any object with the same interface -- the CPU
tests inject an oracle-backed shard to exercise the partition and exchange
logic over gloo without a GPU.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch
import torch.distributed as dist

from . import adaspmv as A

_TORCH = {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64}


def shard_rows(row_offsets, world: int) -> np.ndarray:
    return A.shard_rows(row_offsets, world)


def block(ro, ci, vals, r0, r1):
    """CSR rows [r0, r1) as a standalone CSR (all columns kept)."""
    b, e = int(ro[r0]), int(ro[r1])
    return ro[r0:r1 + 1] - b, ci[b:e], vals[b:e]


class CudaShard:
    """Local compute on this rank's GPU through the CUDA library."""

    def __init__(self, rows, cols, ro, ci, vals, device: int, bundle: Optional[A.SelectorBundle] = None,
                 kernel: Optional[int] = None):
        self.ctx = A.Context(device)
        self.m = A.DualMatrix.from_csr(rows, cols, ro, ci, vals, ctx=self.ctx)
        self.dtype = np.dtype(vals.dtype)
        self.rows = rows
        self.x = A.DeviceVector(cols, self.dtype, self.ctx)
        self.out = A.MultiplyOutput(self.ctx)
        self.bundle = bundle
        self.kernel = kernel
        self.last_kernel = None
        self.stream = torch.cuda.ExternalStream(self.ctx.stream, device=torch.device("cuda", device))

    def multiply(self, xi: Optional[torch.Tensor], xv: torch.Tensor, semiring=A.PLUS_TIMES) -> torch.Tensor:
        """xi int32 / xv values on this GPU (xi None = dense).  Returns the
        dense y block as a torch tensor viewing the library's output."""
        torch.cuda.current_stream().synchronize()  # collectives wrote xi/xv on torch's stream
        if xi is None:
            self.x.set_dense_device(xv.data_ptr())
        else:
            self.x.set_sparse_device(xi.numel(), xi.data_ptr(), xv.data_ptr())
        cfg = A.KernelConfig(semiring=semiring)
        if self.kernel is not None or self.bundle is None:
            k = self.kernel if self.kernel is not None else 1
            A.run_kernel(self.m, k, self.x, cfg, out=self.out)
            self.last_kernel = k
        else:
            _, k = A.run_adaptive(self.m, self.x, self.bundle, cfg, out=self.out)
            self.last_kernel = k.index()
        ptr = self.out.device_dense()
        self.ctx.synchronize()
        if not self.rows:
            return torch.empty(0, dtype=_TORCH[self.dtype], device=xv.device)
        return _device_view(ptr, self.rows, _TORCH[self.dtype], xv.device).clone()


def _device_view(ptr: int, n: int, dtype, device) -> torch.Tensor:
    """A torch tensor aliasing n elements of device memory at ptr."""
    class _Cuda:
        __cuda_array_interface__ = {"shape": (n,), "typestr": torch.empty(0, dtype=dtype).numpy().dtype.str,
                                    "data": (ptr, False), "version": 2}
    return torch.as_tensor(_Cuda(), device=device)


def _bcast(t: Optional[torch.Tensor], dtype, root: int, device) -> torch.Tensor:
    """Broadcast a 1-D tensor of unknown length from root."""
    n = torch.tensor([0 if t is None else t.numel()], dtype=torch.int64, device=device)
    dist.broadcast(n, root)
    buf = torch.empty(int(n.item()), dtype=dtype, device=device)
    if dist.get_rank() == root and t is not None:
        buf.copy_(t.to(device=device, dtype=dtype))
    if buf.numel():
        dist.broadcast(buf, root)
    return buf


def _allgather_var(t: torch.Tensor, device) -> torch.Tensor:
    """all-gather of variable-length 1-D tensors in rank order (all_gatherv by
    padding to the longest block)."""
    world = dist.get_world_size()
    n = torch.tensor([t.numel()], dtype=torch.int64, device=device)
    sizes = [torch.zeros(1, dtype=torch.int64, device=device) for _ in range(world)]
    dist.all_gather(sizes, n)
    sizes = [int(s.item()) for s in sizes]
    mx = max(sizes)
    if mx == 0:
        return torch.zeros(0, dtype=t.dtype, device=device)
    pad = torch.zeros(mx, dtype=t.dtype, device=device)
    pad[:t.numel()] = t.to(device)
    parts = [torch.empty(mx, dtype=t.dtype, device=device) for _ in range(world)]
    dist.all_gather(parts, pad)
    return torch.cat([p[:s] for p, s in zip(parts, sizes)])


@dataclass
class RowPartitioned:
    """This rank's view of a row-partitioned matrix."""

    rows: int
    cols: int
    cuts: np.ndarray
    shard: object        # CudaShard, or a test backend with .multiply(xi, xv, semiring) and .dtype
    device: torch.device  # where the collectives run (cuda for NCCL, cpu for gloo)

    @staticmethod
    def create(rows, cols, ro, ci, vals, make_shard, device) -> "RowPartitioned":
        """Every rank passes identical row_offsets (and at least its own block's
        arrays); make_shard(rows_b, cols, ro_b, ci_b, vals_b) builds the local
        compute."""
        world, rank = dist.get_world_size(), dist.get_rank()
        cuts = shard_rows(ro, world)
        r0, r1 = int(cuts[rank]), int(cuts[rank + 1])
        ro_b, ci_b, v_b = block(ro, ci, vals, r0, r1)
        return RowPartitioned(rows, cols, cuts, make_shard(r1 - r0, cols, ro_b, ci_b, v_b), torch.device(device))

    @property
    def row_range(self):
        r = dist.get_rank()
        return int(self.cuts[r]), int(self.cuts[r + 1])

    def _vdtype(self):
        return _TORCH[np.dtype(self.shard.dtype)]

    def multiply(self, x_dense=None, x_sparse=None, root: int = 0, gather: bool = False,
                 semiring=A.PLUS_TIMES) -> torch.Tensor:
        """y = A x with x given on `root` (dense values, or (indices, values)).
        Returns the local y block, or the full y when gather=True."""
        is_root = dist.get_rank() == root
        kind = torch.tensor([1 if (is_root and x_dense is None) else 0], device=self.device)
        dist.broadcast(kind, root)
        vdt = self._vdtype()
        if int(kind.item()) == 0:
            xv = _bcast(torch.as_tensor(np.asarray(x_dense)) if is_root else None, vdt, root, self.device)
            y = self.shard.multiply(None, xv, semiring)
        else:
            xi = _bcast(torch.as_tensor(np.asarray(x_sparse[0])) if is_root else None, torch.int32, root,
                        self.device)
            xv = _bcast(torch.as_tensor(np.asarray(x_sparse[1])) if is_root else None, vdt, root, self.device)
            y = self.shard.multiply(xi, xv, semiring)
        return _allgather_var(y, self.device) if gather else y

    def bfs(self, source: int, semiring=A.OR_AND):
        """Level-synchronous BFS over the row blocks: the
        frontier is replicated; each rank finds the new vertices among its own
        rows; only the new index lists are all-gathered."""
        r0, r1 = self.row_range
        vdt = self._vdtype()
        levels = torch.full((self.rows,), -1, dtype=torch.int64, device=self.device)
        levels[source] = 0
        frontier = torch.tensor([source], dtype=torch.int32, device=self.device)
        it = 0
        ident = float("inf") if semiring == A.MIN_PLUS else 0.0
        while frontier.numel():
            fill = float(it) if semiring == A.MIN_PLUS else 1.0
            vals = torch.full((frontier.numel(),), fill, dtype=vdt, device=self.device)
            y = self.shard.multiply(frontier, vals, semiring)
            local_new = torch.nonzero((y != ident) & (levels[r0:r1] < 0)).flatten().to(torch.int32) + r0
            frontier = _allgather_var(local_new, self.device)
            it += 1
            levels[frontier.long()] = it
        return levels.cpu().numpy(), it

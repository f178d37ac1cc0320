"""CPU, world size 2 over gloo: the row-partitioned mode's partition and
exchange logic (broadcast of dense / sparse x, all_gatherv of y blocks and of
BFS frontiers).  The local compute is an oracle-backed stand-in for the CUDA
shard (test infrastructure only); the GPU shard is covered by -m gpu tests."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2006_16767_b200 import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class OracleShard:
    def __init__(self, rows, cols, ro, ci, vals):
        from oracle.oracle import Port
        self.port = Port()
        self.rows, self.cols, self.ro, self.ci, self.vals = rows, cols, ro, ci, vals
        self.dtype = vals.dtype
        self.co, self.ri, self.cv = self.port.csr_to_csc(rows, cols, ro, ci, vals)

    def multiply(self, xi, xv, semiring=0):
        xv = xv.cpu().numpy().astype(self.dtype)
        if xi is None:
            xd = xv
        else:
            xd = self.port.sparse_to_dense(self.cols, xi.cpu().numpy().astype(np.int64), xv)
        if semiring == 2:  # min-plus on a pattern matrix: y_i = min_j (x_j + 1)
            y = np.full(self.rows, np.inf)
            for r in range(self.rows):
                for k in range(self.ro[r], self.ro[r + 1]):
                    c = self.ci[k]
                    if np.isfinite(xd[c]) and (xi is None or c in set(xi.tolist())):
                        y[r] = min(y[r], xd[c] + self.vals[k])
            return torch.as_tensor(y.astype(self.dtype))
        y = self.port.reference_multiply(self.rows, self.ro, self.ci, self.vals, xd)
        return torch.as_tensor(y)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2006_16767_b200 import multigpu as MG
        from oracle.oracle import Port
        port_ = Port()
        rows, cols, ro, ci, vals = synth.random_csr(300, 300, 0.03, seed=5, dtype=np.float64)
        rp = MG.RowPartitioned.create(rows, cols, ro, ci, vals, OracleShard, "cpu")
        # dense x from root 0, full y gathered
        xd = np.random.default_rng(1).uniform(-1, 1, cols)
        y = rp.multiply(x_dense=xd if rank == 0 else None, gather=True).numpy()
        ref = port_.reference_multiply(rows, ro, ci, vals, xd)
        ok_dense = np.allclose(y, ref, rtol=0, atol=1e-12)
        # sparse x from root 1, local blocks only
        xi, xv = synth.sparse_vector(cols, 20, seed=3)
        yb = rp.multiply(x_sparse=(xi, xv) if rank == 1 else None, root=1).numpy()
        r0, r1 = rp.row_range
        ref2 = port_.reference_multiply(rows, ro, ci, vals, port_.sparse_to_dense(cols, xi, xv))[r0:r1]
        ok_sparse = np.allclose(yb, ref2, rtol=0, atol=1e-12)
        # BFS on a symmetric pattern graph vs a queue BFS
        n, _, gro, gci, gv = synth.rmat(9, 8, seed=4)
        g = MG.RowPartitioned.create(n, n, gro, gci, gv.astype(np.float64), OracleShard, "cpu")
        levels, nl = g.bfs(0, semiring=1)
        co, ri, _ = port_.csr_to_csc(n, n, gro, gci, np.ones(len(gci)))
        exp, _ = port_.bfs_queue(n, co, ri, 0)
        ok_bfs = np.array_equal(levels, exp)
        balanced = abs(int(ro[rp.cuts[1]]) - int(ro[-1]) // 2) <= int(np.diff(ro).max())
        q.put((rank, ok_dense, ok_sparse, ok_bfs, balanced))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_row_partitioned_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, a, b, c, d in res:
        assert a, f"rank {rank}: dense multiply + all-gather mismatch"
        assert b, f"rank {rank}: sparse broadcast block mismatch"
        assert c, f"rank {rank}: BFS levels differ from queue BFS"
        assert d, f"rank {rank}: row cut not nnz-balanced"

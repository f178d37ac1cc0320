"""CPU, world size 2 over gloo: the host side of the row-partitioned mode
(paper_2006_16767_b200/multigpu.py, csrc/dist.cpp) without a GPU:

* the nnz-balanced row cut (adaspmv_shard_rows, host C-ABI: the segment_of
  search of partition.hpp:30-33 snapped to row starts) is the same on every
  rank, covers every row once and is balanced;
* `host_allgather`, the adaspmv_allgather_fn contract the library's host
  transport calls (every rank's bytes in rank order), over the process group;
* the exchange protocol of adaspmv_dist_bfs restated with the oracle as the
  local compute (test infrastructure): every rank multiplies its row block
  with the replicated frontier, keeps its newly reached rows, and the
  frontier lists are all-gathered in rank order -- the levels equal a queue
  BFS and the gathered frontier is sorted (SparseVector order,
  sparse.hpp:113-130).  The CUDA path of the same protocol is
  tests/test_gpu_dist.py."""
import os
import pickle
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2006_16767_b200 import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.oracle import Port
        from paper_2006_16767_b200 import multigpu as MG
        P = Port()
        # row cut
        rows, cols, ro, ci, vals = synth.random_csr(500, 400, 0.02, seed=5, dtype=np.float64)
        cuts = MG.shard_rows(ro, world)
        all_cuts = MG.host_allgather(cuts.tobytes())
        same = all(c == cuts.tobytes() for c in all_cuts)
        covers = cuts[0] == 0 and cuts[-1] == rows and np.all(np.diff(cuts) >= 0)
        share = np.diff(ro[cuts])
        balanced = share.max() - share.min() <= 2 * int(np.diff(ro).max())
        # the all-gather contract: rank order, byte-exact, equal sizes
        got = MG.host_allgather(bytes([rank]) * 5)
        contract = got == [bytes([r]) * 5 for r in range(world)]
        # the dist BFS protocol with oracle blocks
        n, _, gro, gci, _ = synth.rmat(9, 8, seed=4)
        gc = MG.shard_rows(gro, world)
        r0, r1 = int(gc[rank]), int(gc[rank + 1])
        bro, bci, _ = MG.block(gro, gci, None, r0, r1)
        bvals = np.ones(len(bci))
        lv = np.full(r1 - r0, -1, np.int64)
        src = 3
        if r0 <= src < r1:
            lv[src - r0] = 0
        frontier = np.array([src], np.int64)
        level, sorted_ok = 0, True
        while len(frontier):
            xd = np.zeros(n)
            xd[frontier] = 1.0
            y = P.reference_multiply(r1 - r0, bro, bci, bvals, xd)
            new = np.nonzero((y != 0) & (lv < 0))[0]
            level += 1
            lv[new] = level
            parts = MG.host_allgather(pickle.dumps(new + r0))
            frontier = np.concatenate([pickle.loads(p) for p in parts]).astype(np.int64)
            sorted_ok = sorted_ok and bool(np.all(np.diff(frontier) > 0))
        full = np.concatenate([np.frombuffer(p, np.int64) for p in MG.host_allgather(lv.tobytes())])
        co, ri, _ = P.csr_to_csc(n, n, gro, gci, np.ones(len(gci)))
        exp, _ = P.bfs_queue(n, co, ri, src)
        q.put((rank, bool(same), bool(covers), bool(balanced), bool(contract), bool(np.array_equal(full, exp)),
               sorted_ok))
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_row_partitioned_host_side_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    names = ("cuts identical on all ranks", "cuts cover the rows", "cut nnz-balanced", "all-gather contract",
             "BFS levels == queue BFS", "gathered frontier sorted")
    for r in res:
        assert len(r) == 1 + len(names), r
        for ok, what in zip(r[1:], names):
            assert ok, f"rank {r[0]}: {what}"

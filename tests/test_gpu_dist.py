"""GPU: the row-partitioned mode with one rank per process or thread
(adaspmv_dist_*, csrc/dist.cpp) through the C-ABI.

* world 2 and 3 on the one GPU of the test box, one thread per rank, each rank
  with its own context (stream), its row block as its own matrix, and the
  host transport (an in-process all-gather): x broadcast (dense and sparse)
  + each rank's own kernel + y all-gather vs reference_multiply
  (kernels.hpp:197-209); BFS levels bit-exact vs a queue BFS
  for the three semirings under the built-in policy, the trained selector and
  forced pull / push kernels;
* world 1 over the NCCL transport (NCCL refuses two ranks on one device, so
  more ranks need more GPUs): the same calls;
* world 2 as two processes over gloo (paper_2006_16767_b200/multigpu.py,
  the structure bench.py runs at N > 1 with NCCL), both on cuda:0.
"""
import ctypes as C
import os
import socket
import threading

import numpy as np
import pytest
import torch

from paper_2006_16767_b200 import adaspmv as A
from paper_2006_16767_b200 import selector as S
from paper_2006_16767_b200 import synth
from tests.util import assert_dense_close, ref_and_bound

pytestmark = pytest.mark.gpu


def _cuda_driver():
    """libcuda (the rank threads' current context is the device's primary one)."""
    return C.CDLL("libcuda.so.1")


class ThreadAllgather:
    """adaspmv_allgather_fn over threads: every rank's bytes in rank order."""

    def __init__(self, world):
        self.world = world
        self.buf = [None] * world
        self.b1 = threading.Barrier(world)
        self.b2 = threading.Barrier(world)

    def for_rank(self, rank):
        def ag(data):
            self.buf[rank] = data
            self.b1.wait(timeout=120)
            out = list(self.buf)
            self.b2.wait(timeout=120)
            return out
        return ag


def run_ranks(world, fn):
    """fn(rank, dist_factory) on `world` threads; returns the per-rank results."""
    ag = ThreadAllgather(world)
    res, errs = [None] * world, [None] * world

    def body(r):
        try:
            ctx = A.Context(0)
            d = A.Dist.host(ctx, r, world, ag.for_rank(r))
            try:
                res[r] = fn(r, ctx, d)
            finally:
                d.close()
        except BaseException as e:  # noqa: BLE001
            errs[r] = e
            ag.b1.abort()
            ag.b2.abort()

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for e in errs:
        if e is not None and not isinstance(e, threading.BrokenBarrierError):
            raise e
    for e in errs:
        if e is not None:
            raise e
    return res


def _block(ro, ci, vals, r0, r1):
    b, e = int(ro[r0]), int(ro[r1])
    return ro[r0:r1 + 1] - b, ci[b:e], (None if vals is None else vals[b:e])


def _sym_rmat(scale, seed):
    n, _, ro, ci, _ = synth.rmat(scale, 8, seed=seed)
    return n, ro, ci


@pytest.mark.parametrize("world", [2, 3])
def test_dist_spmv_bcast_allgather(port, world):
    rows, cols, ro, ci, vals = synth.random_csr(2000, 1500, 0.006, seed=7, dtype=np.float64)
    cuts = A.shard_rows(ro, world)
    xd = np.random.default_rng(2).uniform(-1, 1, cols)
    xi, xv = synth.sparse_vector(cols, 60, seed=4)
    y_ref, bound = ref_and_bound(port, rows, ro, ci, vals, xd)
    ys_ref, sbound = ref_and_bound(port, rows, ro, ci, vals, port.sparse_to_dense(cols, xi, xv))

    def rank_fn(r, ctx, d):
        r0, r1 = int(cuts[r]), int(cuts[r + 1])
        bro, bci, bv = _block(ro, ci, vals, r0, r1)
        m = A.DualMatrix.from_csr(r1 - r0, cols, bro, bci, bv, ctx=ctx)
        x = A.DeviceVector(cols, np.float64, ctx)
        out = A.MultiplyOutput(ctx)
        got = {}
        for name, root, kernels in (("dense", 0, (0, 1, 4)), ("sparse", world - 1, (2, 5, 6, 7))):
            for k in kernels:
                if r == root:
                    if name == "dense":
                        x.set_dense(xd)
                    else:
                        x.set_sparse(xi, xv)
                d.bcast_vector(x, root)
                x.prepare(k)
                A.run_kernel(m, k, x, out=out)
                full = torch.empty(rows, dtype=torch.float64, device="cuda:0")
                assert d.allgather_output(out, full.data_ptr()) == rows
                ctx.synchronize()
                got[(name, k)] = full.cpu().numpy()
        return got

    res = run_ranks(world, rank_fn)
    for r in range(world):
        for (name, k), y in res[r].items():
            ref, b = (y_ref, bound) if name == "dense" else (ys_ref, sbound)
            assert_dense_close(y, ref, b, np.float64, f"world {world} rank {r} {name} K{k}")


@pytest.mark.parametrize("world", [2, 3])
def test_dist_peer_allgather(port, world):
    """The y all-gather as peer stores (csrc/peer.cu) into the library's
    IPC-shared full-y buffer: every rank's K0 block lands in every rank's
    buffer, repeated (entry/exit barriers) and with fp32 blocks of odd length
    (the byte tail of the 16-B put)."""
    for dt in (np.float64, np.float32):
        rows, cols, ro, ci, vals = synth.random_csr(3001, 1500, 0.01, seed=world, dtype=dt)
        cuts = np.linspace(0, rows, world + 1).astype(np.int64)
        xd = np.random.default_rng(1).uniform(-1, 1, cols).astype(dt)
        y_ref, bound = ref_and_bound(port, rows, ro, ci, vals, xd)

        def rank_fn(r, ctx, d):
            r0, r1 = int(cuts[r]), int(cuts[r + 1])
            bro, bci, bv = _block(ro, ci, vals, r0, r1)
            m = A.DualMatrix.from_csr(r1 - r0, cols, bro, bci, bv, ctx=ctx)
            x = A.DeviceVector(cols, dt, ctx)
            out = A.MultiplyOutput(ctx)
            ptr = d.alloc_peer_output(rows * np.dtype(dt).itemsize)
            full = []
            for it in range(3):
                x.set_dense(xd * (it + 1))
                A.run_kernel(m, 0, x, out=out)
                assert d.allgather_output(out, ptr) == rows
                ctx.synchronize()
                h = np.empty(rows, dt)
                assert _cuda_driver().cuMemcpyDtoH_v2(C.c_void_p(h.ctypes.data), C.c_uint64(ptr),
                                                      C.c_size_t(h.nbytes)) == 0
                full.append(h)
            return full

        res = run_ranks(world, rank_fn)
        for r in range(world):
            for it in range(3):
                assert_dense_close(res[r][it], y_ref * (it + 1), bound * (it + 1), dt,
                                   f"peer all-gather rank {r} iter {it} {np.dtype(dt).name}")


@pytest.mark.parametrize("world", [2, 3])
def test_dist_fused_allgather_epilogue(port, world):
    """adaspmv_dist_run_allgather: the row-bin K0/K2 store epilogue writes each
    row into every rank's full y (fused = True); K1 (CSR) and K6 (column) are
    followed by the put kernel (fused = False).  Every rank's buffer must hold
    the whole y, three rounds in a row, under all three semirings for K0."""
    dt = np.float32
    rows, cols, ro, ci, vals = synth.random_csr(6007, 4000, 0.004, seed=world + 10, dtype=dt)
    cuts = np.linspace(0, rows, world + 1).astype(np.int64)
    xd = np.random.default_rng(2).uniform(-1, 1, cols).astype(dt)
    y_ref, bound = ref_and_bound(port, rows, ro, ci, vals, xd)
    xi = np.nonzero(xd)[0].astype(np.int64)

    def rank_fn(r, ctx, d):
        r0, r1 = int(cuts[r]), int(cuts[r + 1])
        bro, bci, bv = _block(ro, ci, vals, r0, r1)
        m = A.DualMatrix.from_csr(r1 - r0, cols, bro, bci, bv, ctx=ctx)
        x = A.DeviceVector(cols, dt, ctx)
        ptr = d.alloc_peer_output(rows * 4)
        got = []
        for it, (k, cfg) in enumerate(((0, A.KernelConfig(row_layout=2)), (2, A.KernelConfig(row_layout=2)),
                                       (1, None), (6, None), (0, A.KernelConfig(row_layout=2)))):
            if k == 6:
                x.set_sparse(xi, xd[xi])
            else:
                x.set_dense(xd)
            x.prepare(k)
            try:
                tot, fused = d.run_allgather(m, k, x, ptr, cfg)
            except Exception as e:
                raise AssertionError(f"rank {r} iteration {it} K{k}: {e}") from e
            assert tot == rows
            h = np.empty(rows, dt)
            assert _cuda_driver().cuMemcpyDtoH_v2(C.c_void_p(h.ctypes.data), C.c_uint64(ptr),
                                                  C.c_size_t(h.nbytes)) == 0
            got.append((k, fused, h))
        # semirings through the fused epilogue (OR_AND / MIN_PLUS exact)
        for sr in (A.OR_AND, A.MIN_PLUS):
            xs = np.where(xd > 0, xd, np.inf).astype(dt) if sr == A.MIN_PLUS else xd
            x.set_dense(xs)
            x.prepare(0)
            tot, fused = d.run_allgather(m, 0, x, ptr, A.KernelConfig(row_layout=2, semiring=sr))
            h = np.empty(rows, dt)
            assert _cuda_driver().cuMemcpyDtoH_v2(C.c_void_p(h.ctypes.data), C.c_uint64(ptr),
                                                  C.c_size_t(h.nbytes)) == 0
            got.append((("sr", sr), fused, h, xs))
        return got

    res = run_ranks(world, rank_fn)
    for r in range(world):
        for item in res[r]:
            k, fused, h = item[:3]
            if isinstance(k, tuple):
                sr, xs = k[1], item[3]
                ref = port.semiring_multiply(rows, ro, ci, vals, xs, sr)
                assert fused and h.tobytes() == ref.tobytes(), (r, sr)
            else:
                assert fused == (k in (0, 2)), (r, k, fused)
                assert_dense_close(h, y_ref, bound, dt, f"world {world} rank {r} K{k} fused={fused}")


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("sr", [A.OR_AND, A.MIN_PLUS, A.PLUS_TIMES])
def test_dist_bfs_levels(port, world, sr):
    bundle = A.SelectorBundle.load(S.DEFAULT_PATH)
    for scale, seed in ((10, 3), (12, 8)):
        n, ro, ci = _sym_rmat(scale, seed)
        cuts = A.shard_rows(ro, world)
        co, ri, _ = port.csr_to_csc(n, n, ro, ci, np.ones(len(ci)))
        srcs = sorted({0, n - 1, int(cuts[1])})
        exp = {s: port.bfs_queue(n, co, ri, s) for s in srcs}

        def rank_fn(r, ctx, d):
            r0, r1 = int(cuts[r]), int(cuts[r + 1])
            bro, bci, _ = _block(ro, ci, None, r0, r1)
            m = A.DualMatrix.from_csr(r1 - r0, n, bro, bci, None, dtype=np.float32, ctx=ctx)
            out = {}
            for s in srcs:
                for pol, kw in (("heur", {}), ("sel", {"bundle": bundle}), ("pull", {"force_kernel": 2}),
                                ("push", {"force_kernel": 6}), ("sort", {"force_kernel": 7})):
                    lv, reps = d.bfs(m, r0, s, sr, **kw)
                    out[(s, pol)] = (lv, len(reps))
            return out

        res = run_ranks(world, rank_fn)
        for s in srcs:
            levels, nl = exp[s]
            for pol in ("heur", "sel", "pull", "push", "sort"):
                full = np.concatenate([res[r][(s, pol)][0] for r in range(world)])
                assert np.array_equal(full, levels), (scale, world, sr, s, pol)
                assert all(res[r][(s, pol)][1] == nl for r in range(world)), (scale, world, s, pol)


def test_dist_nccl_world1(port):
    """The NCCL transport end to end with one rank (more ranks need more GPUs)."""
    ctx = A.Context(0)
    d = A.Dist.nccl(ctx, 0, 1, A.dist_unique_id())
    try:
        n, ro, ci = _sym_rmat(11, 5)
        m = A.DualMatrix.from_csr(n, n, ro, ci, None, dtype=np.float32, ctx=ctx)
        co, ri, _ = port.csr_to_csc(n, n, ro, ci, np.ones(len(ci)))
        exp, nl = port.bfs_queue(n, co, ri, 0)
        for kw in ({}, {"force_kernel": 3}, {"force_kernel": 6}):
            lv, reps = d.bfs(m, 0, 0, A.OR_AND, **kw)
            assert np.array_equal(lv, exp) and len(reps) == nl, kw
        rows, cols, cro, cci, cvals = synth.random_csr(700, 500, 0.01, seed=3, dtype=np.float32)
        cm = A.DualMatrix.from_csr(rows, cols, cro, cci, cvals, ctx=ctx)
        xd = np.random.default_rng(5).uniform(-1, 1, cols).astype(np.float32)
        x = A.DeviceVector(cols, np.float32, ctx).set_dense(xd)
        d.bcast_vector(x, 0)
        out = A.MultiplyOutput(ctx)
        A.run_kernel(cm, 0, x, out=out)
        full = torch.empty(rows, dtype=torch.float32, device="cuda:0")
        assert d.allgather_output(out, full.data_ptr()) == rows
        ctx.synchronize()
        y_ref, bound = ref_and_bound(port, rows, cro, cci, cvals, xd)
        assert_dense_close(full.cpu().numpy(), y_ref, bound, np.float32, "nccl world 1")
    finally:
        d.close()


def _proc(rank, world, port_no, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.oracle import Port
        from paper_2006_16767_b200 import multigpu as MG
        P = Port()
        n, ro, ci = _sym_rmat(11, 6)
        g = MG.RowBlockMatrix(n, n, ro, ci, None, 0, dtype=np.float32)
        co, ri, _ = P.csr_to_csc(n, n, ro, ci, np.ones(len(ci)))
        exp, nl = P.bfs_queue(n, co, ri, 5)
        lv, nl2, _ = g.bfs(5, A.OR_AND)
        ok_bfs = bool(np.array_equal(lv, exp) and nl2 == nl)
        rows, cols, cro, cci, cvals = synth.random_csr(900, 800, 0.01, seed=9, dtype=np.float64)
        h = MG.RowBlockMatrix(rows, cols, cro, cci, cvals, 0)
        xi, xv = synth.sparse_vector(cols, 30, seed=1)
        y = h.multiply(x_sparse=(xi, xv), root=1, gather=True, kernel=6).cpu().numpy()
        y_ref, bound = ref_and_bound(P, rows, cro, cci, cvals, P.sparse_to_dense(cols, xi, xv))
        ok_y = bool(np.all(np.abs(y - y_ref) <= 1e-12 * bound + 1e-300))
        yb = h.multiply(x_dense=np.ones(cols), gather=False, kernel=1).cpu().numpy()
        ok_block = yb.shape[0] == h.r1 - h.r0
        # the peer transport across processes: IPC handles opened on the same device
        ptr = h.dist.alloc_peer_output(rows * 8)
        h.multiply(x_sparse=(xi, xv), root=1, gather=False, kernel=6)
        ok_peer = h.dist.allgather_output(h.out, ptr) == rows
        h.ctx.synchronize()
        yp = np.empty(rows, np.float64)
        ok_peer = ok_peer and _cuda_driver().cuMemcpyDtoH_v2(C.c_void_p(yp.ctypes.data), C.c_uint64(ptr),
                                                             C.c_size_t(yp.nbytes)) == 0
        ok_peer = ok_peer and bool(np.all(np.abs(yp - y_ref) <= 1e-12 * bound + 1e-300))
        q.put((rank, ok_bfs, ok_y, ok_block, ok_peer))
        g.close()
        h.close()
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_dist_two_processes_gloo_host_transport():
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port_no = s.getsockname()[1]
    s.close()
    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    ps = [ctxm.Process(target=_proc, args=(r, 2, port_no, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = [q.get(timeout=600) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    for g in got:
        assert len(g) == 5, g
        assert all(g[1:]), g

"""The device-resident BFS level loop (csrc/bfs_graph.cu): levels bit exact
against the queue BFS and the host-driven loop (adaspmv_ctx_set_bfs_loop),
for every semiring on pattern matrices and OR_AND on valued ones, under the
built-in policy and the trained selector (whose trees are walked on the
device: its per-level choices must equal the host selector's on the same
frontiers), on graphs of many WHILE iterations (two levels per iteration),
disconnected graphs, isolated sources and a 3001-level path -- in both
device forms: the cooperative persistent kernel (default) and the CUDA
graph (ADASPMV_BFS_PERSIST=0)."""
import numpy as np
import pytest

from paper_2006_16767_b200 import adaspmv as A
from paper_2006_16767_b200 import selector as S
from paper_2006_16767_b200 import synth

pytestmark = pytest.mark.gpu


def _sym(n, edges):
    a = np.zeros((n, n), bool)
    for u, v in edges:
        a[u, v] = a[v, u] = True
    r, c = np.nonzero(a)
    ro = np.zeros(n + 1, np.int64)
    np.add.at(ro, r + 1, 1)
    return np.cumsum(ro), c.astype(np.int64)


def _graphs():
    out = []
    # path of 40 vertices: 40 levels = 20 iterations of the graph's WHILE body
    out.append(("path40", 40, *_sym(40, [(i, i + 1) for i in range(39)])))
    # two components + an isolated vertex
    out.append(("disconnected", 12, *_sym(12, [(0, 1), (1, 2), (2, 0), (4, 5), (5, 6)])))
    for seed, scale in ((1, 10), (2, 13)):
        n, _, ro, ci, _ = synth.rmat(scale, 8, seed=seed)
        out.append((f"rmat{scale}", n, ro, ci))
    rows, cols, ro, ci, _ = synth.random_csr(3000, 3000, 0.002, seed=4)
    a = np.zeros((3000, 3000), bool)
    r = np.repeat(np.arange(3000), np.diff(ro))
    a[r, ci] = True
    a = a | a.T
    np.fill_diagonal(a, False)
    rr, cc = np.nonzero(a)
    ro2 = np.zeros(3001, np.int64)
    np.add.at(ro2, rr + 1, 1)
    out.append(("random3000", 3000, np.cumsum(ro2), cc.astype(np.int64)))
    # ~120 neighbours per vertex: the pull runs 4 lanes per row (G = 4)
    rows, cols, ro, ci, _ = synth.random_csr(2000, 2000, 0.03, seed=6)
    a = np.zeros((2000, 2000), bool)
    a[np.repeat(np.arange(2000), np.diff(ro)), ci] = True
    a = a | a.T
    np.fill_diagonal(a, False)
    rr, cc = np.nonzero(a)
    ro3 = np.zeros(2001, np.int64)
    np.add.at(ro3, rr + 1, 1)
    out.append(("dense2000", 2000, np.cumsum(ro3), cc.astype(np.int64)))
    return out


GRAPHS = _graphs()


@pytest.fixture(params=["persistent", "graph"])
def device_form(request, monkeypatch):
    # read when a matrix's traversal plan is built (first BFS on it)
    monkeypatch.setenv("ADASPMV_BFS_PERSIST", "1" if request.param == "persistent" else "0")
    return request.param


@pytest.mark.parametrize("name,n,ro,ci", GRAPHS, ids=[g[0] for g in GRAPHS])
@pytest.mark.parametrize("sr", [A.OR_AND, A.MIN_PLUS, A.PLUS_TIMES], ids=["or_and", "min_plus", "plus_times"])
def test_device_loop_levels(ctx, port, device_form, name, n, ro, ci, sr):
    m = A.DualMatrix.from_csr(n, n, ro, ci, None, dtype=np.float32, ctx=ctx)
    co, ri, _ = port.csr_to_csc(n, n, ro, ci, np.ones(len(ci)))
    bundle = A.SelectorBundle.load(S.DEFAULT_PATH)
    bundle_v2 = A.SelectorBundle.load(S.DEFAULT_PATH.parent / "b200_bundle_v2.txt")  # schema 2 on the device
    for src in sorted({0, n - 1, 3 % n}):
        exp, nl = port.bfs_queue(n, co, ri, src)
        for kw in (dict(), dict(bundle=bundle), dict(bundle=bundle_v2)):
            ctx.set_bfs_loop(False)
            lv, reps = A.bfs(m, src, sr, **kw)
            assert np.array_equal(lv, exp), (name, src, kw.keys())
            assert len(reps) == nl
            # the frontier sizes the device logged are the level sizes
            assert [r["nnz_x"] for r in reps] == [int((exp == L).sum()) for L in range(nl)]
            for r in reps:
                assert r["exec_mode"] == (A.EXEC_FUSED_PUSH_LB if r["kernel"] >= 4 else A.EXEC_MASKED_PULL)
            ctx.set_bfs_loop(True)
            lv_h, reps_h = A.bfs(m, src, sr, **kw)
            ctx.set_bfs_loop(False)
            assert np.array_equal(lv_h, exp)
            if "bundle" in kw:
                # device tree walk == host tree walk on the same frontiers
                assert [r["kernel"] for r in reps] == [r["kernel"] for r in reps_h], name


def test_device_loop_valued_or_and_and_levels_download_optional(ctx, port):
    n, _, ro, ci, vals = synth.rmat(12, 8, seed=5, values="uniform")
    m = A.DualMatrix.from_csr(n, n, ro, ci, vals, dtype=np.float64, ctx=ctx)
    co, ri, _ = port.csr_to_csc(n, n, ro, ci, np.ones(len(ci)))
    exp, nl = port.bfs_queue(n, co, ri, 0)
    lv, reps = A.bfs(m, 0, A.OR_AND)
    assert np.array_equal(lv, exp) and len(reps) == nl
    none, reps2 = A.bfs(m, 0, A.OR_AND, download_levels=False)
    assert none is None and len(reps2) == nl
    # valued matrix under plus-times: values decide y_i != 0, so the host loop runs
    lv, reps = A.bfs(m, 0, A.PLUS_TIMES)
    assert all(r["exec_mode"] != A.EXEC_FUSED_PUSH_LB or r["kernel"] >= 4 for r in reps)


def test_device_loop_deep_path(ctx, port, device_form):
    """3001 levels: the graph's WHILE node runs 1501 two-level bodies."""
    n = 3001
    ro, ci = _sym(n, [(i, i + 1) for i in range(n - 1)])
    m = A.DualMatrix.from_csr(n, n, ro, ci, None, dtype=np.float32, ctx=ctx)
    ctx.set_bfs_loop(False)
    lv, reps = A.bfs(m, 0, A.OR_AND)
    assert np.array_equal(lv, np.arange(n)) and len(reps) == n
    lv, reps = A.bfs(m, n // 2, A.MIN_PLUS)
    assert np.array_equal(lv, np.abs(np.arange(n) - n // 2)) and len(reps) == n // 2 + 1


def test_persistent_launch_fallback(ctx, port, monkeypatch):
    # a grid the device cannot co-schedule (test hook ADASPMV_BFS_PERSIST=2):
    # the plan falls back to the graph form and the traversal is still exact
    monkeypatch.setenv("ADASPMV_BFS_PERSIST", "2")
    n, _, ro, ci, _ = synth.rmat(12, 8, seed=9)
    m = A.DualMatrix.from_csr(n, n, ro, ci, None, dtype=np.float32, ctx=ctx)
    co, ri, _ = port.csr_to_csc(n, n, ro, ci, np.ones(len(ci)))
    ctx.set_bfs_loop(False)
    for _ in range(2):  # the second call runs the fallen-back plan directly
        lv, reps = A.bfs(m, 0, A.OR_AND)
        exp, nl = port.bfs_queue(n, co, ri, 0)
        assert np.array_equal(lv, exp) and len(reps) == nl

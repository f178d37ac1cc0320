"""GPU parity of the eight kernels and the operand conversions against the CPU
oracle (oracle/adaspmv_oracle.c), through the C-ABI (ctypes mirror).

Edge cases follow SURVEY.md section 4 (probe-verified reference behaviour) and
SPEC.md:156-186: all-zero matrix, a dense 1x100 row, a 100x1 column, empty x,
dense x, explicit zero in x, rows spanning several LB tiles, empty rows at
tile boundaries.
"""
import numpy as np
import pytest

from paper_2006_16767_b200 import adaspmv as A
from paper_2006_16767_b200 import synth
from tests.util import assert_dense_close, assert_sparse_match, ref_and_bound

pytestmark = pytest.mark.gpu

DTYPES = [np.float64, np.float32]


def _matrix_cases():
    cases = []
    for seed, (r, c, d) in enumerate([(300, 200, 0.05), (1000, 1000, 0.01), (64, 500, 0.2),
                                      (2000, 3000, 0.004), (1, 1, 1.0), (3, 3, 0.0)]):
        cases.append(("rand%d" % seed, synth.random_csr(r, c, d, seed=seed)))
    # all-zero 5x7
    cases.append(("zero5x7", (5, 7, np.zeros(6, np.int64), np.zeros(0, np.int64), np.zeros(0))))
    # one dense row 1x100 and one dense column 100x1
    cases.append(("row1x100", (1, 100, np.array([0, 100]), np.arange(100), np.linspace(-1, 1, 100))))
    cases.append(("col100x1", (100, 1, np.arange(101), np.zeros(100, np.int64), np.linspace(-1, 1, 100))))
    # long rows spanning LB tiles + empty rows around tile boundaries
    rng = np.random.default_rng(7)
    deg = rng.integers(0, 6, size=4000)
    deg[[10, 11, 12, 500]] = 0
    deg[100] = 9000   # spans several 2048-item tiles
    deg[2000] = 5000
    deg[1500:1600] = 0
    cols = 12000
    ro = np.zeros(len(deg) + 1, np.int64)
    ro[1:] = np.cumsum(deg)
    ci = np.concatenate([np.sort(rng.choice(cols, size=d, replace=False)) for d in deg]).astype(np.int64)
    cases.append(("skewed", (len(deg), cols, ro, ci, rng.uniform(-1, 1, ro[-1]))))
    # trailing and leading empty rows
    ro2 = np.array([0, 0, 0, 3, 3, 5, 5, 5], np.int64)
    cases.append(("emptyends", (7, 4, ro2, np.array([0, 1, 3, 0, 2]), np.array([1., 2., 3., 4., 5.]))))
    return cases


CASES = _matrix_cases()


@pytest.mark.parametrize("dt", DTYPES, ids=["f64", "f32"])
@pytest.mark.parametrize("name,case", CASES, ids=[c[0] for c in CASES])
def test_all_kernels_vs_oracle(ctx, port, name, case, dt):
    rows, cols, ro, ci, vals = case
    vals = np.asarray(vals, dt)
    m = A.DualMatrix.from_csr(rows, cols, ro, ci, vals, ctx=ctx)
    for nx in sorted({0, 1, max(1, cols // 50), max(1, cols // 3), cols}):
        xi, xv = synth.sparse_vector(cols, nx, seed=nx + 3, dtype=dt)
        xd = port.sparse_to_dense(cols, xi, xv)
        y_ref, bound = ref_and_bound(port, rows, ro, ci, vals, xd)
        for k in range(8):
            x = A.SparseVector(cols, xi, xv) if k >= 4 else A.DenseVector(xd)
            out = A.run_kernel(m, k, x)
            what = f"{name} k={k} nnz_x={nx} {np.dtype(dt).name}"
            assert_dense_close(out.dense().values, y_ref, bound, dt, what)
            s = out.sparse()
            assert_sparse_match(s.indices, s.values, y_ref, bound, dt, what)


@pytest.mark.parametrize("dt", DTYPES, ids=["f64", "f32"])
def test_lanes_override_and_workers_invariance(ctx, port, dt):
    rows, cols, ro, ci, vals = synth.random_csr(700, 900, 0.02, seed=3, dtype=dt)
    m = A.DualMatrix.from_csr(rows, cols, ro, ci, vals, ctx=ctx)
    xi, xv = synth.sparse_vector(cols, 300, seed=1, dtype=dt)
    xd = port.sparse_to_dense(cols, xi, xv)
    y_ref, bound = ref_and_bound(port, rows, ro, ci, vals, xd)
    for lanes in (1, 2, 4, 8, 16, 32):
        for k in (0, 2, 4, 5):
            x = A.SparseVector(cols, xi, xv) if k >= 4 else A.DenseVector(xd)
            out = A.run_kernel(m, k, x, A.KernelConfig(lanes_per_row=lanes, workers=lanes))
            assert_dense_close(out.dense().values, y_ref, bound, dt, f"lanes={lanes} k={k}")


@pytest.mark.parametrize("dt", DTYPES, ids=["f64", "f32"])
def test_private_accumulators(ctx, port, dt):
    # KernelConfig::atomic_private_accumulators (kernels.hpp:161, :452-478): few rows
    for r, c, d in ((64, 5000, 0.05), (3000, 800, 0.01)):
        rows, cols, ro, ci, vals = synth.random_csr(r, c, d, seed=r, dtype=dt)
        m = A.DualMatrix.from_csr(rows, cols, ro, ci, vals, ctx=ctx)
        for nx in (1, 100, cols):
            xi, xv = synth.sparse_vector(cols, nx, seed=nx, dtype=dt)
            y_ref, bound = ref_and_bound(port, rows, ro, ci, vals, port.sparse_to_dense(cols, xi, xv))
            for k in (4, 6):
                out = A.run_kernel(m, k, A.SparseVector(cols, xi, xv),
                                   A.KernelConfig(atomic_private_accumulators=True))
                assert_dense_close(out.dense().values, y_ref, bound, dt, f"private k={k} rows={r} nnz_x={nx}")
                for sr in (A.OR_AND,):
                    o2 = A.run_kernel(m, k, A.SparseVector(cols, xi, xv),
                                      A.KernelConfig(atomic_private_accumulators=True, semiring=sr))
                    o3 = A.run_kernel(m, k, A.SparseVector(cols, xi, xv), A.KernelConfig(semiring=sr))
                    assert np.array_equal(o2.dense().values, o3.dense().values)


def test_explicit_zero_in_x_drops_zero_sums(ctx):
    # A = {(0,0),(1,1),(2,0)}, x = {0: 0.0, 1: 5.0} -> sparse y = {1}
    ro = np.array([0, 1, 2, 3])
    ci = np.array([0, 1, 0])
    m = A.DualMatrix.from_csr(3, 2, ro, ci, np.array([1.0, 1.0, 1.0]), ctx=ctx)
    for k in range(8):
        out = A.run_kernel(m, k, A.SparseVector(2, [0, 1], [0.0, 5.0]))
        assert out.sparse().indices.tolist() == [1], k
        assert out.sparse().values.tolist() == [5.0], k


def test_sort_writeback_bitwise_deterministic(ctx):
    rows, cols, ro, ci, vals = synth.random_csr(20000, 20000, 0.002, seed=9, dtype=np.float32)
    m = A.DualMatrix.from_csr(rows, cols, ro, ci, vals, ctx=ctx)
    for nx in (50, 5000):  # single-CTA path and multi-kernel radix path
        xi, xv = synth.sparse_vector(cols, nx, seed=2, dtype=np.float32)
        for k in (5, 7):
            runs = [A.run_kernel(m, k, A.SparseVector(cols, xi, xv)).sparse() for _ in range(3)]
            for r in runs[1:]:
                assert np.array_equal(r.indices, runs[0].indices)
                assert r.values.tobytes() == runs[0].values.tobytes()
        # Direct and LB sort paths emit identical pair streams -> identical bits
        a = A.run_kernel(m, 5, A.SparseVector(cols, xi, xv)).sparse()
        b = A.run_kernel(m, 7, A.SparseVector(cols, xi, xv)).sparse()
        assert a.values.tobytes() == b.values.tobytes()


@pytest.mark.parametrize("dt", DTYPES, ids=["f64", "f32"])
def test_device_csc_is_bit_exact_csr_to_csc(ctx, port, dt):
    for seed, (r, c, d) in enumerate([(500, 700, 0.03), (4000, 100, 0.1), (1, 1000, 0.5)]):
        rows, cols, ro, ci, vals = synth.random_csr(r, c, d, seed=seed, dtype=dt)
        m = A.DualMatrix.from_csr(rows, cols, ro, ci, vals, ctx=ctx)
        ro2, ci2, v2, co, ri, cv = m.download()
        eco, eri, ecv = port.csr_to_csc(rows, cols, ro, ci, vals)
        assert np.array_equal(ro2, ro) and np.array_equal(ci2, ci) and v2.tobytes() == vals.tobytes()
        assert np.array_equal(co, eco)
        assert np.array_equal(ri, eri)
        assert cv.tobytes() == ecv.tobytes()
        t = m.transpose()
        tro, tci, tv, tco, tri, tcv = t.download()
        assert np.array_equal(tro, eco) and np.array_equal(tci, eri) and tv.tobytes() == ecv.tobytes()
        assert np.array_equal(tco, ro) and np.array_equal(tri, ci)


@pytest.mark.parametrize("dt", DTYPES, ids=["f64", "f32"])
def test_vector_conversions(ctx, port, dt):
    n = 10000
    rng = np.random.default_rng(4)
    xd = rng.uniform(-1, 1, n).astype(dt)
    xd[rng.random(n) < 0.7] = 0
    xd[5] = -0.0  # negative zero is a zero (sparse.hpp:291)
    v = A.DeviceVector(n, dt, ctx).set_dense(xd)
    s = v.sparse()
    ei, ev = port.dense_to_sparse(xd)
    assert np.array_equal(s.indices, ei) and s.values.tobytes() == ev.tobytes()
    assert np.array_equal(v.bitmask().words, port.build_bitmask_dense(xd))
    assert v.nnz() == len(ei)
    # sparse -> dense, bitmask across the 63/64 word boundary
    v2 = A.DeviceVector(65, dt, ctx).set_sparse([0, 63, 64], np.array([1, 2, 3], dt))
    w = v2.bitmask().words
    assert w.tolist() == [1 | (1 << 63), 1]
    assert v2.dense().values.tolist() == [1] + [0] * 62 + [2, 3]
    # explicit zero stays a structural nonzero in the mask
    v3 = A.DeviceVector(10, dt, ctx).set_sparse([2, 4], np.array([0, 1], dt))
    assert v3.bitmask().words.tolist() == [(1 << 2) | (1 << 4)]


def test_effective_nnz_and_features(ctx, port):
    rows, cols, ro, ci, vals = synth.random_csr(800, 600, 0.02, seed=8)
    m = A.DualMatrix.from_csr(rows, cols, ro, ci, vals, ctx=ctx)
    co, ri, cv = port.csr_to_csc(rows, cols, ro, ci, vals)
    fm = port.matrix_features(rows, cols, ro)
    got = m.features()
    assert np.allclose(got, fm, rtol=1e-12, atol=0)
    for nx in (0, 1, 57, 600):
        xi, xv = synth.sparse_vector(cols, nx, seed=nx)
        assert A.effective_nnz(m, A.SparseVector(cols, xi, xv)) == port.effective_nnz(co, xi)
        f = A.features(m, A.SparseVector(cols, xi, xv))
        exp = np.concatenate([fm, port.vector_features_sparse(cols, co, xi)])
        assert np.allclose(f, exp, rtol=1e-12, atol=0)
    # dense input: nnz_x counts nonzero entries
    xd = np.zeros(cols)
    xd[[3, 7, 100]] = 1.0
    f = A.features(m, A.DenseVector(xd))
    assert np.allclose(f[9:], port.vector_features_dense(co, xd))


def test_selector_cascade_stub_bundles(ctx):
    rows, cols, ro, ci, vals = synth.random_csr(100, 100, 0.05, seed=1)
    m = A.DualMatrix.from_csr(rows, cols, ro, ci, vals, ctx=ctx)
    x = A.SparseVector(cols, [1, 5], [1.0, 2.0])
    # constant (SpMV, Direct, -) -> SpMV/Direct; write-back tree not evaluated
    k, used, nt = A.predict_kernel(m, x, A.SelectorBundle.constant(2, 0, 1))
    assert k.index() == 0 and nt == 2 and used == 0
    # (ColSpMSpV, LoadBalanced, Sort) -> that exact KernelId
    k, used, nt = A.predict_kernel(m, x, A.SelectorBundle.constant(0, 1, 1))
    assert k.name() == "col_lb_sort" and nt == 3
    # a real split on x_sparsity (feature 10): <= 0.05 -> ColSpMSpV else SpMV
    pat = {"feature": [10, -1, -1], "threshold": [0.05, 0, 0], "left": [1, -1, -1],
           "right": [2, -1, -1], "leaf": [0, 0, 2]}
    wl = {"feature": [-1], "threshold": [0.0], "left": [-1], "right": [-1], "leaf": [1]}
    wb = {"feature": [11, -1, -1], "threshold": [10.0, 0, 0], "left": [1, -1, -1],
          "right": [2, -1, -1], "leaf": [1, 1, 0]}
    b = A.SelectorBundle.from_trees([pat, wl, wb])
    k, used, _ = A.predict_kernel(m, x, b)
    assert k.index() == 7 and used == (1 << 10) | (1 << 11)  # lazy: only the features walked
    k, used, _ = A.predict_kernel(m, A.DenseVector(np.ones(cols)), b)
    assert k.index() == 1 and used == (1 << 10)
    out, kk = A.run_adaptive(m, x, b)
    assert kk.index() == 7


def test_execute_iteration_reports_and_forced_override(ctx, port):
    # forced override = each of the 8 KernelIds -> all within tolerance
    rows, cols, ro, ci, vals = synth.random_csr(400, 300, 0.03, seed=12)
    m = A.DualMatrix.from_csr(rows, cols, ro, ci, vals, ctx=ctx)
    xi, xv = synth.sparse_vector(cols, 30, seed=4)
    y_ref, bound = ref_and_bound(port, rows, ro, ci, vals, port.sparse_to_dense(cols, xi, xv))
    for k in range(8):
        out, rep = A.execute_iteration(m, A.SparseVector(cols, xi, xv), force_kernel=k)
        assert rep["kernel"].index() == k and rep["kernel_s"] > 0 and rep["convert_s"] >= 0
        assert_dense_close(out.dense().values, y_ref, bound, np.float64, f"execute k={k}")
    # empty sparse x -> zero output
    out, rep = A.execute_iteration(m, A.SparseVector(cols, [], []), bundle=A.SelectorBundle.load(
        __import__("paper_2006_16767_b200.selector", fromlist=["x"]).DEFAULT_PATH))
    assert not out.dense().values.any()
    with pytest.raises(A.InvalidArgument):  # untrained bundle without override
        A.execute_iteration(m, A.SparseVector(cols, xi, xv))


def test_run_trace_contracts(ctx):
    # identical vectors -> at most 1 switch; empty trace -> overhead 0;
    # an oracle-faithful stub (constant per density class) has regret 1.0 on its own timings
    rows, cols, ro, ci, vals = synth.random_csr(2000, 2000, 0.005, seed=3)
    m = A.DualMatrix.from_csr(rows, cols, ro, ci, vals, ctx=ctx)
    from paper_2006_16767_b200 import selector as S
    b = A.SelectorBundle.load(S.DEFAULT_PATH)
    xi, xv = synth.sparse_vector(cols, 20, seed=1)
    st = A.run_trace(m, [A.SparseVector(cols, xi, xv)] * 4, b)
    assert st["kernel_switches"] <= 1 and 0 <= st["overhead_fraction"] <= 1
    assert A.run_trace(m, [], b)["overhead_fraction"] == 0.0
    sparse = A.SparseVector(cols, xi, xv)
    dense = A.DenseVector(np.random.default_rng(0).uniform(-1, 1, cols))
    st = A.run_trace(m, [sparse, dense, sparse], force_kernel=6, oracle_times=[[2] * 6 + [1, 2]] * 3)
    assert st["regret"] == 1.0 and st["kernel_switches"] == 0


@pytest.mark.parametrize("semiring", [A.PLUS_TIMES, A.OR_AND, A.MIN_PLUS])
def test_bfs_levels_match_queue_bfs(ctx, port, semiring):
    # path graph 0-1-2-3 -> levels [0,1,2,3], 4 iterations
    ro = np.array([0, 1, 3, 5, 6])
    ci = np.array([1, 0, 2, 1, 3, 2])
    m = A.DualMatrix.from_csr(4, 4, ro, ci, None, dtype=np.float32, ctx=ctx)
    lv, reps = A.bfs(m, 0, semiring)
    assert lv.tolist() == [0, 1, 2, 3] and len(reps) == 4
    for seed, scale in ((1, 10), (2, 12)):
        n, _, ro, ci, vals = synth.rmat(scale, 8, seed=seed)
        m = A.DualMatrix.from_csr(n, n, ro, ci, None, dtype=np.float32, ctx=ctx)
        co, ri, _ = port.csr_to_csc(n, n, ro, ci, np.ones(len(ci)))
        exp, nl = port.bfs_queue(n, co, ri, 0)
        for forced in (-1, 1, 3, 4, 7):
            lv, reps = A.bfs(m, 0, semiring, force_kernel=forced)
            assert np.array_equal(lv, exp), (scale, forced)


def test_sort_reduce_pairs_known_answer(ctx):
    # [(2,1.0),(0,2.0),(2,3.0)] -> {0: 2.0, 2: 4.0}
    s = A.sort_reduce_pairs([2, 0, 2], np.array([1.0, 2.0, 3.0]), 3, ctx)
    assert s.indices.tolist() == [0, 2] and s.values.tolist() == [2.0, 4.0]
    # exact-zero sums dropped (kernels.hpp:331)
    s = A.sort_reduce_pairs([1, 1, 0], np.array([1.5, -1.5, 2.0]), 2, ctx)
    assert s.indices.tolist() == [0]


def test_errors_map_to_reference_exceptions(ctx, tmp_path):
    m = A.DualMatrix.from_csr(2, 2, [0, 1, 2], [0, 1], [1.0, 2.0], ctx=ctx)
    with pytest.raises(A.InvalidArgument):
        A.run_kernel(m, 0, A.DenseVector(np.ones(3)))
    with pytest.raises(A.InvalidArgument):
        A.run_kernel(m, 0, A.OperandViews(sparse=A.SparseVector(2, [0], [1.0])))
    with pytest.raises(A.InvalidArgument):
        A.DualMatrix.from_csr(2, 2, [0, 2, 2], [1, 0], [1.0, 2.0], ctx=ctx)  # unsorted columns
    with pytest.raises(A.InvalidArgument):
        A.run_kernel(m, 4, A.SparseVector(2, [1, 0], [1.0, 1.0]))
    p = tmp_path / "bad.mtx"
    p.write_text("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n")
    with pytest.raises(A.ParseError) as e:
        A.load_matrix(p, ctx=ctx)
    assert e.value.line == 3
    with pytest.raises(A.FormatError):
        A.load_matrix(tmp_path / "missing.mtx", ctx=ctx)


def test_matrix_market_and_binary_round_trip(ctx, tmp_path):
    rows, cols, ro, ci, vals = synth.random_csr(50, 40, 0.1, seed=2)
    m = A.DualMatrix.from_csr(rows, cols, ro, ci, vals, ctx=ctx)
    p = tmp_path / "a.mtx"
    m.write_matrix_market(p)
    m2 = A.load_matrix(p, ctx=ctx)
    a, b = m.download(), m2.download()
    for u, v in zip(a, b):
        assert u.tobytes() == v.tobytes()
    pb = tmp_path / "a.bin"
    m.save_binary(pb)
    m3 = A.load_matrix(pb, ctx=ctx)
    for u, v in zip(a, m3.download()):
        assert u.tobytes() == v.tobytes()
    with pytest.raises(A.FormatError):
        A.load_matrix(pb, dtype=np.float32, ctx=ctx)  # width mismatch
    # symmetric + pattern + duplicates
    q = tmp_path / "s.mtx"
    q.write_text("%%MatrixMarket matrix coordinate pattern symmetric\n3 3 3\n2 1\n3 3\n2 1\n")
    s = A.load_matrix(q, ctx=ctx).download()
    assert s[0].tolist() == [0, 1, 2, 3] and s[1].tolist() == [1, 0, 2] and s[2].tolist() == [2.0, 2.0, 1.0]


# ---- row-bin execution of K0/K2 (kernels_binned.cu) ----------------------------
# Overrides exercise many bins (bin_rows), bins split into several tiles whose
# partial y segments are combined with atomics (bin_tile_nnz), and empty bins.
BIN_CFGS = [dict(), dict(bin_rows=7), dict(bin_rows=64, bin_tile_nnz=5), dict(bin_tile_nnz=1000),
            dict(bin_cluster=2), dict(bin_rows=64, bin_cluster=2), dict(bin_rows=9, bin_tile_nnz=7, bin_cluster=2),
            dict(bin_cluster=1), dict(bin_panel_kib=1), dict(bin_panel_kib=1, bin_tile_nnz=500),
            dict(bin_panel_kib=1, bin_rows=64), dict(bin_panel_kib=-1)]


@pytest.mark.parametrize("dt", DTYPES, ids=["f64", "f32"])
@pytest.mark.parametrize("name,case", CASES, ids=[c[0] for c in CASES])
def test_binned_row_layout_vs_oracle(ctx, port, name, case, dt):
    rows, cols, ro, ci, vals = case
    vals = np.asarray(vals, dt)
    m = A.DualMatrix.from_csr(rows, cols, ro, ci, vals, ctx=ctx)
    for nx in sorted({0, 1, max(1, cols // 3), cols}):
        xi, xv = synth.sparse_vector(cols, nx, seed=nx + 5, dtype=dt)
        xd = port.sparse_to_dense(cols, xi, xv)
        y_ref, bound = ref_and_bound(port, rows, ro, ci, vals, xd)
        for cfg in BIN_CFGS:
            for k in (0, 2):
                out = A.run_kernel(m, k, A.DenseVector(xd), A.KernelConfig(row_layout=2, **cfg))
                what = f"binned {name} k={k} nnz_x={nx} {cfg} {np.dtype(dt).name}"
                assert_dense_close(out.dense().values, y_ref, bound, dt, what)
                s = out.sparse()
                assert_sparse_match(s.indices, s.values, y_ref, bound, dt, what)


@pytest.mark.parametrize("dt", DTYPES, ids=["f64", "f32"])
def test_binned_multi_chunk_and_semirings(ctx, port, dt):
    # > 2^17 (f32) / 2^18 (f64) columns: entries of a bin span several column
    # chunks.  PLUS_TIMES against the oracle; OR_AND / MIN_PLUS are order-free
    # and must equal the CSR execution bit for bit.
    rows, cols, ro, ci, vals = synth.random_csr(3000, 600_000, 0.0001, seed=21, dtype=dt)
    m = A.DualMatrix.from_csr(rows, cols, ro, ci, vals, ctx=ctx)
    for nx in (1, 3000, cols // 2, cols):
        xi, xv = synth.sparse_vector(cols, nx, seed=nx, dtype=dt)
        xd = port.sparse_to_dense(cols, xi, xv)
        y_ref, bound = ref_and_bound(port, rows, ro, ci, vals, xd)
        for cfg in BIN_CFGS:
            for k in (0, 2):
                c2 = A.KernelConfig(row_layout=2, **cfg)
                out = A.run_kernel(m, k, A.DenseVector(xd), c2)
                assert_dense_close(out.dense().values, y_ref, bound, dt, f"multichunk k={k} {cfg}")
                for sr in (A.OR_AND, A.MIN_PLUS):
                    xs = A.SparseVector(cols, xi, xv)
                    b = A.run_kernel(m, k, xs, A.KernelConfig(semiring=sr, row_layout=2, **cfg))
                    c = A.run_kernel(m, k, xs, A.KernelConfig(semiring=sr, row_layout=1))
                    assert b.dense().values.tobytes() == c.dense().values.tobytes(), (sr, k, cfg)


def test_binned_auto_layout_large_uniform(ctx, port):
    # auto picks the row bins for a scattered matrix (mean gather distance
    # >> 64 KiB of x) with >= 2^20 nonzeros; results match the oracle
    rows, cols, ro, ci, vals = synth.random_csr(300_000, 300_000, 12 / 300_000, seed=5, dtype=np.float32)
    m = A.DualMatrix.from_csr(rows, cols, ro, ci, vals, ctx=ctx)
    assert m.gather_spread() * 4 > 65536
    xd = np.random.default_rng(1).uniform(-1, 1, cols).astype(np.float32)
    y_ref, bound = ref_and_bound(port, rows, ro, ci, vals, xd)
    for layout in (0, 1, 2):
        out = A.run_kernel(m, 0, A.DenseVector(xd), A.KernelConfig(row_layout=layout))
        assert_dense_close(out.dense().values, y_ref, bound, np.float32, f"layout={layout}")


@pytest.mark.parametrize("dt", DTYPES, ids=["f64", "f32"])
def test_binned_heavy_rows(ctx, port, dt):
    # rows far above the bin's warp window (degree > 4096) run from the CSR as
    # segments; light rows stay in the bins.  Plus-times vs the oracle,
    # OR_AND / MIN_PLUS bitwise vs the CSR execution, masked K2 included.
    rng = np.random.default_rng(9)
    rows, cols = 5000, 60000
    deg = rng.integers(0, 8, size=rows)
    deg[[0, 17, 2500, 4999]] = [30000, 9000, 4097, 20000]
    ro = np.zeros(rows + 1, np.int64)
    ro[1:] = np.cumsum(deg)
    ci = np.concatenate([np.sort(rng.choice(cols, size=d, replace=False)) for d in deg]).astype(np.int64)
    vals = rng.uniform(-1, 1, len(ci)).astype(dt)
    m = A.DualMatrix.from_csr(rows, cols, ro, ci, vals, ctx=ctx)
    for nx in (1, 700, cols // 2, cols):
        xi, xv = synth.sparse_vector(cols, nx, seed=nx + 1, dtype=dt)
        xd = port.sparse_to_dense(cols, xi, xv)
        y_ref, bound = ref_and_bound(port, rows, ro, ci, vals, xd)
        for cfg in (dict(), dict(bin_cluster=2), dict(bin_rows=100, bin_tile_nnz=300)):
            for k in (0, 2):
                out = A.run_kernel(m, k, A.DenseVector(xd), A.KernelConfig(row_layout=2, **cfg))
                assert_dense_close(out.dense().values, y_ref, bound, dt, f"heavy k={k} nx={nx} {cfg}")
                xs = A.SparseVector(cols, xi, xv)
                for sr in (A.OR_AND, A.MIN_PLUS):
                    b = A.run_kernel(m, k, xs, A.KernelConfig(semiring=sr, row_layout=2, **cfg))
                    c = A.run_kernel(m, k, xs, A.KernelConfig(semiring=sr, row_layout=1))
                    assert b.dense().values.tobytes() == c.dense().values.tobytes(), (sr, k, cfg)


@pytest.mark.parametrize("dt", DTYPES, ids=["f64", "f32"])
def test_atomic_output_reuse(ctx, port, dt):
    # one MultiplyOutput reused across supports, kernels, semirings and a
    # second matrix: every result matches the oracle (no stale rows).
    rows, cols, ro, ci, vals = synth.random_csr(20000, 15000, 0.0004, seed=31, dtype=dt)
    m = A.DualMatrix.from_csr(rows, cols, ro, ci, vals, ctx=ctx)
    r2, c2, ro2, ci2, v2 = synth.random_csr(20000, 15000, 0.0003, seed=32, dtype=dt)
    m2 = A.DualMatrix.from_csr(r2, c2, ro2, ci2, v2, ctx=ctx)
    out = A.MultiplyOutput(ctx)
    seq = [(m, 4, 3), (m, 4, 5), (m, 6, 2), (m, 4, 0), (m, 6, 40), (m, 0, 15000), (m, 4, 1), (m2, 4, 7),
           (m, 4, 9), (m, 5, 4), (m, 4, 3), (m, 6, 3000), (m, 4, 2)]
    for i, (mat, k, nx) in enumerate(seq):
        rr, cc, roo, cii, vv = (rows, cols, ro, ci, vals) if mat is m else (r2, c2, ro2, ci2, v2)
        xi, xv = synth.sparse_vector(cc, nx, seed=100 + i, dtype=dt)
        xd = port.sparse_to_dense(cc, xi, xv)
        y_ref, bound = ref_and_bound(port, rr, roo, cii, vv, xd)
        x = A.SparseVector(cc, xi, xv) if k >= 4 else A.DenseVector(xd)
        y = A.run_kernel(mat, k, x, out=out)
        assert_dense_close(y.dense().values, y_ref, bound, dt, f"step {i} k={k} nx={nx}")
    # min-plus after plus-times into the same buffer: identity differs (+inf)
    xi, xv = synth.sparse_vector(cols, 5, seed=7, dtype=dt)
    a = A.run_kernel(m, 4, A.SparseVector(cols, xi, xv), A.KernelConfig(semiring=A.MIN_PLUS), out=out)
    b = A.run_kernel(m, 4, A.SparseVector(cols, xi, xv), A.KernelConfig(semiring=A.MIN_PLUS))
    assert a.dense().values.tobytes() == b.dense().values.tobytes()


@pytest.mark.parametrize("dt", DTYPES, ids=["f64", "f32"])
def test_binned_skewed_rows_in_heavy_bins(ctx, port, dt):
    """A power-law matrix (Gini > 0.5, rows above the 256 cut): its heavy rows
    leave the light bins for the heavy bins (kernels_binned.cu: slot -> row
    map, the light bins skip them at write-back) -- every density, K0 and K2,
    against the oracle; OR_AND and MIN_PLUS bit-equal to the CSR run."""
    rows, cols, ro, ci, vals = synth.rmat(15, 32, seed=5, values="uniform")
    vals = np.asarray(vals, dt)
    assert np.diff(ro).max() > 1024
    m = A.DualMatrix.from_csr(rows, cols, ro, ci, vals, ctx=ctx)
    assert m.features()[8] > 0.5
    for nx in (1, cols // 50, cols // 2, cols):
        xi, xv = synth.sparse_vector(cols, nx, seed=nx + 9, dtype=dt)
        xd = port.sparse_to_dense(cols, xi, xv)
        y_ref, bound = ref_and_bound(port, rows, ro, ci, vals, xd)
        for k in (0, 2):
            out = A.run_kernel(m, k, A.DenseVector(xd), A.KernelConfig(row_layout=2))
            assert_dense_close(out.dense().values, y_ref, bound, dt, f"rmat binned k={k} nnz_x={nx}")
            xs = A.SparseVector(cols, xi, xv)
            b = A.run_kernel(m, k, xs, A.KernelConfig(semiring=A.OR_AND, row_layout=2))
            c = A.run_kernel(m, k, xs, A.KernelConfig(semiring=A.OR_AND, row_layout=1))
            assert b.dense().values.tobytes() == c.dense().values.tobytes(), (k, nx)
            b = A.run_kernel(m, k, xs, A.KernelConfig(semiring=A.MIN_PLUS, row_layout=2))
            c = A.run_kernel(m, k, xs, A.KernelConfig(semiring=A.MIN_PLUS, row_layout=1))
            assert b.dense().values.tobytes() == c.dense().values.tobytes(), ("min_plus", k, nx)


@pytest.mark.parametrize("dt", DTYPES, ids=["f64", "f32"])
def test_kernel_counters(port, dt):
    """KernelCounters (kernels.hpp:106-111) as the reference's counter build
    records them (kernels.hpp:281-283, 447-511): values_read = nnz on the SpMV
    path, nnz_s on the row-SpMSpV and column paths (every entry consumed once
    -- no kernel reads a value twice or skips one); pairs_emitted = nnz_s on
    the sort write-back; cas_retries 0.  CSR and row-bin executions, the
    private-accumulator variant, the small and the radix sort paths."""
    ctx = A.Context(0)
    ctx.set_counters(True)
    for rows, cols, dens, seed in ((700, 500, 0.02, 4), (6000, 5000, 0.004, 5)):
        r_, c_, ro, ci, vals = synth.random_csr(rows, cols, dens, seed=seed, dtype=dt)
        m = A.DualMatrix.from_csr(rows, cols, ro, ci, vals, ctx=ctx)
        nnz = int(ro[-1])
        co = np.bincount(ci, minlength=cols)
        for nx in (1, 30, cols // 3, cols):
            xi, xv = synth.sparse_vector(cols, nx, seed=nx, dtype=dt)
            nnz_s = int(co[xi].sum())
            xd = port.sparse_to_dense(cols, xi, xv)
            cfgs = [A.KernelConfig(), A.KernelConfig(row_layout=2), A.KernelConfig(atomic_private_accumulators=1)]
            for cfg in cfgs:
                for k in range(8):
                    x = A.SparseVector(cols, xi, xv) if k >= 4 else A.DenseVector(xd)
                    out = A.run_kernel(m, k, x, cfg, out=A.MultiplyOutput(ctx))
                    c = out.counters()
                    want = nnz if k <= 1 else nnz_s
                    assert c["values_read"] == want, (k, nx, cfg._c().row_layout, c)
                    assert c["pairs_emitted"] == (nnz_s if k in (5, 7) else 0), (k, nx, c)
                    assert c["cas_retries"] == 0
    ctx.set_counters(False)
    out = A.run_kernel(m, 0, A.DenseVector(xd), out=A.MultiplyOutput(ctx))
    with pytest.raises(A.InvalidArgument):
        out.counters()


def _random_tree(rng, depth, feats, nclasses=3):
    """A random full tree (SelectorBundle.from_trees dict) splitting on `feats`."""
    feature, threshold, left, right, leaf = [], [], [], [], []

    def node(d):
        i = len(feature)
        feature.append(-1), threshold.append(0.0), left.append(-1), right.append(-1), leaf.append(0)
        if d == depth:
            leaf[i] = int(rng.integers(0, nclasses))
            return i
        f = int(rng.choice(feats))
        feature[i] = f
        threshold[i] = float({11: rng.uniform(0, 4000), 12: rng.uniform(0, 0.4), 10: rng.uniform(0, 0.3),
                              9: rng.uniform(0, 300), 2: rng.uniform(0, 40000), 5: rng.uniform(0, 30)}[f])
        left[i] = node(d + 1)
        right[i] = node(d + 1)
        return i

    node(0)
    return {"feature": feature, "threshold": threshold, "left": left, "right": right, "leaf": leaf}


@pytest.mark.gpu
def test_selector_degree_bounds_route_like_exact_features(ctx):
    """nnz_s / m_sparsity splits settled on the column-degree bounds (selector.cpp)
    route exactly as the computed features would, and skip the device reduction
    when the bound interval is on one side."""
    rng = np.random.default_rng(5)
    for mat_seed, (rows, cols, dens) in enumerate([(3000, 2000, 0.004), (500, 4000, 0.01)]):
        r, c, ro, ci, vals = synth.random_csr(rows, cols, dens, seed=mat_seed + 40)
        m = A.DualMatrix.from_csr(r, c, ro, ci, vals, ctx=ctx)
        for t in range(25):
            # the workload tree reads matrix features only
            trees = [_random_tree(rng, 3, [9, 10, 11, 12]), _random_tree(rng, 2, [2, 5], 2),
                     _random_tree(rng, 3, [9, 10, 11, 12], 2)]
            b = A.SelectorBundle.from_trees(trees)
            for nx in (1, 3, 20, 200, cols // 2, cols):
                xi = np.sort(rng.choice(cols, nx, replace=False))
                xv = rng.uniform(-1, 1, nx)
                fresh = A.DeviceVector(cols, np.float64, ctx)
                fresh.set_sparse(xi, xv)
                k_pruned, used_p, _ = A.predict_kernel(m, fresh, b)
                exact = A.DeviceVector(cols, np.float64, ctx)
                exact.set_sparse(xi, xv)
                A.features(m, exact, (1 << 11) | (1 << 12))  # caches the exact nnz_s
                k_exact, used_e, _ = A.predict_kernel(m, exact, b)
                assert k_pruned.index() == k_exact.index(), (mat_seed, t, nx)
                assert used_p == used_e
    # a split far above any possible nnz_s is settled without a launch
    r, c, ro, ci, vals = synth.random_csr(2000, 2000, 0.005, seed=3)
    m = A.DualMatrix.from_csr(r, c, ro, ci, vals, ctx=ctx)
    pat = {"feature": [12, -1, -1], "threshold": [0.5, 0, 0], "left": [1, -1, -1], "right": [2, -1, -1],
           "leaf": [0, 0, 2]}
    one = {"feature": [-1], "threshold": [0.0], "left": [-1], "right": [-1], "leaf": [0]}
    b = A.SelectorBundle.from_trees([pat, one, one])
    x = A.DeviceVector(c, np.float64, ctx)
    x.set_sparse(np.array([4, 9]), np.array([1.0, 2.0]))
    ctx.synchronize()
    l0 = ctx.launches
    k, used, _ = A.predict_kernel(m, x, b)
    assert k.index() == 4 and used == 1 << 12 and ctx.launches == l0


@pytest.mark.gpu
def test_selector_schema2_runtime_matches_host_mirror(ctx):
    """The shipped schema-2 bundle: the runtime's cascade (selector.cpp) and the
    host mirror (selector.predict) pick the same kernel on the same features."""
    from paper_2006_16767_b200 import selector as S
    path = S.DEFAULT_PATH.parent / "b200_bundle_v2.txt"
    trees = S.read_bundle(path)
    assert "workload_col" in trees
    b = A.SelectorBundle.load(path)
    rng = np.random.default_rng(3)
    for seed, (rows, cols, dens) in enumerate([(4000, 4000, 0.002), (20000, 3000, 0.001), (3000, 30000, 0.002)]):
        r, c, ro, ci, vals = synth.random_csr(rows, cols, dens, seed=seed + 60)
        m = A.DualMatrix.from_csr(r, c, ro, ci, vals, ctx=ctx)
        for nx in (1, 10, 100, 1000, cols // 3, cols):
            xi = np.sort(rng.choice(cols, nx, replace=False))
            x = A.SparseVector(cols, xi, rng.uniform(-1, 1, nx))
            f = A.features(m, x)
            k, _, _ = A.predict_kernel(m, x, b)
            assert k.index() == S.predict(trees, f), (seed, nx)


@pytest.mark.parametrize("nx_frac", [1.0, 0.3])
def test_subnormal_products_fp32(ctx, port, nx_frac):
    # the hardware float reduction (REDG.E.ADD.F32.FTZ)
    # flushes subnormals; the reference's float sums keep them.  Entries and x
    # of ~1e-20 give products of ~1e-40 (subnormal in fp32): every kernel must
    # sum them like the reference.  Tolerance: the fp32 rtol of the row bound
    # plus the absolute rounding of subnormal arithmetic (half an ulp of
    # 2^-149 per product and per add).
    rows, cols, ro, ci, vals = synth.random_csr(3000, 2500, 0.004, seed=11, dtype=np.float32)
    rng = np.random.default_rng(5)
    vals = (rng.uniform(1.0, 2.0, len(vals)) * 1e-20).astype(np.float32)
    m = A.DualMatrix.from_csr(rows, cols, ro, ci, vals, ctx=ctx)
    nx = max(1, int(cols * nx_frac))
    xi = np.sort(rng.choice(cols, nx, replace=False)).astype(np.int64)
    xv = (rng.uniform(1.0, 2.0, nx) * 1e-20).astype(np.float32)
    xd = port.sparse_to_dense(cols, xi, xv)
    y_ref, bound = ref_and_bound(port, rows, ro, ci, np.asarray(vals, np.float64),
                                 np.asarray(xd, np.float32).astype(np.float64))
    assert 0 < np.max(np.abs(y_ref)) < 1.17e-38  # the row sums themselves are subnormal
    deg = np.diff(ro)
    allowed = 1e-5 * bound + (2 * deg + 1) * 2.0 ** -149
    for k in range(8):
        x = A.SparseVector(cols, xi, xv) if k >= 4 else A.DenseVector(np.asarray(xd, np.float32))
        y = np.asarray(A.run_kernel(m, k, x).dense().values, np.float64)
        bad = np.abs(y - y_ref) > allowed
        assert not bad.any(), (f"k={k}: {int(bad.sum())} rows flushed/off, e.g. row {int(np.argmax(bad))} "
                               f"y={y[np.argmax(bad)]!r} ref={y_ref[np.argmax(bad)]!r}")

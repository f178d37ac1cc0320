"""GPU parity at BASELINE.json's full sizes: the C2 matrix
(uniform 4M x 4M, 2^26 draws, fp32) against the C oracle at the bench's x
sparsities for all eight kernels, plus size-independent properties --
linearity y(x1 + x2) = y(x1) + y(x2), sparse index sets equal to the
structural support, and the adaptive choice agreeing with its forced kernel
with its forced kernel -- and BFS levels on an R-MAT graph of the C3 class
(scale 20 here to keep the suite short; scale 22 is checked level for level
by tools/bfs_bench.py, profiles/r01_bfs_rmat22.json "levels_match").  The
oracle runs single-threaded C at these sizes in about a second per call.
"""
import numpy as np
import pytest

from paper_2006_16767_b200 import adaspmv as A
from paper_2006_16767_b200 import selector as S
from paper_2006_16767_b200 import synth
from tests.util import assert_dense_close, assert_sparse_match, ref_and_bound

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c2(ctx):
    rows, cols, ro, ci, vals = synth.uniform_random(1 << 22, 1 << 26, seed=1, dtype=np.float32)
    m = A.DualMatrix.from_csr(rows, cols, ro, ci, vals, ctx=ctx)
    return rows, cols, ro, ci, vals, m


@pytest.mark.parametrize("sparsity", [1e-5, 1e-2, 0.5, 1.0])
def test_c2_all_kernels_vs_oracle(c2, port, sparsity):
    rows, cols, ro, ci, vals, m = c2
    nx = max(1, int(round(sparsity * cols)))
    xi, xv = synth.sparse_vector(cols, nx, seed=1000 + nx % 997, dtype=np.float32)
    xd = port.sparse_to_dense(cols, xi, xv)
    y_ref, bound = ref_and_bound(port, rows, ro, ci, vals, xd)
    struct = None
    if nx < 5000:  # structural support = rows of the support's columns
        co, ri, _ = port.csr_to_csc(rows, cols, ro, ci, np.ones(len(ci), np.float32))
        struct = set(np.concatenate([ri[co[j]:co[j + 1]] for j in xi]).tolist())
    for k in range(8):
        if nx == cols and k in (5, 7):
            continue  # sort write-back of 67 M pairs: covered at 50 %
        x = A.SparseVector(cols, xi, xv) if k >= 4 else A.DenseVector(xd)
        out = A.run_kernel(m, k, x)
        what = f"C2 x={sparsity} k={k}"
        assert_dense_close(out.dense().values, y_ref, bound, np.float32, what)
        if k in (5, 7):
            s = out.sparse()
            assert_sparse_match(s.indices, s.values, y_ref, bound, np.float32, what)
            if struct is not None:
                assert set(s.indices.tolist()) <= struct


def test_c2_linearity_and_adaptive_agreement(c2):
    # y(x1 + x2) = y(x1) + y(x2) within fp32 rounding of the three sums (disjoint supports)
    rows, cols, ro, ci, vals, m = c2
    rng = np.random.default_rng(3)
    perm = rng.permutation(cols)
    s1, s2 = np.sort(perm[: cols // 3]), np.sort(perm[cols // 3: 2 * cols // 3])
    x1 = np.zeros(cols, np.float32)
    x2 = np.zeros(cols, np.float32)
    x1[s1] = rng.uniform(-1, 1, len(s1))
    x2[s2] = rng.uniform(-1, 1, len(s2))
    bound = np.abs(A.run_kernel(A_abs(m, c2), 0, A.DenseVector(np.abs(x1) + np.abs(x2))).dense().values)
    for k in (0, 1, 4, 6):
        y12 = A.run_kernel(m, k, A.DenseVector(x1 + x2)).dense().values.astype(np.float64)
        y1 = A.run_kernel(m, k, A.DenseVector(x1)).dense().values.astype(np.float64)
        y2 = A.run_kernel(m, k, A.DenseVector(x2)).dense().values.astype(np.float64)
        assert np.all(np.abs(y12 - (y1 + y2)) <= 3e-5 * bound + 1e-30), k
    # adaptive == its forced kernel: bitwise for the deterministic kernels
    # (spmv_lb, the sort write-backs), within tolerance for the atomic ones
    # (row bins accumulate in shared memory, K4/K6 in L2)
    bundle = A.SelectorBundle.load(S.DEFAULT_PATH)
    for nx in (42, 41943, cols):
        xi, xv = synth.sparse_vector(cols, nx, seed=nx, dtype=np.float32)
        y, kid = A.run_adaptive(m, A.SparseVector(cols, xi, xv), bundle)
        z = A.run_kernel(m, kid.index(), A.SparseVector(cols, xi, xv))
        a, b = y.dense().values, z.dense().values
        if kid.index() in (1, 5, 7):
            assert a.tobytes() == b.tobytes(), kid.name()
        else:
            bx = A.run_kernel(A_abs(m, c2), 0, A.SparseVector(cols, xi, np.abs(xv))).dense().values
            assert np.all(np.abs(a.astype(np.float64) - b) <= 2e-5 * bx + 1e-30), kid.name()


_ABS = {}


def A_abs(m, c2):
    """|A| as a device matrix (bound for the linearity check), built once."""
    if "m" not in _ABS:
        rows, cols, ro, ci, vals, _ = c2
        _ABS["m"] = A.DualMatrix.from_csr(rows, cols, ro, ci, np.abs(vals), ctx=m.ctx)
    return _ABS["m"]


def test_c2_batch_sweep_vs_oracle(c2, port):
    """The e2e path of bench.py: one adaptive_run_batch over the C2 sweep's host
    vectors (int64-indexed sparse points, a dense 100 % point), results in
    their smaller form, each checked against the oracle."""
    rows, cols, ro, ci, vals, m = c2
    bundle = A.SelectorBundle.load(S.DEFAULT_PATH)
    xs, dense = [], []
    for i, sp in enumerate((1e-5, 1e-3, 0.1, 0.5, 1.0)):
        nx = max(1, int(round(sp * cols)))
        xi, xv = synth.sparse_vector(cols, nx, seed=77 + i, dtype=np.float32)
        d = np.zeros(cols, np.float32)
        d[xi] = xv
        dense.append(d)
        xs.append(d if nx == cols else (xi, xv))
    res = A.run_batch(m, xs, bundle=bundle, form=A.RESULT_AUTO, lanes=3)
    for i, (r, d) in enumerate(zip(res, dense)):
        y_ref, bound = ref_and_bound(port, rows, ro, ci, vals, d)
        what = f"batch op {i} kernel {r.kernel.name()}"
        if r.is_sparse:
            assert_sparse_match(r.sparse.indices, r.sparse.values, y_ref, bound, np.float32, what)
        else:
            assert_dense_close(r.dense.values, y_ref, bound, np.float32, what)


def test_c3_class_bfs_levels(ctx, port):
    n, _, ro, ci, _ = synth.rmat(20, 16, seed=2)
    m = A.DualMatrix.from_csr(n, n, ro, ci, None, dtype=np.float32, ctx=ctx)
    co, ri, _ = port.csr_to_csc(n, n, ro, ci, np.ones(len(ci), np.float32))
    exp, nl = port.bfs_queue(n, co, ri, 0)
    for sr in (A.OR_AND, A.MIN_PLUS):
        for forced in (-1, 3, 6):
            lv, reps = A.bfs(m, 0, sr, force_kernel=forced)
            assert np.array_equal(lv, exp), (sr, forced)
            assert len(reps) == nl


@pytest.mark.parametrize("sparsity", [0.01, 1.0])
def test_c1_laplacian_fp64_all_kernels_vs_oracle(ctx, port, sparsity):
    """configs[0]: the 2-D 5-point Laplacian on a 1000 x 1000 grid (10^6 rows,
    4,996,000 nnz, fp64) at x = 100 % (SpMV) and 1 % (SpMSpV), every kernel
    against the oracle at the fp64 tolerance (1e-12 of |A||x|).  x is random
    (an all-ones x would cancel exactly on the interior rows)."""
    rows, cols, ro, ci, vals = synth.laplacian_2d(1000, dtype=np.float64)
    assert rows == 10 ** 6 and int(ro[-1]) == 4_996_000
    m = A.DualMatrix.from_csr(rows, cols, ro, ci, vals, ctx=ctx)
    nx = int(round(sparsity * cols))
    xi, xv = synth.sparse_vector(cols, nx, seed=7, dtype=np.float64)
    xd = port.sparse_to_dense(cols, xi, xv)
    y_ref, bound = ref_and_bound(port, rows, ro, ci, vals, xd)
    for k in range(8):
        x = A.SparseVector(cols, xi, xv) if k >= 4 else A.DenseVector(xd)
        out = A.run_kernel(m, k, x)
        assert_dense_close(out.dense().values, y_ref, bound, np.float64, f"C1 x={sparsity} k={k}")
        if k in (5, 7):
            s = out.sparse()
            assert_sparse_match(s.indices, s.values, y_ref, bound, np.float64, f"C1 sparse k={k}")

"""Incremental PageRank: the oracle against SPEC's known
answers and dense power iteration (CPU), and the CUDA driver against the
oracle through the C-ABI (GPU).  SPEC-only: no reference code exists, so the
oracle is pinned by SPEC's examples and the dense power-iteration identity
(rank = sum_k (dP)^k (1/n) = (I - dP)^-1 (1/n)) only."""
import numpy as np
import pytest

from paper_2006_16767_b200 import synth


def _sym_graph(n, p, seed):
    rng = np.random.default_rng(seed)
    a = rng.random((n, n)) < p
    a = np.triu(a, 1)
    a = a | a.T
    return a


def _csr_csc(a):
    n = a.shape[0]
    r, c = np.nonzero(a)
    ro = np.zeros(n + 1, np.int64)
    np.add.at(ro, r + 1, 1)
    ro = np.cumsum(ro)
    rt, ct = np.nonzero(a.T)  # CSC of a = CSR of a.T
    co = np.zeros(n + 1, np.int64)
    np.add.at(co, rt + 1, 1)
    co = np.cumsum(co)
    return ro, c.astype(np.int64), co, ct.astype(np.int64)


def _dense_power(a, d, iters=2000):
    """rank = sum_k (d P)^k (1/n), P = A^T column-normalised by
    out-degree (row length of A): P[j, i] = a[i, j] / outdeg(i)."""
    n = a.shape[0]
    at = a.T
    deg = at.sum(axis=0).astype(np.float64)  # = out-degree of each source i
    P = np.where(deg > 0, at / np.maximum(deg, 1), 0.0)
    v = np.full(n, 1.0 / n)
    r = v.copy()
    for _ in range(iters):
        r = v + d * P @ r
    return r


def test_oracle_spec_examples(port):
    # 2-vertex symmetric pair -> equal ranks
    a = np.array([[0, 1], [1, 0]], bool)
    ro, ci, co, ri = _csr_csc(a)
    r, it = port.pagerank_incremental(2, ro, ci, 0.85, 1e-6, 300)
    assert r[0] == r[1] and it > 1
    # 3-vertex chain -> middle strictly largest, matches dense oracle
    a = np.array([[0, 1, 0], [1, 0, 1], [0, 1, 0]], bool)
    ro, ci, co, ri = _csr_csc(a)
    r, _ = port.pagerank_incremental(3, ro, ci, 0.85, 0.0, 10000)
    assert r[1] > r[0] and r[1] > r[2]
    assert np.abs(r - _dense_power(a, 0.85)).sum() <= 1e-8


@pytest.mark.parametrize("seed", range(6))
def test_oracle_prune0_is_dense_power_iteration(port, seed):
    # prune = 0, many iterations -> dense power iteration, 1e-8 in L1, n <= 100
    n = 20 + 15 * seed
    a = _sym_graph(n, 0.08, seed)
    a[0, :] = a[:, 0] = False  # a dangling (isolated) vertex: propagates nothing
    ro, ci, co, ri = _csr_csc(a)
    r, it = port.pagerank_incremental(n, ro, ci, 0.85, 0.0, 100000)
    assert np.abs(r - _dense_power(a, 0.85)).sum() <= 1e-8
    # pruning bound: every iteration drops < n*prune of delta mass, each unit of
    # which would have grown to at most 1/(1-d) (P column-substochastic).
    # SPEC.md:500 states n*prune/(1-d) without the iteration factor; that is
    # not a bound (exceeded by 1.3x on these graphs), so the test uses the
    # provable one.
    rp, itp = port.pagerank_incremental(n, ro, ci, 0.85, 1e-4, 300)
    assert 0 < rp.sum() <= r.sum() and itp <= it
    assert np.abs(rp - r).sum() <= itp * n * 1e-4 / 0.15 + 1e-12


def _directed_graph(n, p, seed):
    rng = np.random.default_rng(seed)
    a = rng.random((n, n)) < p
    np.fill_diagonal(a, False)
    a[1, :] = False  # a dangling source (no out-edges)
    return a


@pytest.mark.parametrize("seed", range(3))
def test_oracle_directed_orientation(port, seed):
    # SPEC.md:500 on a directed graph: mass moves along A's edges i -> j
    # (delta' = d * A^T_colnorm * delta); a symmetric graph cannot tell the
    # two orientations apart
    n = 40 + 10 * seed
    a = _directed_graph(n, 0.1, seed)
    ro, ci, co, ri = _csr_csc(a)
    r, _ = port.pagerank_incremental(n, ro, ci, 0.85, 0.0, 100000)
    assert np.abs(r - _dense_power(a, 0.85)).sum() <= 1e-8
    # the opposite orientation is a different answer
    assert np.abs(r - _dense_power(a.T, 0.85)).sum() > 1e-3


def test_oracle_max_iters_counts_multiplies(port):
    a = _sym_graph(30, 0.2, 3)
    ro, ci, _, _ = _csr_csc(a)
    r0, it0 = port.pagerank_incremental(30, ro, ci, 0.85, 0.0, 0)
    assert it0 == 0 and not r0.any()
    r1, it1 = port.pagerank_incremental(30, ro, ci, 0.85, 0.0, 1)
    assert it1 == 1 and np.all(r1 == 1.0 / 30)


# ---------------------------------------------------------------------------
# GPU: the CUDA driver vs the oracle, all kernels + adaptive policies
# ---------------------------------------------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("dt", [np.float64, np.float32], ids=["f64", "f32"])
def test_gpu_pagerank_matches_oracle(ctx, port, dt):
    from paper_2006_16767_b200 import adaspmv as A
    n, _, ro, ci, _ = synth.rmat(11, 8, seed=4)
    m = A.DualMatrix.from_csr(n, n, ro, ci, None, dtype=dt, ctx=ctx)
    for prune in (1e-7, 0.0):
        exp, it = port.pagerank_incremental(n, ro, ci, 0.85, prune, 60)
        # rank entries are sums of positive terms: relative 1e-12 (f64) / 1e-5 (f32)
        # per vertex, plus the pruning-boundary slack of 2 deltas of size <= prune
        rtol = 1e-11 if dt == np.float64 else 2e-5
        for forced in (-1, 0, 1, 2, 3, 4, 5, 6, 7):
            r, reps = A.pagerank_incremental(m, 0.85, prune, 60, force_kernel=forced)
            assert len(reps) == it or dt == np.float32, (forced, len(reps), it)
            err = np.abs(r - exp) - rtol * np.abs(exp) - 4 * prune
            assert np.all(err <= 0), (prune, forced, float(err.max()))
            if forced >= 0:
                assert all(x["kernel"] == forced for x in reps)


@pytest.mark.gpu
@pytest.mark.parametrize("dt", [np.float64, np.float32], ids=["f64", "f32"])
def test_gpu_pagerank_directed(ctx, port, dt):
    # directed graph: the driver's orientation must be SPEC's (edges i -> j
    # of A carry mass from i to j), checked against the dense oracle
    from paper_2006_16767_b200 import adaspmv as A
    n = 120
    a = _directed_graph(n, 0.05, 7)
    ro, ci, co, ri = _csr_csc(a)
    m = A.DualMatrix.from_csr(n, n, ro, ci, None, dtype=dt, ctx=ctx)
    exp = _dense_power(a, 0.85)
    tol = 1e-10 if dt == np.float64 else 2e-5
    for forced in (-1, 0, 1, 4, 5, 6, 7):
        r, _ = A.pagerank_incremental(m, 0.85, 0.0, 5000, force_kernel=forced)
        assert np.abs(r - exp).sum() <= tol, (forced, float(np.abs(r - exp).sum()))
    exp_o, _ = port.pagerank_incremental(n, ro, ci, 0.85, 1e-7, 200)
    r, _ = A.pagerank_incremental(m, 0.85, 1e-7, 200)
    rtol = 1e-11 if dt == np.float64 else 2e-5
    assert np.all(np.abs(r - exp_o) - rtol * np.abs(exp_o) - 4e-7 <= 0)


@pytest.mark.gpu
def test_gpu_pagerank_small_cases(ctx, port):
    from paper_2006_16767_b200 import adaspmv as A
    a = np.array([[0, 1], [1, 0]], bool)
    ro, ci, co, ri = _csr_csc(a)
    m = A.DualMatrix.from_csr(2, 2, ro, ci, None, dtype=np.float64, ctx=ctx)
    r, reps = A.pagerank_incremental(m, 0.85, 1e-6, 300)
    assert r[0] == r[1]
    r0, reps0 = A.pagerank_incremental(m, 0.85, 1e-6, 0)
    assert not r0.any() and reps0 == []
    with pytest.raises(A.InvalidArgument):
        A.pagerank_incremental(m, 1.5)
    a = np.array([[0, 1, 0], [1, 0, 1], [0, 1, 0]], bool)
    ro, ci, co, ri = _csr_csc(a)
    m = A.DualMatrix.from_csr(3, 3, ro, ci, None, dtype=np.float64, ctx=ctx)
    r, _ = A.pagerank_incremental(m, 0.85, 0.0, 5000)
    exp, _ = port.pagerank_incremental(3, ro, ci, 0.85, 0.0, 5000)
    assert np.abs(r - exp).sum() <= 1e-12 and r[1] > r[0]

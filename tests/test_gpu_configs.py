"""Parity at BASELINE.json's configured sizes, run by
the driver with the rest of `-m gpu`:

  C3  R-MAT scale 22 (128 M stored entries), BFS from vertex 0: levels bit
      exact against the queue BFS for OR_AND, MIN_PLUS and PLUS_TIMES (the
      reference BFS), under the built-in policy, the
      trained selector and forced kernels.
  C4  SVM-like 10 M x 2 M (~2e8 nnz), sparse sample rows with nnz_x in
      {200, 2,000, 20,000}: all eight kernels against the oracle's
      reference_multiply (kernels.hpp:197-209) on the downloaded CSR, every
      row; sparse index sets exact (positive values: no cancellation).
  C5  R-MAT scale 26 (2.1 G stored entries) at N = 1: 10^4 sampled rows plus
      the 64 heaviest rows against reference_multiply on those rows, for every
      kernel at x = 0.1 % and the row kernels (+ K4/K6) at x = 100 %; BFS
      levels against the queue BFS.

The matrices are generated on the device (synth_device; host generation of
R-MAT 22 takes ~107 s) and handed to the library as device CSR.
"""
import gc

import numpy as np
import pytest

from paper_2006_16767_b200 import adaspmv as A
from paper_2006_16767_b200 import selector as S
from paper_2006_16767_b200 import synth_device as SD
from tests.util import assert_dense_close, assert_sparse_match

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

torch = pytest.importorskip("torch")


def _free():
    gc.collect()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


# ---------------------------------------------------------------------------
# C3: R-MAT 22 BFS
# ---------------------------------------------------------------------------
@pytest.fixture(scope="module")
def c3(ctx, port):
    n, ro, ci = SD.rmat_device(22)
    nnz = int(ro[-1].item())
    m = A.DualMatrix.from_device(n, n, nnz, ro.data_ptr(), ci.data_ptr(), None, np.float32, ctx)
    ro_h = ro.cpu().numpy()
    ci_h = ci.cpu().numpy()
    del ro, ci
    _free()
    # symmetric graph: the CSR is the CSC; queue BFS over y = A x semantics
    q, nq = port.bfs_queue_i32(n, ro_h, ci_h, 0)
    yield m, q, nq, nnz
    m.close()
    _free()


def test_c3_rmat22_shape(c3):
    m, q, nq, nnz = c3
    assert m.rows() == 1 << 22 and nnz > 120_000_000  # probe: 128,306,762 (host draw)
    assert nq >= 5 and (q >= 0).sum() > 2_000_000


@pytest.mark.parametrize("sr", [A.OR_AND, A.MIN_PLUS, A.PLUS_TIMES], ids=["or_and", "min_plus", "plus_times"])
def test_c3_bfs_levels_bitexact(c3, sr):
    m, q, nq, _ = c3
    bundle = A.SelectorBundle.load(S.DEFAULT_PATH)
    for policy in ("heuristic", "selector", 6, 2, 0):
        kw = dict(semiring=sr)
        if policy == "selector":
            kw["bundle"] = bundle
        elif policy != "heuristic":
            kw["force_kernel"] = policy
        levels, reps = A.bfs(m, 0, **kw)
        assert np.array_equal(levels, q), (sr, policy, int((levels != q).sum()))
        assert len(reps) == nq  # one multiply per level; the last finds nothing
        # what ran is reported beside what was selected (exec_mode)
        for r in reps:
            if r["kernel"] in (2, 3):
                assert r["exec_mode"] == A.EXEC_MASKED_PULL
            if r["kernel"] >= 4 and sr == A.OR_AND and r["exec_mode"] != A.EXEC_AS_SELECTED:
                assert r["exec_mode"] == A.EXEC_FUSED_PUSH_LB


# ---------------------------------------------------------------------------
# C4: SVM-like, all eight kernels vs reference_multiply
# ---------------------------------------------------------------------------
@pytest.fixture(scope="module")
def c4(ctx):
    mr, nc = 10_000_000, 2_000_000
    ro, ci, vals, draw = SD.svm_device(mr, nc, 20, 1.0, 3)
    nnz = int(ro[-1].item())
    m = A.DualMatrix.from_device(mr, nc, nnz, ro.data_ptr(), ci.data_ptr(), vals.data_ptr(), np.float32, ctx)
    host = (ro.cpu().numpy(), ci.cpu().numpy().astype(np.int64), vals.cpu().numpy().astype(np.float64))
    del ro, ci, vals
    _free()
    yield m, host, draw, mr, nc
    m.close()
    _free()


@pytest.mark.parametrize("nnz_x", [200, 2000, 20000])
def test_c4_svm_all_kernels(c4, port, nnz_x):
    m, (ro, ci, vals), draw, mr, nc = c4
    xi, xv = SD.svm_vector(draw, nc, nnz_x, seed=nnz_x)
    xd = np.zeros(nc)
    xd[xi] = xv
    y_ref = port.reference_multiply(mr, ro, ci, vals, xd)
    bound = y_ref  # all values positive: |A||x| = A x
    x = A.DeviceVector(nc, np.float32, m.ctx).set_sparse(xi, xv)
    out = A.MultiplyOutput(m.ctx)
    for k in range(8):
        x.prepare(k)
        y = A.run_kernel(m, k, x, out=out)
        what = f"C4 k={k} nnz_x={nnz_x}"
        assert_dense_close(y.dense().values, y_ref, bound, np.float32, what)
        s = y.sparse()
        assert np.array_equal(s.indices, np.nonzero(y_ref)[0]), what
        assert_sparse_match(s.indices, s.values, y_ref, bound, np.float32, what)


# ---------------------------------------------------------------------------
# C5: R-MAT 26 at N = 1
# ---------------------------------------------------------------------------
@pytest.fixture(scope="module")
def c5(ctx, port):
    free, total = torch.cuda.mem_get_info()
    if total < 150e9:
        pytest.skip("C5 needs a 180 GB B200")
    n, ro, ci = SD.rmat_device(26)
    nnz = int(ro[-1].item())
    g = torch.Generator(device="cuda")
    g.manual_seed(26)
    vals = torch.rand(nnz, generator=g, device="cuda") * 2 - 1
    _free()
    m = A.DualMatrix.from_device(n, n, nnz, ro.data_ptr(), ci.data_ptr(), vals.data_ptr(), np.float32, ctx)
    # sampled rows: 10^4 uniform + the 64 heaviest (hub rows), their CSR segments
    deg = ro[1:] - ro[:-1]
    rng = np.random.default_rng(5)
    rows = np.unique(np.concatenate([rng.choice(n, 10_000, replace=False),
                                     torch.topk(deg, 64).indices.cpu().numpy()]))
    rt = torch.from_numpy(rows).cuda()
    b, e = ro[rt], ro[rt + 1]
    lens = e - b
    sub_ro = torch.zeros(len(rows) + 1, dtype=torch.int64, device="cuda")
    sub_ro[1:] = torch.cumsum(lens, 0)
    pos = torch.repeat_interleave(b - sub_ro[:-1], lens) + torch.arange(int(sub_ro[-1].item()), device="cuda")
    sample = (rows, sub_ro.cpu().numpy(), ci[pos].cpu().numpy().astype(np.int64),
              vals[pos].cpu().numpy().astype(np.float64))
    ro_h = ro.cpu().numpy()
    ci_h = ci.cpu().numpy()
    del ro, ci, vals, deg, rt, b, e, lens, sub_ro, pos
    _free()
    q, nq = port.bfs_queue_i32(n, ro_h, ci_h, 0)
    del ci_h
    yield m, sample, q, nq, n
    m.close()
    _free()


def _c5_x(n, dens, seed):
    nx = max(1, int(round(dens * n)))
    rng = np.random.default_rng(seed)
    if nx == n:
        return None, rng.uniform(-1, 1, n).astype(np.float32)
    xi = np.sort(rng.choice(n, size=nx, replace=False)).astype(np.int64)
    return xi, rng.uniform(-1, 1, nx).astype(np.float32)


@pytest.mark.parametrize("dens,kernels", [(0.001, range(8)), (1.0, (0, 1, 2, 3, 4, 6))], ids=["x0.1pct", "x100pct"])
def test_c5_sampled_rows_vs_oracle(c5, port, dens, kernels):
    m, (rows, sro, sci, svals), _, _, n = c5
    xi, xv = _c5_x(n, dens, 17)
    if xi is None:
        xd = xv.astype(np.float64)
        x = A.DeviceVector(n, np.float32, m.ctx).set_dense(xv)
    else:
        xd = np.zeros(n)
        xd[xi] = xv
        x = A.DeviceVector(n, np.float32, m.ctx).set_sparse(xi, xv)
    y_ref = port.reference_multiply(len(rows), sro, sci, svals, xd)
    bound = port.reference_multiply(len(rows), sro, sci, np.abs(svals), np.abs(xd))
    out = A.MultiplyOutput(m.ctx)
    for k in kernels:
        x.prepare(k)
        y = A.run_kernel(m, k, x, out=out)
        yd = y.dense().values[rows]
        assert_dense_close(yd, y_ref, bound, np.float32, f"C5 k={k} x={dens}")
        if k in (5, 7):  # sparse y: the sampled rows' membership matches
            s = y.sparse()
            got = np.isin(rows, s.indices)
            want = y_ref != 0
            diff = got != want
            assert np.all(np.abs(y_ref[diff]) <= 1e-5 * bound[diff]), f"C5 k={k} sparse index set"


def test_c5_bfs_levels_bitexact(c5):
    m, _, q, nq, _ = c5
    for kw in (dict(), dict(bundle=A.SelectorBundle.load(S.DEFAULT_PATH))):
        levels, reps = A.bfs(m, 0, semiring=A.OR_AND, **kw)
        assert np.array_equal(levels, q), int((levels != q).sum())
        assert len(reps) == nq

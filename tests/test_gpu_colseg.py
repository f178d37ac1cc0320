"""Row-segmented atomic column write-back (csrc/kernels_colseg.cu) against the
oracle: heavy support columns accumulated per row segment in shared memory
(plain stores), light ones through the global atomic write-back.  Forced on
with ADASPMV_COLSEG=1 for K4 and K6; ADASPMV_COLSEG_ROWS shrinks the segments
so small matrices cross many of them.  Same tolerance / bit-exactness as the
atomic kernels (tests/util.py; OR_AND and MIN_PLUS exact)."""
import os

import numpy as np
import pytest

from paper_2006_16767_b200 import adaspmv as A
from tests.util import assert_dense_close, ref_and_bound

pytestmark = pytest.mark.gpu

DTYPES = [np.float64, np.float32]


def _zipf_csr(rows, cols, nnz, seed, dt):
    """Rows uniform, columns Zipf(1.0)-popular (heavy + light columns)."""
    rng = np.random.default_rng(seed)
    w = 1.0 / np.arange(1, cols + 1)
    perm = rng.permutation(cols)
    c = perm[rng.choice(cols, nnz, p=w / w.sum())]
    r = rng.integers(0, rows, nnz)
    key = np.unique(r.astype(np.int64) * cols + c)
    r, c = key // cols, key % cols
    ro = np.zeros(rows + 1, np.int64)
    np.add.at(ro, r + 1, 1)
    ro = np.cumsum(ro)
    return rows, cols, ro, c.astype(np.int64), rng.uniform(-1, 1, len(c)).astype(dt)


@pytest.fixture
def colseg_env():
    old = {k: os.environ.get(k) for k in ("ADASPMV_COLSEG", "ADASPMV_COLSEG_ROWS")}
    yield os.environ
    for k, v in old.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v


def _x(cols, nx, seed, dt, sr):
    rng = np.random.default_rng(seed)
    xi = np.sort(rng.choice(cols, nx, replace=False)).astype(np.int64)
    xv = (rng.uniform(0, 2, nx) if sr == A.MIN_PLUS else rng.uniform(-1, 1, nx)).astype(dt)
    xd = np.full(cols, np.inf if sr == A.MIN_PLUS else 0.0, dt)
    xd[xi] = xv
    return xi, xv, xd


@pytest.mark.parametrize("dt", DTYPES, ids=["f64", "f32"])
@pytest.mark.parametrize("seg_rows", ["97", "1000", ""], ids=["R97", "R1000", "Rdefault"])
def test_colseg_all_semirings_vs_oracle(ctx, port, colseg_env, dt, seg_rows):
    colseg_env["ADASPMV_COLSEG"] = "1"
    if seg_rows:
        colseg_env["ADASPMV_COLSEG_ROWS"] = seg_rows
    else:
        colseg_env.pop("ADASPMV_COLSEG_ROWS", None)
    shape = (5000, 3000, 60000) if seg_rows else (70000, 5000, 400000)
    rows, cols, ro, ci, vals = _zipf_csr(*shape, seed=len(seg_rows), dt=dt)
    m = A.DualMatrix.from_csr(rows, cols, ro, ci, vals, ctx=ctx)
    for nx in (1, 37, cols // 10, cols):
        for sr in (A.PLUS_TIMES, A.OR_AND, A.MIN_PLUS):
            xi, xv, xd = _x(cols, nx, nx + 5, dt, sr)
            for k in (4, 6):
                out = A.run_kernel(m, k, A.SparseVector(cols, xi, xv), A.KernelConfig(semiring=sr))
                y = out.dense().values
                what = f"R={seg_rows or 'auto'} sr={sr} k={k} nnz_x={nx} {np.dtype(dt).name}"
                if sr == A.PLUS_TIMES:
                    y_ref, bound = ref_and_bound(port, rows, ro, ci, vals, xd)
                    assert_dense_close(y, y_ref, bound, dt, what)
                else:
                    y_ref = port.semiring_multiply(rows, ro, ci, vals, xd, sr)
                    assert y.tobytes() == y_ref.tobytes(), (what, np.nonzero(y != y_ref)[0][:5])


def test_colseg_counters_on_and_off(ctx, port, colseg_env):
    # values_read (kernels.hpp:108) == nnz_s through both halves of the split,
    # and the default (unset / 0: the L2-atomic K6) agrees with it
    colseg_env.pop("ADASPMV_COLSEG", None)
    colseg_env["ADASPMV_COLSEG_ROWS"] = "256"
    rows, cols, ro, ci, vals = _zipf_csr(4000, 2000, 80000, seed=4, dt=np.float32)
    m = A.DualMatrix.from_csr(rows, cols, ro, ci, vals, ctx=ctx)
    xi, xv, xd = _x(cols, 600, 1, np.float32, A.PLUS_TIMES)
    y_ref, bound = ref_and_bound(port, rows, ro, ci, vals, xd)
    co = np.zeros(cols + 1, np.int64)
    np.add.at(co, ci + 1, 1)
    nnz_s = int(co[1:][xi].sum())
    ctx.set_counters(True)
    try:
        for mode in ("", "0", "1"):
            if mode:
                colseg_env["ADASPMV_COLSEG"] = mode
            out = A.run_kernel(m, 6, A.SparseVector(cols, xi, xv))
            assert_dense_close(out.dense().values, y_ref, bound, np.float32, f"mode={mode!r}")
            assert out.counters()["values_read"] == nnz_s, mode
    finally:
        ctx.set_counters(False)

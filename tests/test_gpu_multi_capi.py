"""The single-process row-partitioned mode behind the C-ABI (adaspmv_multi_*,
SURVEY.md 8(b)/8(e)): G row blocks of ~nnz/G nonzeros, each on its own
context and stream (here all on device 0, which exercises the same cut,
per-block selection and y assembly as G devices), against the oracle."""
import numpy as np
import pytest

from paper_2006_16767_b200 import adaspmv as A
from paper_2006_16767_b200 import selector as S
from paper_2006_16767_b200 import synth
from tests.util import assert_dense_close, ref_and_bound

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dt", [np.float64, np.float32], ids=["f64", "f32"])
@pytest.mark.parametrize("g", [1, 3])
def test_multi_blocks_vs_oracle(ctx, port, dt, g):
    rows, cols, ro, ci, vals = synth.random_csr(5000, 4000, 0.003, seed=12, dtype=dt)
    mm = A.MultiMatrix(rows, cols, ro, ci, vals, devices=[0] * g)
    cuts = mm.cuts()
    assert cuts[0] == 0 and cuts[-1] == rows and np.all(np.diff(cuts) >= 0)
    assert np.array_equal(cuts, A.shard_rows(ro, g))
    bundle = A.SelectorBundle.load(S.DEFAULT_PATH)
    for nx in (0, 5, 400, cols):
        xi, xv = synth.sparse_vector(cols, nx, seed=nx + 2, dtype=dt)
        xd = port.sparse_to_dense(cols, xi, xv)
        y_ref, bound = ref_and_bound(port, rows, ro, ci, vals, xd)
        for k in (-1, 0, 1, 3, 4, 5, 6, 7):
            x = xd if k in (0, 1) else (xi, xv)
            y, ks = mm.multiply(x, bundle=bundle if k < 0 else None, force_kernel=k)
            assert len(ks) == g
            assert_dense_close(y, y_ref, bound, dt, f"multi g={g} k={k} nx={nx}")
    mm.close()


def test_multi_errors(ctx):
    rows, cols, ro, ci, vals = synth.random_csr(100, 80, 0.05, seed=1)
    with pytest.raises(A.InvalidArgument):
        A.MultiMatrix(rows, cols, ro, ci, vals, devices=[])
    mm = A.MultiMatrix(rows, cols, ro, ci, vals, devices=[0, 0])
    with pytest.raises(A.InvalidArgument):
        mm.multiply((np.array([5, 2]), np.array([1.0, 1.0])), force_kernel=4)  # unsorted
    with pytest.raises(A.InvalidArgument):
        mm.multiply(np.ones(cols))  # no bundle, no forced kernel
    y, _ = mm.multiply(np.ones(cols), force_kernel=0)  # still usable
    assert y.shape == (rows,)

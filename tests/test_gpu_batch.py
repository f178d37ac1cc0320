"""adaspmv_run_batch (pipelined multiplies from host buffers) against the CPU
oracle: every operand of a mixed dense/sparse batch, every result form, forced
kernels and the selector, several lane counts; an invalid operand fails the
batch with the reference's exception type (sparse.hpp:120-129)."""
import numpy as np
import pytest

from paper_2006_16767_b200 import adaspmv as A
from paper_2006_16767_b200 import selector as S
from paper_2006_16767_b200 import synth
from tests.util import assert_dense_close, assert_sparse_match, ref_and_bound

pytestmark = pytest.mark.gpu


def _batch(cols, dt, seeds=(1, 2, 3, 4, 5, 6, 7)):
    xs, dense = [], []
    for i, s in enumerate(seeds):
        nx = [0, 1, cols // 100, cols // 10, cols // 2, cols, cols // 3][i % 7]
        xi, xv = synth.sparse_vector(cols, nx, seed=s, dtype=dt)
        d = np.zeros(cols, dt)
        d[xi] = xv
        dense.append(d)
        xs.append(d if i % 2 else (xi, xv))
    return xs, dense


@pytest.mark.parametrize("dt", [np.float64, np.float32], ids=["f64", "f32"])
@pytest.mark.parametrize("lanes", [1, 3, 5])
def test_batch_forced_and_forms(ctx, port, dt, lanes):
    rows, cols, ro, ci, vals = synth.random_csr(3000, 2000, 0.01, seed=4, dtype=dt)
    m = A.DualMatrix.from_csr(rows, cols, ro, ci, vals, ctx=ctx)
    xs, dense = _batch(cols, dt)
    refs = [ref_and_bound(port, rows, ro, ci, vals, d) for d in dense]
    for k in range(8):
        for form in (A.RESULT_DENSE, A.RESULT_SPARSE, A.RESULT_AUTO):
            res = A.run_batch(m, xs, force_kernel=k, form=form, lanes=lanes)
            assert len(res) == len(xs)
            for i, (r, (y_ref, bound)) in enumerate(zip(res, refs)):
                what = f"k={k} form={form} op={i} lanes={lanes}"
                assert r.kernel.index() == k, what
                if form == A.RESULT_DENSE:
                    assert not r.is_sparse
                if form == A.RESULT_SPARSE:
                    assert r.is_sparse
                if r.is_sparse:
                    assert_sparse_match(r.sparse.indices, r.sparse.values, y_ref, bound, dt, what)
                else:
                    assert_dense_close(r.dense.values, y_ref, bound, dt, what)


def test_batch_selector_matches_single_calls(ctx, port):
    """The selected kernels equal run_adaptive's, operand by operand, and the
    results match the oracle."""
    dt = np.float32
    rows, cols, ro, ci, vals = synth.random_csr(20000, 20000, 0.0008, seed=9, dtype=dt)
    m = A.DualMatrix.from_csr(rows, cols, ro, ci, vals, ctx=ctx)
    bundle = A.SelectorBundle.load(S.DEFAULT_PATH)
    xs, dense = _batch(cols, dt, seeds=range(11, 25))
    res = A.run_batch(m, xs, bundle=bundle, lanes=3)
    for i, (x, d, r) in enumerate(zip(xs, dense, res)):
        v = A.DeviceVector(cols, dt, ctx)
        if isinstance(x, tuple):
            v.set_sparse(*x)
        else:
            v.set_dense(x)
        _, k = A.run_adaptive(m, v, bundle)
        assert k.index() == r.kernel.index(), i
        y_ref, bound = ref_and_bound(port, rows, ro, ci, vals, d)
        if r.is_sparse:
            assert_sparse_match(r.sparse.indices, r.sparse.values, y_ref, bound, dt, str(i))
        else:
            assert_dense_close(r.dense.values, y_ref, bound, dt, str(i))


def test_batch_reused_buffers_and_empty(ctx, port):
    dt = np.float64
    rows, cols, ro, ci, vals = synth.random_csr(500, 400, 0.05, seed=2, dtype=dt)
    m = A.DualMatrix.from_csr(rows, cols, ro, ci, vals, ctx=ctx)
    assert A.run_batch(m, [], force_kernel=0) == []
    xs, dense = _batch(cols, dt)
    bufs = [(np.empty(rows, np.int64), np.empty(rows, dt)) for _ in xs]
    for rep in range(3):
        res = A.run_batch(m, xs, force_kernel=[5, 6, 0][rep], buffers=bufs, lanes=2)
        for r, d in zip(res, dense):
            y_ref, bound = ref_and_bound(port, rows, ro, ci, vals, d)
            if r.is_sparse:
                assert_sparse_match(r.sparse.indices, r.sparse.values, y_ref, bound, dt)
            else:
                assert_dense_close(r.dense.values, y_ref, bound, dt)


def test_batch_invalid_operand_raises(ctx):
    dt = np.float64
    rows, cols, ro, ci, vals = synth.random_csr(100, 100, 0.05, seed=2, dtype=dt)
    m = A.DualMatrix.from_csr(rows, cols, ro, ci, vals, ctx=ctx)
    good = (np.array([1, 5], np.int64), np.array([1.0, 2.0]))
    unsorted = (np.array([5, 1], np.int64), np.array([1.0, 2.0]))
    oob = (np.array([1, 100], np.int64), np.array([1.0, 2.0]))
    with pytest.raises(A.InvalidArgument, match="operand 1"):
        A.run_batch(m, [good, unsorted, good], force_kernel=4, lanes=1)
    with pytest.raises(A.InvalidArgument):
        A.run_batch(m, [good, oob], force_kernel=4, lanes=2)
    with pytest.raises(A.InvalidArgument):
        A.run_batch(m, [good], lanes=1)  # neither a bundle nor a forced kernel
    # the context stays usable
    r = A.run_batch(m, [good], force_kernel=4)
    assert r[0].kernel.index() == 4


def test_batch_many_operands_more_lanes_than_needed(ctx, port):
    """A long batch (60 operands, more lanes than the default) and a batch
    shorter than the lane count both return every result in order."""
    dt = np.float32
    rows, cols, ro, ci, vals = synth.random_csr(4000, 3000, 0.002, seed=8, dtype=dt)
    m = A.DualMatrix.from_csr(rows, cols, ro, ci, vals, ctx=ctx)
    xs, dense = _batch(cols, dt, seeds=range(100, 160))
    for lanes, sub in ((8, slice(None)), (16, slice(0, 3))):
        res = A.run_batch(m, xs[sub], force_kernel=6, lanes=lanes)
        assert len(res) == len(dense[sub])
        for r, d in zip(res, dense[sub]):
            y_ref, bound = ref_and_bound(port, rows, ro, ci, vals, d)
            if r.is_sparse:
                assert_sparse_match(r.sparse.indices, r.sparse.values, y_ref, bound, dt)
            else:
                assert_dense_close(r.dense.values, y_ref, bound, dt)

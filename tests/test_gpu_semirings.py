"""BFS semirings on all eight kernels against the C oracle's
semiring multiply (oracle/oracle_impl.inc or_semiring_multiply, an extension
of reference_multiply, kernels.hpp:197-209).  OR_AND and MIN_PLUS are
order-free (one rounding per term, then OR / min), so every kernel must match
the oracle BIT FOR BIT -- dense views, and the sparse index sets of the sort
write-back.

x is given sparse (explicit zeros and negative values included: under
MIN_PLUS a stored 0.0 is a real distance) and as a user-dense vector whose
absent entries hold the semiring's identity (0 / +inf), which the column
kernels must turn into the same support the oracle sees (a dense
x's sparse / mask views are semiring-keyed)."""
import numpy as np
import pytest

from paper_2006_16767_b200 import adaspmv as A
from paper_2006_16767_b200 import synth
from tests.test_gpu_kernels import CASES, DTYPES

SEMIRINGS = [(A.OR_AND, "or_and"), (A.MIN_PLUS, "min_plus")]


def _dense_x(cols, xi, xv, sr, dt):
    x = np.full(cols, np.inf if sr == A.MIN_PLUS else 0.0, dt)
    x[xi] = xv
    return x


def _sparse_x(cols, nx, seed, dt):
    xi, xv = synth.sparse_vector(cols, nx, seed=seed, dtype=dt)
    xv = xv.copy()
    if nx >= 3:
        xv[::3] = 0.0  # explicit zeros: present (MIN_PLUS), false (OR_AND)
    return xi, xv


def test_oracle_semiring_known_answers(port):
    ro = np.array([0, 2, 3, 3])
    ci = np.array([0, 2, 1])
    v = np.array([1.0, -2.0, 3.0])
    # MIN_PLUS: row 0 = min(1 + 0, -2 + 5) = 1; row 1 sees only +inf -> +inf
    y = port.semiring_multiply(3, ro, ci, v, np.array([0.0, np.inf, 5.0]), 2)
    assert y.tolist() == [1.0, np.inf, np.inf]
    y = port.semiring_multiply(3, ro, ci, v, np.array([0.0, 1.0, 0.0]), 1)
    assert y.tolist() == [0.0, 1.0, 0.0]
    y = port.semiring_multiply(3, ro, ci, v, np.array([2.0, 0.0, 1.0]), 0)
    assert y.tolist() == [0.0, 0.0, 0.0]




@pytest.mark.gpu
@pytest.mark.parametrize("dt", DTYPES, ids=["f64", "f32"])
@pytest.mark.parametrize("sr,srname", SEMIRINGS, ids=[s[1] for s in SEMIRINGS])
@pytest.mark.parametrize("name,case", CASES, ids=[c[0] for c in CASES])
def test_semiring_all_kernels_bitexact(ctx, port, name, case, sr, srname, dt):
    rows, cols, ro, ci, vals = case
    vals = np.asarray(vals, dt)
    m = A.DualMatrix.from_csr(rows, cols, ro, ci, vals, ctx=ctx)
    cfg = A.KernelConfig(semiring=sr)
    for nx in sorted({0, 1, max(1, cols // 50), max(1, cols // 3), cols}):
        xi, xv = _sparse_x(cols, nx, nx + 11, dt)
        xd = _dense_x(cols, xi, xv, sr, dt)
        y_ref = port.semiring_multiply(rows, ro, ci, vals, xd, sr)
        ident = 0.0 if sr == A.OR_AND else np.inf
        ref_idx = np.nonzero(y_ref != ident)[0]
        for k in range(8):
            for form in ("sparse", "dense"):
                x = A.SparseVector(cols, xi, xv) if form == "sparse" else A.DenseVector(xd)
                out = A.run_kernel(m, k, x, cfg)
                y = out.dense().values
                what = f"{name} {srname} k={k} nnz_x={nx} x={form} {np.dtype(dt).name}"
                assert y.tobytes() == y_ref.tobytes(), (what, np.nonzero(y != y_ref)[0][:5])
                s = out.sparse()
                assert np.array_equal(s.indices, ref_idx), what
                assert s.values.tobytes() == y_ref[ref_idx].tobytes(), what


@pytest.mark.gpu
@pytest.mark.parametrize("dt", DTYPES, ids=["f64", "f32"])
def test_min_plus_user_dense_zeros_every_kernel(ctx, port, dt):
    # ADVICE r01 (vector.cu): a user-dense x under MIN_PLUS whose zeros are
    # real values (a source distance of 0) -- row kernels read them from the
    # dense values, column kernels and the mask must keep them too
    rows, cols, ro, ci, vals = synth.random_csr(3000, 2500, 0.003, seed=41, dtype=dt)
    m = A.DualMatrix.from_csr(rows, cols, ro, ci, vals, ctx=ctx)
    rng = np.random.default_rng(3)
    xd = np.full(cols, np.inf, dt)
    sup = rng.choice(cols, 400, replace=False)
    xd[sup] = rng.uniform(0, 2, 400).astype(dt)
    xd[sup[:150]] = 0.0
    y_ref = port.semiring_multiply(rows, ro, ci, vals, xd, 2)
    res = []
    dv = A.DeviceVector(cols, dt, ctx).set_dense(xd)
    # the same vector object serves a plus-times run in between: its derived
    # views must be rebuilt for each semiring, not reused
    xpt = np.where(np.isinf(xd), 0.0, xd).astype(dt)
    dpt = A.DeviceVector(cols, dt, ctx).set_dense(xpt)
    for k in range(8):
        out = A.run_kernel(m, k, dv, A.KernelConfig(semiring=A.MIN_PLUS))
        res.append(out.dense().values.copy())
        A.run_kernel(m, k, dpt)
    for k, y in enumerate(res):
        assert y.tobytes() == y_ref.tobytes(), (k, np.nonzero(y != y_ref)[0][:5])


@pytest.mark.gpu
@pytest.mark.parametrize("k", [5, 7])
def test_sort_writeback_all_support_on_empty_columns(ctx, k):
    # ADVICE r01 (kernels_col.cu:627): > 4096 support entries whose columns are
    # all empty (nnz_s = 0) skip the single-CTA path; the result is an empty y
    rows, cols = 100, 20000
    ro = np.zeros(rows + 1, np.int64)
    ro[1:] = np.cumsum(np.full(rows, 3))
    rng = np.random.default_rng(1)
    ci = np.concatenate([np.sort(rng.choice(100, 3, replace=False)) for _ in range(rows)]).astype(np.int64)
    m = A.DualMatrix.from_csr(rows, cols, ro, ci, rng.uniform(-1, 1, len(ci)), ctx=ctx)
    xi = np.arange(1000, 1000 + 6000, dtype=np.int64)
    for sr in (A.PLUS_TIMES, A.OR_AND, A.MIN_PLUS):
        out = A.run_kernel(m, k, A.SparseVector(cols, xi, np.ones(len(xi))), A.KernelConfig(semiring=sr))
        assert out.nnz() == 0
        ident = np.inf if sr == A.MIN_PLUS else 0.0
        assert np.all(out.dense().values == ident)


@pytest.mark.gpu
def test_device_input_validation(ctx):
    # ADVICE r01 (capi.cpp:295): caller device arrays are validated like the host ones
    import torch
    dev = torch.device("cuda", 0)
    ro = torch.tensor([0, 2, 3], dtype=torch.int64, device=dev)
    good = torch.tensor([0, 2, 1], dtype=torch.int32, device=dev)
    vals = torch.ones(3, dtype=torch.float64, device=dev)
    m = A.DualMatrix.from_device(2, 3, 3, ro.data_ptr(), good.data_ptr(), vals.data_ptr(), np.float64, ctx=ctx)
    assert m.nnz() == 3
    for bad_ci, bad_ro in ((torch.tensor([0, 5, 1], dtype=torch.int32, device=dev), ro),
                           (torch.tensor([2, 0, 1], dtype=torch.int32, device=dev), ro),
                           (good, torch.tensor([0, 2, 1], dtype=torch.int64, device=dev)),
                           (good, torch.tensor([0, 2, 4], dtype=torch.int64, device=dev))):
        with pytest.raises(A.InvalidArgument):
            A.DualMatrix.from_device(2, 3, 3, bad_ro.data_ptr(), bad_ci.data_ptr(), vals.data_ptr(),
                                     np.float64, ctx=ctx)
    v = A.DeviceVector(3, np.float64, ctx)
    xv = torch.ones(2, dtype=torch.float64, device=dev)
    for idx in ([0, 3], [2, 1], [1, 1]):
        t = torch.tensor(idx, dtype=torch.int32, device=dev)
        with pytest.raises(A.InvalidArgument):
            v.set_sparse_device(2, t.data_ptr(), xv.data_ptr())
    t = torch.tensor([0, 2], dtype=torch.int32, device=dev)
    v.set_sparse_device(2, t.data_ptr(), xv.data_ptr())
    assert v.nnz() == 2

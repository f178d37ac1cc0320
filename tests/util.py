"""Parity helpers (SURVEY.md section 8(c) parity rules).

Dense y: |y_i - y_ref_i| <= rtol * (|A||x|)_i + tiny, rtol 1e-12 (fp64) /
1e-5 (fp32) -- the magnitude-scaled form of BASELINE.json's tolerances; the
reference (fp64) is the oracle's multiply in float64 of the same inputs.
Sparse y: exact index-set equality except where |y_ref_i| <= rtol*(|A||x|)_i.
"""
import numpy as np

RTOL = {np.dtype(np.float64): 1e-12, np.dtype(np.float32): 1e-5}


def ref_and_bound(port, rows, ro, ci, vals, xd):
    v64 = np.asarray(vals, np.float64)
    x64 = np.asarray(xd, np.float64)
    y = port.reference_multiply(rows, ro, ci, v64, x64)
    b = port.reference_multiply(rows, ro, ci, np.abs(v64), np.abs(x64))
    return y, b


def assert_dense_close(y, y_ref, bound, dtype, what=""):
    rtol = RTOL[np.dtype(dtype)]
    y = np.asarray(y, np.float64)
    excess = np.abs(y - y_ref) - (rtol * bound + 1e-300)
    if np.any(excess > 0):
        i = int(np.argmax(excess))
        raise AssertionError(f"{what}: row {i} y={y[i]!r} ref={y_ref[i]!r} bound={bound[i]!r} "
                             f"({int((excess > 0).sum())} rows out of tolerance)")


def assert_sparse_match(idx, val, y_ref, bound, dtype, what=""):
    rtol = RTOL[np.dtype(dtype)]
    idx = np.asarray(idx)
    ref_idx = np.nonzero(y_ref)[0]
    a = set(idx.tolist())
    b = set(ref_idx.tolist())
    for i in a ^ b:  # allowed only at near-cancellation
        assert abs(y_ref[i]) <= rtol * bound[i], f"{what}: index {i} differs (ref {y_ref[i]!r})"
    assert np.all(np.diff(idx) > 0), f"{what}: sparse indices not strictly increasing"
    dense = np.zeros_like(y_ref)
    dense[idx] = np.asarray(val, np.float64)
    assert_dense_close(dense, y_ref, bound, dtype, what)

"""The C++ drop-in against the reference, in one program (VERDICT r01 "next" 3).

`oracle/_ref/dropin_vs_ref_{f64,f32}` (built by oracle/Makefile from
`oracle/dropin_vs_ref.cpp`) includes the unmodified reference headers
(kernels.hpp, matrix_market.hpp) and `include/adaspmv_cuda.hpp`, loads the same
Matrix Market file through both `load_matrix`s (matrix_market.hpp:228-238)
and runs all 8 KernelIds through both `run_kernel`s (kernels.hpp:520-535):
dense results within the 8(c) tolerance of the magnitude bound, sparse index
sets of the sort write-back identical.
"""
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
BIN = ROOT / "oracle" / "_ref"


def _write_mtx(path, rows, cols, r, c, v):
    with open(path, "w") as f:
        f.write("%%MatrixMarket matrix coordinate real general\n")
        f.write(f"% drop-in check matrix\n{rows} {cols} {len(r)}\n")
        for a, b, x in zip(r, c, v):
            f.write(f"{int(a) + 1} {int(b) + 1} {float(x)!r}\n")


def _random_mtx(path, rows, cols, nnz, seed, skew=False):
    rng = np.random.default_rng(seed)
    if skew:  # power-law rows and columns, empty rows and columns at the ends
        r = np.minimum((rng.pareto(1.2, nnz) * 8).astype(np.int64), rows - 40)
        c = np.minimum((rng.pareto(1.2, nnz) * 8).astype(np.int64), cols - 40)
    else:
        r = rng.integers(0, rows, nnz)
        c = rng.integers(0, cols, nnz)
    v = rng.uniform(-1.0, 1.0, nnz)
    _write_mtx(path, rows, cols, r, c, v)  # duplicates are summed by both loaders


@pytest.mark.gpu
@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("shape", ["uniform", "skewed", "tall", "wide"])
def test_dropin_matches_reference(tmp_path, prec, shape):
    exe = BIN / f"dropin_vs_ref_{prec}"
    assert exe.exists(), f"{exe} not built (build() compiles it next to the reference checkers)"
    mtx = tmp_path / f"{shape}.mtx"
    if shape == "uniform":
        _random_mtx(mtx, 3000, 2500, 40000, 1)
    elif shape == "skewed":
        _random_mtx(mtx, 4000, 4000, 60000, 2, skew=True)
    elif shape == "tall":
        _random_mtx(mtx, 20000, 64, 30000, 3)
    else:
        _random_mtx(mtx, 64, 20000, 30000, 4)
    res = subprocess.run([str(exe), str(mtx), "7", "0.0005", "0.02", "0.3", "1.0"],
                         capture_output=True, text=True, timeout=600)
    out = res.stdout + res.stderr
    assert res.returncode == 0 and "DROPIN OK" in out, out[-4000:]
    assert out.count(" ok ") == 4 * 8, out[-4000:]

"""Ingestion at scale: DualMatrix::from_triplets on the
device and the parallel Matrix Market parser, bit-exact against fixtures the
reference itself produced (tests/golden/make_golden.py: triplets.npz,
mm_cases.npz), plus the reference's error behaviour on large files (the
parallel parser hands any irregular file to the serial one)."""
import hashlib
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_2006_16767_b200 import adaspmv as A

sys.path.insert(0, str(Path(__file__).resolve().parent / "golden"))
from make_golden import TRIPLET_CASES, big_mm_text, triplet_case  # noqa: E402

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"


def test_from_triplets_matches_reference(ctx):
    z = np.load(GOLD / "triplets.npz")
    for k in range(int(z["nt"][0])):
        rows, cols, n, seed, bits = (int(v) for v in z[f"t{k}_meta"])
        dt = np.float64 if bits == 64 else np.float32
        tr, tc, tv = triplet_case(rows, cols, n, seed, dt)
        m = A.DualMatrix.from_triplets(rows, cols, tr, tc, tv, dtype=dt, ctx=ctx)
        ro, ci, v = m.download()[:3]
        assert np.array_equal(ro, z[f"t{k}_ro"]), k
        assert np.array_equal(ci, z[f"t{k}_ci"]), k
        ref_v = z[f"t{k}_v"].astype(dt)
        if n == 0 or np.bincount(tr, minlength=rows).max() <= 16:
            # rows of <= 16 triplets: libstdc++'s std::sort is an insertion
            # sort there (stable), so duplicates are summed in input order
            # like ours: bit-exact
            assert v.astype(dt).tobytes() == ref_v.tobytes(), k
        else:
            # longer rows: the reference's introsort may sum duplicates in
            # another order; the BASELINE tolerance relative to sum |v|
            key = tr * cols + tc
            uk, inv = np.unique(key, return_inverse=True)
            absum = np.zeros(len(uk))
            np.add.at(absum, inv, np.abs(tv.astype(np.float64)))
            rtol = 1e-12 if dt == np.float64 else 1e-5
            assert np.all(np.abs(v.astype(np.float64) - ref_v.astype(np.float64)) <= rtol * absum + 1e-300), k


def test_from_triplets_errors(ctx):
    with pytest.raises(A.InvalidArgument, match="out of range"):
        A.DualMatrix.from_triplets(3, 3, [0, 3], [0, 0], [1.0, 2.0], ctx=ctx)
    with pytest.raises(A.InvalidArgument, match="out of range"):
        A.DualMatrix.from_triplets(3, 3, [0, 1], [0, -1], [1.0, 2.0], ctx=ctx)
    with pytest.raises(A.InvalidArgument, match="negative"):
        A.DualMatrix.from_triplets(-1, 3, [], [], [], ctx=ctx)
    m = A.DualMatrix.from_triplets(4, 5, [], [], [], ctx=ctx)
    assert m.nnz() == 0 and m.rows() == 4


def test_mm_golden_small(ctx, tmp_path):
    z = np.load(GOLD / "mm_cases.npz")
    for i in range(int(z["nmm"][0])):
        p = tmp_path / f"m{i}.mtx"
        p.write_text(str(z[f"mm{i}_text"]))
        ro, ci, v = A.load_matrix(p, ctx=ctx).download()[:3]
        assert np.array_equal(ro, z[f"mm{i}_ro"]) and np.array_equal(ci, z[f"mm{i}_ci"]), i
        assert v.tobytes() == z[f"mm{i}_v"].tobytes(), i


@pytest.mark.parametrize("dt", [np.float64, np.float32], ids=["f64", "f32"])
@pytest.mark.parametrize("sym", [1, 0])
def test_large_mm_parallel_parser_matches_reference(ctx, tmp_path, dt, sym):
    z = np.load(GOLD / "triplets.npz")
    p = tmp_path / "big.mtx"
    p.write_text(big_mm_text(symmetric=bool(sym)))
    assert p.stat().st_size > (1 << 20)  # takes the parallel path
    ro, ci, v = A.load_matrix(p, dtype=dt, ctx=ctx).download()[:3]
    key = f"big_{np.dtype(dt).name}_{sym}"
    assert len(ci) == int(z[key + "_nnz"][0])
    h = hashlib.sha256(ro.tobytes() + ci.tobytes() + v.astype(dt).tobytes()).hexdigest()
    assert h == str(z[key + "_sha"])


@pytest.mark.parametrize("dt", [np.float64, np.float32], ids=["f64", "f32"])
def test_large_pattern_mm_matches_reference(ctx, tmp_path, dt):
    z = np.load(GOLD / "triplets.npz")
    p = tmp_path / "bigp.mtx"
    p.write_text(big_mm_text(pattern=True))
    assert p.stat().st_size > (1 << 20)
    ro, ci, v = A.load_matrix(p, dtype=dt, ctx=ctx).download()[:3]
    key = f"bigp_{np.dtype(dt).name}"
    assert len(ci) == int(z[key + "_nnz"][0])
    h = hashlib.sha256(ro.tobytes() + ci.tobytes() + v.astype(dt).tobytes()).hexdigest()
    assert h == str(z[key + "_sha"])


def test_large_mm_errors_report_reference_line(ctx, tmp_path):
    text = big_mm_text(symmetric=False)
    lines = text.split("\n")
    # a bad entry late in the file: ParseError at its 1-based line
    bad = len(lines) - 10
    lines[bad - 1] = "3 x 1.0"
    p = tmp_path / "bad.mtx"
    p.write_text("\n".join(lines))
    with pytest.raises(A.ParseError) as e:
        A.load_matrix(p, ctx=ctx)
    assert e.value.line == bad
    # out-of-range coordinate
    lines = text.split("\n")
    lines[bad - 1] = "99999999 1 1.0"
    p.write_text("\n".join(lines))
    with pytest.raises(A.ParseError, match="out of range") as e:
        A.load_matrix(p, ctx=ctx)
    assert e.value.line == bad
    # fewer entries than declared
    lines = text.split("\n")
    del lines[bad - 1]
    p.write_text("\n".join(lines))
    with pytest.raises(A.ParseError, match="does not match declared"):
        A.load_matrix(p, ctx=ctx)

"""Generates the golden fixtures in tests/golden/ from THE REFERENCE ITSELF
(oracle/_ref/libadaspmv_ref_{f64,f32}.so, i.e. /root/reference's headers
compiled unmodified by oracle/Makefile).  Run here, where the reference is
mounted:  python tests/golden/make_golden.py

Fixtures (npz):
  kernels_{f64,f32}.npz   small matrices x vectors x all 8 kernels (workers 1
                          and 3): CSR, CSC, x, dense y, sparse y, counters
  prims.npz               make_partition / segment_of / dense_to_sparse /
                          bitmask / sort_reduce_pairs examples
  mm_cases.npz            Matrix Market texts and the CSR the reference loads
  triplets.npz            from_triplets cases (duplicates, unsorted, -0.0,
                          empty rows) and a >1 MB Matrix Market file (text
                          regenerated from its seed by big_mm_text) with the
                          sha256 of the CSR the reference loads
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle.oracle import Ref  # noqa: E402
from paper_2006_16767_b200 import synth  # noqa: E402

OUT = Path(__file__).resolve().parent

SHAPES = [(30, 30, 0.1), (60, 40, 0.05), (1, 50, 0.5), (50, 1, 0.5), (5, 7, 0.0), (200, 150, 0.03),
          (100, 100, 0.2)]


def kernels(dt):
    ref = Ref(dt, counters=True)
    ref.set_threads(4)
    rec = {}
    case = 0
    for si, (r, c, d) in enumerate(SHAPES):
        rows, cols, ro, ci, vals = synth.random_csr(r, c, d, seed=100 + si, dtype=dt)
        M = ref.matrix(rows, cols, ro, ci, vals)
        ro2, ci2, v2, co, ri, cv = M.export()
        for nx in sorted({0, 1, max(1, cols // 4), cols}):
            xi, xv = synth.sparse_vector(cols, nx, seed=7 * nx + si, dtype=dt)
            p = f"c{case}_"
            rec[p + "dims"] = np.array([rows, cols], np.int64)
            rec[p + "ro"], rec[p + "ci"], rec[p + "vals"] = ro, ci, vals
            rec[p + "co"], rec[p + "ri"], rec[p + "cv"] = co, ri, cv
            rec[p + "xi"], rec[p + "xv"] = xi, xv
            xd = ref.sparse_to_dense(cols, xi, xv)
            rec[p + "y_oracle"] = M.reference_multiply(xd)
            rec[p + "eff"] = np.array([M.effective_nnz(xi)], np.int64)
            for w in (1, 3):
                for k in range(8):
                    yd, (yi, yv), cnt = M.run_kernel(k, x_sparse=(xi, xv), workers=w)
                    q = f"{p}k{k}_w{w}_"
                    rec[q + "yd"], rec[q + "yi"], rec[q + "yv"], rec[q + "cnt"] = yd, yi, yv, cnt
            case += 1
    rec["ncases"] = np.array([case])
    np.savez_compressed(OUT / f"kernels_{np.dtype(dt).name}.npz", **rec)
    return case


def prims():
    ref = Ref(np.float64)
    rec = {}
    offs = [[0, 0, 0, 9, 10], list(range(8)), [0, 3, 3, 3, 7, 12, 12], [0, 5]]
    tot = [10, 7, 12, 5]
    i = 0
    for o, t in zip(offs, tot):
        for w in (1, 2, 3, 5, 16):
            rec[f"part{i}_off"] = np.array(o, np.int64)
            rec[f"part{i}_meta"] = np.array([t, w], np.int64)
            rec[f"part{i}_out"] = ref.make_partition(o, t, w)
            i += 1
    rec["npart"] = np.array([i])
    seg_off = np.array([0, 0, 2, 2, 2, 7, 9], np.int64)
    rec["seg_off"] = seg_off
    rec["seg_pos"] = np.arange(0, 9)
    rec["seg_out"] = np.array([ref.segment_of(seg_off, p) for p in range(9)], np.int64)
    rng = np.random.default_rng(5)
    v = rng.uniform(-1, 1, 1000)
    v[rng.random(1000) < 0.6] = 0.0
    v[3] = -0.0
    rec["d2s_in"] = v
    rec["d2s_idx"], rec["d2s_val"] = ref.dense_to_sparse(v)
    rec["mask_dense"] = ref.build_bitmask_dense(v)
    rec["mask_sparse_idx"] = np.array([0, 63, 64, 127, 128, 200], np.int64)
    rec["mask_sparse"] = ref.build_bitmask_sparse(201, rec["mask_sparse_idx"])
    pr = np.array([2, 0, 2, 5, 5, 1, 0], np.int64)
    pv = np.array([1.0, 2.0, 3.0, 0.5, -0.5, 4.0, 1.0])
    rec["srp_rows"], rec["srp_vals"] = pr, pv
    rec["srp_idx"], rec["srp_val"] = ref.sort_reduce_pairs(pr, pv, 6)
    np.savez_compressed(OUT / "prims.npz", **rec)


MM_TEXTS = [
    "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 5.0\n2 2 7.0\n",
    "%%MatrixMarket matrix coordinate real symmetric\n% comment\n\n3 3 2\n2 1 3.0\n3 3 1.5\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n1 1 2.0\n",
    "%%MatrixMarket matrix coordinate pattern general\n3 4 3\n1 4\n3 1\n2 2\n",
    "%%MatrixMarket matrix coordinate integer general\n2 3 2\n1 3 -4\n2 1 9\n",
    "%%MATRIXMARKET Matrix Coordinate Real General\n1 1 1\n1 1 0.1\n",
]


def mm_cases(tmp: Path):
    ref = Ref(np.float64)
    rec = {}
    for i, t in enumerate(MM_TEXTS):
        p = tmp / f"m{i}.mtx"
        p.write_text(t)
        M = ref.load_matrix(p)
        ro, ci, cv, *_ = M.export()
        rec[f"mm{i}_text"] = np.array(t)
        rec[f"mm{i}_dims"] = np.array([M.rows, M.cols], np.int64)
        rec[f"mm{i}_ro"], rec[f"mm{i}_ci"], rec[f"mm{i}_v"] = ro, ci, cv
    rec["nmm"] = np.array([len(MM_TEXTS)])
    np.savez_compressed(OUT / "mm_cases.npz", **rec)


TRIPLET_CASES = [(5, 4, 12, 0), (40, 30, 400, 1), (1, 1, 3, 2), (300, 200, 6000, 3), (2000, 1500, 40000, 4),
                 (7, 9, 0, 5)]


def triplet_case(rows, cols, n, seed, dt):
    """Triplets with many duplicates (coordinates drawn from a small pool),
    input order random, some -0.0 and exact zeros."""
    rng = np.random.default_rng(seed)
    pool = max(1, n // 3)
    pr = rng.integers(0, rows, pool)
    pc = rng.integers(0, cols, pool)
    pick = rng.integers(0, pool, n)
    tr, tc = pr[pick].astype(np.int64), pc[pick].astype(np.int64)
    tv = rng.uniform(-1, 1, n).astype(dt)
    if n:
        tv[rng.random(n) < 0.05] = -0.0
        tv[rng.random(n) < 0.05] = 0.0
    return tr, tc, tv


def big_mm_text(seed=11, rows=20000, cols=15000, n=70000, symmetric=True, pattern=False):
    """A ~1.7 MB Matrix Market file: comments and blank lines between
    entries, CRLF line ends, duplicates, mixed number formats."""
    if pattern:  # ~1.4 MB pattern file
        rng = np.random.default_rng(seed + 1)
        n = 2 * n
        r = rng.integers(1, rows + 1, n)
        c = rng.integers(1, cols + 1, n)
        lines = ["%%MatrixMarket matrix coordinate pattern general", f"{rows} {cols} {n}"]
        lines += [f"{r[i]} {c[i]}" + ("\r" if i % 5 == 0 else "") for i in range(n)]
        return "\n".join(lines) + "\n"
    rng = np.random.default_rng(seed)
    r = rng.integers(1, rows + 1, n)
    c = rng.integers(1, cols + 1, n)
    if symmetric:
        cols = rows
        c = rng.integers(1, rows + 1, n)
    v = rng.uniform(-10, 10, n)
    lines = ["%%MatrixMarket matrix coordinate real " + ("symmetric" if symmetric else "general"),
             "% generated", f"{rows} {cols} {n}"]
    for i in range(n):
        fmt = ("%.17g", "%.6e", "%.3f")[i % 3]
        lines.append(f"{r[i]} {c[i]} " + fmt % v[i] + ("\r" if i % 7 == 0 else ""))
        if i % 997 == 0:
            lines.append("% a comment line")
        if i % 1499 == 0:
            lines.append("   ")
    return "\n".join(lines) + "\n"


def triplets(tmp: Path):
    import hashlib
    rec = {}
    k = 0
    for dt in (np.float64, np.float32):
        ref = Ref(dt)
        for rows, cols, n, seed in TRIPLET_CASES:
            tr, tc, tv = triplet_case(rows, cols, n, seed, dt)
            M = ref.from_triplets(rows, cols, tr, tc, tv)
            ro, ci, cv, *_ = M.export()
            p = f"t{k}_"
            rec[p + "meta"] = np.array([rows, cols, n, seed, 64 if dt == np.float64 else 32], np.int64)
            rec[p + "ro"], rec[p + "ci"], rec[p + "v"] = ro, ci, cv
            k += 1
    rec["nt"] = np.array([k])
    for dt in (np.float64, np.float32):
        ref = Ref(dt)
        for sym in (True, False):
            p = tmp / "big.mtx"
            p.write_text(big_mm_text(symmetric=sym))
            M = ref.load_matrix(p)
            ro, ci, cv, *_ = M.export()
            h = hashlib.sha256(ro.tobytes() + ci.tobytes() + cv.tobytes()).hexdigest()
            rec[f"big_{np.dtype(dt).name}_{int(sym)}_sha"] = np.array(h)
            rec[f"big_{np.dtype(dt).name}_{int(sym)}_nnz"] = np.array([len(ci)], np.int64)
    for dt in (np.float64, np.float32):
        p = tmp / "bigp.mtx"
        p.write_text(big_mm_text(pattern=True))
        M = Ref(dt).load_matrix(p)
        ro, ci, cv, *_ = M.export()
        rec[f"bigp_{np.dtype(dt).name}_sha"] = np.array(
            hashlib.sha256(ro.tobytes() + ci.tobytes() + cv.tobytes()).hexdigest())
        rec[f"bigp_{np.dtype(dt).name}_nnz"] = np.array([len(ci)], np.int64)
    np.savez_compressed(OUT / "triplets.npz", **rec)


if __name__ == "__main__":
    import tempfile

    n64 = kernels(np.float64)
    n32 = kernels(np.float32)
    prims()
    with tempfile.TemporaryDirectory() as d:
        mm_cases(Path(d))
        triplets(Path(d))
    print(f"golden: {n64} f64 + {n32} f32 kernel cases, prims, {len(MM_TEXTS)} MM files")

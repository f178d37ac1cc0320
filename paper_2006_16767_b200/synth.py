"""Deterministic synthetic inputs for the BASELINE.json configurations
(SURVEY.md section 8(d) "Concrete synthetic inputs").  Host-side numpy; the
same arrays feed the CUDA path, the oracle and the reference CPU baseline, so
every arm sees identical bytes.

All matrices are returned as (rows, cols, row_offsets int64, col_indices
int64, values) in the reference layout (types.hpp:9), rows sorted, columns
strictly increasing within a row, duplicates summed (sparse.hpp:220-258).
"""
from __future__ import annotations

import numpy as np


def laplacian_2d(g: int = 1000, dtype=np.float64):
    """C1: 2-D 5-point Laplacian on a g x g grid; row r = i*g + j; diagonal 4,
    N/W/E/S = -1, columns sorted (r-g, r-1, r, r+1, r+g)."""
    n = g * g
    r = np.arange(n, dtype=np.int64)
    i, j = r // g, r % g
    cols, vals, rows_ = [], [], []
    for dc, ok, v in ((-g, i > 0, -1.0), (-1, j > 0, -1.0), (0, np.ones(n, bool), 4.0),
                      (1, j < g - 1, -1.0), (g, i < g - 1, -1.0)):
        rows_.append(r[ok])
        cols.append(r[ok] + dc)
        vals.append(np.full(int(ok.sum()), v))
    rr = np.concatenate(rows_)
    cc = np.concatenate(cols)
    vv = np.concatenate(vals)
    order = np.lexsort((cc, rr))
    rr, cc, vv = rr[order], cc[order], vv[order].astype(dtype)
    ro = np.zeros(n + 1, np.int64)
    ro[1:] = np.bincount(rr, minlength=n)
    np.cumsum(ro, out=ro)
    return n, n, ro, cc, vv


def uniform_random(n: int = 1 << 22, draws: int = 1 << 26, seed: int = 1, dtype=np.float32):
    """C2: `draws` iid (row, col) cells over n x n, values U[-1,1), duplicate
    cells summed (each draw contributes its own value)."""
    rng = np.random.default_rng(seed)
    keys = rng.integers(0, n * n, size=draws, dtype=np.int64)
    keys.sort()
    uniq, first, counts = np.unique(keys, return_index=True, return_counts=True)
    vals = rng.uniform(-1.0, 1.0, size=len(uniq)).astype(dtype)
    dup = np.nonzero(counts > 1)[0]
    for d in dup:  # rare: ~draws^2 / (2 n^2)
        extra = rng.uniform(-1.0, 1.0, size=int(counts[d]) - 1).astype(dtype)
        s = vals[d]
        for e in extra:
            s = dtype(s + e)
        vals[d] = s
    del keys, first, counts
    r = uniq // n
    c = uniq - r * n
    ro = np.zeros(n + 1, np.int64)
    ro[1:] = np.bincount(r, minlength=n)
    np.cumsum(ro, out=ro)
    return n, n, ro, c.astype(np.int64), vals


def rmat(scale: int, edge_factor: int = 16, abcd=(0.57, 0.19, 0.19, 0.05), seed: int = 2,
         symmetric: bool = True, values: str = "pattern", dtype=np.float32):
    """C3/C5: R-MAT (Graph500 parameters), edge_factor * 2^scale draws,
    self-loops dropped, symmetrised, deduplicated.  values='pattern' -> 1.0,
    'uniform' -> U[-1,1)."""
    n = 1 << scale
    m = edge_factor * n
    rng = np.random.default_rng(seed)
    a, b, c, _ = abcd
    src = np.zeros(m, np.int64)
    dst = np.zeros(m, np.int64)
    chunk = 1 << 24
    for s0 in range(0, m, chunk):
        s1 = min(m, s0 + chunk)
        k = s1 - s0
        rs = np.zeros(k, np.int64)
        cs = np.zeros(k, np.int64)
        for _lvl in range(scale):
            u = rng.random(k, dtype=np.float32)
            rbit = u >= a + b
            cbit = ((u >= a) & (u < a + b)) | (u >= a + b + c)
            rs = (rs << 1) | rbit
            cs = (cs << 1) | cbit
        src[s0:s1] = rs
        dst[s0:s1] = cs
    keep = src != dst
    src, dst = src[keep], dst[keep]
    if symmetric:
        src, dst = np.concatenate([src, dst]), np.concatenate([dst, src])
    keys = src * n + dst
    del src, dst
    keys = np.unique(keys)
    r = keys // n
    cc = keys - r * n
    ro = np.zeros(n + 1, np.int64)
    ro[1:] = np.bincount(r, minlength=n)
    np.cumsum(ro, out=ro)
    if values == "pattern":
        vals = np.ones(len(cc), dtype)
    else:
        vals = np.random.default_rng(seed + 1).uniform(-1.0, 1.0, len(cc)).astype(dtype)
    return n, n, ro, cc.astype(np.int64), vals


def svm_like(m: int = 10_000_000, n: int = 2_000_000, nnz_per_row: int = 20, zipf: float = 1.0,
             seed: int = 3, dtype=np.float32):
    """C4: m samples x n features, ~nnz_per_row per row, column popularity
    Zipf(zipf) over a random column permutation, values U(0,1]."""
    rng = np.random.default_rng(seed)
    ranks = np.arange(1, n + 1, dtype=np.float64)
    p = ranks ** (-zipf)
    p /= p.sum()
    cdf = np.cumsum(p)
    perm = rng.permutation(n)
    total = m * nnz_per_row
    rows = np.repeat(np.arange(m, dtype=np.int64), nnz_per_row)
    cols = perm[np.searchsorted(cdf, rng.random(total), side="right").clip(0, n - 1)]
    keys = np.unique(rows * n + cols)
    r = keys // n
    c = keys - r * n
    ro = np.zeros(m + 1, np.int64)
    ro[1:] = np.bincount(r, minlength=m)
    np.cumsum(ro, out=ro)
    vals = (1.0 - rng.random(len(c))).astype(dtype)  # (0, 1]
    return m, n, ro, c.astype(np.int64), vals


def random_csr(rows: int, cols: int, density: float, seed: int = 0, dtype=np.float64,
               positive: bool = False):
    """Small random matrices for the property tests."""
    rng = np.random.default_rng(seed)
    cells = rows * cols
    k = int(round(density * cells))
    k = min(k, cells)
    if cells and k:
        keys = np.sort(rng.choice(cells, size=k, replace=False)).astype(np.int64)
    else:
        keys = np.zeros(0, np.int64)
    r = keys // max(cols, 1)
    c = keys - r * max(cols, 1)
    ro = np.zeros(rows + 1, np.int64)
    if rows:
        ro[1:] = np.bincount(r, minlength=rows)
    np.cumsum(ro, out=ro)
    if positive:
        vals = (1.0 - rng.random(k)).astype(dtype)
    else:
        vals = rng.uniform(-1.0, 1.0, k).astype(dtype)
    return rows, cols, ro, c.astype(np.int64), vals


def sparse_vector(n: int, nnz: int, seed: int = 0, dtype=np.float64, positive: bool = False):
    """nnz distinct indices uniform without replacement, sorted; U[-1,1)."""
    rng = np.random.default_rng(seed)
    nnz = min(int(nnz), n)
    if nnz == n:
        idx = np.arange(n, dtype=np.int64)
    elif nnz > n // 8:
        idx = np.sort(rng.permutation(n)[:nnz]).astype(np.int64)
    else:
        idx = np.sort(rng.choice(n, size=nnz, replace=False)).astype(np.int64)
    if positive:
        val = (1.0 - rng.random(nnz)).astype(dtype)
    else:
        val = rng.uniform(-1.0, 1.0, nnz).astype(dtype)
    return idx, val


def sweep_nnz(n: int, sparsities=(0.00001, 0.0001, 0.001, 0.01, 0.1, 0.5, 1.0)):
    """nnz_x = round(s * n) for the C2 x-sparsity sweep (0.001 % .. 100 %)."""
    return [max(1, int(round(s * n))) for s in sparsities]

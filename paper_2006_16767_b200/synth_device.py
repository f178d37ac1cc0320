"""Device-side generators for the large BASELINE.json configurations
(SURVEY.md section 8(d) "Concrete synthetic inputs"): measurement and test
INPUTS only, produced with torch on the GPU because the host generators take
minutes at these sizes (R-MAT 22 on the host: ~107 s).  The result is handed
to the library as device CSR (adaspmv_matrix_create_csr_device), which
validates it and builds the CSC on the device.

  rmat_device   C3 (scale 22) / C5 (scale 26): Graph500 R-MAT, edge factor
                16, (a,b,c,d) = (.57,.19,.19,.05), self-loops dropped,
                symmetrised, deduplicated
  svm_device    C4: m samples x n features, ~per_row nnz per row, feature
                popularity Zipf(zipf) over a random feature permutation,
                values U(0,1]

Same parameters as the host generators in synth.py; the random streams
differ (torch vs numpy), so the graphs are different draws of the same law.
"""
from __future__ import annotations


def rmat_device(scale, edge_factor=16, abcd=(0.57, 0.19, 0.19, 0.05), seed=2, chunk=1 << 26):
    """-> (n, row_offsets int64 [n+1], col_indices int32 [nnz]) device tensors,
    rows sorted, columns strictly increasing within a row."""
    import torch
    n = 1 << scale
    m = edge_factor * n
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    a, b, c, _ = abcd
    keys = []
    for s0 in range(0, m, chunk):
        k = min(chunk, m - s0)
        rs = torch.zeros(k, dtype=torch.int64, device="cuda")
        cs = torch.zeros(k, dtype=torch.int64, device="cuda")
        for _ in range(scale):
            u = torch.rand(k, generator=g, device="cuda")
            rbit = (u >= a + b).long()
            cbit = (((u >= a) & (u < a + b)) | (u >= a + b + c)).long()
            rs = (rs << 1) | rbit
            cs = (cs << 1) | cbit
        keep = rs != cs
        rs, cs = rs[keep], cs[keep]
        keys.append(rs * n + cs)
        keys.append(cs * n + rs)
        del rs, cs, keep
    keys = torch.cat(keys)
    keys = torch.unique(keys)  # sorted, deduplicated
    rows = keys >> scale
    cols = (keys & (n - 1)).to(torch.int32)
    del keys
    ro = torch.zeros(n + 1, dtype=torch.int64, device="cuda")
    ro[1:] = torch.cumsum(torch.bincount(rows, minlength=n), 0)
    del rows
    torch.cuda.empty_cache()
    return n, ro, cols


def zipf_sampler(n, zipf, seed):
    """Draws feature ids with P(rank r) ~ r^-zipf over a random permutation."""
    import torch
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    ranks = torch.arange(1, n + 1, dtype=torch.float64, device="cuda")
    p = ranks.pow(-zipf)
    cdf = torch.cumsum(p / p.sum(), 0)
    perm = torch.randperm(n, generator=g, device="cuda")

    def draw(k):
        u = torch.rand(k, generator=g, device="cuda", dtype=torch.float64)
        return perm[torch.searchsorted(cdf, u, right=True).clamp_(0, n - 1)]
    return draw, g


def svm_device(m=10_000_000, n=2_000_000, per_row=20, zipf=1.0, seed=3):
    """-> (row_offsets int64, col_indices int32, values fp32 (0,1], draw) device
    tensors; `draw(k)` samples k feature ids from the same popularity law
    (the support of a sample row vector x)."""
    import torch
    draw, g = zipf_sampler(n, zipf, seed)
    keys = []
    chunk = 1 << 22  # rows per chunk
    for r0 in range(0, m, chunk):
        k = min(chunk, m - r0)
        rows = torch.arange(r0, r0 + k, dtype=torch.int64, device="cuda").repeat_interleave(per_row)
        keys.append(torch.unique(rows * n + draw(k * per_row)))
        del rows
    keys = torch.cat(keys)  # chunks are row-disjoint and each sorted -> globally sorted
    rows = keys // n
    cols = (keys - rows * n).to(torch.int32)
    del keys
    ro = torch.zeros(m + 1, dtype=torch.int64, device="cuda")
    ro[1:] = torch.cumsum(torch.bincount(rows, minlength=m), 0)
    del rows
    vals = 1.0 - torch.rand(cols.numel(), generator=g, device="cuda", dtype=torch.float32)  # (0, 1]
    torch.cuda.empty_cache()
    return ro, cols, vals, draw


def svm_vector(draw, n, nnz_x, seed):
    """Sample row vector for C4: nnz_x distinct features drawn from the
    popularity law, values U(0,1] -> host (int64 indices sorted, fp32 values)."""
    import numpy as np
    import torch
    got = torch.unique(draw(4 * nnz_x + 64))
    while got.numel() < nnz_x:
        got = torch.unique(torch.cat([got, draw(4 * nnz_x)]))
    rng = np.random.default_rng(seed)
    idx = got.cpu().numpy()
    idx = np.sort(rng.choice(idx, nnz_x, replace=False)).astype(np.int64)
    val = (1.0 - rng.random(nnz_x)).astype(np.float32)
    return idx, val

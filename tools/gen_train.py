"""generate_training_data on the B200: for a corpus of
synthetic matrices x an x-density sweep ("geometric:k" + "uniform:k"), record
the 13 Table-1 features and the device time of all 8 kernels (1 warm-up, then
the median of `--repeats`, CUDA events recorded by the library, L2 flushed
before every timed multiply).  Writes one CSV row per (matrix, vector):

  matrix, dtype, density, f0..f12, t0..t7      (seconds)

Usage (GPU):  python tools/gen_train.py --out gpurun_out/train_samples.csv
"""
from __future__ import annotations

import argparse
import csv
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2006_16767_b200 import adaspmv as A  # noqa: E402
from paper_2006_16767_b200 import synth  # noqa: E402


def banded(n, half_bw, seed, dtype):
    rng = np.random.default_rng(seed)
    r = np.repeat(np.arange(n, dtype=np.int64), 2 * half_bw + 1)
    off = np.tile(np.arange(-half_bw, half_bw + 1, dtype=np.int64), n)
    c = r + off
    keep = (c >= 0) & (c < n) & (rng.random(len(c)) < 0.6)
    r, c = r[keep], c[keep]
    ro = np.zeros(n + 1, np.int64)
    ro[1:] = np.bincount(r, minlength=n)
    np.cumsum(ro, out=ro)
    return n, n, ro, c, rng.uniform(-1, 1, len(c)).astype(dtype)


def rectangular(m, n, deg, seed, dtype):
    rng = np.random.default_rng(seed)
    keys = np.unique(rng.integers(0, m * n, size=m * deg, dtype=np.int64))
    r = keys // n
    c = keys - r * n
    ro = np.zeros(m + 1, np.int64)
    ro[1:] = np.bincount(r, minlength=m)
    np.cumsum(ro, out=ro)
    return m, n, ro, c, rng.uniform(-1, 1, len(c)).astype(dtype)


def corpus(scale: str):
    f32, f64 = np.float32, np.float64
    big = scale == "full"
    items = [
        ("uniform_n16_d16", lambda: synth.uniform_random(1 << 16, 16 << 16, seed=11, dtype=f32)),
        ("uniform_n18_d4", lambda: synth.uniform_random(1 << 18, 4 << 18, seed=12, dtype=f32)),
        ("uniform_n18_d64", lambda: synth.uniform_random(1 << 18, 64 << 18, seed=13, dtype=f32)),
        ("uniform_n20_d16", lambda: synth.uniform_random(1 << 20, 16 << 20, seed=14, dtype=f32)),
        ("uniform_n20_d8_f64", lambda: synth.uniform_random(1 << 20, 8 << 20, seed=15, dtype=f64)),
        ("rmat_s16_e16", lambda: synth.rmat(16, 16, seed=21, values="uniform")),
        ("rmat_s18_e8", lambda: synth.rmat(18, 8, seed=22, values="uniform")),
        ("rmat_s20_e16", lambda: synth.rmat(20, 16, seed=23, values="uniform")),
        ("lap2d_512_f64", lambda: synth.laplacian_2d(512, dtype=f64)),
        ("lap2d_1000_f64", lambda: synth.laplacian_2d(1000, dtype=f64)),
        ("lap2d_2048_f32", lambda: synth.laplacian_2d(2048, dtype=f32)),
        ("banded_1m_bw8", lambda: banded(1 << 20, 8, 31, f32)),
        ("banded_256k_bw64", lambda: banded(1 << 18, 64, 32, f32)),
        ("svm_1m_200k", lambda: synth.svm_like(1_000_000, 200_000, 20, 1.0, seed=41)),
        ("rect_4m_64k_d8", lambda: rectangular(1 << 22, 1 << 16, 8, 51, f32)),
        ("rect_64k_4m_d64", lambda: rectangular(1 << 16, 1 << 22, 64, 52, f32)),
    ]
    if big:
        items += [
            ("uniform_n22_d16", lambda: synth.uniform_random(1 << 22, 16 << 22, seed=1, dtype=f32)),
            ("rmat_s22_e16", lambda: synth.rmat(22, 16, seed=24, values="uniform")),
            ("svm_10m_2m", lambda: synth.svm_like(10_000_000, 2_000_000, 20, 1.0, seed=3)),
        ]
    return items


def biased_vector(col_deg, nnz, seed, dtype):
    """Support drawn without replacement with probability proportional to the
    column degree (+1): the shape of BFS frontiers and PageRank deltas on
    power-law graphs (their nonzeros sit on high-degree vertices), which
    uniform supports never produce.  Values U[-1,1)."""
    rng = np.random.default_rng(seed)
    n = len(col_deg)
    nnz = min(int(nnz), n)
    w = col_deg.astype(np.float64) + 1.0
    # Efraimidis-Spirakis weighted sampling without replacement: top-k of u^(1/w)
    keys = np.log(rng.random(n)) / w
    idx = np.sort(np.argpartition(-keys, nnz - 1)[:nnz]).astype(np.int64) if nnz < n else np.arange(n)
    return idx, rng.uniform(-1.0, 1.0, nnz).astype(dtype)


def densities(n, geo=16, uni=8):
    """geometric:k and uniform:k density points (nnz_x)."""
    g = np.unique(np.round(np.geomspace(1, n, geo)).astype(np.int64))
    u = np.unique(np.round(np.linspace(1, n, uni)).astype(np.int64))
    return sorted(set(g.tolist()) | set(u.tolist()))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/train_samples.csv")
    ap.add_argument("--scale", choices=("small", "full"), default="full")
    ap.add_argument("--repeats", type=int, default=3)
    a = ap.parse_args()
    import torch

    ctx = A.Context(0)
    ctx.set_timing(True)
    stream = torch.cuda.ExternalStream(ctx.stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    sink = torch.zeros(1, dtype=torch.int64, device="cuda")

    def l2_flush():
        with torch.cuda.stream(stream):
            flush.add_(1)                # write > L2 ...
            sink.add_(flush[::4096].sum())  # ... then touch it again (clean lines)

    out = A.MultiplyOutput(ctx)
    Path(a.out).parent.mkdir(parents=True, exist_ok=True)
    with open(a.out, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["matrix", "dtype", "nnz_x"] + [f"f{i}" for i in range(13)] + [f"t{k}" for k in range(8)])
        for name, gen in corpus(a.scale):
            t0 = time.time()
            rows, cols, ro, ci, vals = gen()
            m = A.DualMatrix.from_csr(rows, cols, ro, ci, vals, ctx=ctx)
            dt = np.dtype(vals.dtype)
            col_deg = np.bincount(ci, minlength=cols)
            skewed = col_deg.max() > 8 * max(col_deg.mean(), 1.0)
            pts = [(nx, False) for nx in densities(cols)]
            if skewed:  # degree-biased supports (BFS / PageRank shapes) on skewed matrices
                pts += [(nx, True) for nx in densities(cols, geo=10, uni=4) if nx < cols]
            for k_idx, (nx, biased) in enumerate(pts):
                if biased:
                    xi, xv = biased_vector(col_deg, nx, seed=5000 + k_idx, dtype=dt)
                else:
                    xi, xv = synth.sparse_vector(cols, nx, seed=1000 + k_idx, dtype=dt)
                x = A.DeviceVector(cols, dt, ctx)
                if nx == cols:
                    d = np.zeros(cols, dt)
                    d[xi] = xv
                    x.set_dense(d)
                else:
                    x.set_sparse(xi, xv)
                f = A.features(m, x)
                ts = []
                for k in range(8):
                    x.prepare(k)
                    A.run_kernel(m, k, x, out=out)  # warm-up
                    rep = []
                    for _ in range(a.repeats):
                        l2_flush()
                        with torch.cuda.stream(stream):
                            torch.cuda._sleep(400_000)  # host enqueue overlaps: device time only
                        A.run_kernel(m, k, x, out=out)
                        rep.append(out.elapsed())
                    ts.append(float(np.median(rep)))
                w.writerow([name + ("/biased" if biased else ""), dt.name, nx] + [repr(float(v)) for v in f] + [repr(t) for t in ts])
                fh.flush()
            print(f"{name}: {rows}x{cols} nnz={ro[-1]} in {time.time() - t0:.1f}s", flush=True)
            del m


if __name__ == "__main__":
    main()

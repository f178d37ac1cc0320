"""C4 (BASELINE.json configs[3]): SVM-style skinny sparse data matrix (10 M
samples x 2 M features, ~20 nnz per sample row, feature popularity Zipf(1.0)
over a random feature permutation, values U(0,1]) times a sparse sample row
vector with nnz_x in {200, 2,000, 20,000} (0.01 / 0.1 / 1 % of the features)
drawn from the same popularity law.

The matrix is generated ON THE DEVICE with torch (measurement input only)
and handed to the library as device CSR.  Every kernel and the adaptive
selector are timed with CUDA events (the library's own, on its stream),
after an L2 flush; y is checked against the CPU oracle
(oracle/adaspmv_oracle.c reference_multiply on the downloaded CSR, fp64)
with the magnitude-scaled tolerance of SURVEY.md 8(c).

  python tools/c4_bench.py --out gpurun_out/c4.json
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2006_16767_b200 import adaspmv as A  # noqa: E402
from paper_2006_16767_b200 import selector as S  # noqa: E402


def zipf_sampler(n, zipf, seed):
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


def svm_device(m, n, per_row, zipf, seed):
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
    return ro, cols, vals, draw


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=10_000_000)
    ap.add_argument("--cols", type=int, default=2_000_000)
    ap.add_argument("--per-row", type=int, default=20)
    ap.add_argument("--nnz-x", default="200,2000,20000")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--no-oracle", action="store_true")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    m, n = a.rows, a.cols
    t0 = time.time()
    ro, ci, vals, draw = svm_device(m, n, a.per_row, 1.0, 3)
    nnz = int(ro[-1].item())
    gen_s = time.time() - t0
    ctx = A.Context(0)
    t0 = time.time()
    mat = A.DualMatrix.from_device(m, n, nnz, ro.data_ptr(), ci.data_ptr(), vals.data_ptr(), np.float32, ctx)
    build_s = time.time() - t0
    res = {"config": "C4 SVM-like %d x %d, Zipf(1.0) feature popularity, %d nnz, fp32" % (m, n, nnz),
           "rows": m, "cols": n, "nnz": nnz, "generate_s": round(gen_s, 1), "device_csr_to_dual_s": round(build_s, 2),
           "features": mat.features().tolist(), "points": []}
    print(json.dumps({k: res[k] for k in ("config", "generate_s", "device_csr_to_dual_s")}), flush=True)
    host = None
    port = None
    if not a.no_oracle:
        from oracle.oracle import Port
        port = Port()
        host = (ro.cpu().numpy(), ci.cpu().numpy().astype(np.int64), vals.cpu().numpy().astype(np.float64))
    del ci, vals
    torch.cuda.empty_cache()
    ctx.set_timing(True)
    stream = torch.cuda.ExternalStream(ctx.stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    out = A.MultiplyOutput(ctx)
    bundle = A.SelectorBundle.load(S.DEFAULT_PATH)
    hbm = 6532.9e9
    for nx in [int(s) for s in a.nnz_x.split(",")]:
        # support from the popularity law (distinct features), values U(0,1]
        sup = torch.unique(draw(4 * nx))[:nx]
        while sup.numel() < nx:
            sup = torch.unique(torch.cat([sup, draw(4 * nx)]))[:nx]
        xi = torch.sort(sup).values.cpu().numpy().astype(np.int64)
        xv = (1.0 - np.random.default_rng(nx).random(nx)).astype(np.float32)
        x = A.DeviceVector(n, np.float32, ctx)
        x.set_sparse(xi, xv)
        nnz_s = A.effective_nnz(mat, x)
        b_col_atomic = nx * 8 + 2 * nx * 8 + nnz_s * 8 + m * 4
        pt = {"nnz_x": nx, "x_sparsity": nx / n, "nnz_s": nnz_s, "kernels": {}}
        y_ref = absy = None
        if host is not None:
            xd = np.zeros(n)
            xd[xi] = xv
            y_ref = port.reference_multiply(m, host[0], host[1], host[2], xd)
            absy = y_ref  # all values positive: |A||x| == A x
        times = {}
        for k in list(range(8)) + ["adaptive"]:
            ts = []
            for r in range(a.reps + 1):
                with torch.cuda.stream(stream):
                    flush.add_(1)
                    torch.cuda._sleep(200_000)
                if k == "adaptive":
                    y, kk = A.run_adaptive(mat, x, bundle, out=out)
                else:
                    x.prepare(k)
                    y = A.run_kernel(mat, k, x, out=out)
                if r:
                    ts.append(y.elapsed())
            t = float(np.median(ts))
            ent = {"t_us": round(t * 1e6, 2), "gflops": round(2 * nnz_s / t / 1e9, 2),
                   "pct_hbm_col_atomic_bytes": round(100 * b_col_atomic / t / hbm, 1)}
            if k == "adaptive":
                ent["selected"] = kk.name()
            else:
                times[k] = t
            if y_ref is not None:
                yd = y.dense().values.astype(np.float64)
                ent["parity"] = bool(np.all(np.abs(yd - y_ref) <= 1e-5 * absy + 1e-30))
            pt["kernels"][str(k) if k == "adaptive" else A.KernelId.from_index(k).name()] = ent
            print(nx, k, ent, flush=True)
        best = min(times, key=times.get)
        pt["best"] = A.KernelId.from_index(best).name()
        pt["regret"] = round(pt["kernels"]["adaptive"]["t_us"] / (times[best] * 1e6), 3)
        res["points"].append(pt)
        print(json.dumps({"nnz_x": nx, "nnz_s": nnz_s, "best": pt["best"], "selected":
                          pt["kernels"]["adaptive"]["selected"], "regret": pt["regret"]}), flush=True)
    if a.out:
        Path(a.out).write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()

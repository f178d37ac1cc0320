"""Per-point breakdown of the selection overhead on C2 (SPEC.md:561 bound):
feature pull (device reduction + host wait), tree walk, conversion, kernel,
for fresh operands exactly as bench.py's overhead leg sets them.

  python tools/select_probe.py [--reps 5]
"""
import argparse
import statistics
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2006_16767_b200 import adaspmv as A  # noqa: E402
from paper_2006_16767_b200 import selector as S  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    ctx = A.Context(0)
    (rows, cols, ro, ci, vals), _ = bench.make_matrix()
    m = A.DualMatrix.from_csr(rows, cols, ro, ci, vals, ctx=ctx)
    bundle = A.SelectorBundle.load(S.DEFAULT_PATH)
    vecs = bench.make_vectors(cols)
    out = A.MultiplyOutput(ctx)
    fresh = A.DeviceVector(cols, np.float32, ctx)
    tot = {"feature": 0.0, "predict": 0.0, "convert": 0.0, "kernel": 0.0}
    for i, (xi, xv) in enumerate(vecs):
        f, p, c, k = [], [], [], []
        for _ in range(a.reps + 1):
            if len(xi) == cols:
                d = np.zeros(cols, np.float32)
                d[xi] = xv
                fresh.set_dense(d)
            else:
                fresh.set_sparse(xi, xv)
            ctx.synchronize()
            _, rep = A.execute_iteration(m, fresh, bundle, out=out)
            f.append(rep["feature_s"]), p.append(rep["predict_s"]), c.append(rep["convert_s"]), k.append(rep["kernel_s"])
        med = [statistics.median(v[1:]) * 1e6 for v in (f, p, c, k)]
        for key, v in zip(tot, med):
            tot[key] += v
        print(f"x={bench.SPARSITIES[i]:<8g} nnz_x={len(xi):>8d} kernel={rep['kernel'].name():18s} "
              f"feature {med[0]:7.1f} us  predict {med[1]:6.1f}  convert {med[2]:6.1f}  kernel {med[3]:7.1f}")
    over = tot["feature"] + tot["predict"] + tot["convert"]
    print(f"total: feature {tot['feature']:.1f} predict {tot['predict']:.1f} convert {tot['convert']:.1f} "
          f"kernel {tot['kernel']:.1f} us -> overhead fraction {over / (over + tot['kernel']):.3f}")


if __name__ == "__main__":
    main()

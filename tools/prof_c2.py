"""Profiling driver: C2 (uniform 4M x 4M, 2^26 draws, fp32) and one x
density; runs the chosen kernels `--reps` times each (for ncu / launch lists)."""
import argparse
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2006_16767_b200 import adaspmv as A  # noqa: E402
from paper_2006_16767_b200 import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--density", type=float, default=1.0)
ap.add_argument("--kernels", default="0,1")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--log2n", type=int, default=22)
ap.add_argument("--lanes", type=int, default=0)
a = ap.parse_args()
n = 1 << a.log2n
rows, cols, ro, ci, vals = synth.uniform_random(n, 16 * n, seed=1, dtype=np.float32)
ctx = A.Context(0)
m = A.DualMatrix.from_csr(rows, cols, ro, ci, vals, ctx=ctx)
xi, xv = synth.sparse_vector(cols, max(1, int(round(a.density * cols))), seed=7, dtype=np.float32)
x = A.DeviceVector(cols, np.float32, ctx)
if len(xi) == cols:
    d = np.zeros(cols, np.float32); d[xi] = xv; x.set_dense(d)
else:
    x.set_sparse(xi, xv)
out = A.MultiplyOutput(ctx)
cfg = A.KernelConfig(lanes_per_row=a.lanes)
for k in [int(s) for s in a.kernels.split(",")]:
    x.prepare(k)
    ctx.synchronize()
    for _ in range(a.reps):
        A.run_kernel(m, k, x, cfg, out=out)
    ctx.synchronize()
print("done", time.time())

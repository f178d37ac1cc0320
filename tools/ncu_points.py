"""One multiply per (input, kernel, x density) inside an NVTX range "measure",
for ncu captures of the kernels a point runs (launch lists and --set full of
the dominant kernel), e.g.

  ncu --nvtx --nvtx-include "measure/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,\
dram__bytes_write.sum --clock-control none --csv python tools/ncu_points.py --input c2 --kernel 5 --density 0.001

Each point is run once untimed first (lazy layouts, operand views), then once
inside the range.  Inputs: c2 (BASELINE configs[1]), c4 (configs[3], device
generator, sample row of --nnz-x), rmat22 (configs[2] graph, device generator).
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2006_16767_b200 import adaspmv as A  # noqa: E402
from paper_2006_16767_b200 import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--input", default="c2")
    ap.add_argument("--kernel", type=int, required=True)
    ap.add_argument("--density", type=float, default=1.0, help="x density (c2, rmat22)")
    ap.add_argument("--nnz-x", type=int, default=2000, help="sample-row nnz (c4)")
    a = ap.parse_args()
    ctx = A.Context(0)
    keep = None
    if a.input == "c2":
        rows, cols, ro, ci, vals = synth.uniform_random(1 << 22, 1 << 26, seed=1, dtype=np.float32)
        m = A.DualMatrix.from_csr(rows, cols, ro, ci, vals, ctx=ctx)
    else:
        from paper_2006_16767_b200 import synth_device as SD
        if a.input in ("rmat22", "rmat26"):
            n, ro, ci = SD.rmat_device(26 if a.input == "rmat26" else 22)
            rows = cols = n
            vals = torch.rand(ci.numel(), device="cuda", dtype=torch.float32) + 0.5
        elif a.input == "c4":
            rows, cols = 10_000_000, 2_000_000
            ro, ci, vals, draw = SD.svm_device(rows, cols, 20, 1.0, 3)
        else:
            raise SystemExit(f"unknown input {a.input}")
        torch.cuda.synchronize()
        m = A.DualMatrix.from_device(rows, cols, ci.numel(), ro.data_ptr(), ci.data_ptr(), vals.data_ptr(),
                                     np.float32, ctx)
        ctx.synchronize()
        keep = (ro, ci, vals)
    x = A.DeviceVector(cols, np.float32, ctx)
    if a.input == "c4":
        xi, xv = SD.svm_vector(draw, cols, a.nnz_x, seed=a.nnz_x)
        xi = xi.cpu().numpy() if hasattr(xi, "cpu") else xi
        xv = xv.cpu().numpy() if hasattr(xv, "cpu") else xv
        x.set_sparse(xi, xv)
    else:
        nx = max(1, int(round(a.density * cols)))
        xi, xv = synth.sparse_vector(cols, nx, seed=9, dtype=np.float32)
        if nx == cols:
            d = np.zeros(cols, np.float32)
            d[xi] = xv
            x.set_dense(d)
        else:
            x.set_sparse(xi, xv)
    out = A.MultiplyOutput(ctx)
    x.prepare(a.kernel)
    A.run_kernel(m, a.kernel, x, out=out)
    ctx.synchronize()
    torch.cuda.nvtx.range_push("measure")
    A.run_kernel(m, a.kernel, x, out=out)
    ctx.synchronize()
    torch.cuda.nvtx.range_pop()
    del keep
    print(f"ok {a.input} kernel {a.kernel}")


if __name__ == "__main__":
    main()

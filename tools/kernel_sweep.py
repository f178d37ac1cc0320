"""Device time of chosen kernels on the BASELINE inputs, for tuning
(lanes_per_row sweep of the direct kernels, LB vs direct).  Prints a table.

  python tools/kernel_sweep.py --inputs c2,c1,rmat20 --kernels 0,1,4,6 --lanes 0,2,4,8,16
"""
import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2006_16767_b200 import adaspmv as A  # noqa: E402
from paper_2006_16767_b200 import synth  # noqa: E402

INPUTS = {
    "c1": lambda: synth.laplacian_2d(1000, dtype=np.float64),
    "c2": lambda: synth.uniform_random(1 << 22, 1 << 26, seed=1, dtype=np.float32),
    "rmat20": lambda: synth.rmat(20, 16, seed=23, values="uniform"),
    "rmat22": lambda: synth.rmat(22, 16, seed=2, values="uniform"),
}


def main():
    import torch
    ap = argparse.ArgumentParser()
    ap.add_argument("--inputs", default="c2,c1")
    ap.add_argument("--kernels", default="0,1")
    ap.add_argument("--lanes", default="0")
    ap.add_argument("--densities", default="1.0")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--layouts", default="0", help="row_layout values for K0/K2 (0 auto, 1 csr, 2 bins)")
    ap.add_argument("--bin-rows", default="0", help="bin_rows overrides (rows per bin, 0 = auto)")
    ap.add_argument("--tile-nnz", type=int, default=0, help="bin_tile_nnz override (0 = auto)")
    a = ap.parse_args()
    ctx = A.Context(0)
    ctx.set_timing(True)
    stream = torch.cuda.ExternalStream(ctx.stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    out = A.MultiplyOutput(ctx)
    for name in a.inputs.split(","):
        rows, cols, ro, ci, vals = INPUTS[name]()
        m = A.DualMatrix.from_csr(rows, cols, ro, ci, vals, ctx=ctx)
        hbm = 6532.9e9
        for dens in [float(s) for s in a.densities.split(",")]:
            nx = max(1, int(round(dens * cols)))
            xi, xv = synth.sparse_vector(cols, nx, seed=9, dtype=vals.dtype)
            x = A.DeviceVector(cols, vals.dtype, ctx)
            if nx == cols:
                d = np.zeros(cols, vals.dtype)
                d[xi] = xv
                x.set_dense(d)
            else:
                x.set_sparse(xi, xv)
            V = vals.dtype.itemsize
            b_spmv = (rows + 1) * 8 + ro[-1] * (4 + V) + cols * V + rows * V
            yfirst = None
            for k in [int(s) for s in a.kernels.split(",")]:
                for lanes, lay, br in [(int(s), int(l), int(b)) for s in a.lanes.split(",")
                                       for l in a.layouts.split(",") for b in a.bin_rows.split(",")]:
                    x.prepare(k)
                    cfg = A.KernelConfig(lanes_per_row=lanes, row_layout=lay, bin_rows=br, bin_tile_nnz=a.tile_nnz)
                    A.run_kernel(m, k, x, cfg, out=out)
                    y = out.dense().values.astype(np.float64)
                    if yfirst is None:
                        yfirst = y
                    dev = float(np.max(np.abs(y - yfirst)) / max(np.max(np.abs(yfirst)), 1e-300))
                    ts = []
                    for _ in range(a.reps):
                        with torch.cuda.stream(stream):
                            flush.add_(1)
                            torch.cuda._sleep(400_000)
                        A.run_kernel(m, k, x, cfg, out=out)
                        ts.append(out.elapsed())
                    t = float(np.median(ts))
                    print(f"{name:7s} x={dens:<8g} k={k} lanes={lanes:2d} layout={lay} bin_rows={br} {t * 1e6:9.2f} us  "
                          f"maxdev={dev:.1e} "
                          f"B_spmv/t={b_spmv / t / 1e9:8.1f} GB/s ({100 * b_spmv / t / hbm:5.1f}% of HBM)",
                          flush=True)


if __name__ == "__main__":
    main()

"""A/B of the row-bin K0 kernels (bin_cluster 1 = register-streaming,
3 = warp-specialised bulk-copy ring) on C2 / R-MAT inputs: device time
(library events), agreement of the two results, and vs the CSR kernel.
  python tools/ws_ab.py [c2,rmat22] [densities]"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2006_16767_b200 import adaspmv as A  # noqa: E402
from paper_2006_16767_b200 import synth  # noqa: E402

INPUTS = {
    "c2": lambda: synth.uniform_random(1 << 22, 1 << 26, seed=1, dtype=np.float32),
    "rmat20": lambda: synth.rmat(20, 16, seed=23, values="uniform"),
    "rmat22": lambda: synth.rmat(22, 16, seed=2, values="uniform"),
    "c2f64": lambda: synth.uniform_random(1 << 22, 1 << 26, seed=1, dtype=np.float64),
}
names = (sys.argv[1] if len(sys.argv) > 1 else "c2").split(",")
dens = [float(d) for d in (sys.argv[2] if len(sys.argv) > 2 else "1.0").split(",")]
ctx = A.Context(0)
ctx.set_timing(True)
stream = torch.cuda.ExternalStream(ctx.stream)
out = A.MultiplyOutput(ctx)
for name in names:
    rows, cols, ro, ci, vals = INPUTS[name]()
    m = A.DualMatrix.from_csr(rows, cols, ro, ci, vals, ctx=ctx)
    V = vals.dtype.itemsize
    b_spmv = (rows + 1) * 8 + ro[-1] * (4 + V) + cols * V + rows * V
    for d in dens:
        nx = max(1, int(round(d * cols)))
        xi, xv = synth.sparse_vector(cols, nx, seed=9, dtype=vals.dtype)
        xd = np.zeros(cols, vals.dtype)
        xd[xi] = xv
        x = A.DeviceVector(cols, vals.dtype, ctx).set_dense(xd)
        ys = {}
        for label, cfg in (("csr", A.KernelConfig(row_layout=1)),
                           ("bins-regs", A.KernelConfig(row_layout=2, bin_cluster=1)),
                           ("bins-ws", A.KernelConfig(row_layout=2, bin_cluster=3))):
            try:
                A.run_kernel(m, 0, x, cfg, out=out)
            except Exception as e:  # noqa: BLE001
                print(f"{name} x={d} {label}: {e}")
                continue
            ts = []
            for _ in range(7):
                with torch.cuda.stream(stream):
                    torch.cuda._sleep(400_000)
                A.run_kernel(m, 0, x, cfg, out=out)
                ts.append(out.elapsed())
            ys[label] = out.dense().values.astype(np.float64)
            t = float(np.median(ts))
            print(f"{name} x={d} {label:10s} {t * 1e6:8.1f} us  {b_spmv / t / 6554.2e9 * 100:5.1f} % of HBM (B_spmv)",
                  flush=True)
        if "bins-ws" in ys:
            ref = ys["csr"]
            for k, v in ys.items():
                tol = 1e-4 * (np.abs(ref).max() + 1e-30)
                print(f"   {k}: max|y - y_csr| = {np.abs(v - ref).max():.3e} (scale {np.abs(ref).max():.3e})")

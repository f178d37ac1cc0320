"""Device time of binned K0 on C2 vs rows per bin, tile cap and CTAs per bin
tile (tuning aid).   python tools/bin_rows_sweep.py 0:0:1,0:0:2,57344:0:1 """
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2006_16767_b200 import adaspmv as A, synth  # noqa: E402

ctx = A.Context(0)
ctx.set_timing(True)
rows, cols, ro, ci, vals = synth.uniform_random(1 << 22, 1 << 26, seed=1, dtype=np.float32)
m = A.DualMatrix.from_csr(rows, cols, ro, ci, vals, ctx=ctx)
xd = np.random.default_rng(0).uniform(-1, 1, cols).astype(np.float32)
x = A.DeviceVector(cols, np.float32, ctx).set_dense(xd)
out = A.MultiplyOutput(ctx)
stream = torch.cuda.ExternalStream(ctx.stream)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ref = None
for spec in (sys.argv[1] if len(sys.argv) > 1 else "0:0").split(","):
    r, c, cl = (int(v) for v in spec.split(":"))
    cfg = A.KernelConfig(row_layout=2, bin_rows=r, bin_tile_nnz=c, bin_cluster=cl)
    y = A.run_kernel(m, 0, x, cfg, out=out).dense().values.astype(np.float64)
    ref = y if ref is None else ref
    ts = []
    for _ in range(9):
        with torch.cuda.stream(stream):
            flush.add_(1)
            torch.cuda._sleep(400_000)
        A.run_kernel(m, 0, x, cfg, out=out)
        ts.append(out.elapsed())
    print(f"bin_rows {r:7d} tile_cap {c:8d} cluster {cl}: {np.median(ts) * 1e6:7.1f} us  max|dy| {np.abs(y - ref).max():.2e}",
          flush=True)

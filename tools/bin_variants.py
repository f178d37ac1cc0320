"""Device time of the binned K0 variants on C2 (tuning aid)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2006_16767_b200 import adaspmv as A, synth  # noqa: E402

ctx = A.Context(0)
ctx.set_timing(True)
rows, cols, ro, ci, vals = synth.uniform_random(1 << 22, 1 << 26, seed=1, dtype=np.float32)
m = A.DualMatrix.from_csr(rows, cols, ro, ci, vals, ctx=ctx)
x = A.DeviceVector(cols, np.float32, ctx).set_dense(np.random.default_rng(0).uniform(-1, 1, cols).astype(np.float32))
out = A.MultiplyOutput(ctx)
stream = torch.cuda.ExternalStream(ctx.stream)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
variants = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "0,1,2,3,4").split(",")]
for var in variants:
    cfg = A.KernelConfig(row_layout=2, lanes_per_row=var)
    A.run_kernel(m, 0, x, cfg, out=out)
    ts = []
    for _ in range(7):
        with torch.cuda.stream(stream):
            flush.add_(1)
            torch.cuda._sleep(400_000)
        A.run_kernel(m, 0, x, cfg, out=out)
        ts.append(out.elapsed())
    print("variant", var, "%.1f us" % (np.median(ts) * 1e6), flush=True)

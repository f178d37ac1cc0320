"""K0 (row bins) and K1 (LB) device time on R-MAT graphs generated on the
device (scales from argv), x = 100 % / 50 % / 10 %, y checked K0 vs K1.

  python tools/rmat_spmv_probe.py 22 26
"""
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2006_16767_b200 import adaspmv as A  # noqa: E402
from paper_2006_16767_b200 import synth_device as SD  # noqa: E402


def main():
    import os
    panels = [int(v) for v in os.environ.get("PANELS_KIB", "0").split(",")]
    for scale in [int(a) for a in sys.argv[1:]] or [22]:
        ctx = A.Context(0)
        n, ro, ci = SD.rmat_device(scale)
        vals = torch.rand(ci.numel(), device="cuda", dtype=torch.float32) + 0.5
        torch.cuda.synchronize()
        m = A.DualMatrix.from_device(n, n, ci.numel(), ro.data_ptr(), ci.data_ptr(), vals.data_ptr(), np.float32, ctx)
        ctx.synchronize()
        del ro, ci, vals
        torch.cuda.empty_cache()
        ctx.set_timing(True)
        stream = torch.cuda.ExternalStream(ctx.stream)
        out = A.MultiplyOutput(ctx)
        for d in (1.0, 0.5, 0.1):
            g = torch.Generator(device="cuda")
            g.manual_seed(3)
            xd = (torch.rand(n, generator=g, device="cuda") < d).float() * (torch.rand(n, generator=g, device="cuda") + 0.5)
            x = A.DeviceVector(n, np.float32, ctx)
            x.set_dense_device(xd.data_ptr())
            ys, ts, names = [], [], []
            for k, pk in [(0, pk) for pk in panels] + [(1, 0)]:
                cfg = A.KernelConfig(bin_panel_kib=pk)
                x.prepare(k)
                A.run_kernel(m, k, x, cfg, out=out)
                t = []
                for _ in range(5):
                    with torch.cuda.stream(stream):
                        torch.cuda._sleep(400_000)
                    A.run_kernel(m, k, x, cfg, out=out)
                    t.append(out.elapsed())
                ts.append(statistics.median(t))
                names.append(f"K{k}" + (f"/panel {pk} KiB" if pk else ""))
                ys.append(out.dense().values.astype(np.float64))
            dev = max(float(np.max(np.abs(y - ys[-1]) / (np.abs(ys[-1]) + 1e-3))) for y in ys)
            print(f"rmat{scale} x={d}: " + "  ".join(f"{nm} {t * 1e6:9.1f} us" for nm, t in zip(names, ts))
                  + f"  max rel dev {dev:.1e}", flush=True)
        del m, out, x, ctx
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

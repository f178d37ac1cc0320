"""Where the end-to-end time of one C2 sweep step goes (bench.py e2e leg):
per point, host wall time of set_{sparse,dense} (H2D + validation), the
adaptive select + run, and the result read (D2H), plus raw pinned copy
bandwidth for reference.   python tools/e2e_profile.py"""
import ctypes as C
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2006_16767_b200 import adaspmv as A  # noqa: E402
from paper_2006_16767_b200 import selector as S  # noqa: E402


def main():
    (rows, cols, ro, ci, vals), _ = bench.make_matrix()
    ctx = A.Context(0)
    m = A.DualMatrix.from_csr(rows, cols, ro, ci, vals, ctx=ctx)
    bundle = A.SelectorBundle.load(S.DEFAULT_PATH)
    vecs = bench.make_vectors(cols)
    out = A.MultiplyOutput(ctx)
    x = A.DeviceVector(cols, np.float32, ctx)
    pinned = []
    for xi, xv in vecs:
        if len(xi) == cols:
            d = torch.zeros(cols, dtype=torch.float32).pin_memory()
            d[torch.from_numpy(xi)] = torch.from_numpy(xv)
            pinned.append(("dense", d.numpy()))
        else:
            pinned.append(("sparse", (torch.from_numpy(xi).pin_memory().numpy(),
                                      torch.from_numpy(xv).pin_memory().numpy())))
    ybuf = torch.zeros(rows, dtype=torch.float32).pin_memory().numpy()
    yidx = torch.zeros(rows, dtype=torch.int64).pin_memory().numpy()
    # raw copy bandwidth
    dev = torch.empty(rows, dtype=torch.float32, device="cuda")
    hst = torch.zeros(rows, dtype=torch.float32).pin_memory()
    for name, fn in (("h2d", lambda: dev.copy_(hst, non_blocking=True)), ("d2h", lambda: hst.copy_(dev, non_blocking=True))):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(20):
            fn()
        torch.cuda.synchronize()
        print(f"raw pinned {name}: {20 * rows * 4 / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
    for rep in range(4):
        tot = 0
        line = []
        for i, (kind, payload) in enumerate(pinned):
            t0 = time.perf_counter()
            if kind == "dense":
                x.set_dense(payload)
            else:
                x.set_sparse(*payload)
            ctx.synchronize()
            t1 = time.perf_counter()
            y, k = A.run_adaptive(m, x, bundle, out=out)
            ctx.synchronize()
            t2 = time.perf_counter()
            ns = A.effective_nnz(m, x)
            if k.index() in (5, 7) or 4 * ns < rows:
                ny = C.c_int64()
                A._check(A._lib.adaspmv_output_sparse(ctx.h, y.h, rows, A._ptr(yidx), A._ptr(ybuf), C.byref(ny)))
            else:
                A._check(A._lib.adaspmv_output_dense(ctx.h, y.h, A._ptr(ybuf)))
            t3 = time.perf_counter()
            tot += t3 - t0
            line.append(f"{kind[0]} set {1e3 * (t1 - t0):6.3f} run {1e3 * (t2 - t1):6.3f} get {1e3 * (t3 - t2):6.3f}")
        if rep == 3:
            print("\n".join(line))
            print(f"step {1e3 * tot:.3f} ms")


if __name__ == "__main__":
    main()

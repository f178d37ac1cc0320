"""Timeline of one end-to-end C2 sweep through adaspmv_run_batch (the bench's
e2e leg) with ADASPMV_BATCH_TRACE=1, and the step time for several lane
counts.

  python tools/e2e_trace.py
"""
import os
import statistics
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
    ctx = A.Context(0)
    (rows, cols, ro, ci, vals), _ = bench.make_matrix()
    m = A.DualMatrix.from_csr(rows, cols, ro, ci, vals, ctx=ctx)
    bundle = A.SelectorBundle.load(S.DEFAULT_PATH)
    vecs = bench.make_vectors(cols)
    pinned = []
    for xi, xv in vecs:
        if len(xi) == cols:
            d = torch.zeros(cols, dtype=torch.float32).pin_memory()
            d[torch.from_numpy(xi)] = torch.from_numpy(xv)
            pinned.append(d.numpy())
        else:
            pinned.append((torch.from_numpy(xi).pin_memory().numpy(), torch.from_numpy(xv).pin_memory().numpy()))
    bufs = [(torch.zeros(rows, dtype=torch.int64).pin_memory().numpy(),
             torch.zeros(rows, dtype=torch.float32).pin_memory().numpy()) for _ in pinned]
    flops = None
    for lanes in (1, 2, 3, 4, 7):
        ts = []
        for it in range(8):
            t0 = time.perf_counter()
            res = A.run_batch(m, pinned, bundle=bundle, form=A.RESULT_AUTO, lanes=lanes, buffers=bufs)
            ts.append(time.perf_counter() - t0)
        print(f"lanes {lanes}: {statistics.median(ts[3:]) * 1e3:.3f} ms per sweep  kernels "
              f"{[r.kernel.index() for r in res]}  forms {['S' if r.is_sparse else 'D' for r in res]}", flush=True)
    os.environ["ADASPMV_BATCH_TRACE"] = "1"
    A.run_batch(m, pinned, bundle=bundle, form=A.RESULT_AUTO, lanes=3, buffers=bufs)


if __name__ == "__main__":
    main()

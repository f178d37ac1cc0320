"""Where the C3 BFS wall time goes (R-MAT 22, OR_AND, source 0): wall per call
for several report sizes, device time per level, launches per call.

  python tools/bfs_probe.py
"""
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
    n, ro, ci, _ = bench.c3_inputs()
    nnz = int(ro[-1].item())
    ctx = A.Context(0)
    m = A.DualMatrix.from_device(n, n, nnz, ro.data_ptr(), ci.data_ptr(), None, np.float32, ctx)
    ctx.synchronize()
    del ro, ci
    torch.cuda.empty_cache()
    bundle = A.SelectorBundle.load(S.DEFAULT_PATH)
    q = None
    for host_loop in (True, False):
      ctx.set_bfs_loop(host_loop)
      lv, _ = A.bfs(m, 0, A.OR_AND, bundle=bundle)
      if q is None:
          q = lv
      print(f"== host_loop={host_loop} levels identical to the host loop: {bool(np.array_equal(lv, q))}")
      for name, kw in (("selector", dict(bundle=bundle)), ("heuristic", {})):
        for mr in (4096, 16):
            A.bfs(m, 0, A.OR_AND, max_reports=mr, download_levels=False, **kw)
            walls = []
            for _ in range(7):
                ctx.synchronize()
                l0 = ctx.launches
                t1 = time.perf_counter()
                _, rep = A.bfs(m, 0, A.OR_AND, max_reports=mr, download_levels=False, **kw)
                walls.append(time.perf_counter() - t1)
                nl = ctx.launches - l0
            dev = sum(r["kernel_s"] + r["convert_s"] for r in rep)
            print(f"{name:9s} max_reports={mr:5d} wall {statistics.median(walls) * 1e3:.3f} ms  device {dev * 1e3:.3f} ms"
                  f"  launches {nl}  levels {len(rep)}")
        for r in rep:
          if True:
            print(f"   level {r['iteration']} nnz_x {r['nnz_x']:>8d} k {r['kernel']} mode {r['exec_mode']} "
                  f"predict {r['predict_s'] * 1e6:6.1f} us convert {r['convert_s'] * 1e6:6.1f} kernel {r['kernel_s'] * 1e6:7.1f}")


if __name__ == "__main__":
    main()

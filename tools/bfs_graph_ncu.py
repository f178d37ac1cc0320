"""One device-loop (graph) BFS on C3 inside an NVTX range, for an ncu launch list."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2006_16767_b200 import adaspmv as A  # noqa: E402

n, ro, ci, _ = bench.c3_inputs()
ctx = A.Context(0)
m = A.DualMatrix.from_device(n, n, int(ro[-1].item()), ro.data_ptr(), ci.data_ptr(), None, np.float32, ctx)
ctx.synchronize()
ctx.set_bfs_loop(sys.argv[1] == "host" if len(sys.argv) > 1 else False)
A.bfs(m, 0, A.OR_AND, download_levels=False)
ctx.synchronize()
torch.cuda.nvtx.range_push("measure")
A.bfs(m, 0, A.OR_AND, download_levels=False)
ctx.synchronize()
torch.cuda.nvtx.range_pop()

"""GPU: the row-partitioned mode's CUDA shard on one device (world size 1 over
NCCL) -- the broadcast lands in device buffers handed to the library by
pointer, y comes back as a torch view of the library's output."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

from paper_2006_16767_b200 import adaspmv as A
from paper_2006_16767_b200 import multigpu as MG
from paper_2006_16767_b200 import synth
from tests.util import assert_dense_close, ref_and_bound

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pg():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


def test_cuda_shard_multiply_and_bfs(pg, port):
    rows, cols, ro, ci, vals = synth.random_csr(3000, 2500, 0.004, seed=3, dtype=np.float32)
    for kernel in (None, 1, 4, 7):
        rp = MG.RowPartitioned.create(rows, cols, ro, ci, vals,
                                      lambda r, c, a, b, v: MG.CudaShard(r, c, a, b, v, 0, kernel=kernel),
                                      "cuda")
        xd = np.random.default_rng(1).uniform(-1, 1, cols).astype(np.float32)
        y = rp.multiply(x_dense=xd, gather=True).cpu().numpy()
        y_ref, bound = ref_and_bound(port, rows, ro, ci, vals, xd)
        assert_dense_close(y, y_ref, bound, np.float32, f"dense kernel={kernel}")
        xi, xv = synth.sparse_vector(cols, 40, seed=2, dtype=np.float32)
        y = rp.multiply(x_sparse=(xi, xv)).cpu().numpy()
        y_ref, bound = ref_and_bound(port, rows, ro, ci, vals, port.sparse_to_dense(cols, xi, xv))
        assert_dense_close(y, y_ref, bound, np.float32, f"sparse kernel={kernel}")
    n, _, gro, gci, gv = synth.rmat(11, 8, seed=5)
    g = MG.RowPartitioned.create(n, n, gro, gci, gv, lambda r, c, a, b, v: MG.CudaShard(r, c, a, b, v, 0, kernel=3),
                                 "cuda")
    levels, _ = g.bfs(0, A.OR_AND)
    co, ri, _ = port.csr_to_csc(n, n, gro, gci, np.ones(len(gci)))
    exp, _ = port.bfs_queue(n, co, ri, 0)
    assert np.array_equal(levels, exp)

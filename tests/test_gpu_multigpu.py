"""GPU: paper_2006_16767_b200/multigpu.py on one device over the NCCL backend
(world size 1): the library's NCCL transport (uid handed over by
torch.distributed), x broadcast into the library's operand, per-rank
selection, y all-gathered into a device tensor, and the library's dist BFS."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

from paper_2006_16767_b200 import adaspmv as A
from paper_2006_16767_b200 import multigpu as MG
from paper_2006_16767_b200 import selector as S
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


def test_row_block_matrix_nccl_world1(pg, port):
    rows, cols, ro, ci, vals = synth.random_csr(3000, 2500, 0.004, seed=3, dtype=np.float32)
    bundle = A.SelectorBundle.load(S.DEFAULT_PATH)
    rp = MG.RowBlockMatrix(rows, cols, ro, ci, vals, 0, bundle=bundle)
    xd = np.random.default_rng(1).uniform(-1, 1, cols).astype(np.float32)
    y_ref, bound = ref_and_bound(port, rows, ro, ci, vals, xd)
    xi, xv = synth.sparse_vector(cols, 40, seed=2, dtype=np.float32)
    ys_ref, sbound = ref_and_bound(port, rows, ro, ci, vals, port.sparse_to_dense(cols, xi, xv))
    for kernel in (None, 1, 4, 7):
        y = rp.multiply(x_dense=xd, gather=True, kernel=kernel).cpu().numpy()
        assert_dense_close(y, y_ref, bound, np.float32, f"dense kernel={kernel}")
        y = rp.multiply(x_sparse=(xi, xv), kernel=kernel).cpu().numpy()
        assert_dense_close(y, ys_ref, sbound, np.float32, f"sparse kernel={kernel}")
    rp.close()
    n, _, gro, gci, _ = synth.rmat(11, 8, seed=5)
    g = MG.RowBlockMatrix(n, n, gro, gci, None, 0, dtype=np.float32)
    co, ri, _ = port.csr_to_csc(n, n, gro, gci, np.ones(len(gci)))
    exp, nl = port.bfs_queue(n, co, ri, 0)
    for kernel in (-1, 3, 6):
        levels, nl2, _ = g.bfs(0, A.OR_AND, kernel=kernel)
        assert np.array_equal(levels, exp) and nl2 == nl, kernel
    g.close()

"""Multi-GPU layer (paper_1710_08538_b200/mg.py).

CPU (gloo, world size 2): the row partition and the slab all-gather.
GPU (one device): the sharded compute path -- every "rank" computes H, T in full and its
row slab of Q, Z (ht_options.row_begin/row_end); the assembled slabs must equal the
single-call Q, Z bitwise (rows of Q and Z are independent under right multiplication,
PAPER.md P:886).
"""
import os

import numpy as np
import pytest

import ht_inputs
from paper_1710_08538_b200 import mg


@pytest.mark.parametrize("n,world", [(0, 1), (1, 3), (7, 2), (100, 8), (8192, 8), (16384, 3)])
def test_row_range_partition(n, world):
    rs = [mg.row_range(n, world, r) for r in range(world)]
    assert rs[0][0] == 0 and rs[-1][1] == n
    for (b0, e0), (b1, e1) in zip(rs, rs[1:]):
        assert e0 == b1 and b0 <= e0
    sizes = [e - b for b, e in rs]
    assert max(sizes) - min(sizes) <= 1


def _gather_worker(rank, world, port, n, out):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # column-major M held as t = M^T; rank r knows only its rows of M (columns of t)
    full = torch.arange(n * n, dtype=torch.float64).reshape(n, n)
    t = torch.full((n, n), -1.0, dtype=torch.float64)
    b, e = mg.row_range(n, world, rank)
    t[:, b:e] = full[:, b:e]
    mg.gather_rows(t, n, world, rank)
    out[rank] = bool(torch.equal(t, full))
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [5, 64])
def test_gather_rows_gloo_world2(n):
    import socket
    import torch.multiprocessing as tmp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mgr = tmp.Manager()
    out = mgr.dict()
    tmp.spawn(_gather_worker, args=(2, port, n, out), nprocs=2, join=True)
    assert out[0] and out[1]


@pytest.mark.gpu
@pytest.mark.parametrize("world,n,nb", [(2, 300, 32), (3, 257, 16), (4, 130, 64)])
def test_sharded_qz_slabs_match_single_call(world, n, nb):
    torch = pytest.importorskip("torch")
    from test_gpu import gpu_reduce, from_dev
    A, B = ht_inputs.pencil("qrnormal", n, 11 + world)
    H, T, Q, Z, _ = gpu_reduce(A, B, nb=nb)
    Qs, Zs = np.zeros_like(Q), np.zeros_like(Z)
    for r in range(world):
        b, e = mg.row_range(n, world, r)
        Hr, Tr, Qr, Zr, _ = gpu_reduce(A, B, nb=nb, row_range=(b, e))
        assert np.array_equal(Hr, H) and np.array_equal(Tr, T)  # replicated part: bitwise
        Qs[b:e], Zs[b:e] = Qr[b:e], Zr[b:e]
    assert np.array_equal(Qs, Q) and np.array_equal(Zs, Z)

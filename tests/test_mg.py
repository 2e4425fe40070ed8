"""Multi-GPU layer (ht_reduce_mg, paper_1710_08538_b200/mg.py).

CPU (gloo, world size 2): the library's slab partition as every rank sees it (disjoint,
covering, balanced) and the NCCL-id bootstrap of mg.init_comm.
GPU (one device): the sharded compute path in LOOPBACK mode -- ht_reduce_mg with no
communicator plays P ranks on one GPU (A's right-hand applies on row slabs, left-hand
applies on column slabs, the packed all-gathers of both layout switches, Q/Z row slabs
and their final gather); the result must equal the single-GPU call bitwise, because every
element receives the same transforms in the same order (rows/columns are independent
under right/left multiplication, PAPER.md eq. commuteQ, commuteQ2 P:1083-1134).
"""
import os

import numpy as np
import pytest

import ht_inputs
import paper_1710_08538_b200 as ht
from paper_1710_08538_b200 import mg


@pytest.mark.parametrize("n,world", [(0, 1), (1, 3), (7, 2), (100, 8), (8192, 8), (16384, 3)])
def test_row_range_partition(n, world):
    rs = [mg.row_range(n, world, r) for r in range(world)]
    assert rs[0][0] == 0 and rs[-1][1] == n
    for (b0, e0), (b1, e1) in zip(rs, rs[1:]):
        assert e0 == b1 and b0 <= e0
    sizes = [e - b for b, e in rs]
    assert max(sizes) - min(sizes) <= 1
    # the library's partition (used for A, Q, Z slabs) is the same
    assert rs == [ht.ht_mg_slab(0, n, world, r) for r in range(world)]


def test_slab_argument_errors():
    with pytest.raises(ht.HTError):
        ht.ht_mg_slab(0, 10, 0, 0)
    with pytest.raises(ht.HTError):
        ht.ht_mg_slab(0, 10, 2, 2)


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # every rank's view of the slabs of one absorption (rows [0, n), columns [J, n))
    n, J = 1000, 379
    mine = {"rows": ht.ht_mg_slab(0, n, world, rank), "cols": ht.ht_mg_slab(J, n, world, rank)}
    allv = [None] * world
    dist.all_gather_object(allv, mine)
    ok = True
    for key, (b, e) in (("rows", (0, n)), ("cols", (J, n))):
        cover = np.zeros(e - b, dtype=int)
        for v in allv:
            lo, hi = v[key]
            cover[lo - b:hi - b] += 1
        ok &= bool(np.all(cover == 1))
    # NCCL bootstrap: rank 0's unique id (from the library) reaches every rank unchanged
    uid = mg.share_unique_id()
    ids = [None] * world
    dist.all_gather_object(ids, uid)
    ok &= len(uid) == 128 and all(x == ids[0] for x in ids)
    out[rank] = ok
    dist.destroy_process_group()


def test_partition_and_bootstrap_gloo_world2():
    import torch.multiprocessing as tmp
    mgr = tmp.Manager()
    out = mgr.dict()
    tmp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    assert out[0] and out[1]


@pytest.mark.gpu
@pytest.mark.parametrize("world,n,nb,kind", [(2, 300, 32, "qrnormal"), (3, 257, 16, "qruniform"),
                                             (4, 700, 64, "shifted"), (2, 1100, 128, "qruniform")])
def test_loopback_sharded_path_matches_single_call(world, n, nb, kind):
    torch = pytest.importorskip("torch")
    from test_gpu import gpu_reduce, to_dev, from_dev
    A, B = ht_inputs.pencil(kind, n, 11 + world)
    H, T, Q, Z, rep1 = gpu_reduce(A, B, nb=nb)
    dA, dB = to_dev(A), to_dev(B)
    dQ, dZ = torch.empty_like(dA), torch.empty_like(dA)
    rep = mg.reduce_mg(dA, dB, dQ, dZ, nb=nb, comm=None, world=world)
    torch.cuda.synchronize()
    for X, t in ((H, dA), (T, dB), (Q, dQ), (Z, dZ)):
        assert np.array_equal(X, from_dev(t))
    assert rep["flops"] == pytest.approx(rep1["flops"], rel=1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("world,n,nb", [(2, 300, 32), (3, 257, 16), (4, 130, 64)])
def test_sharded_qz_slabs_match_single_call(world, n, nb):
    torch = pytest.importorskip("torch")
    from test_gpu import gpu_reduce
    A, B = ht_inputs.pencil("qrnormal", n, 11 + world)
    H, T, Q, Z, _ = gpu_reduce(A, B, nb=nb)
    Qs, Zs = np.zeros_like(Q), np.zeros_like(Z)
    for r in range(world):
        b, e = mg.row_range(n, world, r)
        Hr, Tr, Qr, Zr, _ = gpu_reduce(A, B, nb=nb, row_range=(b, e))
        assert np.array_equal(Hr, H) and np.array_equal(Tr, T)  # replicated part: bitwise
        Qs[b:e], Zs[b:e] = Qr[b:e], Zr[b:e]
    assert np.array_equal(Qs, Q) and np.array_equal(Zs, Z)

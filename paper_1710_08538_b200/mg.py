"""Multi-GPU HouseHT: one process per GPU of one node.

Argument marshalling over the C ABI's ht_reduce_mg (include/ht.h): every rank passes its
own device buffers and an NCCL communicator built by the library's NCCL bootstrap
(ht_nccl_unique_id on rank 0 -> torch.distributed broadcast of the 128 id bytes ->
ht_nccl_comm_init on every rank).  The sharding lives in the library:
  * A, B replicated on entry; the panel, B and the staircase factorizations are
    computed redundantly (bitwise identical on every rank);
  * A's right-hand applies (R2, R3, Remark 2) on row slabs, its left-hand applies (L2,
    L3) on column slabs, one packed ncclAllGather per layout switch (twice per absorption);
  * Q and Z (right multiplications only) on row slabs,
    all-gathered at the end.
torch.distributed is plumbing here (process group for the id broadcast); the data path
collectives are the library's NCCL calls on the reduction's stream.
"""
from __future__ import annotations


def row_range(n: int, world: int, rank: int):
    """Balanced contiguous split of rows [0, n) over `world` ranks: (begin, end) of `rank`
    (the same partition as the library's ht_mg_slab; tests check they agree)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def share_unique_id(group=None) -> bytes:
    """Collective: rank 0's NCCL unique id (from the library) on every rank of the group."""
    import torch.distributed as dist
    import paper_1710_08538_b200 as ht
    obj = [ht.ht_nccl_unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def init_comm(group=None):
    """Collective: an NCCL communicator over the ranks of the torch.distributed group (one
    per process/GPU), created by the library.  Returns (comm, rank, world)."""
    import torch.distributed as dist
    import paper_1710_08538_b200 as ht
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    uid = share_unique_id(group)
    return ht.ht_nccl_comm_init(world, uid, rank), rank, world


def layout(A, B, Q=None, Z=None, gather_qz=True):
    """ht_mg_layout of torch CUDA tensors holding column-major n x n matrices (t = M^T)."""
    import paper_1710_08538_b200 as ht
    n = A.shape[0]
    p = lambda t: t.data_ptr() if t is not None else None
    return ht.HTMgLayout(p(A), n, p(B), n, p(Q), n, p(Z), n, int(bool(gather_qz)))


def reduce_mg(A, B, Q=None, Z=None, nb=0, comm=None, rank=0, world=1, stream=None, gather=True, **kw):
    """Collective HT reduction of the replicated device pencil A, B (torch CUDA tensors,
    t = M^T).  comm None with world > 1 runs the loopback mode (all ranks on this GPU).
    Returns the report."""
    import paper_1710_08538_b200 as ht
    if stream is None:
        import torch
        stream = torch.cuda.current_stream().cuda_stream
    n = A.shape[0]
    opt = ht.make_options(nb=nb, stream=stream, **kw)
    return ht.ht_reduce_mg(n, layout(A, B, Q, Z, gather), comm, rank, world, Q is not None, Z is not None, opt)

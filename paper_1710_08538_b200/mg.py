"""Multi-GPU HouseHT: one process per GPU of one node, torch.distributed (NCCL) process group.

Layout:
  * A and B are replicated.  Every rank runs the panel (sec. 3.2), the staircase
    factorizations and all updates of A and B (sec. 3.3).  The kernels are deterministic,
    so H and T come out bitwise identical on every rank.
  * Q and Z are split into contiguous row slabs.  They only ever receive right
    multiplications (Q(:, .) <- Q * (window transforms); Z likewise,
    P:886), so their rows are independent: rank r computes rows row_range(n, P, r)
    and nothing crosses the network until the final all-gather of the slabs (C6).
  * The panel, the factorization chains and the A/B updates are not sharded ("replicas"):
    the B-solve is a sequential chain and sharding A's right/left chains
    needs a layout switch per absorption (future work).

The product path is the C ABI (ht_reduce_ex with ht_options.row_begin/row_end); this
module only marshals arguments and runs the collective.
"""
from __future__ import annotations


def row_range(n: int, world: int, rank: int):
    """Balanced contiguous split of rows [0, n) over `world` ranks: (begin, end) of `rank`."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def gather_rows(t, n: int, world: int, rank: int, group=None):
    """All-gather the row slabs of a column-major n x n matrix M held as the torch tensor
    t = M^T (so rows of M are columns of t).  In place; returns t."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return t
    ranges = [row_range(n, world, r) for r in range(world)]
    width = max(e - b for b, e in ranges)
    b0, e0 = ranges[rank]
    send = torch.zeros((n, width), dtype=t.dtype, device=t.device)
    send[:, : e0 - b0] = t[:, b0:e0]
    recv = [torch.empty_like(send) for _ in range(world)]
    dist.all_gather(recv, send, group=group)
    for r, (b, e) in enumerate(ranges):
        if r != rank:
            t[:, b:e] = recv[r][:, : e - b]
    return t


def reduce_mg(A, B, Q=None, Z=None, nb=0, group=None, stream=None, gather=True, **kw):
    """Collective HT reduction of the (replicated) device pencil A, B on every rank.
    A, B, Q, Z: torch CUDA tensors holding column-major n x n matrices (t = M^T).
    Each rank computes H, T in full and its row slab of Q and Z; with gather=True the
    slabs are all-gathered so every rank ends with the full Q, Z.  Returns the report."""
    import torch.distributed as dist
    import paper_1710_08538_b200 as ht
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    n = A.shape[0]
    rr = row_range(n, world, rank) if world > 1 else None
    rep = ht.reduce_device(A, B, Q, Z, nb=nb, stream=stream, row_range=rr, **kw)
    if gather and world > 1:
        for M in (Q, Z):
            if M is not None:
                gather_rows(M, n, world, rank, group)
    return rep

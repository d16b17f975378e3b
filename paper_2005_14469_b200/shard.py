"""Column sharding of B/C across ranks.

GCOOSpDM's output tiles (row group x column strip) are independent and every
C element's accumulation order is fixed by A alone, so splitting B and C into
contiguous column blocks changes nothing numerically: the G-rank C is bitwise
the 1-rank C.  A is replicated.  There is no collective on the data path.
"""
from __future__ import annotations

from typing import List, Tuple


def column_shards(n_total: int, world: int, align: int = 64) -> List[Tuple[int, int]]:
    """Contiguous [lo, hi) column blocks, one per rank; every boundary is a
    multiple of `align` (the reference's strip width b=64, so per-rank
    KernelStats sum to the single-call counters), the last block takes the
    remainder.  Ranks past the data get empty blocks."""
    if world < 1 or n_total < 0 or align < 1:
        raise ValueError("column_shards: bad arguments")
    units = -(-n_total // align)
    base, extra = divmod(units, world)
    out, lo = [], 0
    for r in range(world):
        w = (base + (1 if r < extra else 0)) * align
        hi = min(n_total, lo + w)
        out.append((lo, hi))
        lo = hi
    return out


def weak_block(n_per_rank: int, rank: int) -> Tuple[int, int]:
    """Weak scaling: rank r owns columns [r*n, (r+1)*n) of a B/C that is
    world*n columns wide (per-rank work fixed as the world grows)."""
    return rank * n_per_rank, (rank + 1) * n_per_rank


def gather_columns(c_local, shards: List[Tuple[int, int]], root: int = 0, group=None):
    """The optional gather of a column-sharded C onto `root` (the
    north star's only use of NCCL): every rank sends its contiguous m x w_r
    block point to point (one NCCL group over NVLink/NVSwitch on GPUs, gloo on
    CPU), and root places each block into row-major m x N.  Returns the full C
    on root, None elsewhere.  Not on the multiply's timed path."""
    import torch
    import torch.distributed as dist

    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    if len(shards) != world:
        raise ValueError("gather_columns: one shard per rank")
    lo, hi = shards[rank]
    if c_local.dim() != 2 or c_local.shape[1] != hi - lo:
        raise ValueError("gather_columns: local block width does not match its shard")
    m = c_local.shape[0]
    if rank != root:
        if hi > lo:
            for req in dist.batch_isend_irecv([dist.P2POp(dist.isend, c_local.contiguous(), root, group)]):
                req.wait()
        return None
    out = torch.empty((m, shards[-1][1]), dtype=c_local.dtype, device=c_local.device)
    out[:, lo:hi].copy_(c_local)
    bufs, ops = {}, []
    for r, (rl, rh) in enumerate(shards):
        if r == root or rh == rl:
            continue
        bufs[r] = torch.empty((m, rh - rl), dtype=c_local.dtype, device=c_local.device)
        ops.append(dist.P2POp(dist.irecv, bufs[r], r, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    for r, buf in bufs.items():
        out[:, shards[r][0]:shards[r][1]].copy_(buf)
    return out

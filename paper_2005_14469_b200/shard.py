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

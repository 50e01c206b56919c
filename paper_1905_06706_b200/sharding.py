"""Multi-GPU partitioning of one GIRG.

Every event (type-I or type-II cell pair of a layer pair) is owned by the Morton block of its
A cell at a split level `sl` (coarser events by the block of their first descendant).  Rank r
of N owns the contiguous block range [r*B/N, (r+1)*B/N), B = 2^(d*sl), and calls
girg_edges_shard with it: no exchange is needed on the data path, the shards are disjoint and
their union is the single-GPU edge set for any N (the Philox keys do not depend on placement).
"""
from __future__ import annotations


def split_level(d: int, world: int, blocks_per_rank: int = 64) -> int:
    """Smallest level with at least `blocks_per_rank` Morton blocks per rank (d*sl <= 30)."""
    sl = 0
    while (1 << (d * sl)) < blocks_per_rank * world and d * (sl + 1) <= 30:
        sl += 1
    return sl


def shard_for_rank(d: int, world: int, rank: int, blocks_per_rank: int = 64):
    """(shard_level, blk_lo, blk_hi) of `rank` for girg_edges_shard."""
    if world <= 1:
        return (0, 0, 1)
    sl = split_level(d, world, blocks_per_rank)
    nb = 1 << (d * sl)
    return (sl, nb * rank // world, nb * (rank + 1) // world)

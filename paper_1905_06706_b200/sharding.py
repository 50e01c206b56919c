"""Multi-GPU partitioning of one GIRG.

Every event (type-I or type-II cell pair of a layer pair) is owned by one rank, decided from its
A cell alone, so the ranks need no exchange on the data path: the shards are disjoint and their
union is the single-GPU edge set for any N (the Philox keys do not depend on placement).

Default ("ranked", include/girg.h girg_options.nranks): interleaved ownership -- an event whose A
cell is on a level l >= sl belongs to rank (Morton block of A at the split level sl) mod N; a
coarser event (l < sl) to rank (A + 7 j + 13 i + 31 l) mod N.  Interleaving the >= 4096 blocks per
rank balances the spatially varying cost (a contiguous block range puts a whole region on one
rank), and spreading the coarse events by identity avoids giving all of them to the first block.
The block-range mode (girg_edges_shard) remains available as ``shard_for_rank(..., mode="range")``.
"""
from __future__ import annotations


def split_level(d: int, world: int, blocks_per_rank: int = 4096) -> int:
    """Smallest level with at least `blocks_per_rank` Morton blocks per rank (d*sl <= 30)."""
    sl = 0
    while (1 << (d * sl)) < blocks_per_rank * world and d * (sl + 1) <= 30:
        sl += 1
    return sl


def shard_for_rank(d: int, world: int, rank: int, blocks_per_rank: int = 4096, mode: str = "ranked"):
    """The `shard` argument of paper_1905_06706_b200.edges for `rank` of `world`:
    ("ranked", sl, world, rank) (interleaved, default) or (sl, blk_lo, blk_hi) (mode="range")."""
    if world <= 1:
        return (0, 0, 1)
    sl = split_level(d, world, blocks_per_rank)
    if mode == "ranked":
        return ("ranked", sl, world, rank)
    nb = 1 << (d * sl)
    return (sl, nb * rank // world, nb * (rank + 1) // world)

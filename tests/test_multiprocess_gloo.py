"""World-size-2 test of the multi-GPU partitioning on CPU (gloo, 127.0.0.1).

Each rank samples its shard (paper_1905_06706_b200.sharding, the same partition bench.py
--mode shard uses) with the oracle, the ranks exchange edge counts and edge sets through
torch.distributed (gloo), and the union must equal the single-process edge set, disjointly.
The CUDA kernels apply the identical ownership rule (tests/test_gpu_parity.py shard tests)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def worker(rank, world, port, d, T, q, mode="ranked"):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_1905_06706_b200.sharding import shard_for_rank
    from workloads import synth_inputs

    n = 6000
    w, x = synth_inputs(n, d, 2.4, 90 + d)
    kappa = oracle.scale_weights(w, 10.0, d, T, 2.4)
    e = oracle.edges(w, x, d, T, kappa, 11, shard=shard_for_rank(d, world, rank, mode=mode))
    keys = oracle.sort_edges(e).astype(np.int64)
    cnt = torch.tensor([len(keys)], dtype=torch.int64)
    counts = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(counts, cnt)
    gathered = [None] * world
    dist.all_gather_object(gathered, keys)
    total = torch.tensor([len(keys)], dtype=torch.int64)
    dist.all_reduce(total, op=dist.ReduceOp.SUM)
    if rank == 0:
        full = oracle.sort_edges(oracle.edges(w, x, d, T, kappa, 11)).astype(np.int64)
        union = np.sort(np.concatenate(gathered))
        q.put((int(total.item()), [int(c.item()) for c in counts], len(full),
               bool(np.array_equal(union, full)), bool(len(np.unique(union)) == len(union))))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["ranked", "range"])
@pytest.mark.parametrize("d,T", [(1, 0.5), (2, 0.8), (3, 0.0)])
def test_two_rank_shards_cover_the_graph(d, T, mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, 2, port, d, T, q, mode)) for r in range(2)]
    for p in procs:
        p.start()
    total, counts, m_full, equal, disjoint = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert total == m_full == sum(counts)
    assert all(c > 0 for c in counts)
    assert equal and disjoint


def test_shard_ranges_partition_blocks():
    from paper_1905_06706_b200.sharding import shard_for_rank, split_level

    for d in (1, 2, 3, 5):
        for world in (1, 2, 3, 4, 8):
            assert [shard_for_rank(d, world, r)[2:] for r in range(world) if world > 1] == \
                [(world, r) for r in range(world) if world > 1]
            rs = [shard_for_rank(d, world, r, mode="range") for r in range(world)]
            if world == 1:
                assert rs == [(0, 0, 1)]
                continue
            sl = split_level(d, world)
            assert all(r[0] == sl for r in rs)
            assert rs[0][1] == 0 and rs[-1][2] == 1 << (d * sl)
            assert all(a[2] == b[1] for a, b in zip(rs, rs[1:]))
            assert (1 << (d * sl)) >= 4096 * world or d * (sl + 1) > 30


@pytest.mark.parametrize("scheme", [0, 1, 2])
def test_ranked_shards_partition_and_spread_coarse_events(scheme):
    """Interleaved ownership (SURVEY 8(e) "Balance"), oracle only: for N = 3 and 4 the shards are
    disjoint, their union is the full edge set, and no rank is starved or overloaded -- the
    coarse events (levels below the split level) are spread by identity, not given to rank 0."""
    import sys

    sys.path.insert(0, ROOT)
    import oracle
    from paper_1905_06706_b200.sharding import shard_for_rank
    from workloads import synth_inputs

    n, d, T = 8000, 2, 0.7
    w, x = synth_inputs(n, d, 2.3, 17)
    kappa = oracle.scale_weights(w, 12.0, d, T, 2.3)
    if scheme == 2:
        oracle.set_ref_x(-1)  # REFINED (R27) on every level below CL: refined jobs are owned by their A cell too
    try:
        full = oracle.sort_edges(oracle.edges(w, x, d, T, kappa, 5, scheme=scheme))
        for world in (3, 4):
            parts = [oracle.sort_edges(oracle.edges(w, x, d, T, kappa, 5, shard=shard_for_rank(d, world, r),
                                                    scheme=scheme)) for r in range(world)]
            union = np.sort(np.concatenate(parts))
            assert np.array_equal(union, full)
            sizes = [len(p) for p in parts]
            assert max(sizes) < 1.25 * min(sizes), sizes
    finally:
        oracle.set_ref_x(0)

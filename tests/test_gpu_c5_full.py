"""BASELINE config 5 (n = 2^24, d = 3, T = 0.9) in FULL against the oracle, and the headline ABI
call ``girg_edges`` on its success path.

The oracle would need ~10 CPU-minutes for all of C5, so it runs as 64 shards (A-cell blocks at
level 2, SURVEY 8(e) ownership; ``test_shards_partition_the_edge_set`` pins that shards partition
the edge set) in a process pool over the host's cores.  Every shard's edges must be in the GPU's
full edge set (production kernels, the bench's launch configuration), and the shards together
must have exactly the GPU's edge count and key sum -- i.e. the union is the GPU set.  The
oracle's near-tie counters must be zero on every shard, and the device's counting build must see
zero near-ties and zero fast-path disagreements on the whole graph.
"""
import ctypes as C
import json
import multiprocessing as mp
import os

import numpy as np
import pytest
import torch

import oracle as O
from workloads import BY_NAME, synth_inputs

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1905_06706_b200 as girg  # noqa: E402

_G = {}  # inherited by the forked oracle workers: inputs and the GPU's sorted keys


def _shard(blk):
    c = _G["cfg"]
    e, so = O.edges(_G["w"], _G["x"], c.d, c.T, _G["kappa"], c.seed, shard=(2, blk, blk + 1), cap=8_000_000,
                    with_stats=True, scheme=_G["scheme"])
    k = O.sort_edges(e)
    g = _G["keys"]
    pos = np.minimum(np.searchsorted(g, k), len(g) - 1)
    subset = bool((g[pos] == k).all())
    return (blk, len(k), int(np.sum(k, dtype=np.uint64)), subset, so["nt1"] + so["nt2acc"], so["landings"],
            so["cand1"], so["nt2jump"])


@pytest.mark.parametrize("scheme", [girg.SCHEME_MERGED, girg.SCHEME_REFINED], ids=["merged", "refined"])
def test_C5_full_parity_all_shards(scheme):
    """scheme = refined: GIRG_SCHEME_REFINED with its default level rule (R27), the
    configuration ``bench.py --scheme refined`` times.  The type-I and acceptance near-tie counters
    must be zero on both sides.  Jump near-ties (R21: z within 1e-15 max(1, |z|) of an integer) are
    a diagnostic since R26 -- both sides compute z with the same deterministic log, bit for bit --
    and their window grows with |z| ~ 1 / pbar; MERGED has none on C5, REFINED's smaller bounds
    leave one: the two sides must count the same number, and the edge sets must be equal."""
    c = BY_NAME["C5"]
    w, x = synth_inputs(c.n, c.d, c.beta, c.seed)
    with open(os.path.join(os.path.dirname(__file__), "golden", "oracle_kappa.json")) as f:
        kappa = json.load(f)["C5"]
    wd, xd = torch.from_numpy(w).cuda(), torch.from_numpy(x).cuda()
    out = torch.empty((180_000_000, 2), dtype=torch.int32, device="cuda")
    e = girg.edges(wd, xd, c.T, kappa, c.seed, out=out, scheme=scheme)  # production kernels
    m = e.shape[0]
    keys = girg.edge_keys(e)
    assert bool((keys[1:] != keys[:-1]).all())
    gsum = int(keys.sum().item()) % (1 << 64)  # int64 wrap-around sum == uint64 sum mod 2^64
    _G.update(cfg=c, w=w, x=x, kappa=kappa, keys=keys.cpu().numpy().astype(np.uint64), scheme=scheme)
    del keys, e
    _, st = girg.edges(wd, xd, c.T, kappa, c.seed, out=out, stats=True, scheme=scheme)  # counting build
    assert st["neartie1"] == st["neartie2"] == st["fast_mismatch"] == 0, st
    if scheme == girg.SCHEME_MERGED:
        assert st["neartie_jump"] == 0, st
    del out
    torch.cuda.empty_cache()
    ncpu = max(1, min(32, os.cpu_count() or 1))
    with mp.get_context("fork").Pool(ncpu) as pool:
        res = pool.map(_shard, range(64), chunksize=1)
    tot = sum(r[1] for r in res)
    ksum = sum(r[2] for r in res) % (1 << 64)
    assert all(r[3] for r in res), [r[0] for r in res if not r[3]]
    assert sum(r[4] for r in res) == 0  # oracle type-I / acceptance near-ties over all of C5
    assert sum(r[7] for r in res) == st["neartie_jump"] <= 2, (sum(r[7] for r in res), st["neartie_jump"])
    assert tot == m, (tot, m)
    assert ksum == gsum
    assert sum(r[5] for r in res) == st["landings"] and sum(r[6] for r in res) == st["cand1"]


def test_girg_edges_abi_success_path():
    """The headline call girg_edges (merged scheme, whole graph) through the raw C ABI, on C2-sized
    inputs: OK status, m_out, and the edge set equals the oracle's."""
    c = BY_NAME["C2"]
    w, x = synth_inputs(c.n, c.d, c.beta, c.seed)
    kappa = O.scale_weights(w, c.avg_deg, c.d, c.T, c.beta)
    wd, xd = torch.from_numpy(w).cuda(), torch.from_numpy(x).cuda()
    cap = 6_000_000
    buf = torch.empty((cap, 2), dtype=torch.int32, device="cuda")
    m = C.c_uint64(0)
    rc = girg._lib.girg_edges(wd.data_ptr(), xd.data_ptr(), c.n, c.d, c.T, kappa, c.seed, buf.data_ptr(), cap,
                              C.byref(m), torch.cuda.current_stream().cuda_stream)
    assert rc == girg.OK
    got = girg.edge_keys(buf[: m.value]).cpu().numpy().astype(np.uint64)
    eo, so = O.edges(w, x, c.d, c.T, kappa, c.seed, with_stats=True)
    assert so["nt1"] + so["nt2acc"] + so["nt2jump"] == 0
    assert np.array_equal(got, O.sort_edges(eo))

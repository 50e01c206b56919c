"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle, element by element.

Inputs come from workloads.synth_inputs (numpy PCG64, shared by both sides) or from each side's
own generator (H1/H2 parity).  kappa always comes from the oracle's estimator, never from the
CUDA path.  T = 0: bit-exact edge sets.  T > 0: identical edge sets, with the oracle's near-tie
counters (|r - p| < 1e-12, |r_acc - p/pbar| < 1e-12, jump z within 1e-15 max(1,|z|) of an
integer, R14/R21) required to be zero, and the device's own counters of the same
near-ties and of fast-path disagreements too.  Every parity case runs both the production
kernels (stats=False) and the counting build (stats=True).
"""
import numpy as np
import pytest
import torch

import oracle as O
from workloads import BY_NAME, synth_inputs

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # CPU-only host: the -m gpu suite cannot run here
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1905_06706_b200 as girg  # noqa: E402  (fails loudly if libgirg.so is missing)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def gpu_keys(e):
    return girg.edge_keys(e).cpu().numpy().astype(np.uint64)


def run_both(w, x, d, T, kappa, seed, shard=(0, 0, 1), scheme=girg.SCHEME_MERGED):
    """The production kernels (stats=False: the float fast paths decide) and the counting build
    (stats=True: every decision also taken canonically, disagreements counted) against the
    oracle on the same inputs."""
    wd, xd = dev(w), dev(x)
    e, st = girg.edges(wd, xd, T, kappa, seed, shard=shard, stats=True, scheme=scheme)
    ep = girg.edges(wd, xd, T, kappa, seed, shard=shard, stats=False, scheme=scheme)
    eo, so = O.edges(w, x, d, T, kappa, seed, shard=shard, with_stats=True, scheme=scheme)
    return gpu_keys(e), O.sort_edges(eo), st, so, gpu_keys(ep)


def assert_device_clean(st):
    """Device-side near-tie counters (type-I, acceptance, jump) and fast-path disagreements."""
    assert st["neartie1"] == 0 and st["neartie2"] == 0 and st["neartie_jump"] == 0, st
    assert st["fast_mismatch"] == 0, st


def assert_parity(w, x, d, T, kappa, seed, shard=(0, 0, 1), scheme=girg.SCHEME_MERGED):
    g, o, st, so, gp = run_both(w, x, d, T, kappa, seed, shard, scheme)
    assert so["nt1"] + so["nt2acc"] + so["nt2jump"] == 0, so
    assert len(g) == len(o), (len(g), len(o))
    assert np.array_equal(g, o)
    assert np.array_equal(gp, o)  # the production (stats=False) kernels too
    assert_device_clean(st)
    # the device's own work counters agree with the oracle's
    assert st["cand1"] == so["cand1"]
    assert st["landings"] == so["landings"] and st["draws"] == so["draws"]
    assert st["edges1"] == so["acc1"] and st["edges2"] == so["acc2"]
    return g, st, so


# ----------------------------------------------------------------- generators (H1, H2) ----
def test_positions_bit_exact():
    for n, d, seed in ((1, 1, 3), (1000, 3, 5), (100_003, 2, 9), (70_001, 5, 1)):
        xg = girg.positions(n, d, seed).cpu().numpy()
        assert np.array_equal(xg, O.positions(n, d, seed))


def test_weights_within_2ulp():
    for n, beta, seed in ((1, 2.5, 1), (200_001, 2.2, 4), (50_000, 2.9, 5)):
        wg = girg.weights(n, beta, seed).cpu().numpy()
        wo = O.weights(n, beta, seed)
        ulps = np.abs(wg.view(np.int64) - wo.view(np.int64))
        assert ulps.max() <= 2, ulps.max()
        assert (wg >= 1.0).all()


# ----------------------------------------------------------------- estimator --------------
@pytest.mark.parametrize("cfg", ["C1", "C2", "C3", "C5"])
def test_scale_weights_matches_oracle(cfg):
    c = BY_NAME[cfg]
    n = min(c.n, 200_000)
    w, _ = synth_inputs(n, c.d, c.beta, c.seed)
    kg = girg.scale_weights(dev(w), c.avg_deg, c.d, c.T, c.beta)
    ko = O.scale_weights(w, c.avg_deg, c.d, c.T, c.beta)
    assert abs(kg - ko) <= 1e-12 * ko, (kg, ko)
    assert O.f(w, c.d, c.T, kg) == pytest.approx(c.avg_deg, rel=1e-10)


# ----------------------------------------------------------------- T = 0 -----------------
def test_C1_bit_exact_and_bruteforce():
    """BASELINE config 1 in full: GPU == oracle == O(n^2) brute force."""
    c = BY_NAME["C1"]
    w, x = synth_inputs(c.n, c.d, c.beta, c.seed)
    kappa = O.scale_weights(w, c.avg_deg, c.d, c.T, c.beta)
    g, st, so = assert_parity(w, x, c.d, 0.0, kappa, c.seed)
    assert np.array_equal(g, O.sort_edges(O.bruteforce_t0(w, x, c.d, kappa)))


@pytest.mark.parametrize("d", [1, 2, 3, 4, 5])
def test_threshold_parity_all_dims(d):
    for n, seed in ((3001, 1), (40_000, 2)):
        w, x = synth_inputs(n, d, 2.4, 100 * d + seed)
        kappa = O.scale_weights(w, 8.0, d, 0.0, 2.4)
        g, _, _ = assert_parity(w, x, d, 0.0, kappa, seed)
        if n <= 3001:
            assert np.array_equal(g, O.sort_edges(O.bruteforce_t0(w, x, d, kappa)))


# ----------------------------------------------------------------- T > 0 -----------------
SCHEMES = pytest.mark.parametrize("scheme", [girg.SCHEME_EVENT, girg.SCHEME_MERGED], ids=["event", "merged"])


@SCHEMES
@pytest.mark.parametrize("d,T,beta", [(1, 0.5, 2.5), (2, 0.8, 2.2), (3, 0.9, 2.9), (1, 0.2, 2.1),
                                      (2, 0.3, 3.0), (4, 0.6, 2.5), (5, 0.5, 2.7)])
def test_binomial_parity_small(d, T, beta, scheme):
    for n, seed in ((1, 1), (2, 2), (997, 3), (30_011, 4)):
        w, x = synth_inputs(n, d, beta, 7 * d + seed)
        kappa = O.scale_weights(w, min(10.0, max(n - 1.5, 0.5)), d, T, beta) if n > 2 else 0.7
        g, st, so = assert_parity(w, x, d, T, kappa, seed, scheme=scheme)
        if n > 1000:
            assert so["landings"] > 0


@pytest.mark.parametrize("cfg,scheme", [("C2", girg.SCHEME_MERGED), ("C3", girg.SCHEME_MERGED),
                                        ("C4", girg.SCHEME_MERGED), ("C2", girg.SCHEME_EVENT)])
def test_baseline_config_full_parity(cfg, scheme):
    """BASELINE configs 2-4 in full: identical edge sets, zero near-ties, degree on target."""
    c = BY_NAME[cfg]
    w, x = synth_inputs(c.n, c.d, c.beta, c.seed)
    kappa = O.scale_weights(w, c.avg_deg, c.d, c.T, c.beta)
    g, st, so = assert_parity(w, x, c.d, c.T, kappa, c.seed, scheme=scheme)
    assert abs(2 * len(g) / c.n - c.avg_deg) < 0.01 * c.avg_deg


def test_C5_sampled_shard_parity():
    """BASELINE config 5 (n = 2^24, d = 3): the oracle cannot run all ~10^10 events in a test,
    so parity is checked on sampled shards (SURVEY 8(e) ownership by A-cell block at level 3)
    in the same launch configuration; the full GPU run is checked for its degree and structure.
    kappa is the oracle's (tests/golden/oracle_kappa.json, written by tools/oracle_kappas.py)."""
    import json
    import os

    c = BY_NAME["C5"]
    w, x = synth_inputs(c.n, c.d, c.beta, c.seed)
    with open(os.path.join(os.path.dirname(__file__), "golden", "oracle_kappa.json")) as f:
        kappa = json.load(f)["C5"]
    wd, xd = dev(w), dev(x)
    full, st = girg.edges(wd, xd, c.T, kappa, c.seed, stats=True)
    m = full.shape[0]
    assert abs(2 * m / c.n - c.avg_deg) < 0.01 * c.avg_deg
    assert_device_clean(st)
    k = girg.edge_keys(full)  # sorted int64 keys on the device
    assert bool((k[1:] != k[:-1]).all())  # no duplicates
    u, v = k >> 32, k & 0xFFFFFFFF
    assert bool((u < v).all()) and bool((v < c.n).all())
    total = 0
    for lo, hi in ((0, 1), (137, 138), (511, 512)):
        g, o, stg, so, gp = run_both(w, x, c.d, c.T, kappa, c.seed, shard=(3, lo, hi))
        assert so["nt1"] + so["nt2acc"] + so["nt2jump"] == 0, so
        assert np.array_equal(g, o) and np.array_equal(gp, o)
        gd = torch.from_numpy(g.astype(np.int64)).cuda()
        pos = torch.searchsorted(k, gd).clamp(max=m - 1)
        assert bool((k[pos] == gd).all())  # the shard is a subset of the full graph
        total += len(g)
    assert total > 0


# ----------------------------------------------------------------- edge cases -------------
def test_degenerate_inputs():
    # n = 1: no edges; all weights equal: one layer; coincident points (D = 0 -> p = 1)
    w1, x1 = np.ones(1), np.full((2, 1), 0.3)
    assert girg.edges(dev(w1), dev(x1), 0.5, 1.0, 1).shape[0] == 0
    n = 5000
    w = np.full(n, 3.0)
    _, x = synth_inputs(n, 2, 2.5, 3)
    for T in (0.0, 0.7):
        assert_parity(w, x, 2, T, 0.3, 5)
    xc = np.zeros((1, 64))
    g, _, _ = assert_parity(np.ones(64), xc, 1, 0.5, 1e-3, 1)
    assert len(g) == 64 * 63 // 2


@SCHEMES
@pytest.mark.parametrize("d", [1, 2, 3])
def test_extreme_kappa(d, scheme):
    """kappa so large that every level is coarse (CL <= 2: the whole-level regions of the job
    setup, lg <= 1) or so small that only the finest cells matter."""
    n = 800
    w, x = synth_inputs(n, d, 2.5, 4)
    g, _, _ = assert_parity(w, x, d, 0.5, 1e6, 2, scheme=scheme)  # every pair saturated: complete graph
    assert len(g) == n * (n - 1) // 2
    g, _, _ = assert_parity(w, x, d, 0.0, 1e-12, 2, scheme=scheme)
    assert len(g) == 0
    assert_parity(w, x, d, 0.9, 1e-9, 2, scheme=scheme)
    for kappa in (3e-2, 0.3, 3.0, 30.0):  # CL of the heavy layers through 0, 1, 2
        assert_parity(w, x, d, 0.6, kappa, 5, scheme=scheme)


@pytest.mark.parametrize("d,T", [(1, 0.0), (1, 0.5), (2, 0.7), (3, 0.9)])
def test_parity_over_edge_seeds(d, T):
    """Several edge seeds on one graph (the draws differ per seed, the events do not)."""
    n = 20_000
    w, x = synth_inputs(n, d, 2.4, 90 + d)
    kappa = O.scale_weights(w, 12.0, d, T, 2.4)
    for seed in (1, 2, 3, 2**33 + 5):
        assert_parity(w, x, d, T, kappa, seed)


def test_capacity_and_determinism():
    n, d, T = 50_000, 2, 0.7
    w, x = synth_inputs(n, d, 2.3, 8)
    kappa = O.scale_weights(w, 10.0, d, T, 2.3)
    wd, xd = dev(w), dev(x)
    import ctypes as C

    buf = torch.empty((10, 2), dtype=torch.int32, device="cuda")
    m = C.c_uint64(0)
    rc = girg._lib.girg_edges(wd.data_ptr(), xd.data_ptr(), n, d, T, kappa, 3, buf.data_ptr(), 10, C.byref(m),
                              torch.cuda.current_stream().cuda_stream)
    assert rc == girg.ECAPACITY
    a = gpu_keys(girg.edges(wd, xd, T, kappa, 3, cap=int(m.value)))
    assert len(a) == m.value
    assert np.array_equal(a, gpu_keys(girg.edges(wd, xd, T, kappa, 3)))
    assert not np.array_equal(a, gpu_keys(girg.edges(wd, xd, T, kappa, 4)))


def test_invalid_inputs_rejected():
    n = 100
    w, x = synth_inputs(n, 1, 2.5, 1)
    bad_x = x.copy()
    bad_x[0, 5] = 1.0
    with pytest.raises(girg.GirgError) as ei:
        girg.edges(dev(w), dev(bad_x), 0.5, 1.0, 1)
    assert ei.value.code == girg.EINVAL
    for bad in (0.0, -1.0, np.nan, np.inf):
        bw = w.copy()
        bw[3] = bad
        with pytest.raises(girg.GirgError) as ei:
            girg.edges(dev(bw), dev(x), 0.5, 1.0, 1)
        assert ei.value.code == girg.EINVAL
    wide = w.copy()
    wide[0] = 2.0**70  # 71 layers
    with pytest.raises(girg.GirgError) as ei:
        girg.edges(dev(wide), dev(x), 0.5, 1.0, 1)
    assert ei.value.code == girg.ERANGE


def test_shards_union_equals_full():
    n, d, T = 60_000, 2, 0.8
    w, x = synth_inputs(n, d, 2.2, 12)
    kappa = O.scale_weights(w, 12.0, d, T, 2.2)
    wd, xd = dev(w), dev(x)
    full = gpu_keys(girg.edges(wd, xd, T, kappa, 9))
    parts = [gpu_keys(girg.edges(wd, xd, T, kappa, 9, shard=(2, a, b))) for a, b in ((0, 5), (5, 11), (11, 16))]
    assert np.array_equal(np.sort(np.concatenate(parts)), full)


def test_host_buffer_call_matches_device_call():
    n, d, T = 30_000, 3, 0.6
    w, x = synth_inputs(n, d, 2.6, 2)
    kappa = O.scale_weights(w, 10.0, d, T, 2.6)
    ref = gpu_keys(girg.edges(dev(w), dev(x), T, kappa, 5))
    wh = torch.from_numpy(w).pin_memory()
    xh = torch.from_numpy(x).pin_memory()
    out = torch.empty((len(ref) + 10, 2), dtype=torch.int32).pin_memory()  # kernels write into it directly
    m = girg.edges_host(wh, xh, d, T, kappa, 5, out)
    assert m == len(ref)
    assert np.array_equal(girg.edge_keys(out[:m]).numpy().astype(np.uint64), ref)
    pageable = torch.empty((len(ref) + 10, 2), dtype=torch.int32)  # copy-back path
    m = girg.edges_host(torch.from_numpy(w), torch.from_numpy(x), d, T, kappa, 5, pageable)
    assert m == len(ref)
    assert np.array_equal(girg.edge_keys(pageable[:m]).numpy().astype(np.uint64), ref)


# ------------------------------------------------------- batched small graphs (NEXT-4) ----
@pytest.mark.parametrize("d,T", [(1, 0.0), (2, 0.5), (3, 0.8)])
def test_batch_equals_single_calls_and_oracle(d, T):
    """girg_edges_batch: every graph of the batch equals its own girg_edges call (and, for two of
    them, the oracle), with mixed seeds and kappas, more graphs than streams, and one graph whose
    capacity is too small (ECAPACITY for that graph only, re-issued by the binding)."""
    n, beta, B = 5003, 2.5, 7
    ws, xs, kap, seeds = [], [], [], []
    for g in range(B):
        w, x = synth_inputs(n, d, beta, 100 + 7 * g + d)
        ws.append(w)
        xs.append(x)
        kap.append(O.scale_weights(w, 4.0 + g, d, T, beta))
        seeds.append(1000 + g)
    caps = [16 * n + 1024] * B
    caps[3] = 5  # too small: the library reports the exact count, the binding re-issues graph 3
    out = girg.edges_batch([dev(w) for w in ws], [dev(x) for x in xs], T, kap, seeds, caps=caps, nstreams=3)
    assert len(out) == B
    for g in range(B):
        single = girg.edges(dev(ws[g]), dev(xs[g]), T, kap[g], seeds[g])
        assert np.array_equal(gpu_keys(out[g]), gpu_keys(single)), g
    for g in (0, 3):
        eo, so = O.edges(ws[g], xs[g], d, T, kap[g], seeds[g], with_stats=True)
        assert so["nt1"] + so["nt2acc"] + so["nt2jump"] == 0, so
        assert np.array_equal(gpu_keys(out[g]), O.sort_edges(eo)), g


def test_batch_single_graph_and_status():
    """B = 1 through the raw ABI: status_out and m_out per graph, and a capacity failure."""
    import ctypes as C
    n, d, T, beta = 2000, 2, 0.3, 2.4
    w, x = synth_inputs(n, d, beta, 5)
    kappa = O.scale_weights(w, 6.0, d, T, beta)
    wd, xd = dev(w), dev(x)
    buf = torch.empty((4, 2), dtype=torch.int32, device="cuda")
    P1 = C.c_void_p * 1
    mo, so = (C.c_uint64 * 1)(), (C.c_int * 1)()
    rc = girg._lib.girg_edges_batch(1, P1(wd.data_ptr()), P1(xd.data_ptr()), n, d, T, (C.c_double * 1)(kappa),
                                    (C.c_uint64 * 1)(9), P1(buf.data_ptr()), (C.c_uint64 * 1)(4), mo, so, 0, None)
    ref = girg.edges(wd, xd, T, kappa, 9)
    assert rc == girg.ECAPACITY and so[0] == girg.ECAPACITY
    assert mo[0] == ref.shape[0] > 4


@pytest.mark.parametrize("d", [1, 2, 3])
@pytest.mark.parametrize("T,beta", [(0.99, 2.5), (0.02, 2.5), (0.5, 2.05), (0.0, 2.05), (0.7, 6.0)])
def test_parameter_extremes(d, T, beta):
    """Temperatures near 1 (flat p, pbar near 1 on coarse levels) and near 0 (p close to a step),
    beta near 2 (huge hub weights, many layers) and a light tail (beta = 6: few layers)."""
    n = 20_000
    w, x = synth_inputs(n, d, beta, 300 + d)
    kappa = O.scale_weights(w, 10.0, d, T, beta)
    g, st, so = assert_parity(w, x, d, T, kappa, 11)
    if beta >= 2.5:  # degree near target (for beta ~ 2 the realised degree is dominated by a few hubs)
        assert abs(2 * len(g) / n - 10.0) < 2.0


def test_big_job_items_and_queue_regrowth(monkeypatch):
    """Every job split into 1-unit k_big items (development thresholds GIRG_BIG_WORK /
    GIRG_ITEM_WORK): far more items than the initial queue holds, so the library must grow the
    queue and re-run the sampler; the edge set is unchanged (schedule independence)."""
    n, d, T, beta = 20_000, 2, 0.6, 2.3
    w, x = synth_inputs(n, d, beta, 77)
    kappa = O.scale_weights(w, 12.0, d, T, beta)
    ref, st0 = girg.edges(dev(w), dev(x), T, kappa, 5, stats=True)
    monkeypatch.setenv("GIRG_BIG_WORK", "2")
    monkeypatch.setenv("GIRG_ITEM_WORK", "1")
    got, st1 = girg.edges(dev(w), dev(x), T, kappa, 5, stats=True)
    assert np.array_equal(gpu_keys(got), gpu_keys(ref))
    assert st1["landings"] == st0["landings"] and st1["cand1"] == st0["cand1"]
    assert st1["cand1"] + st1["chunks"] > (1 << 18)  # more 1-unit items than the initial queue


@pytest.mark.parametrize("d,T,nc,kappa", [(1, 0.0, 30_000, 1e-9), (2, 0.6, 3_000, 1e-19)])
def test_crowded_cell_linear_order(d, T, nc, kappa):
    """One cell holding nc points (a tight cluster, far more than the insertion level expects):
    k_order lists it and k_order_big radix-sorts its ids in linear time (several 256-point
    tiles, 3 digit passes for n = 10^5); the in-cell id order (R11) and so the edge set must
    still equal the oracle's."""
    n, beta = 100_000, 2.5
    w, x = synth_inputs(n, d, beta, 606)
    rng = np.random.default_rng(5)
    idx = rng.choice(n, nc, replace=False)
    for k in range(d):
        x[k, idx] = 0.5 + rng.integers(0, 1 << 20, size=idx.size) * 2.0**-53  # width 1.2e-10
    g, st, so = assert_parity(w, x, d, T, kappa, 3)
    assert len(g) > 1000


@pytest.mark.parametrize("d,T,scheme", [(2, 0.8, girg.SCHEME_MERGED), (3, 0.9, girg.SCHEME_MERGED),
                                        (1, 0.5, girg.SCHEME_EVENT), (2, 0.0, girg.SCHEME_MERGED)])
def test_ranked_shards_equal_oracle_and_union(d, T, scheme):
    """Interleaved multi-GPU ownership (girg_options.nranks, sharding.shard_for_rank): every rank's
    shard equals the oracle's shard of the same rank, and the N shards partition the full graph."""
    from paper_1905_06706_b200.sharding import shard_for_rank

    n = 40_000
    w, x = synth_inputs(n, d, 2.4, 70 + d)
    kappa = O.scale_weights(w, 12.0, d, T, 2.4)
    wd, xd = dev(w), dev(x)
    full = gpu_keys(girg.edges(wd, xd, T, kappa, 4, scheme=scheme))
    world = 3
    parts = []
    for r in range(world):
        sh = shard_for_rank(d, world, r)
        g = gpu_keys(girg.edges(wd, xd, T, kappa, 4, shard=sh, scheme=scheme))
        eo, so = O.edges(w, x, d, T, kappa, 4, shard=sh, with_stats=True, scheme=scheme)
        assert so["nt1"] + so["nt2acc"] + so["nt2jump"] == 0
        assert np.array_equal(g, O.sort_edges(eo)), r
        parts.append(g)
    assert np.array_equal(np.sort(np.concatenate(parts)), full)


def test_batch_binomial_d3_many_graphs_and_overflowing_capacity():
    """Fused batch at T > 0, d = 3 with more graphs than one block row per SM and two graphs whose
    capacity is too small: every graph equals its single call, the small ones report their count."""
    n, d, T, beta, B = 4000, 3, 0.9, 2.9, 40
    ws = [girg.weights(n, beta, 500 + g) for g in range(B)]
    xs = [girg.positions(n, d, 900 + g) for g in range(B)]
    kap = [girg.scale_weights(w, 12.0, d, T, beta) for w in ws]
    seeds = [77 + g for g in range(B)]
    caps = [16 * n] * B
    caps[5] = caps[31] = 3
    out = girg.edges_batch(ws, xs, T, kap, seeds, caps=caps)
    for g in range(B):
        assert np.array_equal(gpu_keys(out[g]), gpu_keys(girg.edges(ws[g], xs[g], T, kap[g], seeds[g]))), g


@pytest.mark.parametrize("d,T", [(1, 0.0), (2, 0.7), (3, 0.9)])
def test_edge_set_independent_of_tile_size(d, T, monkeypatch):
    """The sampler's schedule (sorted points per tile: 8 below 2^17 points, else 32; any 1..32 by
    GIRG_TILE_PTS) does not change the edge set -- the randomness is keyed by vertex pair and
    cell-pair chunk (R17, R22), not by warp or lane -- and equals the oracle's."""
    n, beta, seed = 40_000, 2.5, 31 + d
    w, x = synth_inputs(n, d, beta, seed)
    kappa = O.scale_weights(w, 10.0, d, T, beta)
    eo = O.sort_edges(O.edges(w, x, d, T, kappa, seed))
    wd, xd = dev(w), dev(x)
    for tp in (None, "32", "13", "4", "1"):
        if tp is None:
            monkeypatch.delenv("GIRG_TILE_PTS", raising=False)
        else:
            monkeypatch.setenv("GIRG_TILE_PTS", tp)
        g = gpu_keys(girg.edges(wd, xd, T, kappa, seed))
        assert np.array_equal(g, eo), (tp, len(g), len(eo))

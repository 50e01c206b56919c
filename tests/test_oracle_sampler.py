"""Pins for the oracle's edge sampler (Algorithm 1, type-I/type-II) -- CPU only.

T = 0: the method computes exactly the plain threshold graph, so the oracle must equal the O(n^2)
brute force bit for bit.  T > 0: the result is random; the oracle is pinned by per-pair
frequencies against Eq. 1, expected edge counts against sum_{u<v} p_uv, exact coverage of the
candidate pairs by events, the T -> 0 limit and structural invariants.
"""
import math

import numpy as np
import pytest

from workloads import synth_inputs


def keys(e):
    return np.sort((e[:, 0].astype(np.uint64) << np.uint64(32)) | e[:, 1].astype(np.uint64))


@pytest.mark.parametrize("d", [1, 2, 3])
@pytest.mark.parametrize("beta", [2.2, 2.5, 2.8, 3.0])
def test_threshold_equals_bruteforce(oracle, d, beta):
    """T=0 sampler == O(n^2) brute force for n in {200,1000,2000}, several seeds."""
    for n, seed in ((200, 1), (1000, 2), (2000, 3), (2000, 4)):
        w, x = synth_inputs(n, d, beta, 1000 * d + seed)
        kappa = oracle.scale_weights(w, 10.0, d, 0.0, beta)
        e = oracle.edges(w, x, d, 0.0, kappa, seed)
        b = oracle.bruteforce_t0(w, x, d, kappa)
        assert np.array_equal(keys(e), keys(b)), (n, seed)


def test_threshold_C1_full_bruteforce(oracle):
    """BASELINE config 1 itself (n = 10^4, d = 1, beta = 2.8, T = 0), all 5*10^7 pairs."""
    w, x = synth_inputs(10_000, 1, 2.8, 1)
    kappa = oracle.scale_weights(w, 10.0, 1, 0.0, 2.8)
    e, st = oracle.edges(w, x, 1, 0.0, kappa, 1, with_stats=True)
    b = oracle.bruteforce_t0(w, x, 1, kappa)
    assert np.array_equal(keys(e), keys(b))
    assert abs(2 * len(e) / 10_000 - 10.0) < 0.6
    assert st["ev2"] == 0  # no type-II events at T = 0


# "refined_all": R27 on every level l < CL(i,j) (the ref_x test hook), so that the small pin
# graphs exercise the refined sequences, which the default threshold (4096 points per cell) only
# reaches at larger n
SCHEMES = pytest.mark.parametrize("scheme", [0, 1, 2, "refined_all"], ids=["event", "merged", "refined", "refined_all"],
                                  indirect=True)


@pytest.fixture
def scheme(request, oracle):
    if request.param == "refined_all":
        oracle.set_ref_x(-1)
        yield 2
        oracle.set_ref_x(0)
    else:
        yield request.param


@SCHEMES
@pytest.mark.parametrize("d,T", [(1, 0.5), (2, 0.8), (3, 0.9), (1, 0.2)])
def test_coverage_each_pair_exactly_once(oracle, d, T, scheme):
    """every unordered vertex pair is a candidate of exactly one (cell pair, bucket pair)
    event -- instrumented oracle on n <= 600.  Merged sequences (R22) regroup the same events,
    so the same exact cover must hold."""
    n = 600 if d < 3 else 400
    w, x = synth_inputs(n, d, 2.3, 77 + d)
    kappa = oracle.scale_weights(w, 4.0, d, T, 2.3)
    cov, st = oracle.coverage(w, x, d, T, kappa, scheme=scheme)
    sym = cov.astype(np.int64) + cov.T.astype(np.int64)
    assert (np.diag(cov) == 0).all()
    off = ~np.eye(n, dtype=bool)
    assert (sym[off] == 1).all()
    assert st["ev2_nonempty"] > 0 and st["ev1_nonempty"] > 0
    assert st["cand1"] + st["cand2"] == n * (n - 1) // 2
    # the type-II bound of every candidate's sequence holds: p_uv <= pbar (R9, R27)
    assert st["bound_viol"] == 0


@SCHEMES
@pytest.mark.parametrize("d,T,runs", [(1, 0.5, 20000), (2, 0.8, 20000), (1, 0.3, 8000), (3, 0.9, 8000)])
def test_per_pair_frequency(oracle, d, T, runs, scheme):
    """with fixed w and x, each pair's empirical edge frequency over independent edge
    seeds is within 5 sigma of p_uv (Eq. 1), and the chi-square over pairs is plausible."""
    per_pair_check(oracle, 40, d, T, runs, 3.0, scheme)


def test_refined_per_pair_frequency_d3(oracle):
    """The same pin for R27 in d = 3 on a graph where its rows are split (n = 64, low degree:
    CL(0,0) = 3, so level 2 is refined under the every-level hook; the n = 40 graph above has no
    level below CL)."""
    oracle.set_ref_x(-1)
    try:
        w, x = synth_inputs(64, 3, 2.5, 8)
        kappa = oracle.scale_weights(w, 1.0, 3, 0.9, 2.5)
        sm = oracle.edges(w, x, 3, 0.9, kappa, 1, with_stats=True, scheme=1)[1]
        sr = oracle.edges(w, x, 3, 0.9, kappa, 1, with_stats=True, scheme=2)[1]
        assert sr["ev2_nonempty"] > sm["ev2_nonempty"]  # refined sequences exist
        per_pair_check(oracle, 64, 3, 0.9, 5000, 1.0, 2)
    finally:
        oracle.set_ref_x(0)


def per_pair_check(oracle, n, d, T, runs, deg, scheme):
    w, x = synth_inputs(n, d, 2.5, 5 + d)
    kappa = oracle.scale_weights(w, deg, d, T, 2.5)
    W = oracle.exact_sum(w)
    s = kappa / W
    P = np.zeros((n, n))
    for u in range(n):
        for v in range(u + 1, n):
            D = oracle.dpow(oracle.torus_dist(x[:, u], x[:, v]), d)
            P[u, v] = oracle.prob(w[u], w[v], s, D, T)
    cnt = np.zeros((n, n))
    land = 0
    for seed in range(runs):
        e, st = oracle.edges(w, x, d, T, kappa, seed + 1, with_stats=True, scheme=scheme)
        land += st["landings"]
        cnt[e[:, 0], e[:, 1]] += 1
    assert land > 0  # type-II jumps were exercised
    iu = np.triu_indices(n, 1)
    p, f = P[iu], cnt[iu] / runs
    sure = p >= 1.0
    assert (f[sure] == 1.0).all()
    q = p[~sure]
    c = cnt[iu][~sure]
    assert (c[q == 0] == 0).all()
    # exact two-sided binomial p-value per pair, Bonferroni over pairs (normal z is wrong for
    # pairs with expected counts << 1)
    from scipy import stats
    pv = np.minimum(1.0, 2 * np.minimum(stats.binom.cdf(c, runs, q), stats.binom.sf(c - 1, runs, q)))
    assert pv[q > 0].min() * (q > 0).sum() > 1e-4, pv[q > 0].min()
    sig = np.sqrt(q * (1 - q) / runs)
    z = np.abs(f[~sure] - q) / np.maximum(sig, 1e-300)
    live = (q > 1e-3) & (q < 1 - 1e-3)
    chi2 = float(np.sum(z[live] ** 2))
    k = int(live.sum())
    assert abs(chi2 - k) < 6 * math.sqrt(2 * k), (chi2, k)


@SCHEMES
def test_expected_edge_count(oracle, scheme):
    """mean of m over independent edge seeds vs sum_{u<v} p_uv (brute force), z < 4."""
    n, d, T = 3000, 2, 0.5
    w, x = synth_inputs(n, d, 2.5, 9)
    kappa = oracle.scale_weights(w, 8.0, d, T, 2.5)
    mu = oracle.expected_edges_bf(w, x, d, T, kappa)
    ms = np.array([len(oracle.edges(w, x, d, T, kappa, s, scheme=scheme)) for s in range(1, 61)])
    # var(m) = sum p(1-p) <= mu
    z = abs(ms.mean() - mu) / math.sqrt(mu / len(ms))
    assert z < 4, (ms.mean(), mu)


@SCHEMES
def test_structure_and_determinism(oracle, scheme):
    for d, T in ((1, 0.5), (2, 0.8), (3, 0.6)):
        n = 5000
        w, x = synth_inputs(n, d, 2.4, 31 + d)
        kappa = oracle.scale_weights(w, 10.0, d, T, 2.4)
        e = oracle.edges(w, x, d, T, kappa, 7, scheme=scheme)
        assert (e[:, 0] < e[:, 1]).all() and (e[:, 1] < n).all()
        k = keys(e)
        assert len(np.unique(k)) == len(k)
        assert np.array_equal(k, keys(oracle.edges(w, x, d, T, kappa, 7, scheme=scheme)))
        assert not np.array_equal(k, keys(oracle.edges(w, x, d, T, kappa, 8, scheme=scheme)))


def test_merged_scheme_reduces_draws(oracle):
    """R22 does what it is for: same landings in expectation, far fewer Philox draws (the
    per-cell-pair terminating draws disappear), and the same type-I work."""
    n, d, T = 20000, 3, 0.9
    w, x = synth_inputs(n, d, 2.9, 5)
    kappa = oracle.scale_weights(w, 20.0, d, T, 2.9)
    _, se = oracle.edges(w, x, d, T, kappa, 3, with_stats=True, scheme=0)
    _, sm = oracle.edges(w, x, d, T, kappa, 3, with_stats=True, scheme=1)
    assert se["cand1"] == sm["cand1"] and se["acc1"] == sm["acc1"]  # type-I keyed by (u, v)
    assert se["cand2"] == sm["cand2"]  # the same candidate pairs, regrouped
    assert sm["draws"] < 0.7 * se["draws"]
    z = abs(sm["landings"] - se["landings"]) / math.sqrt(se["landings"] + sm["landings"])
    assert z < 5, (se["landings"], sm["landings"])


@pytest.mark.parametrize("d,T,beta,deg", [(3, 0.9, 2.9, 20.0), (2, 0.8, 2.2, 20.0)])
def test_refined_scheme_cuts_landings(oracle, d, T, beta, deg):
    """R27: the same candidate pairs and type-I work as R22; on the refined
    levels (l < CL(i,j), here >= 8 points of layer i per cell) sequences per (child of A, distance
    class) instead of per (A, delta_max), and markedly fewer landings for the same edges in
    expectation (the bound of a far child is (2/3)^(d/T) of A's)."""
    n = 60000
    w, x = synth_inputs(n, d, beta, 5)
    kappa = oracle.scale_weights(w, deg, d, T, beta)
    em, sm = oracle.edges(w, x, d, T, kappa, 3, with_stats=True, scheme=1)
    oracle.set_ref_x(8)  # the level rule at 8 points per cell (the default, 4096, refines nothing at this n)
    try:
        er, sr = oracle.edges(w, x, d, T, kappa, 3, with_stats=True, scheme=2)
    finally:
        oracle.set_ref_x(0)
    assert sm["cand1"] == sr["cand1"] and sm["acc1"] == sr["acc1"]
    assert sm["cand2"] == sr["cand2"]
    assert sr["ev2_nonempty"] > 1.4 * sm["ev2_nonempty"]  # the children's sequences exist
    assert sr["landings"] < (0.87 if d == 3 else 0.92) * sm["landings"], (sm["landings"], sr["landings"])
    z = abs(sr["acc2"] - sm["acc2"]) / math.sqrt(sr["acc2"] + sm["acc2"])
    assert z < 5, (sm["acc2"], sr["acc2"])
    assert sr["nt1"] + sr["nt2acc"] + sr["nt2jump"] == 0


@SCHEMES
@pytest.mark.parametrize("d", [1, 2, 3])
def test_shards_partition_the_edge_set(oracle, d, scheme):
    """events are owned by the block of their A cell; shards are disjoint and
    their union is the full edge set (also exercised by the gloo multi-process test)."""
    n, T = 4000, 0.7
    w, x = synth_inputs(n, d, 2.3, 51 + d)
    kappa = oracle.scale_weights(w, 10.0, d, T, 2.3)
    full = keys(oracle.edges(w, x, d, T, kappa, 3, scheme=scheme))
    for sl in (1, 2, 3):
        nb = 1 << (d * sl)
        cuts = sorted(set([0, nb // 3, nb // 2, nb]))
        parts = [keys(oracle.edges(w, x, d, T, kappa, 3, shard=(sl, a, b), scheme=scheme))
                 for a, b in zip(cuts, cuts[1:])]
        allp = np.concatenate(parts)
        assert len(allp) == len(full)
        assert np.array_equal(np.sort(allp), full)


def test_capacity_error_and_rerun(oracle):
    """ECAPACITY reports the true m; re-running with enough capacity gives the same set."""
    import ctypes as C

    n, d, T = 3000, 1, 0.5
    w, x = synth_inputs(n, d, 2.5, 3)
    kappa = oracle.scale_weights(w, 10.0, d, T, 2.5)
    full = oracle.edges(w, x, d, T, kappa, 5)
    out = np.empty((10, 2), dtype=np.uint32)
    m = C.c_uint64(0)
    rc = oracle.lib().or_edges(oracle._dp(w), oracle._dp(x), n, d, T, kappa, 5, 0, 0, 1, oracle.SCHEME_MERGED,
                               oracle._u32p(out), 10, C.byref(m), None)
    assert rc == oracle.ECAPACITY and int(m.value) == len(full)
    assert np.array_equal(keys(oracle.edges(w, x, d, T, kappa, 5, cap=len(full))), keys(full))


@pytest.mark.parametrize("d", [1, 2])
def test_T_to_zero_limit(oracle, d):
    """P:319-320 / P:107-108: as T -> 0 the binomial model becomes the threshold model.  For
    fixed kappa the symmetric difference E_T ^ E_0 consists of the long pairs (D > q) that
    happen to be T-edges: expected sum_{D>q} (q/D)^(1/T) = sum_{u<v} p_uv - |E_0|, -> 0."""
    n = 1500
    w, x = synth_inputs(n, d, 2.5, 61 + d)
    kappa = oracle.scale_weights(w, 10.0, d, 0.0, 2.5)
    E0 = set(keys(oracle.edges(w, x, d, 0.0, kappa, 1)).tolist())
    sizes = []
    for T in (1e-2, 1e-3, 1e-4):
        mu = oracle.expected_edges_bf(w, x, d, T, kappa) - len(E0)
        ET = set(keys(oracle.edges(w, x, d, T, kappa, 2)).tolist())
        assert E0 <= ET  # every short pair has p = 1
        diff = len(ET ^ E0)
        assert abs(diff - mu) <= 5 * math.sqrt(mu) + 1, (T, diff, mu)
        sizes.append(diff)
    assert sizes[0] >= sizes[-1]
    assert sizes[-1] <= 3


@SCHEMES
def test_near_tie_detector_fires_inside_window_only(oracle, scheme):
    """O12 pin (north-star parity rule; R14, R21): the near-tie detector must fire on
    EVERY decision whose variable lies inside its window and on none outside it.  The test hook
    moves each decision variable to threshold + delta: type-I r := p_uv + delta (window 1e-12),
    type-II acceptance r_acc := p_uv/pbar + delta (window 1e-12 in r_acc), jump quotient
    z := round(z) + delta*max(1,|z|) (window 1e-15 relative).  Without the hook the counters are
    zero on the same graph, so "zero near-ties" in the parity runs is evidence, not a detector
    that never fires."""
    w, x = synth_inputs(3000, 2, 2.4, 501)
    kappa = oracle.scale_weights(w, 10.0, 2, 0.6, 2.4)
    try:
        _, base = oracle.edges(w, x, 2, 0.6, kappa, 9, with_stats=True, scheme=scheme)
        assert base["nt1"] == base["nt2acc"] == base["nt2jump"] == 0
        assert base["rnd1"] > 100 and base["landings"] > 100 and base["jchk"] > 100
        for delta in (0.0, 0.25e-12, -0.25e-12, 0.9e-12):  # inside the 1e-12 windows
            oracle.set_tie_hook(1, delta)
            _, s = oracle.edges(w, x, 2, 0.6, kappa, 9, with_stats=True, scheme=scheme)
            assert s["nt1"] == s["rnd1"] > 0, (delta, s)
            oracle.set_tie_hook(2, delta)
            _, s = oracle.edges(w, x, 2, 0.6, kappa, 9, with_stats=True, scheme=scheme)
            assert s["nt2acc"] == s["landings"] > 0, (delta, s)
        for delta in (1.1e-12, -1.1e-12, 4e-12, 1e-9):  # outside
            oracle.set_tie_hook(1, delta)
            _, s = oracle.edges(w, x, 2, 0.6, kappa, 9, with_stats=True, scheme=scheme)
            assert s["nt1"] == 0 and s["rnd1"] > 0, (delta, s)
            oracle.set_tie_hook(2, delta)
            _, s = oracle.edges(w, x, 2, 0.6, kappa, 9, with_stats=True, scheme=scheme)
            assert s["nt2acc"] == 0 and s["landings"] > 0, (delta, s)
        for delta in (0.0, 0.25e-15, -0.5e-15):  # jump: inside 1e-15 |z|
            oracle.set_tie_hook(4, delta)
            _, s = oracle.edges(w, x, 2, 0.6, kappa, 9, with_stats=True, scheme=scheme)
            assert s["nt2jump"] == s["jchk"] > 0, (delta, s)
        for delta in (2e-15, -4e-15, 1e-9):
            oracle.set_tie_hook(4, delta)
            _, s = oracle.edges(w, x, 2, 0.6, kappa, 9, with_stats=True, scheme=scheme)
            assert s["nt2jump"] == 0 and s["jchk"] > 0, (delta, s)
    finally:
        oracle.set_tie_hook(0, 0.0)

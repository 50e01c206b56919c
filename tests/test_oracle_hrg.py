"""Pins for the oracle's hyperbolic random graphs (Sec. 3.2) sampled through
the dominating GIRG of Sec. 3.3 and exact thinning (R25) -- CPU only.

The generator is pinned by closed forms and a KS test, the geometry by the two closed-form ends
of the hyperbolic law of cosines, the dominance p_HRG <= p_GIRG' by brute force over all pairs,
the threshold model by an O(n^2) brute force (exact edge-set equality), and the binomial model by
per-pair frequencies against p_T(d) over many seeds."""
import math

import numpy as np
import pytest
from scipy import stats


def keys(e):
    return np.sort((e[:, 0].astype(np.uint64) << np.uint64(32)) | e[:, 1].astype(np.uint64))


def test_radius_law_and_angles(oracle):
    """r = acosh(1 + U (cosh(alpha R) - 1)) / alpha has CDF (cosh(alpha r) - 1)/(cosh(alpha R) - 1)
    on [0, R) (density alpha sinh(alpha r)/(cosh(alpha R) - 1)); angles uniform."""
    n, alpha, C = 100_000, 0.75, -1.0
    r, x = oracle.hrg_points(n, alpha, C, 11)
    R = oracle.hrg_R(n, C)
    assert R == pytest.approx(2 * math.log(n) + C)
    assert (r >= 0).all() and (r < R).all()
    cdf = lambda t: (np.cosh(alpha * np.asarray(t)) - 1) / (math.cosh(alpha * R) - 1)  # noqa: E731
    assert stats.kstest(r, cdf).pvalue > 1e-3
    assert stats.kstest(x, "uniform").pvalue > 1e-3
    assert ((x * 2.0**53) % 1 == 0).all()  # on the 2^-53 grid


def test_hyperbolic_distance_closed_forms(oracle):
    """Law of cosines ends: equal angles give cosh(r_u - r_v), opposite angles cosh(r_u + r_v);
    symmetric; p_T(R) = 1/2; T = 0 is the strict threshold d < R."""
    for ru, rv in ((0.3, 2.0), (5.0, 7.5), (10.0, 1e-3)):
        assert oracle.hrg_cosh_dist(ru, rv, 0.25, 0.25) == pytest.approx(math.cosh(ru - rv), rel=1e-12)
        assert oracle.hrg_cosh_dist(ru, rv, 0.1, 0.6) == pytest.approx(math.cosh(ru + rv), rel=1e-12)
        assert oracle.hrg_cosh_dist(ru, rv, 0.1, 0.35) == oracle.hrg_cosh_dist(rv, ru, 0.35, 0.1)
    R = 20.0
    for T in (0.1, 0.5, 0.9):
        assert oracle.hrg_prob(math.cosh(R), R, T) == pytest.approx(0.5, rel=1e-12)
        assert oracle.hrg_prob(math.cosh(R - 4 * T), R, T) == pytest.approx(1 / (math.exp(-2) + 1), rel=1e-12)
    assert oracle.hrg_prob(math.cosh(R) * (1 - 1e-12), R, 0.0) == 1.0
    assert oracle.hrg_prob(math.cosh(R), R, 0.0) == 0.0


@pytest.mark.parametrize("alpha", [0.6, 0.75, 1.0])
@pytest.mark.parametrize("T", [0.0, 0.2, 0.5, 0.9])
def test_dominating_girg_bounds_every_pair(oracle, alpha, T):
    """R25: with w' = e^((R-r)/2)/sqrt(1-e^(-2r)) and s' = e^(-R/2)/sqrt 2, p_HRG <= p_GIRG' for
    EVERY pair (brute force, the canonical GIRG arithmetic), so thinning with p_HRG/p_GIRG' is a
    probability."""
    for C, seed in ((-1.0, 1), (1.5, 2)):
        r, x = oracle.hrg_points(1500, alpha, C, seed)
        w = oracle.hrg_dom_weights(r, C)
        assert oracle.hrg_max_ratio(r, x, w, C, T) <= 1.0


@pytest.mark.parametrize("alpha", [0.6, 0.75, 1.0])
def test_threshold_hrg_equals_bruteforce(oracle, alpha):
    """threshold HRG through the dominating GIRG == O(n^2) brute force, bit for bit."""
    for n, C, seed in ((500, -0.5, 1), (2000, -1.0, 2), (2000, 2.0, 3)):
        r, x = oracle.hrg_points(n, alpha, C, seed)
        w = oracle.hrg_dom_weights(r, C)
        e, st = oracle.hrg_edges(r, x, w, C, 0.0, seed, with_stats=True)
        assert np.array_equal(keys(e), keys(oracle.hrg_bruteforce_t0(r, x, C)))
        assert st["nt"] == 0 and st["violations"] == 0 and st["super_edges"] >= len(e)


@pytest.mark.parametrize("T", [0.3, 0.7])
def test_binomial_hrg_per_pair_frequencies(oracle, T):
    """n = 30, many edge seeds: every pair's frequency within 5 sigma of p_T(d),
    and the mean edge count within 4 standard errors of sum p_T(d)."""
    n, alpha, C, runs = 30, 0.75, 1.0, 6000
    r, x = oracle.hrg_points(n, alpha, C, 5)
    w = oracle.hrg_dom_weights(r, C)
    R = oracle.hrg_R(n, C)
    P = np.zeros((n, n))
    for u in range(n):
        for v in range(u + 1, n):
            P[u, v] = oracle.hrg_prob(oracle.hrg_cosh_dist(r[u], r[v], x[u], x[v]), R, T)
    cnt = np.zeros((n, n))
    ms = []
    for s in range(runs):
        e = oracle.hrg_edges(r, x, w, C, T, 1000 + s)
        cnt[e[:, 0], e[:, 1]] += 1
        ms.append(len(e))
    iu = np.triu_indices(n, 1)
    p, f = P[iu], cnt[iu] / runs
    sd = np.sqrt(np.maximum(p * (1 - p), 1e-12) / runs)
    assert (np.abs(f - p) <= 5 * sd + 1e-12).all(), np.max(np.abs(f - p) / sd)
    assert 0.05 < p.mean() < 0.95  # a graph with both edges and non-edges
    em = oracle.hrg_expected_edges(r, x, C, T)
    assert em == pytest.approx(p.sum(), rel=1e-12)
    assert abs(np.mean(ms) - em) < 4 * np.std(ms) / math.sqrt(runs)

"""Pins for the oracle's average-degree estimator (Sec. 5.1, App. B.2)."""
import json
import math
import os

import numpy as np
import pytest

from workloads import synth_inputs

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_worked_example(oracle):
    """n=2, d=1, T=0, w=(1,1), c=0.25 -> average degree 0.25."""
    with open(os.path.join(GOLD, "worked_examples.json")) as f:
        ex = json.load(f)["estimator"][0]
    w = np.array(ex["w"])
    assert oracle.f(w, ex["d"], ex["T"], ex["kappa"]) == pytest.approx(ex["avg_degree"], rel=1e-15)
    assert oracle.f_bruteforce(w, ex["d"], ex["T"], ex["kappa"]) == pytest.approx(ex["avg_degree"], rel=1e-15)


@pytest.mark.parametrize("d,T", [(1, 0.5), (2, 0.8), (3, 0.3), (1, 0.0), (2, 0.0)])
def test_g_is_the_expectation_over_positions(oracle, d, T):
    """Eq. 4 vs the model: for two uniform points on T^d the torus distance
    satisfies P(dist <= t) = (2t)^d, so E[p_uv] can be sampled directly; g(y) must
    match within 5 sigma for saturated, mixed and unsaturated y."""
    rng = np.random.default_rng(10 * d + int(10 * T))
    N = 200_000
    dist = rng.uniform(0, 0.5, size=(N, d)).max(axis=1)
    D = dist ** d
    for q in (1e-4, 0.01, 0.3 * 2.0**-d, 2.0**-d * 0.999, 2.0**-d * 1.5):
        y = 2.0**d * q
        if T == 0:
            vals = (D <= q).astype(float)
        else:
            vals = np.array([oracle.prob(1.0, 1.0, q, Dk, T) for Dk in D[:50_000]])
        est, se = vals.mean(), vals.std() / math.sqrt(len(vals)) + 1e-12
        assert abs(oracle.g(y, T) - est) < 5 * se + 1e-9, (q, oracle.g(y, T), est)


@pytest.mark.parametrize("d", [1, 2, 3])
@pytest.mark.parametrize("T", [0.0, 0.3, 0.5, 0.8])
def test_f_linear_equals_bruteforce(oracle, d, T):
    """P:1141-1150 closed form (with E_R in O(|R|)) == the plain O(n^2) sum of g, including
    regimes where E_R is empty and where it is large."""
    w, _ = synth_inputs(2000, d, 2.2, 3 * d + 1)
    base = oracle.scale_weights(w, 10.0, d, T, 2.2)
    # at 30x the target most heavy pairs saturate (|E_R| large): R12's grouping keeps full accuracy
    for kappa, rel in ((base * 0.01, 1e-11), (base, 1e-11), (base * 30.0, 1e-11)):
        a = oracle.f(w, d, T, kappa)
        b = oracle.f_bruteforce(w, d, T, kappa)
        assert a == pytest.approx(b, rel=rel), (kappa, a, b)


def test_ER_linear_equals_quadratic(oracle):
    """S:601 / P:1156-1158: the O(|R|) error term equals the O(|R|^2) one."""
    for d, T in ((1, 0.5), (2, 0.8), (3, 0.0), (1, 0.3)):
        w, _ = synth_inputs(20_000, d, 2.1, 7 + d)
        kappa = oracle.scale_weights(w, 50.0, d, T, 2.1)
        q = oracle.ER_quadratic(w, d, T, kappa)
        l = oracle.ER_linear(w, d, T, kappa)
        assert q != 0.0
        assert l == pytest.approx(q, rel=1e-9, abs=1e-9)


def test_equal_weights_closed_form(oracle):
    """All weights equal: f = (n-1) g(2^d kappa / n) (every pair identical)."""
    n = 500
    w = np.full(n, 3.0)
    for d, T in ((1, 0.5), (2, 0.0), (3, 0.9)):
        for kappa in (0.01, 1.0, 100.0, 1e4):
            y = 2.0**d * kappa * 9.0 / (3.0 * n)
            assert oracle.f(w, d, T, kappa) == pytest.approx((n - 1) * oracle.g(y, T), rel=1e-11)


def test_f_monotone_and_search(oracle):
    """P:639 f monotone in c; the search returns kappa with f(kappa) = target."""
    for d, T, beta, deg in ((1, 0.5, 2.5, 10.0), (2, 0.8, 2.2, 20.0), (3, 0.9, 2.9, 20.0), (1, 0.0, 2.8, 10.0)):
        w, _ = synth_inputs(30_000, d, beta, 11 * d)
        ks = np.geomspace(1e-3, 1e2, 30)
        fs = [oracle.f(w, d, T, k) for k in ks]
        assert all(a < b for a, b in zip(fs, fs[1:]))
        kappa = oracle.scale_weights(w, deg, d, T, beta)
        assert oracle.f(w, d, T, kappa) == pytest.approx(deg, rel=1e-10)


@pytest.mark.parametrize("d,T", [(1, 0.5), (2, 0.8), (1, 0.0)])
def test_degree_control_montecarlo(oracle, d, T):
    """S:600 / Sec. 5.1: the sampler's average degree over independent positions and edge seeds
    matches the target f(kappa) (f is the exact expectation given the weights)."""
    n, beta, deg = 20_000, 2.5, 10.0
    w, _ = synth_inputs(n, d, beta, 100 + d)
    kappa = oracle.scale_weights(w, deg, d, T, beta)
    degs = []
    for r in range(10):
        _, x = synth_inputs(n, d, beta, 1000 + r)
        degs.append(2 * len(oracle.edges(w, x, d, T, kappa, r + 1)) / n)
    assert abs(np.mean(degs) - deg) < 0.02 * deg, degs
    assert all(abs(v - deg) < 0.05 * deg for v in degs)

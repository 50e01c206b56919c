"""Pins for the oracle's model, randomness, grid, levels and index (CPU only).

Each test checks the oracle against something other than itself: values printed in / hand
derived from the paper (tests/golden/), a library routine (curand's Philox, math.fsum, scipy
distributions), closed forms, invariants and exhaustive brute force.
"""
import json
import math
import os
import subprocess
import ctypes as C

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ---------------------------------------------------------------- Philox4x32-10 ----------
def test_philox_published_kat(oracle):
    for v in gold("philox_kat.json")["vectors"]:
        ctr = [int(h, 16) for h in v["ctr"]]
        k0, k1 = (int(h, 16) for h in v["key"])
        out = oracle.philox(ctr, k0 | (k1 << 32))
        assert [int(o) for o in out] == [int(h, 16) for h in v["out"]]


@pytest.fixture(scope="module")
def curand_philox(tmp_path_factory):
    """The CUDA toolkit's own curand_Philox4x32_10 (host path of curand_philox4x32_x.h)."""
    inc = "/usr/local/cuda/include"
    if not os.path.exists(os.path.join(inc, "curand_philox4x32_x.h")):
        pytest.skip("CUDA headers not present")
    d = tmp_path_factory.mktemp("curand")
    src = d / "cp.cpp"
    src.write_text(
        '#define QUALIFIERS static inline\n#include <cuda_runtime.h>\n#include <curand_philox4x32_x.h>\n'
        'extern "C" void ref(const unsigned* c, unsigned long long s, unsigned* o){\n'
        ' uint4 ctr={c[0],c[1],c[2],c[3]}; uint2 k={(unsigned)s,(unsigned)(s>>32)};\n'
        ' uint4 r=curand_Philox4x32_10(ctr,k); o[0]=r.x;o[1]=r.y;o[2]=r.z;o[3]=r.w;}\n')
    so = d / "libcp.so"
    subprocess.check_call(["g++", "-O1", "-shared", "-fPIC", f"-I{inc}", str(src), "-o", str(so)])
    lib = C.CDLL(str(so))
    lib.ref.argtypes = [C.POINTER(C.c_uint32), C.c_uint64, C.POINTER(C.c_uint32)]
    return lib


def test_philox_matches_curand(oracle, curand_philox):
    rng = np.random.default_rng(123)
    for _ in range(2000):
        ctr = rng.integers(0, 2**32, size=4, dtype=np.uint64).astype(np.uint32)
        seed = int(rng.integers(0, 2**63))
        out = np.zeros(4, dtype=np.uint32)
        curand_philox.ref(ctr.ctypes.data_as(C.POINTER(C.c_uint32)), seed, out.ctypes.data_as(C.POINTER(C.c_uint32)))
        assert np.array_equal(oracle.philox(ctr, seed), out)


def test_u53_grid_and_range(oracle):
    assert oracle.u53(0, 0) == 0.0
    assert oracle.u53(0xFFFFFFFF, 0xFFFFFFFF) == 1.0 - 2.0**-53
    assert oracle.u53(0, 1 << 11) == 2.0**-53
    assert oracle.u53(0x80000000, 0) == 0.5


# ---------------------------------------------------------------- generators -------------
def test_inverse_transform_worked_examples(oracle):
    """u=0 -> w=1 (any beta); u=0.75, beta=3 -> w=2."""
    for ex in gold("worked_examples.json")["inverse_transform"]:
        assert oracle.weight_of_uniform(ex["u"], ex["beta"]) == ex["w"]


def test_weights_pareto_law(oracle):
    """w >= 1; KS test against P(w >= x) = x^(1-beta); Hill estimator."""
    from scipy import stats

    n, beta = 1 << 18, 2.5
    w = oracle.weights(n, beta, 11)
    assert w.min() >= 1.0
    ks = stats.kstest(w, lambda x: 1.0 - np.power(x, 1.0 - beta))
    assert ks.pvalue > 1e-3
    top = np.sort(w)[-n // 10:]
    hill = 1.0 + 1.0 / np.mean(np.log(top / top[0]))
    assert 2.35 <= hill <= 2.65
    # determinism and seed dependence
    assert np.array_equal(w[:100], oracle.weights(100, beta, 11))
    assert not np.array_equal(w[:100], oracle.weights(100, beta, 12))


def test_weights_use_documented_stream(oracle):
    """weights[v] uses Philox counter (v,0,0,1) words (o0,o1) through the pinned transform."""
    beta, seed = 2.8, 99
    w = oracle.weights(16, beta, seed)
    for v in range(16):
        o = oracle.philox([v, 0, 0, 1], seed)
        assert w[v] == oracle.weight_of_uniform(oracle.u53(int(o[0]), int(o[1])), beta)


def test_positions_uniform(oracle):
    from scipy import stats

    x = oracle.positions(100_000, 2, 5)
    assert x.shape == (2, 100_000)
    assert (x >= 0).all() and (x < 1).all()
    assert np.all(np.floor(x * 2.0**53) == x * 2.0**53)  # on the 2^-53 grid
    for k in range(2):
        assert 0.495 <= x[k].mean() <= 0.505
        assert stats.kstest(x[k], "uniform").pvalue > 1e-3
    # coordinate 2k / 2k+1 come from the two halves of one Philox call (v, k, 0, 2)
    o = oracle.philox([7, 0, 0, 2], 5)
    assert x[0, 7] == oracle.u53(int(o[0]), int(o[1]))
    assert x[1, 7] == oracle.u53(int(o[2]), int(o[3]))
    x3 = oracle.positions(10, 3, 5)
    o = oracle.philox([4, 1, 0, 2], 5)
    assert x3[2, 4] == oracle.u53(int(o[0]), int(o[1]))


# ---------------------------------------------------------------- exact W ----------------
def test_exact_sum_matches_fsum(oracle):
    """R3: W is the correctly rounded sum; math.fsum is a correctly rounded library routine."""
    rng = np.random.default_rng(0)
    cases = [
        rng.pareto(1.5, 100_000) + 1.0,
        np.concatenate([[2.0**60], np.ones(1000), [2.0**-30] * 7]),
        np.array([1.0, 2.0**-53, 2.0**-53]),            # exact tie -> round to even
        np.array([1.0, 2.0**-53, 2.0**-53, 2.0**-80]),  # sticky bit breaks the tie
        np.array([1.0 + 2.0**-52, 2.0**-53]),           # tie to even (up)
        rng.random(5000) * 1e-300,
        np.array([5e-324, 5e-324, 1e-310]),
    ]
    for w in cases:
        assert oracle.exact_sum(w) == math.fsum(w.tolist())


# ---------------------------------------------------------------- model ------------------
def test_torus_distance_examples_and_properties(oracle):
    for ex in gold("worked_examples.json")["torus_distance"]:
        assert oracle.torus_dist(ex["x"], ex["y"]) == pytest.approx(ex["dist"], abs=1e-15)
    rng = np.random.default_rng(1)
    for _ in range(500):
        d = int(rng.integers(1, 6))
        a, b, c = rng.random(d), rng.random(d), rng.random(d)
        dab = oracle.torus_dist(a, b)
        assert dab == oracle.torus_dist(b, a)
        assert 0.0 <= dab <= 0.5
        assert dab <= oracle.torus_dist(a, c) + oracle.torus_dist(c, b) + 1e-15
        assert oracle.torus_dist(a, a) == 0.0


def test_dpow_left_to_right(oracle):
    assert oracle.dpow(0.5, 1) == 0.5
    assert oracle.dpow(0.5, 3) == 0.125
    assert oracle.dpow(0.1, 2) == 0.1 * 0.1


def test_edge_probability_example(oracle):
    """S:69 / Eq. 1: (0.01 / 0.25)^(1/0.5) = 0.0016 (kappa = c^T = 1)."""
    ex = gold("worked_examples.json")["edge_probability"][0]
    p = oracle.prob(1.0, 1.0, ex["wuwv_over_W"] * ex["kappa"], oracle.dpow(ex["dist"], ex["d"]), ex["T"])
    assert p == pytest.approx(ex["p"], rel=1e-14)
    # saturation and the coincident-point case (R15)
    assert oracle.prob(1.0, 1.0, 0.5, 0.25, 0.5) == 1.0
    assert oracle.prob(1.0, 1.0, 0.5, 0.0, 0.5) == 1.0
    # monotone: non-increasing in D, non-decreasing in s
    Ds = np.linspace(0.01, 0.5, 50)
    ps = [oracle.prob(1.0, 2.0, 0.01, D, 0.7) for D in Ds]
    assert all(a >= b for a, b in zip(ps, ps[1:]))


def test_threshold_boundary_inclusive(oracle):
    """P:284 '<=': D == q is an edge."""
    assert oracle.thresh_edge(1.0, 1.0, 0.25, 0.25)
    assert not oracle.thresh_edge(1.0, 1.0, 0.25, np.nextafter(0.25, 1))


def test_weight_scaling_equivalence(oracle):
    """App. B.2 P:1073-1075 'scaling all weights by c^T emulates' c: with kappa = c^T, the
    probability of Eq. 1 with c outside the power equals the kappa form (R1)."""
    rng = np.random.default_rng(3)
    for _ in range(200):
        T = float(rng.uniform(0.1, 0.9))
        c = float(rng.uniform(0.1, 3))
        wu, wv, W = 1 + rng.pareto(1.5, 2)[0], 1 + rng.pareto(1.5, 2)[1], 1000.0
        D = float(rng.uniform(0.01, 0.5))
        paper = min(1.0, c * ((wu * wv / W) / D) ** (1 / T))
        assert oracle.prob(wu, wv, c**T / W, D, T) == pytest.approx(paper, rel=1e-12)


# ---------------------------------------------------------------- Morton / grid ----------
def test_morton_example_and_roundtrip(oracle):
    ex = gold("worked_examples.json")["morton"][0]
    assert oracle.morton_encode(ex["coord"], ex["d"], ex["level"]) == ex["code"]
    assert list(oracle.morton_decode(ex["code"], ex["d"], ex["level"])) == ex["coord"]
    # exhaustive d=3, level 4 and d*level <= 16 for all d
    for d in range(1, 6):
        level = 16 // d
        if d == 3:
            level = 4
        codes = set()
        for code in range(1 << (d * level)):
            c = oracle.morton_decode(code, d, level)
            assert oracle.morton_encode(c, d, level) == code
            codes.add(tuple(c))
        assert len(codes) == 1 << (d * level)


def test_morton_descendants_contiguous(oracle):
    """Sec. 4.4 property (I) P:583-584: descendants of a level-l cell occupy the code range
    [z 2^(dk), (z+1) 2^(dk)) at level l+k -- checked by brute force on coordinates."""
    for d in (1, 2, 3):
        l, k = 2, 2
        for z in range(1 << (d * l)):
            cz = oracle.morton_decode(z, d, l)
            desc = []
            for code in range(1 << (d * (l + k))):
                c = oracle.morton_decode(code, d, l + k)
                if all((c[t] >> k) == cz[t] for t in range(d)):
                    desc.append(code)
            assert desc == list(range(z << (d * k), (z + 1) << (d * k)))


def test_cell_of_point(oracle):
    for ex in gold("worked_examples.json")["cell_of_point"]:
        assert oracle.cell_of_point(ex["x"], ex["level"]) == ex["cell"]
    rng = np.random.default_rng(5)
    for _ in range(300):
        d = int(rng.integers(1, 4))
        x = rng.random(d)
        for l in range(1, 8):
            # parent(cell at l+1) == cell at l
            assert oracle.cell_of_point(x, l + 1) >> d == oracle.cell_of_point(x, l)
            c = oracle.morton_decode(oracle.cell_of_point(x, l), d, l)
            assert list(c) == [int(math.floor(v * 2**l)) for v in x]


def test_neighbors_and_min_distance(oracle):
    g = gold("worked_examples.json")
    for ex in g["neighbors"]:
        assert oracle.are_neighbors(ex["A"], ex["B"], ex["d"], ex["level"]) == ex["neighbors"]
    for ex in g["min_cell_distance"]:
        dm = oracle.delta_max(ex["A"], ex["B"], ex["d"], ex["level"])
        assert (dm - 1) * 2.0 ** -ex["level"] == ex["mind"]
    # R9 is a lower bound of point distances (random points inside the cells), and tight-ish
    rng = np.random.default_rng(7)
    for _ in range(300):
        d = int(rng.integers(1, 4))
        l = int(rng.integers(2, 5))
        A, B = (int(v) for v in rng.integers(0, 1 << (d * l), 2))
        dm = oracle.delta_max(A, B, d, l)
        ca, cb = oracle.morton_decode(A, d, l), oracle.morton_decode(B, d, l)
        for _ in range(20):
            xa = (ca + rng.random(d)) / 2**l
            xb = (cb + rng.random(d)) / 2**l
            assert oracle.torus_dist(xa, xb) >= max(dm - 1, 0) * 2.0**-l - 1e-15
        assert oracle.are_neighbors(A, B, d, l) == (dm <= 1)
    # R8: levels 0 and 1 -> every pair neighbours
    for d in (1, 2, 3):
        for A in range(1 << d):
            for B in range(1 << d):
                assert oracle.are_neighbors(A, B, d, 1)


# ---------------------------------------------------------------- levels / index ---------
def test_buckets_example(oracle):
    ex = gold("worked_examples.json")["buckets"][0]
    lv = oracle.levels(np.array(ex["w"]), 1, 1.0)
    assert lv["cnt"] == ex["counts"]


def test_comparison_level_example(oracle):
    """qbar = 0.1 -> CL = 3.  All weights 1 (wbar_0 = 2): qbar = 4 kappa / n."""
    n = 64
    lv = oracle.levels(np.ones(n), 1, 0.1 * n / 4)
    assert lv["CL"][0][0] == 3
    assert lv["I"] == [3]


def test_levels_invariants(oracle):
    """CL symmetric, non-increasing in each bucket (weights up -> coarser), I(i) = max CL(i,.);
    and the T=0 safety of R6: for every layer pair, qbar <= 2^(-d CL)."""
    for d in (1, 2, 3):
        w = oracle.weights(50_000, 2.3, d)
        lv = oracle.levels(w, d, 0.7)
        CL = lv["CL"]
        L = lv["L"]
        assert (CL == CL.T).all()
        assert (np.diff(CL, axis=1) <= 0).all()
        for i in range(L):
            ne = [j for j in range(L) if lv["cnt"][j]]
            if lv["cnt"][i]:
                assert lv["I"][i] == max(CL[i][j] for j in ne)
            for j in range(L):
                qbar = 2.0 ** (2 * lv["e_min"] + i + j + 2) * lv["s"]
                if CL[i][j] > 0:
                    assert qbar <= 2.0 ** (-d * CL[i][j])
                if CL[i][j] < lv["Lmax"]:
                    assert qbar > 2.0 ** (-d * (CL[i][j] + 1))
        assert lv["Lmax"] <= 32 // d


def test_index_hand_instance(oracle):
    ex = gold("worked_examples.json")["index_hand_instance"][0]
    xs = np.array([ex["positions"]])
    order, lstart, P, lv = oracle.index(np.ones(4), xs, 1, 0.4)  # qbar = 4*0.4/4 = 0.4 -> I = 1
    assert lv["I"] == [ex["I"]]
    assert list(xs[0][order]) == ex["sorted_positions"]
    assert list(P[0]) == ex["prefix"]


def test_index_partition_property(oracle):
    """for every layer i and level l <= I(i), the Lemma-1 ranges of the level-l
    cells partition V_i, and each range holds exactly the vertices whose cell matches
    (brute-force membership)."""
    for d in (1, 2):
        n = 3000
        w = oracle.weights(n, 2.4, 40 + d)
        x = oracle.positions(n, d, 41 + d)
        order, lstart, P, lv = oracle.index(w, x, d, 0.5)
        layer = np.array([math.floor(math.log2(v)) for v in w]) - lv["e_min"]
        for i in range(lv["L"]):
            Vi = order[lstart[i]: lstart[i + 1]]
            assert set(Vi.tolist()) == set(np.nonzero(layer == i)[0].tolist())
            # in-cell order by id (R11)
            Ii = lv["I"][i]
            cells = np.array([oracle.cell_of_point(x[:, v], Ii) for v in Vi], dtype=np.int64)
            assert (np.diff(cells) >= 0).all()
            same = cells[1:] == cells[:-1]
            assert (np.diff(Vi.astype(np.int64))[same] > 0).all()
            for l in range(0, Ii + 1):
                sh = d * (Ii - l)
                for A in range(1 << (d * l)):
                    lo, hi = P[i][A << sh], P[i][(A + 1) << sh]
                    members = [v for v in Vi if oracle.cell_of_point(x[:, v], l) == A]
                    assert sorted(Vi[lo:hi].tolist()) == sorted(members)
                if l >= 3:
                    break  # keep the brute force small


def test_cell_pair_counts_closed_forms(oracle):
    """SURVEY 8(c) K1 / Fig. 8b / App. B.5: unordered counts of
    cell pairs enumerated by Algorithm 1, per level, against closed forms."""
    g = gold("worked_examples.json")["cell_pairs_d1"]
    nb, ds, ds2, ds3 = oracle.count_pairs(1, 6)
    assert nb[g[0]["level"]] == g[0]["neighbouring_unordered"]
    assert ds[g[1]["level"]] == g[1]["distant_unordered"]
    for l in range(3, 7):
        assert ds[l] == 3 * 2 ** (l - 1)
        assert nb[l] == 2**l + 2**l  # 2^l heavy (A,A) + 2^l light (A,A+1) tasks
    for d, depth in ((1, 8), (2, 5), (3, 3)):
        nb, ds, ds2, ds3 = oracle.count_pairs(d, depth)
        assert nb[0] == 1 and ds[0] == 0
        assert nb[1] == (4**d + 2**d) // 2 and ds[1] == 0
        if depth >= 2:
            assert nb[2] == (3**d * 4**d + 4**d) // 2
            assert ds[2] == (4**d - 3**d) * 4**d // 2
        for l in range(3, depth + 1):
            assert nb[l] == (3**d + 1) * 2 ** (d * l) // 2
            assert ds[l] == (6**d - 3**d) * 2 ** (d * l) // 2
            assert ds2[l] == (5**d - 3**d) * 2 ** (d * l) // 2
            assert ds3[l] == (6**d - 5**d) * 2 ** (d * l) // 2
    # coverage identity: every ordered pair of finest cells lies under exactly one event
    for d, L in ((1, 4), (2, 4)):
        nb, ds, _, _ = oracle.count_pairs(d, L)
        nb_ord = 2 * nb[L] - 2 ** (d * L)          # ordered neighbour pairs at level L
        tot = nb_ord + sum(2 * ds[l] * 4 ** (d * (L - l)) for l in range(2, L + 1))
        assert tot == 2 ** (2 * d * L)


def test_geometric_skip(oracle):
    ex = gold("worked_examples.json")["geometric_jump"]
    assert oracle.geometric_skip(ex[0]["p"], ex[0]["u"]) == ex[0]["skip"]
    assert oracle.geometric_skip(1.0, 0.999) == 0
    # mean skip at p = 0.01 is 99; use the oracle's own uniforms
    skips = [oracle.geometric_skip(0.01, oracle.u53(*map(int, oracle.philox([k, 0, 0, 9], 1)[:2])))
             for k in range(100_000)]
    assert abs(np.mean(skips) - ex[1]["mean_skip"]) < 0.02 * 99
    # P(skip = 0) = p
    skips = np.array([oracle.geometric_skip(0.3, oracle.u53(*map(int, oracle.philox([k, 1, 0, 9], 1)[:2])))
                      for k in range(50_000)])
    assert abs((skips == 0).mean() - 0.3) < 5 * math.sqrt(0.3 * 0.7 / 50_000)


def test_deterministic_log_exp_pow(oracle):
    """R26: the decisions' log / exp / pow are written with + - * / only (so the CUDA library's
    independent copy computes the same bits); pinned against the C library: log within 2 ulp,
    exp within 2 ulp on the normal range, pow within 2e-13 relative on the decisions' range
    (x in (1e-30, 1), y = 1/T in [1, 50]); exact special values."""
    import math

    rng = np.random.default_rng(7)

    def ulp(a, b):
        return abs(int(np.float64(a).view(np.int64)) - int(np.float64(b).view(np.int64)))

    xs = np.concatenate([rng.random(20000), 10.0 ** rng.uniform(-300, 300, 20000),
                         1 + 1e-10 * rng.standard_normal(2000), [5e-324, 1e-310, 1.7e308, 2.0**-53, 1 - 2.0**-53]])
    assert max(ulp(oracle.det_log(x), math.log(x)) for x in xs if x > 0) <= 2
    ts = np.concatenate([rng.uniform(-708, 709, 20000), rng.uniform(-1e-3, 1e-3, 2000)])
    assert max(ulp(oracle.det_exp(t), math.exp(t)) for t in ts) <= 2
    worst = 0.0
    for _ in range(20000):
        x, y = 10 ** rng.uniform(-30, 0), rng.uniform(1.0, 50.0)
        e = x**y
        if e > 1e-300:
            worst = max(worst, abs(oracle.det_pow(x, y) - e) / e)
    assert worst < 2e-13
    assert oracle.det_log(1.0) == 0.0 and oracle.det_exp(0.0) == 1.0
    assert oracle.det_log(2.0) == pytest.approx(math.log(2.0), rel=1e-16)
    assert oracle.det_pow(0.3, 1.0) == pytest.approx(0.3, rel=1e-15)
    assert oracle.det_exp(-800.0) == 0.0 and math.isinf(oracle.det_exp(710.0))

"""CPU oracle for the GIRG hot path (ctypes wrapper around oracle/girg_oracle.c).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The product package
``paper_1905_06706_b200`` never imports it and shares no code with it.

Every function follows a passage of PAPER.md (arXiv:1905.06706); citations are in
``girg_oracle.h`` / ``girg_oracle.c``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "girg_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OK, EINVAL, ECAPACITY, ERANGE, ENOMEM = 0, -1, -2, -3, -4
SCHEME_EVENT, SCHEME_MERGED, SCHEME_REFINED = 0, 1, 2  # type-II: per cell pair (Alg. 1 as written) / merged (R22) / refined bound (R27)


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2, no FMA contraction, glibc libm)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "girg_oracle.h"))
    ):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-std=gnu99", "-ffp-contract=off", "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"]
        )
        os.replace(tmp, _LIB)
    return _LIB


class Stats(C.Structure):
    _fields_ = [(name, C.c_uint64) for name in (
        "visits", "ev1", "ev1_nonempty", "cand1", "acc1",
        "ev2", "ev2_nonempty", "chunks", "draws", "landings", "acc2",
        "nt1", "nt2acc", "nt2jump", "cand2", "ns_pre", "ns_edges", "rnd1", "jchk", "bound_viol")]

    def as_dict(self):
        return {k: int(getattr(self, k)) for k, _ in self._fields_}


class HrgStats(C.Structure):
    _fields_ = [(name, C.c_uint64) for name in ("super_edges", "nt", "violations")]

    def as_dict(self):
        return {k: int(getattr(self, k)) for k, _ in self._fields_}


class Levels(C.Structure):
    _fields_ = [
        ("L", C.c_int), ("e_min", C.c_int), ("Lmax", C.c_int), ("maxCL", C.c_int),
        ("W", C.c_double), ("s", C.c_double),
        ("cnt", C.c_uint64 * 64), ("CL", (C.c_int * 64) * 64), ("I", C.c_int * 64),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        d, u64, u32p, dp, i32 = C.c_double, C.c_uint64, C.POINTER(C.c_uint32), C.POINTER(C.c_double), C.c_int
        L = _lib
        L.or_philox4x32_10.argtypes = [u32p, u64, u32p]
        L.or_u53.argtypes = [C.c_uint32, C.c_uint32]; L.or_u53.restype = d
        L.or_weights.argtypes = [u64, d, u64, dp]; L.or_weights.restype = i32
        L.or_weight_of_uniform.argtypes = [d, d]; L.or_weight_of_uniform.restype = d
        L.or_positions.argtypes = [u64, i32, u64, dp]; L.or_positions.restype = i32
        L.or_exact_sum.argtypes = [dp, u64]; L.or_exact_sum.restype = d
        L.or_torus_dist.argtypes = [dp, dp, i32]; L.or_torus_dist.restype = d
        L.or_dpow.argtypes = [d, i32]; L.or_dpow.restype = d
        L.or_prob.argtypes = [d, d, d, d, d]; L.or_prob.restype = d
        L.or_thresh_edge.argtypes = [d, d, d, d]; L.or_thresh_edge.restype = i32
        L.or_morton_encode.argtypes = [u32p, i32, i32]; L.or_morton_encode.restype = C.c_uint32
        L.or_morton_decode.argtypes = [C.c_uint32, i32, i32, u32p]
        L.or_cell_of_point.argtypes = [dp, i32, i32]; L.or_cell_of_point.restype = C.c_uint32
        L.or_are_neighbors.argtypes = [C.c_uint32, C.c_uint32, i32, i32]; L.or_are_neighbors.restype = i32
        L.or_delta_max.argtypes = [C.c_uint32, C.c_uint32, i32, i32]; L.or_delta_max.restype = i32
        L.or_levels.argtypes = [dp, u64, i32, d, C.POINTER(Levels)]; L.or_levels.restype = i32
        L.or_edges.argtypes = [dp, dp, u64, i32, d, d, u64, i32, u64, u64, i32, u32p, u64,
                               C.POINTER(C.c_uint64), C.POINTER(Stats)]
        L.or_edges.restype = i32
        L.or_edges_ranked.argtypes = [dp, dp, u64, i32, d, d, u64, i32, C.c_uint32, C.c_uint32, i32, u32p, u64,
                                      C.POINTER(C.c_uint64), C.POINTER(Stats)]
        L.or_edges_ranked.restype = i32
        L.or_bruteforce_t0.argtypes = [dp, dp, u64, i32, d, u32p, u64, C.POINTER(C.c_uint64)]
        L.or_bruteforce_t0.restype = i32
        L.or_expected_edges_bf.argtypes = [dp, dp, u64, i32, d, d]; L.or_expected_edges_bf.restype = d
        L.or_g.argtypes = [d, d]; L.or_g.restype = d
        for fn in ("or_f_bruteforce", "or_f", "or_ER_quadratic", "or_ER_linear"):
            getattr(L, fn).argtypes = [dp, u64, i32, d, d]
            getattr(L, fn).restype = d
        L.or_scale_weights.argtypes = [dp, u64, d, i32, d, d, dp]; L.or_scale_weights.restype = i32
        L.or_geometric_skip.argtypes = [d, d]; L.or_geometric_skip.restype = C.c_int64
        u64p = C.POINTER(C.c_uint64)
        L.or_coverage.argtypes = [dp, dp, u64, i32, d, d, i32, u32p, C.POINTER(Stats)]; L.or_coverage.restype = i32
        L.or_index.argtypes = [dp, dp, u64, i32, d, u32p, u64p, u32p, u64p, u64]; L.or_index.restype = i32
        L.or_count_pairs.argtypes = [i32, i32, u64p, u64p, u64p, u64p]; L.or_count_pairs.restype = i32
        L.or_set_tie_hook.argtypes = [i32, d]
        L.or_set_ref_x.argtypes = [i32]
        L.or_det_log.argtypes = [d]; L.or_det_log.restype = d
        L.or_det_exp.argtypes = [d]; L.or_det_exp.restype = d
        L.or_det_pow.argtypes = [d, d]; L.or_det_pow.restype = d
        L.or_hrg_R.argtypes = [u64, d]; L.or_hrg_R.restype = d
        L.or_hrg_points.argtypes = [u64, d, d, u64, dp, dp]; L.or_hrg_points.restype = i32
        L.or_hrg_cosh_dist.argtypes = [d, d, d, d]; L.or_hrg_cosh_dist.restype = d
        L.or_hrg_prob.argtypes = [d, d, d]; L.or_hrg_prob.restype = d
        L.or_hrg_dom_weight.argtypes = [d, d]; L.or_hrg_dom_weight.restype = d
        L.or_hrg_dom_s.argtypes = [d]; L.or_hrg_dom_s.restype = d
        L.or_hrg_dom_weights.argtypes = [dp, u64, d, dp]; L.or_hrg_dom_weights.restype = i32
        L.or_hrg_edges.argtypes = [dp, dp, dp, u64, d, d, u64, u32p, u64, C.POINTER(C.c_uint64), C.POINTER(HrgStats)]
        L.or_hrg_edges.restype = i32
        L.or_hrg_bruteforce_t0.argtypes = [dp, dp, u64, d, u32p, u64, C.POINTER(C.c_uint64)]
        L.or_hrg_bruteforce_t0.restype = i32
        L.or_hrg_expected_edges.argtypes = [dp, dp, u64, d, d]; L.or_hrg_expected_edges.restype = d
        L.or_hrg_max_ratio.argtypes = [dp, dp, dp, u64, d, d]; L.or_hrg_max_ratio.restype = d
    return _lib


def _dp(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _u32p(a: np.ndarray):
    assert a.dtype == np.uint32 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_uint32))


class OracleError(RuntimeError):
    def __init__(self, code):
        super().__init__(f"oracle status {code}")
        self.code = code


def philox(ctr, seed: int) -> np.ndarray:
    c = np.asarray(ctr, dtype=np.uint32).copy()
    out = np.zeros(4, dtype=np.uint32)
    lib().or_philox4x32_10(_u32p(c), C.c_uint64(seed), _u32p(out))
    return out


def u53(hi: int, lo: int) -> float:
    return lib().or_u53(hi, lo)


def weights(n: int, beta: float, seed: int) -> np.ndarray:
    w = np.empty(n, dtype=np.float64)
    rc = lib().or_weights(n, beta, seed, _dp(w))
    if rc:
        raise OracleError(rc)
    return w


def weight_of_uniform(U: float, beta: float) -> float:
    return lib().or_weight_of_uniform(U, beta)


def positions(n: int, d: int, seed: int) -> np.ndarray:
    x = np.empty((d, n), dtype=np.float64)
    rc = lib().or_positions(n, d, seed, _dp(x))
    if rc:
        raise OracleError(rc)
    return x


def exact_sum(w: np.ndarray) -> float:
    w = np.ascontiguousarray(w, dtype=np.float64)
    return lib().or_exact_sum(_dp(w), w.size)


def torus_dist(xu, xv) -> float:
    a = np.ascontiguousarray(xu, dtype=np.float64)
    b = np.ascontiguousarray(xv, dtype=np.float64)
    return lib().or_torus_dist(_dp(a), _dp(b), a.size)


def dpow(dist: float, d: int) -> float:
    return lib().or_dpow(dist, d)


def prob(wu, wv, s, D, T) -> float:
    return lib().or_prob(wu, wv, s, D, T)


def thresh_edge(wu, wv, s, D) -> bool:
    return bool(lib().or_thresh_edge(wu, wv, s, D))


def morton_encode(coord, d: int, level: int) -> int:
    c = np.ascontiguousarray(coord, dtype=np.uint32)
    return int(lib().or_morton_encode(_u32p(c), d, level))


def morton_decode(code: int, d: int, level: int) -> np.ndarray:
    c = np.zeros(d, dtype=np.uint32)
    lib().or_morton_decode(code, d, level, _u32p(c))
    return c


def cell_of_point(x, level: int) -> int:
    a = np.ascontiguousarray(x, dtype=np.float64)
    return int(lib().or_cell_of_point(_dp(a), a.size, level))


def are_neighbors(A: int, B: int, d: int, level: int) -> bool:
    return bool(lib().or_are_neighbors(A, B, d, level))


def delta_max(A: int, B: int, d: int, level: int) -> int:
    return int(lib().or_delta_max(A, B, d, level))


def levels(w: np.ndarray, d: int, kappa: float) -> dict:
    w = np.ascontiguousarray(w, dtype=np.float64)
    lv = Levels()
    rc = lib().or_levels(_dp(w), w.size, d, kappa, C.byref(lv))
    if rc:
        raise OracleError(rc)
    L = lv.L
    return {
        "L": L, "e_min": lv.e_min, "Lmax": lv.Lmax, "maxCL": lv.maxCL, "W": lv.W, "s": lv.s,
        "cnt": [int(lv.cnt[i]) for i in range(L)],
        "CL": np.array([[lv.CL[i][j] for j in range(L)] for i in range(L)], dtype=np.int64),
        "I": [int(lv.I[i]) for i in range(L)],
    }


def edges(w, x, d, T, kappa, seed, shard=(0, 0, 1), cap=None, with_stats=False, scheme=SCHEME_MERGED):
    """Run the oracle sampler.  Returns a (m, 2) uint32 array of (u<v) pairs, unsorted
    (and the work counters when with_stats).  scheme: SCHEME_MERGED (R22, default) or
    SCHEME_EVENT (one type-II sequence per distant cell pair, Alg. 1 as written)."""
    w = np.ascontiguousarray(w, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(d, -1)
    n = w.size
    if cap is None:
        cap = max(1024, 16 * n)
    while True:
        out = np.empty((cap, 2), dtype=np.uint32)
        m = C.c_uint64(0)
        st = Stats()
        if len(shard) == 4 and shard[0] == "ranked":  # ("ranked", shard_level, nranks, rank)
            rc = lib().or_edges_ranked(_dp(w), _dp(x), n, d, float(T), float(kappa), C.c_uint64(seed),
                                       shard[1], shard[2], shard[3], scheme, _u32p(out), cap, C.byref(m),
                                       C.byref(st))
        else:
            rc = lib().or_edges(_dp(w), _dp(x), n, d, float(T), float(kappa), C.c_uint64(seed),
                                shard[0], C.c_uint64(shard[1]), C.c_uint64(shard[2]), scheme, _u32p(out),
                                cap, C.byref(m), C.byref(st))
        if rc == ECAPACITY:
            cap = int(m.value) + 1
            continue
        if rc:
            raise OracleError(rc)
        e = out[: m.value]
        return (e, st.as_dict()) if with_stats else e


def bruteforce_t0(w, x, d, kappa) -> np.ndarray:
    w = np.ascontiguousarray(w, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(d, -1)
    cap = max(1024, 8 * w.size)
    while True:
        out = np.empty((cap, 2), dtype=np.uint32)
        m = C.c_uint64(0)
        rc = lib().or_bruteforce_t0(_dp(w), _dp(x), w.size, d, float(kappa), _u32p(out), cap, C.byref(m))
        if rc == ECAPACITY:
            cap = int(m.value) + 1
            continue
        if rc:
            raise OracleError(rc)
        return out[: m.value]


def expected_edges_bf(w, x, d, T, kappa) -> float:
    w = np.ascontiguousarray(w, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(d, -1)
    return lib().or_expected_edges_bf(_dp(w), _dp(x), w.size, d, float(T), float(kappa))


def g(y, T) -> float:
    return lib().or_g(y, T)


def _wfun(name):
    def f(w, d, T, kappa):
        w = np.ascontiguousarray(w, dtype=np.float64)
        return getattr(lib(), name)(_dp(w), w.size, d, float(T), float(kappa))
    f.__name__ = name
    return f


f_bruteforce = _wfun("or_f_bruteforce")
f = _wfun("or_f")
ER_quadratic = _wfun("or_ER_quadratic")
ER_linear = _wfun("or_ER_linear")


def scale_weights(w, avg_deg, d, T, beta) -> float:
    w = np.ascontiguousarray(w, dtype=np.float64)
    k = C.c_double(0.0)
    rc = lib().or_scale_weights(_dp(w), w.size, float(avg_deg), d, float(T), float(beta), C.byref(k))
    if rc:
        raise OracleError(rc)
    return k.value


def geometric_skip(p, u) -> int:
    return int(lib().or_geometric_skip(p, u))


def det_log(x):
    return lib().or_det_log(float(x))


def det_exp(t):
    return lib().or_det_exp(float(t))


def det_pow(x, y):
    return lib().or_det_pow(float(x), float(y))


def set_tie_hook(mode: int, delta: float = 0.0):
    """TEST HOOK (O12 pin): perturb decision variables to threshold + delta (0 = off)."""
    lib().or_set_tie_hook(int(mode), float(delta))


def set_ref_x(x: int):
    """TEST HOOK (R27 pins at small n): REFINED threshold, 0 = default (4096 points per cell),
    k > 0 = k points, -1 = every level l < CL(i,j)."""
    lib().or_set_ref_x(int(x))


def sort_edges(e: np.ndarray) -> np.ndarray:
    """Edges as sorted uint64 keys (u<<32|v) for set comparison."""
    k = (e[:, 0].astype(np.uint64) << np.uint64(32)) | e[:, 1].astype(np.uint64)
    return np.sort(k)


def coverage(w, x, d, T, kappa, scheme=SCHEME_MERGED):
    """Instrumented oracle: (n, n) matrix of how often each ordered candidate (u, v) occurs."""
    w = np.ascontiguousarray(w, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(d, -1)
    n = w.size
    cov = np.zeros((n, n), dtype=np.uint32)
    st = Stats()
    rc = lib().or_coverage(_dp(w), _dp(x), n, d, float(T), float(kappa), scheme, _u32p(cov), C.byref(st))
    if rc:
        raise OracleError(rc)
    return cov, st.as_dict()


def index(w, x, d, kappa):
    """Lemma-1 index: (order, lstart[L+1], [P_i arrays], levels)."""
    w = np.ascontiguousarray(w, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(d, -1)
    n = w.size
    lv = levels(w, d, kappa)
    pcap = sum((1 << (d * lv["I"][i])) + 1 for i in range(lv["L"]))
    order = np.zeros(n, dtype=np.uint32)
    lstart = np.zeros(65, dtype=np.uint64)
    P = np.zeros(max(pcap, 1), dtype=np.uint32)
    poff = np.zeros(65, dtype=np.uint64)
    rc = lib().or_index(_dp(w), _dp(x), n, d, float(kappa), _u32p(order),
                        lstart.ctypes.data_as(C.POINTER(C.c_uint64)), _u32p(P),
                        poff.ctypes.data_as(C.POINTER(C.c_uint64)), pcap)
    if rc:
        raise OracleError(rc)
    L = lv["L"]
    Ps = [P[int(poff[i]): int(poff[i]) + (1 << (d * lv["I"][i])) + 1] for i in range(L)]
    return order, lstart[: L + 1].astype(np.int64), Ps, lv


def count_pairs(d, depth):
    """Per-level unordered cell-pair counts of Algorithm 1 on a full tree:
    (neighbouring, distant, distant with delta_max=2, distant with delta_max=3)."""
    arrs = [np.zeros(depth + 1, dtype=np.uint64) for _ in range(4)]
    rc = lib().or_count_pairs(d, depth, *[a.ctypes.data_as(C.POINTER(C.c_uint64)) for a in arrs])
    if rc:
        raise OracleError(rc)
    return [a.astype(np.int64) for a in arrs]


# ------------------------------------------------------------------ hyperbolic random graphs --
def hrg_R(n, C_):
    return lib().or_hrg_R(n, float(C_))


def hrg_points(n, alpha, C_, seed):
    """HRG radii r[n] and torus positions x[n] = theta / (2 pi)."""
    r = np.empty(n, dtype=np.float64)
    x = np.empty(n, dtype=np.float64)
    rc = lib().or_hrg_points(n, float(alpha), float(C_), C.c_uint64(seed), _dp(r), _dp(x))
    if rc:
        raise OracleError(rc)
    return r, x


def hrg_cosh_dist(ru, rv, xu, xv):
    return lib().or_hrg_cosh_dist(ru, rv, xu, xv)


def hrg_prob(cosh_d, R, T):
    return lib().or_hrg_prob(cosh_d, R, T)


def hrg_dom_weight(r, R):
    return lib().or_hrg_dom_weight(r, R)


def hrg_dom_s(R):
    return lib().or_hrg_dom_s(R)


def hrg_dom_weights(r, C_):
    r = np.ascontiguousarray(r, dtype=np.float64)
    w = np.empty_like(r)
    rc = lib().or_hrg_dom_weights(_dp(r), r.size, float(C_), _dp(w))
    if rc:
        raise OracleError(rc)
    return w


def hrg_edges(r, x, w, C_, T, seed, cap=None, with_stats=False):
    """HRG edges through the dominating GIRG and exact thinning (R25)."""
    r = np.ascontiguousarray(r, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
    w = np.ascontiguousarray(w, dtype=np.float64)
    n = r.size
    cap = cap or max(1024, 16 * n)
    while True:
        out = np.empty((cap, 2), dtype=np.uint32)
        m = C.c_uint64(0)
        st = HrgStats()
        rc = lib().or_hrg_edges(_dp(r), _dp(x), _dp(w), n, float(C_), float(T), C.c_uint64(seed), _u32p(out), cap,
                                C.byref(m), C.byref(st))
        if rc == ECAPACITY:
            cap = int(m.value) + 1
            continue
        if rc:
            raise OracleError(rc)
        e = out[: m.value]
        return (e, st.as_dict()) if with_stats else e


def hrg_bruteforce_t0(r, x, C_):
    r = np.ascontiguousarray(r, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
    cap = max(1024, 16 * r.size)
    while True:
        out = np.empty((cap, 2), dtype=np.uint32)
        m = C.c_uint64(0)
        rc = lib().or_hrg_bruteforce_t0(_dp(r), _dp(x), r.size, float(C_), _u32p(out), cap, C.byref(m))
        if rc == ECAPACITY:
            cap = int(m.value) + 1
            continue
        if rc:
            raise OracleError(rc)
        return out[: m.value]


def hrg_expected_edges(r, x, C_, T):
    r = np.ascontiguousarray(r, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
    return lib().or_hrg_expected_edges(_dp(r), _dp(x), r.size, float(C_), float(T))


def hrg_max_ratio(r, x, w, C_, T):
    r = np.ascontiguousarray(r, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
    w = np.ascontiguousarray(w, dtype=np.float64)
    return lib().or_hrg_max_ratio(_dp(r), _dp(x), _dp(w), r.size, float(C_), float(T))

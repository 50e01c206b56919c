"""paper_1905_06706_b200 -- B200-native (sm_100a) GIRG edge generator (arXiv:1905.06706).

Thin ctypes binding over the C ABI in ``include/girg.h`` (``libgirg.so``, built in-tree).
The functions below only marshal arguments: every step of the path runs in the library's
CUDA kernels.  PyTorch provides device memory and the current CUDA stream.  There is no CPU
fallback: if ``libgirg.so`` cannot be loaded, the import fails loudly.

    w = girg.weights(n, beta, seed)                    # torch.float64 [n] on cuda
    x = girg.positions(n, d, seed)                     # torch.float64 [d, n] on cuda
    kappa = girg.scale_weights(w, avg_deg, d, T, beta) # float
    e = girg.edges(w, x, T, kappa, seed)               # torch.int32 view of uint32 [m, 2], u < v
"""
from __future__ import annotations

import ctypes as C
import os

import torch

from ._build import LIB as _LIB_PATH

if os.environ.get("GIRG_LIBRARY"):  # e.g. the bounds-checked libgirg_debug.so
    _LIB_PATH = os.environ["GIRG_LIBRARY"]

OK, EINVAL, ECAPACITY, ERANGE, ENOMEM, ECUDA = 0, -1, -2, -3, -4, -5
SCHEME_EVENT, SCHEME_MERGED, SCHEME_REFINED = 0, 1, 2  # include/girg.h GIRG_SCHEME_*

if not os.path.exists(_LIB_PATH):
    raise ImportError(
        f"libgirg.so not built ({_LIB_PATH}); run `python -c 'import __graft_entry__ as g; g.build()'`")

_lib = C.CDLL(_LIB_PATH)


class Stats(C.Structure):
    _fields_ = [(k, C.c_uint64) for k in (
        "cand1", "ev2", "chunks", "draws", "landings", "edges1", "edges2",
        "neartie1", "neartie2", "layers", "key_space", "fast_fallback", "fast_mismatch", "neartie_jump")]

    def as_dict(self):
        return {k: int(getattr(self, k)) for k, _ in self._fields_}


class Options(C.Structure):
    _fields_ = [("scheme", C.c_int), ("shard_level", C.c_int), ("blk_lo", C.c_uint64), ("blk_hi", C.c_uint64),
                ("nranks", C.c_uint32), ("rank", C.c_uint32)]


class Timings(C.Structure):
    _fields_ = [("ms_total", C.c_double), ("ms_wstats", C.c_double), ("ms_index", C.c_double),
                ("ms_sample", C.c_double), ("launches", C.c_uint64), ("n", C.c_uint64), ("m", C.c_uint64),
                ("key_space", C.c_uint64), ("d", C.c_int), ("pad", C.c_int)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "pad"}


_u64, _d, _i, _vp = C.c_uint64, C.c_double, C.c_int, C.c_void_p
_lib.girg_weights.argtypes = [_u64, _d, _u64, _vp, _vp]
_lib.girg_positions.argtypes = [_u64, _i, _u64, _vp, _vp]
_lib.girg_scale_weights.argtypes = [_vp, _u64, _d, _i, _d, _d, C.POINTER(_d), _vp]
_lib.girg_edges.argtypes = [_vp, _vp, _u64, _i, _d, _d, _u64, _vp, _u64, C.POINTER(_u64), _vp]
_lib.girg_edges_shard.argtypes = [_vp, _vp, _u64, _i, _d, _d, _u64, _i, _u64, _u64, _vp, _u64,
                                  C.POINTER(_u64), C.POINTER(Stats), _vp]
_lib.girg_edges_ex.argtypes = [_vp, _vp, _u64, _i, _d, _d, _u64, C.POINTER(Options), _vp, _u64,
                               C.POINTER(_u64), C.POINTER(Stats), _vp]
_lib.girg_edges_host.argtypes = [_vp, _vp, _u64, _i, _d, _d, _u64, _vp, _u64, C.POINTER(_u64), _vp]
_lib.girg_edges_batch.argtypes = [_i, _vp, _vp, _u64, _i, _d, _vp, _vp, _vp, _vp, _vp, _vp, _i, _vp]
_lib.girg_last_timings.argtypes = [C.POINTER(Timings)]
_lib.girg_hrg_points.argtypes = [_u64, _d, _d, _u64, _vp, _vp, _vp, _vp]
_lib.girg_hrg_edges.argtypes = [_vp, _vp, _vp, _u64, _d, _d, _u64, _vp, _u64, C.POINTER(_u64), C.c_void_p, _vp]
_lib.girg_strerror.argtypes = [_i]
_lib.girg_strerror.restype = C.c_char_p
_lib.girg_last_cuda_error.restype = C.c_char_p
for _f in ("girg_weights", "girg_positions", "girg_scale_weights", "girg_edges", "girg_edges_shard",
           "girg_edges_ex", "girg_edges_host", "girg_edges_batch", "girg_version", "girg_last_timings",
           "girg_hrg_points", "girg_hrg_edges", "girg_debug_set_ref_x", "girg_debug_index"):
    getattr(_lib, _f).restype = C.c_int
_lib.girg_debug_set_ref_x.argtypes = [_i]
_lib.girg_debug_index.argtypes = [_vp, _vp, _u64, _i, _d, _d, _vp, _vp, _u64, C.POINTER(_u64), C.POINTER(_i), _vp, _vp,
                                  _vp, _vp]

EXPORTS = ("girg_weights", "girg_positions", "girg_scale_weights", "girg_edges", "girg_edges_shard",
           "girg_edges_ex", "girg_edges_host", "girg_edges_batch", "girg_strerror", "girg_last_cuda_error", "girg_version",
           "girg_last_timings", "girg_hrg_points", "girg_hrg_edges", "girg_debug_set_ref_x",
           "girg_debug_index")


class GirgError(RuntimeError):
    def __init__(self, code: int):
        msg = _lib.girg_strerror(code).decode()
        if code == ECUDA:
            msg += ": " + _lib.girg_last_cuda_error().decode()
        super().__init__(f"girg status {code}: {msg}")
        self.code = code


def _check(rc: int):
    if rc != OK:
        raise GirgError(rc)


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _dev_f64(t: torch.Tensor, name: str) -> torch.Tensor:
    if not (t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
        raise ValueError(f"{name} must be a contiguous float64 CUDA tensor")
    return t


def _edge_buf(t: torch.Tensor, name: str, cuda: bool) -> int:
    """An edge buffer must be a contiguous int32 [cap, 2] tensor (the kernels write 2*cap words)."""
    if not (t.dtype == torch.int32 and t.dim() == 2 and t.shape[1] == 2 and t.is_contiguous()):
        raise ValueError(f"{name} must be a contiguous int32 tensor of shape [cap, 2]")
    if t.is_cuda != cuda:
        raise ValueError(f"{name} must be a {'CUDA' if cuda else 'host'} tensor")
    return t.shape[0]


def _host_f64(t: torch.Tensor, name: str, numel: int) -> torch.Tensor:
    if not (not t.is_cuda and t.dtype == torch.float64 and t.is_contiguous() and t.numel() == numel):
        raise ValueError(f"{name} must be a contiguous float64 host tensor with {numel} elements")
    return t


def library_path() -> str:
    return _LIB_PATH


def version() -> int:
    return _lib.girg_version()


def debug_index(w: torch.Tensor, x: torch.Tensor, T: float, kappa: float, stream=None):
    """TEST HOOK (include/girg.h girg_debug_index): the Lemma-1 index of a girg_edges call as
    (sid [n] int32 view of uint32, P [K+1], base [L+1], lstart [L+1], I [L])."""
    import numpy as np

    _dev_f64(w, "w")
    _dev_f64(x, "x")
    n = w.numel()
    d = x.numel() // n
    base = np.zeros(65, dtype=np.uint32)
    lstart = np.zeros(65, dtype=np.uint32)
    Il = np.zeros(64, dtype=np.uint8)
    K, L = _u64(0), _i(0)
    with torch.cuda.device(w.device):
        sid = torch.empty(n, dtype=torch.int32, device=w.device)
        _check(_lib.girg_debug_index(w.data_ptr(), x.data_ptr(), n, d, T, kappa, sid.data_ptr(), None, 0, C.byref(K),
                                     C.byref(L), base.ctypes.data, lstart.ctypes.data, Il.ctypes.data, _stream(stream)))
        P = torch.empty(K.value + 1, dtype=torch.int32, device=w.device)
        _check(_lib.girg_debug_index(w.data_ptr(), x.data_ptr(), n, d, T, kappa, None, P.data_ptr(), K.value + 1,
                                     C.byref(K), C.byref(L), base.ctypes.data, lstart.ctypes.data, Il.ctypes.data,
                                     _stream(stream)))
    return sid, P, base[: L.value + 1].copy(), lstart[: L.value + 1].copy(), Il[: L.value].copy()


def debug_set_ref_x(x: int) -> None:
    """TEST HOOK (include/girg.h girg_debug_set_ref_x): SCHEME_REFINED's level threshold."""
    _check(_lib.girg_debug_set_ref_x(int(x)))


def weights(n: int, beta: float, seed: int, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Power-law weights (include/girg.h girg_weights)."""
    w = out if out is not None else torch.empty(n, dtype=torch.float64, device="cuda")
    _dev_f64(w, "out")
    _check(_lib.girg_weights(n, beta, seed, w.data_ptr(), _stream(stream)))
    return w


def positions(n: int, d: int, seed: int, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Uniform torus positions, SoA [d, n] (include/girg.h girg_positions)."""
    x = out if out is not None else torch.empty((d, n), dtype=torch.float64, device="cuda")
    _dev_f64(x, "out")
    _check(_lib.girg_positions(n, d, seed, x.data_ptr(), _stream(stream)))
    return x


def scale_weights(w: torch.Tensor, avg_deg: float, d: int, T: float, beta: float, stream=None) -> float:
    """kappa for a target expected average degree (include/girg.h girg_scale_weights)."""
    _dev_f64(w, "w")
    k = C.c_double(0.0)
    _check(_lib.girg_scale_weights(w.data_ptr(), w.numel(), avg_deg, d, T, beta, C.byref(k), _stream(stream)))
    return k.value


def edges(w: torch.Tensor, x: torch.Tensor, T: float, kappa: float, seed: int, cap: int | None = None,
          out: torch.Tensor | None = None, shard=(0, 0, 1), stats: bool = False, stream=None,
          scheme: int = SCHEME_MERGED):
    """Sample the edge list (include/girg.h girg_edges_ex; scheme SCHEME_MERGED = girg_edges).

    Returns an int32 CUDA tensor [m, 2] holding the uint32 pairs (u < v) (and the work counters
    when ``stats``).  If ``cap`` (or ``out``) is too small the call is re-issued once with the
    exact capacity the library reports."""
    _dev_f64(w, "w")
    _dev_f64(x, "x")
    n = w.numel()
    d = x.numel() // n
    if x.numel() != d * n:
        raise ValueError("x must have d*n elements")
    if x.device != w.device:
        raise ValueError("w and x must be on the same device")
    if out is not None:
        cap = _edge_buf(out, "out", cuda=True)
        if out.device != w.device:
            raise ValueError("out must be on the device of w")
    elif cap is None:
        cap = 16 * n + 1024
    with torch.cuda.device(w.device):
        return _edges_on_device(w, x, n, d, T, kappa, seed, cap, out, shard, stats, stream, scheme)


def _edges_on_device(w, x, n, d, T, kappa, seed, cap, out, shard, stats, stream, scheme):
    for _ in range(2):
        buf = out if out is not None else torch.empty((cap, 2), dtype=torch.int32, device=w.device)
        m = C.c_uint64(0)
        st = Stats()
        if len(shard) == 4 and shard[0] == "ranked":  # ("ranked", shard_level, nranks, rank)
            opt = Options(scheme, shard[1], 0, 1, shard[2], shard[3])
        else:
            opt = Options(scheme, shard[0], shard[1], shard[2], 0, 0)
        rc = _lib.girg_edges_ex(w.data_ptr(), x.data_ptr(), n, d, T, kappa, seed, C.byref(opt), buf.data_ptr(), cap,
                                C.byref(m), C.byref(st) if stats else None, _stream(stream))
        if rc == ECAPACITY and out is None:
            cap = int(m.value)
            continue
        _check(rc)
        e = buf[: m.value]
        return (e, st.as_dict()) if stats else e
    raise GirgError(ECAPACITY)


def edges_host(w_host, x_host, d: int, T: float, kappa: float, seed: int, out_host, stream=None) -> int:
    """End-to-end call with HOST (ideally pinned) tensors: returns m; edges in out_host[:m]."""
    n = w_host.numel()
    _host_f64(w_host, "w_host", n)
    _host_f64(x_host, "x_host", d * n)
    cap = _edge_buf(out_host, "out_host", cuda=False)
    m = C.c_uint64(0)
    _check(_lib.girg_edges_host(w_host.data_ptr(), x_host.data_ptr(), n, d, T, kappa, seed, out_host.data_ptr(),
                                cap, C.byref(m), _stream(stream)))
    return int(m.value)


def edges_batch(ws, xs, T: float, kappas, seeds, caps=None, nstreams: int = 8, stream=None):
    """Many independent graphs in one call (include/girg.h girg_edges_batch): graph g equals
    edges(ws[g], xs[g], T, kappas[g], seeds[g]).  Returns a list of int32 CUDA tensors [m_g, 2];
    graphs whose capacity was too small are re-issued once, individually, with the exact size."""
    B = len(ws)
    if not (len(xs) == len(kappas) == len(seeds) == B) or B < 1:
        raise ValueError("ws, xs, kappas, seeds must have the same length >= 1")
    n = ws[0].numel()
    d = xs[0].numel() // n
    for w, x in zip(ws, xs):
        _dev_f64(w, "w")
        _dev_f64(x, "x")
        if w.numel() != n or x.numel() != d * n:
            raise ValueError("all graphs must share n and d")
    if caps is None:
        caps = [16 * n + 1024] * B
    bufs = [torch.empty((int(c), 2), dtype=torch.int32, device=ws[0].device) for c in caps]
    P = C.c_void_p * B
    pw, px, pe = P(*[w.data_ptr() for w in ws]), P(*[x.data_ptr() for x in xs]), P(*[b.data_ptr() for b in bufs])
    ka, se = (_d * B)(*[float(k) for k in kappas]), (_u64 * B)(*[int(s) for s in seeds])
    ca, mo, so = (_u64 * B)(*[int(c) for c in caps]), (_u64 * B)(), (_i * B)()
    rc = _lib.girg_edges_batch(B, pw, px, n, d, T, ka, se, pe, ca, mo, so, nstreams, _stream(stream))
    out = []
    for g in range(B):
        if so[g] == ECAPACITY:
            out.append(edges(ws[g], xs[g], T, kappas[g], seeds[g], cap=int(mo[g]), stream=stream))
            continue
        _check(so[g])
        out.append(bufs[g][: mo[g]])
    if rc not in (0, ECAPACITY):
        _check(rc)
    return out


class HrgStats(C.Structure):
    _fields_ = [("super_edges", C.c_uint64), ("neartie", C.c_uint64), ("violations", C.c_uint64)]

    def as_dict(self):
        return {k: int(getattr(self, k)) for k, _ in self._fields_}


def hrg_points(n: int, alpha: float, C_: float, seed: int, stream=None):
    """HRG points (include/girg.h girg_hrg_points): radii r, torus positions x = theta/(2 pi) and
    the dominating GIRG weights w' (float64 CUDA tensors [n])."""
    r = torch.empty(n, dtype=torch.float64, device="cuda")
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    w = torch.empty(n, dtype=torch.float64, device="cuda")
    _check(_lib.girg_hrg_points(n, alpha, C_, seed, r.data_ptr(), x.data_ptr(), w.data_ptr(), _stream(stream)))
    return r, x, w


def hrg_edges(r: torch.Tensor, x: torch.Tensor, w: torch.Tensor, C_: float, T: float, seed: int,
              cap: int | None = None, stats: bool = False, stream=None):
    """HRG edge list (include/girg.h girg_hrg_edges): int32 CUDA tensor [m, 2] of uint32 pairs u < v."""
    for t, nm in ((r, "r"), (x, "x"), (w, "w")):
        _dev_f64(t, nm)
    n = r.numel()
    if x.numel() != n or w.numel() != n:
        raise ValueError("r, x, w must have n elements each")
    cap = cap if cap is not None else 16 * n + 1024
    with torch.cuda.device(r.device):
        for _ in range(2):
            buf = torch.empty((cap, 2), dtype=torch.int32, device=r.device)
            m = C.c_uint64(0)
            st = HrgStats()
            rc = _lib.girg_hrg_edges(r.data_ptr(), x.data_ptr(), w.data_ptr(), n, C_, T, seed, buf.data_ptr(), cap,
                                     C.byref(m), C.cast(C.pointer(st), C.c_void_p), _stream(stream))
            if rc == ECAPACITY:
                cap = int(m.value)
                continue
            _check(rc)
            e = buf[: m.value]
            return (e, st.as_dict()) if stats else e
    raise GirgError(ECAPACITY)


def last_timings() -> dict:
    """Phase timings (CUDA events on the call's stream) of this thread's last edges call."""
    t = Timings()
    _check(_lib.girg_last_timings(C.byref(t)))
    return t.as_dict()


def edge_keys(e: torch.Tensor) -> torch.Tensor:
    """uint32 pairs as sorted int64 keys u*2^32+v (for set comparison)."""
    u = e[:, 0].to(torch.int64) & 0xFFFFFFFF
    v = e[:, 1].to(torch.int64) & 0xFFFFFFFF
    return torch.sort(u * (1 << 32) + v).values

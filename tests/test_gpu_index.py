"""H5 parity: the Lemma-1 index the library builds (layers, Morton cells on the
insertion level, counting sort, in-cell id order, prefix arrays; App. A) against the
oracle's, array by array, through the girg_debug_index test hook of the C ABI."""
import numpy as np
import pytest
import torch

import oracle as O
from workloads import BY_NAME, synth_inputs

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1905_06706_b200 as girg  # noqa: E402


def check_index(w, x, d, T, kappa):
    wd = torch.from_numpy(np.ascontiguousarray(w)).cuda()
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    sid, P, base, lstart, Il = girg.debug_index(wd, xd, T, kappa)
    sid = sid.cpu().numpy().view(np.uint32)
    P = P.cpu().numpy().view(np.uint32).astype(np.int64)
    order, lstart_o, Ps, lv = O.index(w, x, d, kappa)
    L = lv["L"]
    assert len(Il) == L and list(Il) == list(lv["I"][:L])
    assert np.array_equal(lstart.astype(np.int64), lstart_o)
    assert np.array_equal(sid, order)  # the sorted array, element by element (in-cell order by id, R11)
    n = len(w)
    assert P[-1] == n and base[L] == len(P) - 1
    for i in range(L):
        cells = 1 << (d * int(Il[i]))
        assert int(base[i + 1]) - int(base[i]) == cells
        g = P[int(base[i]): int(base[i]) + cells + 1]  # global sorted positions; the next layer starts where this one ends
        o = Ps[i].astype(np.int64)
        assert g[0] == lstart_o[i] and g[-1] == lstart_o[i + 1]
        assert np.array_equal(g - g[0], o - o[0])  # the layer's prefix array P_C (Lemma 1)


@pytest.mark.parametrize("d", [1, 2, 3, 4, 5])
def test_index_equals_oracle_small(d):
    for n, beta, deg, seed in ((1, 2.5, 0.5, 1), (257, 2.2, 6.0, 2), (20_011, 2.8, 10.0, 3)):
        w, x = synth_inputs(n, d, beta, 11 * d + seed)
        kappa = O.scale_weights(w, deg, d, 0.5, beta) if n > 2 else 0.7
        check_index(w, x, d, 0.5, kappa)
        check_index(w, x, d, 0.0, kappa)


def test_index_crowded_cells():
    """Flat weights and a large kappa: few, crowded insertion-level cells (the k_order_big path)."""
    n, d = 50_000, 2
    _, x = synth_inputs(n, d, 2.5, 5)
    w = np.full(n, 1.5)
    check_index(w, x, d, 0.4, 3000.0)


@pytest.mark.parametrize("cfg", ["C2", "C3"])
def test_index_equals_oracle_baseline_configs(cfg):
    c = BY_NAME[cfg]
    w, x = synth_inputs(c.n, c.d, c.beta, c.seed)
    kappa = O.scale_weights(w, c.avg_deg, c.d, c.T, c.beta)
    check_index(w, x, c.d, c.T, kappa)

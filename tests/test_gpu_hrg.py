"""GPU parity of the hyperbolic random graphs (girg_hrg_points / girg_hrg_edges, R25)
against the oracle: generator within a few ulps (positions bit-exact), edge sets identical on
shared inputs with zero near-ties and zero dominance violations, the threshold model equal to an
O(n^2) brute force."""
import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1905_06706_b200 as girg  # noqa: E402


def ulps(a, b):
    return np.abs(a.view(np.int64) - b.view(np.int64))


@pytest.mark.parametrize("alpha,C", [(0.6, -1.0), (0.75, 0.5), (1.0, 2.0)])
def test_hrg_points_match_oracle(alpha, C):
    n, seed = 100_003, 7
    r, x, w = (t.cpu().numpy() for t in girg.hrg_points(n, alpha, C, seed))
    ro, xo = O.hrg_points(n, alpha, C, seed)
    assert np.array_equal(x, xo)
    assert ulps(r, ro).max() <= 8
    wo = O.hrg_dom_weights(r, C)  # the oracle's weights of the GPU radii
    assert ulps(w, wo).max() <= 8


@pytest.mark.parametrize("alpha", [0.6, 0.75, 1.0])
@pytest.mark.parametrize("T", [0.0, 0.3, 0.8])
def test_hrg_edges_equal_oracle(alpha, T):
    for n, C, seed in ((3000, -1.0, 1), (60_000, 0.5, 2)):
        r, x, w = girg.hrg_points(n, alpha, C, seed)
        e, st = girg.hrg_edges(r, x, w, C, T, seed + 5, stats=True)
        rh, xh, wh = r.cpu().numpy(), x.cpu().numpy(), w.cpu().numpy()
        eo, so = O.hrg_edges(rh, xh, wh, C, T, seed + 5, with_stats=True)
        assert so["nt"] == 0 and so["violations"] == 0
        assert st["neartie"] == 0 and st["violations"] == 0, st
        assert st["super_edges"] == so["super_edges"]
        got = girg.edge_keys(e).cpu().numpy().astype(np.uint64)
        assert np.array_equal(got, O.sort_edges(eo))
        if T == 0.0 and n <= 3000:
            assert np.array_equal(got, O.sort_edges(O.hrg_bruteforce_t0(rh, xh, C)))


def test_hrg_capacity_rerun():
    n = 20_000
    r, x, w = girg.hrg_points(n, 0.75, 0.0, 3)
    full = girg.hrg_edges(r, x, w, 0.0, 0.5, 9)
    small = girg.hrg_edges(r, x, w, 0.0, 0.5, 9, cap=10)  # ECAPACITY, re-issued with the exact size
    assert torch.equal(girg.edge_keys(full), girg.edge_keys(small))

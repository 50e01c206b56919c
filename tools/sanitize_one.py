"""One girg pipeline run for compute-sanitizer: a BASELINE config (scaled to n <= 2e5 for the
slow racecheck/synccheck tools) through weights, positions, scale and edges (both schemes, stats
and production builds), or a small batch.  python tools/sanitize_one.py C1|C2|C3|batch"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1905_06706_b200 as girg  # noqa: E402
from workloads import BY_NAME  # noqa: E402

arg = sys.argv[1]
if arg == "batch":
    n, d, T = 5000, 2, 0.5
    ws = [girg.weights(n, 2.5, g) for g in range(6)]
    xs = [girg.positions(n, d, 100 + g) for g in range(6)]
    ks = [girg.scale_weights(w, 8.0, d, T, 2.5) for w in ws]
    out = girg.edges_batch(ws, xs, T, ks, list(range(6)), nstreams=3)
    print("batch", [o.shape[0] for o in out])
else:
    c = BY_NAME[arg]
    n = min(c.n, 200_000)
    w = girg.weights(n, c.beta, c.seed)
    x = girg.positions(n, c.d, c.seed + 1)
    kappa = girg.scale_weights(w, c.avg_deg, c.d, c.T, c.beta)
    for scheme in (girg.SCHEME_MERGED, girg.SCHEME_EVENT):
        e = girg.edges(w, x, c.T, kappa, c.seed, scheme=scheme)
        e2, st = girg.edges(w, x, c.T, kappa, c.seed, scheme=scheme, stats=True)
        print(arg, n, scheme, e.shape[0], e2.shape[0], st["fast_mismatch"])
    torch.cuda.synchronize()

"""Quick GPU parity smoke over a few small cases (both type-II schemes); prints per-case status.

    python tools/quick_parity.py [--big]
Test infrastructure (calls oracle/); used during development before the full -m gpu suite."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_1905_06706_b200 as girg  # noqa: E402
from workloads import BY_NAME, synth_inputs  # noqa: E402

print("lib", girg.library_path(), flush=True)
cases = [(2000, 1, 0.0, 2.5), (3000, 2, 0.0, 2.4), (3000, 3, 0.0, 2.4), (997, 1, 0.5, 2.5), (5000, 2, 0.8, 2.2),
         (5000, 3, 0.9, 2.9), (30011, 1, 0.2, 2.1), (30011, 3, 0.9, 2.9), (4000, 4, 0.6, 2.5), (3000, 5, 0.5, 2.7)]
if "--big" in sys.argv:
    cases += [(200_000, 3, 0.9, 2.9), (300_000, 2, 0.8, 2.2)]
bad = 0
for (n, d, T, beta) in cases:
    w, x = synth_inputs(n, d, beta, 7 * d + n % 13)
    kappa = O.scale_weights(w, min(10.0, n - 1.5), d, T, beta)
    for scheme in ((0, 1) if T > 0 else (1,)):
        t0 = time.time()
        e, st = girg.edges(torch.from_numpy(w).cuda(), torch.from_numpy(x).cuda(), T, kappa, 3, stats=True,
                           scheme=scheme)
        torch.cuda.synchronize()
        t1 = time.time()
        g = girg.edge_keys(e).cpu().numpy().astype(np.uint64)
        eo, so = O.edges(w, x, d, T, kappa, 3, with_stats=True, scheme=scheme)
        o = O.sort_edges(eo)
        ok = len(g) == len(o) and np.array_equal(g, o)
        cnt = {k: (st[k], so[k2]) for k, k2 in (("cand1", "cand1"), ("landings", "landings"), ("draws", "draws"),
                                                  ("edges1", "acc1"), ("edges2", "acc2"), ("chunks", "chunks"))}
        cok = all(a == b for a, b in cnt.values())
        bad += (not ok) or (not cok)
        extra = ""
        if not ok:
            sg, so_ = set(g.tolist()), set(o.tolist())
            extra = f" gpu-only {len(sg - so_)} oracle-only {len(so_ - sg)} dup {len(g) - len(sg)}"
        print(f"n={n} d={d} T={T} scheme={scheme}: {'OK' if ok else 'MISMATCH'} m={len(g)}/{len(o)} "
              f"counters {'ok' if cok else cnt} fb {st['fast_fallback']} mm {st['fast_mismatch']} "
              f"gpu {1e3 * (t1 - t0):.1f} ms{extra}", flush=True)
        bad += st["fast_mismatch"] != 0
print("FAILURES", bad)

"""girg_scale_weights timing and attempts (GIRG_SCALE_DEBUG=1) for a few sizes:  python tools/scale_probe.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1905_06706_b200 as girg  # noqa: E402

for n, d, T in ((1 << 15, 1, 0.0), (1 << 20, 1, 0.0), (1 << 20, 1, 0.5), (1 << 24, 1, 0.0), (1 << 24, 3, 0.9)):
    w = girg.weights(n, 2.5, 1)
    torch.cuda.synchronize()
    for rep in range(3):
        t0 = time.perf_counter()
        k = girg.scale_weights(w, 10.0, d, T, 2.5)
        t1 = time.perf_counter()
    print(f"n={n} d={d} T={T} kappa={k:.12g} host_ms={1e3 * (t1 - t0):.3f}", flush=True)

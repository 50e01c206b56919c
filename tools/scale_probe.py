"""Time girg_scale_weights phases (GIRG_SCALE_DEBUG=1 prints the attempts)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1905_06706_b200 as girg
for n in (1 << 15, 1 << 20, 1 << 24):
    w = girg.weights(n, 2.5, 1)
    girg.scale_weights(w, 10.0, 1, 0.0, 2.5)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        k = girg.scale_weights(w, 10.0, 1, 0.0, 2.5)
    print(n, "scale ms %.3f" % ((time.perf_counter() - t) / 5 * 1e3), k, flush=True)

"""Summarise a GIRG_WARP_PROFILE dump (per-warp cycles, jobs, engine iterations, lane steps).
The counters exist only in libraries built with -DGIRG_PROFILE (development builds)."""
import sys

import numpy as np

for path in sys.argv[1:]:
    raw = np.fromfile(path, dtype=np.uint64)
    nw, grid, gbig, wpb = (int(v) for v in raw[:4])
    d = raw[4:].reshape(2, nw, 4).astype(np.float64)
    print(path, f"warps {nw} grid {grid} big-grid {gbig} wpb {wpb}")
    for name, a in (("k_sample", d[0, : grid * wpb]), ("k_big", d[1, : gbig * wpb])):
        cyc, jobs, it, steps = a.T
        if cyc.max() == 0:
            print(f"  {name}: idle")
            continue
        util = steps.sum() / max(1.0, 32 * it.sum())
        print(f"  {name}: max {cyc.max()/1.9e6:.2f} ms  mean {cyc.mean()/1.9e6:.2f}  p50 {np.median(cyc)/1.9e6:.2f} "
              f"p99 {np.percentile(cyc, 99)/1.9e6:.2f} | jobs {jobs.sum():.3g} iters {it.sum():.3g} lane-util {util:.2f} "
              f"| cycles/iter {cyc.sum()/max(1, it.sum()):.0f} | argmax warp jobs {jobs[cyc.argmax()]:.0f} iters {it[cyc.argmax()]:.0f}")

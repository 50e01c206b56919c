"""REFINED level-threshold sweep (experiment): sampling time and type-II work of GIRG_SCHEME_REFINED
for several thresholds x (points of layer i per level-l cell, girg_debug_set_ref_x) vs MERGED."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1905_06706_b200 as girg
from workloads import BY_NAME

cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["C3", "C5"]
xs = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [8, 64, 512, 4096]
for name in cfgs:
    c = BY_NAME[name]
    w = girg.weights(c.n, c.beta, c.seed); x = girg.positions(c.n, c.d, c.seed + 1)
    k = girg.scale_weights(w, c.avg_deg, c.d, c.T, c.beta)
    out = torch.empty((int(0.6 * c.avg_deg * c.n) + 100000, 2), dtype=torch.int32, device="cuda")
    for scheme, xv in [(girg.SCHEME_MERGED, 0)] + [(girg.SCHEME_REFINED, v) for v in xs]:
        girg.debug_set_ref_x(xv)
        ts = []
        for _ in range(4):
            e = girg.edges(w, x, c.T, k, c.seed, out=out, scheme=scheme); ts.append(girg.last_timings()["ms_sample"])
        _, st = girg.edges(w, x, c.T, k, c.seed, out=out, scheme=scheme, stats=True)
        print(name, "merged" if scheme == 1 else "refined x=%d" % xv, "m", e.shape[0], "sample ms %.2f" % min(ts[1:]),
              "landings %.3e draws %.3e chunks %.3e seqs %.3e fallbacks %.3e" % (st["landings"], st["draws"], st["chunks"], st["ev2"], st["fast_fallback"]), flush=True)
girg.debug_set_ref_x(0)

"""T = 0 timing probe (experiment): girg_edges sampling time on threshold graphs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1905_06706_b200 as girg
for n, d in ((1 << 24, 1), (1 << 22, 2), (1 << 20, 3), (10000, 1)):
    w = girg.weights(n, 2.5, 1); x = girg.positions(n, d, 2)
    k = girg.scale_weights(w, 10.0, d, 0.0, 2.5)
    out = torch.empty((8 * n + 10000, 2), dtype=torch.int32, device="cuda")
    ts = []
    for _ in range(4):
        e = girg.edges(w, x, 0.0, k, 3, out=out); ts.append(girg.last_timings()["ms_sample"])
    print(n, d, e.shape[0], "sample ms %.3f" % min(ts[1:]), girg.edge_keys(e)[:3].tolist(), flush=True)

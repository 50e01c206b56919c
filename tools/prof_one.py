"""One girg_edges call on a BASELINE config (product generators, kappa from girg_scale_weights),
for profiling under ncu:  python tools/prof_one.py C4 [merged|event|refined] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1905_06706_b200 as girg  # noqa: E402
from workloads import BY_NAME  # noqa: E402

c = BY_NAME[sys.argv[1] if len(sys.argv) > 1 else "C4"]
scheme = {"event": girg.SCHEME_EVENT, "refined": girg.SCHEME_REFINED}.get(sys.argv[2] if len(sys.argv) > 2 else "", girg.SCHEME_MERGED)
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
stats = not (len(sys.argv) > 4 and sys.argv[4] == "nostats")
w = girg.weights(c.n, c.beta, c.seed)
x = girg.positions(c.n, c.d, c.seed + 1)
kappa = girg.scale_weights(w, c.avg_deg, c.d, c.T, c.beta)
out = torch.empty((int(0.6 * c.avg_deg * c.n) + 100_000, 2), dtype=torch.int32, device="cuda")
for _ in range(reps):
    r = girg.edges(w, x, c.T, kappa, c.seed, out=out, scheme=scheme, stats=stats)
    e, st = r if stats else (r, {})
    t = girg.last_timings()
    print(c.name, "m", e.shape[0], "ms_sample %.3f ms_index %.3f" % (t["ms_sample"], t["ms_index"]), st, flush=True)

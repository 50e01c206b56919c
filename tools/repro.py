"""Debug helper: run girg.edges with/without stats on synth and Philox inputs of a config."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1905_06706_b200 as girg  # noqa: E402
from workloads import BY_NAME, synth_inputs  # noqa: E402

c = BY_NAME[sys.argv[1] if len(sys.argv) > 1 else "C2"]
mode = sys.argv[2] if len(sys.argv) > 2 else "synth"
stats = (sys.argv[3] == "stats") if len(sys.argv) > 3 else False
if mode == "synth":
    w, x = synth_inputs(c.n, c.d, c.beta, c.seed)
    w, x = torch.from_numpy(w).cuda(), torch.from_numpy(x).cuda()
else:
    w = girg.weights(c.n, c.beta, c.seed)
    x = girg.positions(c.n, c.d, c.seed + 1)
kappa = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "oracle_kappa.json")))[c.name]
try:
    r = girg.edges(w, x, c.T, kappa, c.seed, stats=stats)
    e = r[0] if stats else r
    print(c.name, mode, "stats" if stats else "nostats", "OK m=", e.shape[0], girg.last_timings()["ms_sample"])
except Exception as ex:
    print(c.name, mode, "stats" if stats else "nostats", "FAIL", ex)

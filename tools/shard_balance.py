"""Multi-GPU balance evidence on one GPU (SURVEY 8(e) "Balance"): run every rank's shard of one
graph back to back and report per-rank edge counts and device-timed sampling time, for the
interleaved ownership (default) and the contiguous block ranges.
    python tools/shard_balance.py [C3 C5 ...] > profiles/r02/shard_balance.json"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1905_06706_b200 as girg  # noqa: E402
from paper_1905_06706_b200.sharding import shard_for_rank  # noqa: E402
from workloads import BY_NAME  # noqa: E402

out = {}
BPR = int(os.environ.get("GIRG_BLOCKS_PER_RANK", "4096"))
for name in (sys.argv[1:] or ["C3", "C4", "C5"]):
    c = BY_NAME[name]
    w = girg.weights(c.n, c.beta, c.seed)
    x = girg.positions(c.n, c.d, c.seed + 1)
    kappa = girg.scale_weights(w, c.avg_deg, c.d, c.T, c.beta)
    buf = torch.empty((int(0.6 * c.avg_deg * c.n) + 100_000, 2), dtype=torch.int32, device="cuda")
    full = girg.edges(w, x, c.T, kappa, c.seed, out=buf).shape[0]
    t_full = girg.last_timings()["ms_sample"]
    res = {"m_full": full, "ms_sample_full": t_full}
    for world in (2, 4, 8):
        for mode in ("ranked", "range"):
            ms, es = [], []
            for r in range(world):
                girg.edges(w, x, c.T, kappa, c.seed, out=buf, shard=shard_for_rank(c.d, world, r, BPR, mode=mode))
                e = girg.edges(w, x, c.T, kappa, c.seed, out=buf, shard=shard_for_rank(c.d, world, r, BPR, mode=mode))
                ms.append(girg.last_timings()["ms_sample"])
                es.append(int(e.shape[0]))
            assert sum(es) == full, (sum(es), full)
            res[f"N{world}_{mode}"] = {
                "edges": es, "ms_sample": ms,
                "edges_max_over_min": max(es) / max(1, min(es)),
                "ms_max_over_mean": max(ms) / (sum(ms) / len(ms)),
                "strong_scaling_eff_model": t_full / (world * max(ms))}
    out[name] = res
    print(name, json.dumps({k: (v if not isinstance(v, dict) else {kk: vv for kk, vv in v.items()
                                                                    if kk != "edges" and kk != "ms_sample"})
                            for k, v in res.items()}), file=sys.stderr, flush=True)
print(json.dumps(out, indent=1))

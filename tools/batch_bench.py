"""Batched small graphs: throughput of girg_edges_batch on C1-sized graphs
(BASELINE config 1 shape) against the same graphs generated one girg_edges call at a time.

    python tools/batch_bench.py [--B 64] [--reps 3] [--out profiles/r01/batch_c1.json]

Each graph has its own product-generated weights/positions and seed; kappa per graph from
girg_scale_weights (outside the timed region).  Timed: CUDA events on the caller's stream around
the whole call (the call synchronises), after one warm-up; edges/s = total edges / time."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1905_06706_b200 as girg  # noqa: E402
from workloads import BY_NAME  # noqa: E402


def timed(fn):
    st = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(st)
    r = fn()
    b.record(st)
    torch.cuda.synchronize()
    return r, a.elapsed_time(b)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--B", type=int, default=64)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--config", default="C1")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    c = BY_NAME[args.config]
    ws = [girg.weights(c.n, c.beta, c.seed + 17 * g) for g in range(args.B)]
    xs = [girg.positions(c.n, c.d, c.seed + 17 * g + 1) for g in range(args.B)]
    kap = [girg.scale_weights(w, c.avg_deg, c.d, c.T, c.beta) for w in ws]
    seeds = [c.seed + 1000 + g for g in range(args.B)]
    caps = [int(0.6 * c.avg_deg * c.n) + 10_000] * args.B
    outs = [torch.empty((k, 2), dtype=torch.int32, device="cuda") for k in caps]
    rows = []

    def seq():
        return sum(girg.edges(ws[g], xs[g], c.T, kap[g], seeds[g], out=outs[g]).shape[0] for g in range(args.B))

    seq()
    best = min(timed(seq)[1] for _ in range(args.reps))
    m = seq()
    rows.append({"mode": "sequential girg_edges", "B": args.B, "ms": best, "m_total": m,
                 "edges_per_s": m / (best * 1e-3), "graphs_per_s": args.B / (best * 1e-3)})
    print(json.dumps(rows[-1]), flush=True)
    for ns in (0, -8):  # 0: the fused batch (one launch per kernel for all graphs); -8: per-graph pipelines
        def bat():
            return sum(e.shape[0] for e in girg.edges_batch(ws, xs, c.T, kap, seeds, caps=caps, nstreams=ns))

        bat()
        best = min(timed(bat)[1] for _ in range(args.reps))
        mb = bat()
        assert mb == m, (mb, m)
        rows.append({"mode": "girg_edges_batch " + ("fused" if ns >= 0 else f"per-graph pipelines x{-ns}"),
                     "nstreams": ns, "B": args.B, "ms": best, "m_total": mb,
                     "edges_per_s": mb / (best * 1e-3), "graphs_per_s": args.B / (best * 1e-3)})
        print(json.dumps(rows[-1]), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump({"config": args.config, "n": c.n, "d": c.d, "T": c.T, "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()

"""Per-step GPU run times in the style of the paper's Fig. 3: weights, positions,
scale (average-degree estimation, "Binary"), preprocessing (weight statistics + Lemma-1 index)
and edge sampling, each device-timed with CUDA events on the launching stream, as ns per edge.

Base point as in §6.1: d = 1, n = 2^15, T = 0, beta = 2.5, average degree 10;
sweeps over n (2^15 .. 2^24), T and d (the paper's plot values are not recoverable, R19).
Inputs come from the product's own generators; mean of `--reps` runs after one warm-up.

    python tools/fig3.py [--reps 5] [--out profiles/r01/fig3.json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1905_06706_b200 as girg  # noqa: E402


def timed(fn):
    st = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(st)
    r = fn()
    b.record(st)
    torch.cuda.synchronize()
    return r, a.elapsed_time(b)


def one(n, d, T, beta, deg, seed, reps):
    out = torch.empty((int(0.6 * deg * n) + 100_000, 2), dtype=torch.int32, device="cuda")
    acc = {}
    m = 0
    for k in range(reps + 1):
        w, tw = timed(lambda: girg.weights(n, beta, seed))
        x, tx = timed(lambda: girg.positions(n, d, seed + 1))
        kappa, ts = timed(lambda: girg.scale_weights(w, deg, d, T, beta))
        e, te = timed(lambda: girg.edges(w, x, T, kappa, seed + 2, out=out))
        t = girg.last_timings()
        m = e.shape[0]
        if k == 0:
            continue  # warm-up
        for key, v in (("weights", tw), ("positions", tx), ("scale", ts), ("pre", t["ms_wstats"] + t["ms_index"]),
                       ("edges", t["ms_sample"]), ("total_edges_call", te)):
            acc[key] = acc.get(key, 0.0) + v / reps
    row = {"n": n, "d": d, "T": T, "beta": beta, "avg_deg": deg, "m": m, "ms": acc,
           "ns_per_edge": {k: 1e6 * v / max(m, 1) for k, v in acc.items()}}
    print(json.dumps(row), flush=True)
    return row


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    rows = []
    for lg in range(15, 25):  # n sweep at the base point
        rows.append(one(1 << lg, 1, 0.0, 2.5, 10.0, 1, args.reps))
    for T in (0.25, 0.5, 0.75):  # temperature sweep, n = 2^20
        rows.append(one(1 << 20, 1, T, 2.5, 10.0, 1, args.reps))
    for d in (2, 3, 4):  # dimension sweep, n = 2^20, T = 0.5
        rows.append(one(1 << 20, d, 0.5, 2.5, 10.0, 1, args.reps))
    if args.out:
        with open(args.out, "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()

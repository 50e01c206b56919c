"""Hyperbolic random graphs on B200 (girg_hrg_points / girg_hrg_edges, R25): edges/s,
device-timed (CUDA events around girg_hrg_edges: the dominating GIRG and its thinning), after a
search for the C giving the target average degree at a small n (R = 2 ln n + C keeps the
average degree n-independent).
    python tools/hrg_bench.py [--n 16777216] [--alpha 0.75] [--deg 10] [--T 0 0.5] [--out x.json]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1905_06706_b200 as girg  # noqa: E402


def find_C(alpha, T, deg, n=1 << 17, seed=1):
    lo, hi = -10.0, 10.0
    for _ in range(30):
        C = 0.5 * (lo + hi)
        r, x, w = girg.hrg_points(n, alpha, C, seed)
        m = girg.hrg_edges(r, x, w, C, T, seed).shape[0]
        if 2 * m / n > deg:
            lo = C
        else:
            hi = C
    return 0.5 * (lo + hi)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 24)
    ap.add_argument("--alpha", type=float, default=0.75)
    ap.add_argument("--deg", type=float, default=10.0)
    ap.add_argument("--T", type=float, nargs="+", default=[0.0, 0.5])
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    rows = []
    st = torch.cuda.current_stream()
    for T in a.T:
        C = find_C(a.alpha, T, a.deg)
        r, x, w = girg.hrg_points(a.n, a.alpha, C, 5)
        e, s = girg.hrg_edges(r, x, w, C, T, 5, stats=True)
        m = e.shape[0]
        ts = []
        for _ in range(a.reps):
            b, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            b.record(st)
            girg.hrg_edges(r, x, w, C, T, 5, cap=m + 1024)
            c.record(st)
            torch.cuda.synchronize()
            ts.append(b.elapsed_time(c))
        ms = sorted(ts)[len(ts) // 2]
        row = {"n": a.n, "alpha": a.alpha, "beta": 2 * a.alpha + 1, "T": T, "C": C, "m": m, "avg_deg": 2 * m / a.n,
               "super_edges": s["super_edges"], "super_over_hrg": s["super_edges"] / max(1, m), "ms": ms,
               "edges_per_s": m / (ms * 1e-3), "neartie": s["neartie"], "violations": s["violations"]}
        rows.append(row)
        print(json.dumps(row), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()

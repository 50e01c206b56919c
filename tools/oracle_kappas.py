"""Writes tests/golden/oracle_kappa.json: the ORACLE's kappa (oracle.scale_weights, App. B.2)
for each BASELINE config on workloads.synth_inputs.  Calls only oracle/ (never the CUDA path).
Used by bench.py's CPU baseline (--impl reference / cpu_baseline) to avoid re-running the
O(n)-per-evaluation search on the host at bench time."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from workloads import CONFIGS, synth_inputs  # noqa: E402


def main():
    out = {"_about": "kappa = oracle.scale_weights(w, avg_deg, d, T, beta) on workloads.synth_inputs(n, d, beta, seed); "
                     "written by tools/oracle_kappas.py (oracle only)"}
    for c in CONFIGS:
        t = time.time()
        w, _ = synth_inputs(c.n, c.d, c.beta, c.seed)
        out[c.name] = oracle.scale_weights(w, c.avg_deg, c.d, c.T, c.beta)
        print(c.name, out[c.name], f"{time.time() - t:.1f}s", flush=True)
    with open(os.path.join(ROOT, "tests", "golden", "oracle_kappa.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()

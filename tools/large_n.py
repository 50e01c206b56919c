"""Large-n runs on one B200 (scale evidence): weights, positions, kappa and girg_edges at n up to
2^30, device-timed, with the device memory in use at the peak.
    python tools/large_n.py [n_log2 d T beta deg] ..."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1905_06706_b200 as girg  # noqa: E402

cases = [(27, 3, 0.9, 2.9, 20.0), (30, 1, 0.5, 2.5, 10.0)]
if len(sys.argv) > 1:
    a = sys.argv[1:]
    cases = [(int(a[0]), int(a[1]), float(a[2]), float(a[3]), float(a[4]))]
st = torch.cuda.current_stream()
for lg, d, T, beta, deg in cases:
    n = 1 << lg
    w = girg.weights(n, beta, 1)
    x = girg.positions(n, d, 2)
    t0 = time.perf_counter()
    kappa = girg.scale_weights(w, deg, d, T, beta)
    t_scale = time.perf_counter() - t0
    cap = int(0.55 * deg * n) + (1 << 20)
    out = torch.empty((cap, 2), dtype=torch.int32, device="cuda")
    free0, total = torch.cuda.mem_get_info()
    ms = []
    for _ in range(2):
        b, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        b.record(st)
        e = girg.edges(w, x, T, kappa, 3, out=out)
        c.record(st)
        torch.cuda.synchronize()
        ms.append(b.elapsed_time(c))
        tim = girg.last_timings()
    m = e.shape[0]
    print(f"n=2^{lg} d={d} T={T} beta={beta}: m={m} avg_deg={2 * m / n:.3f} edges call {min(ms):.1f} ms "
          f"({m / (min(ms) * 1e-3):.3g} edges/s; phases index {tim['ms_index']:.1f} sample {tim['ms_sample']:.1f} ms) "
          f"scale {t_scale * 1e3:.1f} ms; device memory: inputs {(d + 1) * 8 * n / 2**30:.1f} GiB + edge buffer "
          f"{8 * cap / 2**30:.1f} GiB, free before the call {free0 / 2**30:.1f} of {total / 2**30:.1f} GiB", flush=True)
    del w, x, out, e
    torch.cuda.empty_cache()

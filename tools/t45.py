import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import oracle as O, paper_1905_06706_b200 as girg
from workloads import synth_inputs
for d, T, beta in ((4, 0.6, 2.5), (5, 0.5, 2.7)):
    for n, seed in ((997, 3), (30011, 4)):
        w, x = synth_inputs(n, d, beta, 7 * d + seed)
        kappa = O.scale_weights(w, min(10.0, max(n - 1.5, 0.5)), d, T, beta)
        for scheme in (0, 1):
            t = time.time()
            e, st = girg.edges(torch.from_numpy(w).cuda(), torch.from_numpy(x).cuda(), T, kappa, seed, stats=True, scheme=scheme)
            torch.cuda.synchronize(); tg = time.time() - t
            print(f"d={d} n={n} scheme={scheme} gpu {tg:.2f}s m={e.shape[0]}", flush=True)
            t = time.time()
            eo, so = O.edges(w, x, d, T, kappa, seed, with_stats=True, scheme=scheme)
            print(f"   oracle {time.time()-t:.2f}s m={len(eo)} equal={np.array_equal(girg.edge_keys(e).cpu().numpy().astype(np.uint64), O.sort_edges(eo))}", flush=True)

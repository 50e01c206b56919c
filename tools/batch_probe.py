import os, sys
sys.path.insert(0, os.getcwd())
import torch, paper_1905_06706_b200 as girg
from workloads import BY_NAME
c = BY_NAME["C1"]; B = 64
ws = [girg.weights(c.n, c.beta, c.seed + 17 * g) for g in range(B)]
xs = [girg.positions(c.n, c.d, c.seed + 17 * g + 1) for g in range(B)]
kap = [girg.scale_weights(w, c.avg_deg, c.d, c.T, c.beta) for w in ws]
for r in range(3):
    out = girg.edges_batch(ws, xs, c.T, kap, list(range(B)))
    torch.cuda.synchronize(); print("----", flush=True)

"""bench.py's CPU oracle baseline (host logic, no GPU): the per-core shards of a whole-graph sample
add up to exactly the oracle's whole edge set, and the process count honours the request."""
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import oracle as O  # noqa: E402
from workloads import BY_NAME, synth_inputs  # noqa: E402


def test_parallel_oracle_sample_is_the_whole_graph():
    c = BY_NAME["C1"]
    rate, secs, desc, used = bench.oracle_sample(c, workers=3)
    assert used == 3 and rate > 0 and secs > 0
    m_sample = int(re.search(r"; (\d+) edges, slowest worker", desc).group(1))
    with open(os.path.join(ROOT, "tests", "golden", "oracle_kappa.json")) as f:
        kappa = json.load(f)[c.name]
    w, x = synth_inputs(c.n, c.d, c.beta, c.seed)
    assert m_sample == len(O.edges(w, x, c.d, c.T, kappa, c.seed))


def test_oracle_workers_bounded_by_cores():
    n_cores = len(os.sched_getaffinity(0))
    assert 1 <= bench.oracle_workers(1 << 24) <= n_cores
    assert 1 <= bench.oracle_workers(10_000) <= n_cores

"""Workload definitions and the seeded synthetic input generator shared by tests and bench.

This module holds NONE of the method's arithmetic: it only names the BASELINE.json configs and
draws seeded inputs (weights, positions) with numpy's own PCG64 generator, so that the CPU
oracle (``oracle/``) and the CUDA path (``paper_1905_06706_b200``) can be run on identical
inputs without either side producing the other's inputs.

Input recipe:
  * weights: Pareto with w_min = 1 and tail P(w >= x) = x^(1-beta)  (numpy ``pareto(beta-1)+1``),
    the law the configs state (BASELINE.json configs; "power law with
    exponent beta > 2");
  * positions: i.i.d. uniform on [0,1)^d on the 2^-53 grid (``integers(0, 2^53) * 2^-53``),
    structure-of-arrays ``x[d][n]``;
  * all draws from ``numpy.random.Generator(PCG64(seed))``.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    d: int
    T: float
    beta: float
    avg_deg: float
    seed: int


# BASELINE.json "configs" (in order)
CONFIGS = [
    Config("C1", 10_000, 1, 0.0, 2.8, 10.0, 1),
    Config("C2", 1_000_000, 1, 0.5, 2.5, 10.0, 2),
    Config("C3", 1_000_000, 2, 0.8, 2.2, 20.0, 3),
    Config("C4", 10_000_000, 1, 0.5, 2.5, 10.0, 4),
    Config("C5", 16_777_216, 3, 0.9, 2.9, 20.0, 5),
]
BY_NAME = {c.name: c for c in CONFIGS}


def synth_inputs(n: int, d: int, beta: float, seed: int):
    """Seeded weights (n,) float64 and positions (d, n) float64 (see module docstring)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    w = rng.pareto(beta - 1.0, size=n) + 1.0
    x = rng.integers(0, 1 << 53, size=(d, n), dtype=np.int64).astype(np.float64) * 2.0 ** -53
    return np.ascontiguousarray(w), np.ascontiguousarray(x)

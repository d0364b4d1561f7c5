"""Shared helpers for the parity tests (test infrastructure)."""
from __future__ import annotations

import numpy as np

from paper_2505_20719_b200 import problems

F3R16 = "F100:f64/f64 > F8:f32/f32 > F4:f16/f32 > R2:f16,c=64 > identity"
F3R32 = "F100:f64/f64 > F8:f32/f32 > F4:f32/f32 > R2:f32,c=64 > identity"
F3R64 = "F100:f64/f64 > F8:f64/f64 > F4:f64/f64 > R2:f64,c=64 > identity"

# relative normwise tolerances of BASELINE.json north_star, per precision tag
TOL = {0: 2e-3, 1: 1e-5, 2: 1e-12}


def small_problems():
    """(name, Problem) at sizes the CPU oracle finishes in seconds."""
    return [
        ("hpcg16", problems.problem(2, grid=16)),
        ("poisson24", problems.problem(1, grid=24)),
        ("convdiff16", problems.problem(3, grid=16)),
        ("aniso16", problems.problem(4, grid=16)),
        ("unstructured6000", problems.problem(5, grid=6000)),
    ]


def rand_vec(oracle, p, n, seed, lo=-1.0, hi=1.0):
    rng = np.random.default_rng(seed)
    return oracle.round_vec(p, rng.uniform(lo, hi, n))


def normwise(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (den if den > 0 else 1.0)

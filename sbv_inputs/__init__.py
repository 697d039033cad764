"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

This module holds NONE of the method's arithmetic (no scaling, clustering,
distances, covariance or likelihood): it only draws the inputs {X, y} and names
the workload shapes of BASELINE.json's configs.  Recipes (DESIGN.md "Input
recipe"):

* X ~ U[0,1]^d i.i.d. (PCG64 via numpy.random.default_rng(seed_x)) — the
  paper's synthetic design "x in [0,1]^10" and "inputs scaled into
  [0,1]" for MetaRVM.
* y: a smooth random function of the inputs plus a small noise term
  (``smooth``), or i.i.d. N(0,1) (``iid``).  The log-likelihood's cost does not
  depend on y; ``smooth`` gives a GP-like response with two relevant
  dimensions as in the paper's beta = (0.05, 0.05, 5 x 8).
* ``lattice``: coordinates on a k/8 grid (exactly representable) for
  tie-rule tests of RAC/kNN, where every distance is computed exactly.
"""
from __future__ import annotations

import numpy as np

# The paper's Section 6.1 truth: beta_1 = beta_2 = 0.05, beta_3..10 = 5.
PAPER_BETA_D10 = (0.05, 0.05) + (5.0,) * 8

CONFIGS = {
    # name: (n, d, bs, m, nu) — BASELINE.json configs
    "cfg1": dict(n=20_000, d=10, bs=20, m=60, nu=2.5),
    "cfg2": dict(n=1_000_000, d=10, bs=100, m=200, nu=2.5),
    "cfg3": dict(n=2_000_000, d=10, bs=100, m=200, nu=2.5),
    "cfg4": dict(n=50_000_000, d=10, bs=100, m=400, nu=3.5),
    "cfg5": dict(n=5_000_000, d=10, bs=100, m=200, nu=2.5),
}

# MetaRVM input bounds, Table 4, normalised to [0,1] on ingestion.
METARVM_BOUNDS = [(0.1, 0.9), (0.1, 0.9), (30, 90), (1, 5), (1, 3), (1, 9), (1, 9),
                  (1, 5), (30, 90), (0.3, 0.8)]


def make_X(n: int, d: int, seed: int = 1, kind: str = "uniform") -> np.ndarray:
    """n x d row-major float64 inputs."""
    rng = np.random.default_rng(seed)
    if kind == "uniform":
        return rng.random((n, d))
    if kind == "lattice":
        return rng.integers(0, 9, size=(n, d)).astype(np.float64) / 8.0
    if kind == "duplicates":
        X = rng.random((n, d))
        X[n // 2] = X[0]
        return X
    raise ValueError(kind)


def make_y(X: np.ndarray, seed: int = 2, kind: str = "smooth") -> np.ndarray:
    """Responses for the inputs X (float64, length n)."""
    n, d = X.shape
    rng = np.random.default_rng(seed)
    if kind == "iid":
        return rng.standard_normal(n)
    if kind == "zero":
        return np.zeros(n)
    if kind == "smooth":
        # sum of F random cosines; dims 0,1 carry high frequencies, the rest low
        F = 32
        freq_scale = np.full(d, 0.2)
        freq_scale[: min(2, d)] = 4.0
        W = rng.standard_normal((F, d)) * freq_scale
        b = rng.random(F) * 2 * np.pi
        a = rng.standard_normal(F) * np.sqrt(2.0 / F)
        y = np.zeros(n)
        for f in range(F):
            y += a[f] * np.cos(2 * np.pi * (X @ W[f]) + b[f])
        return y + 0.01 * rng.standard_normal(n)
    raise ValueError(kind)


def default_theta(d: int, nu: float = 2.5, sigma2: float = 1.0, tau2: float = 1e-4,
                  beta=None) -> np.ndarray:
    """theta = {sigma2, beta_1..beta_d, nu, tau2} (S:34-35 order)."""
    if beta is None:
        beta = PAPER_BETA_D10 if d == 10 else tuple([0.25] * d)
    return np.array([sigma2, *beta, nu, tau2], dtype=np.float64)


def default_scale(d: int) -> np.ndarray:
    return np.array(PAPER_BETA_D10 if d == 10 else [0.25] * d, dtype=np.float64)

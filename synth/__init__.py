"""Seeded synthetic inputs shared by the oracle side (tests) and the CUDA side (tests, bench).

This module holds NO arithmetic of the method (no covariance, no factorisation): only the
configurations of BASELINE.json (`configs[0..4]` = C1..C5) with the readings of DESIGN.md
(seeds R13, nugget R2, C3 cluster R14, C2 grid R16), and seeded random draws:
locations s (n x 2, external order) and standard-normal vectors xi.

The paper's experiments are synthetic (locations sampled, data Z = L xi);
its "moisture" data set is not available and is not reconstructed.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Tuple

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    sigma2: float
    ell: float
    nu: float
    nugget: float
    eps: Tuple[float, ...]
    kmax: int                      # 0 = no rank cap
    geometry: str = "uniform"      # "uniform" | "clustered"
    ell_grid: Tuple[float, ...] = field(default_factory=tuple)
    seed_points: int = 0
    seed_xi: int = 0
    seed_cluster: int = 0


def _ell_grid_c2() -> Tuple[float, ...]:
    # DESIGN.md R16: 64 log-spaced ell on [0.01, 0.3]: ell_i = 0.01 * 30^(i/63)
    return tuple(float(0.01 * 30.0 ** (i / 63.0)) for i in range(64))


CONFIGS = {
    "C1": Config("C1", 2000, 1.0, 0.1, 0.5, 1e-6, (1e-8,), 0,
                 seed_points=1001, seed_xi=2001),
    "C2": Config("C2", 16384, 1.0, 0.05, 1.5, 1e-6, (1e-4, 1e-8), 0,
                 ell_grid=_ell_grid_c2(), seed_points=1002, seed_xi=2002),
    "C3": Config("C3", 131072, 1.0, 0.0864, 0.5, 1e-6, (1e-6,), 16, geometry="clustered",
                 seed_points=1003, seed_xi=2003, seed_cluster=3003),
    "C4": Config("C4", 524288, 1.0, 0.1, 0.5, 1e-6, (1e-6,), 20,
                 seed_points=1004, seed_xi=2004),
    "C5": Config("C5", 2097152, 1.0, 0.05, 1.0, 1e-6, (1e-5,), 20,
                 seed_points=1005, seed_xi=2005),
}


# eps of the tight H-Cholesky factor whose samples Z = L~ xi are the data of
# C3 / C4 / C5 (no rank cap for C3 / C4).  C5: 1e-8, "if memory forbids, 1e-7" (bench.py).
EPS_GEN = {"C3": 1e-10, "C4": 1e-10, "C5": 1e-8}

def uniform_points(n: int, seed: int) -> np.ndarray:
    """n points U[0,1]^2, (n, 2) float64, external order."""
    return np.random.default_rng(seed).random((n, 2))


def uniform_points_3d(n: int, seed: int) -> np.ndarray:
    """n points U[0,1]^3, (n, 3) float64 (the 3-D variant)."""
    return np.random.default_rng(seed).random((n, 3))


def clustered_points(n: int, seed: int, seed_cluster: int, frac: float = 0.05,
                     lo: float = 0.40, hi: float = 0.45) -> np.ndarray:
    """DESIGN.md R14: U[0,1]^2 with floor(frac*n) seeded indices moved to U[lo,hi]^2."""
    s = uniform_points(n, seed)
    rng = np.random.default_rng(seed_cluster)
    m = int(np.floor(frac * n))
    idx = rng.choice(n, size=m, replace=False)
    s[idx] = lo + (hi - lo) * rng.random((m, 2))
    return s


def points(cfg: Config) -> np.ndarray:
    if cfg.geometry == "clustered":
        return clustered_points(cfg.n, cfg.seed_points, cfg.seed_cluster)
    return uniform_points(cfg.n, cfg.seed_points)


def xi(n: int, seed: int) -> np.ndarray:
    """Standard-normal vector (the xi of Z = L xi)."""
    return np.random.default_rng(seed).standard_normal(n)


def collinear_points(n: int, seed: int) -> np.ndarray:
    """Points on the segment y = 0, x ~ U[0,1] (sorted order not assumed)."""
    x = np.random.default_rng(seed).random(n)
    return np.stack([x, np.zeros(n)], axis=1)

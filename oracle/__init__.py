"""ORACLE — test infrastructure only.

Plain, slow, obviously-correct CPU implementation of what the hot path computes.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import this package.  It shares no code, headers,
tables or helpers with ``paper_1709_08625_b200`` (the CUDA path) and never imports it.

Functions and the passages they follow (PAPER.md = the paper's LaTeX text):

* ``besselk``, ``matern``  — Eq. (3), PAPER.md:185-191 (C(h;theta)); K_nu from the
  integral representation (C code in ``matern.c``); half-integer closed forms
  (read with Eq. (3)'s argument h/ell — DESIGN.md reading R1).
* ``cov_dense``            — C_ij = C(s_i - s_j; theta) (Eq. (1) text)
  + nugget tau^2 on the diagonal (listing).
* ``loglik_dense``         — Eq. (1), PAPER.md:109-114:
  L = -n/2 log(2 pi) - 1/2 log det C - 1/2 Z^T C^{-1} Z, computed through the Cholesky
  factor C = L L^T exactly as Eq. (2) / Def. 1 writes it with the
  exact factor: log det C = 2 sum log L_ii, v = L^{-1} Z, Z^T C^{-1} Z = v^T v.
  The factorisation and the triangular solve are LAPACK library primitives (MKL, through
  plain PyTorch CPU ops: the OpenBLAS builds of numpy/scipy in this image return a spurious
  "not positive definite" (scipy, 32-bit LAPACK) or crash (numpy) for n >= 32,768).
* ``loglik_ou_collinear``  — Eq. (1) in closed form for nu = 1/2, tau^2 = 0 on collinear
  points: the exponential covariance (Eq. (3) at nu = 1/2) on a line is the
  Ornstein-Uhlenbeck process, which is Markov, so the joint density factorises into
  one-step conditionals.  O(n) exact L at any n (used at 2M).
* ``sample_dense``         — Z = L xi with the exact dense factor (Sec. 5.1, PAPER.md:573-577,
  with the exact factor in place of the H-factor; configs C1/C2 of BASELINE.json).

Parity pins for every function are in ``tests/test_oracle.py`` (none unpinned).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import contextlib

import numpy as np
import torch

# Host threads used by the oracle (OpenMP fill + MKL LAPACK): every host core by default.
THREADS = int(os.environ.get("HCOV_ORACLE_THREADS", os.cpu_count() or 1))


@contextlib.contextmanager
def lapack_threads(k: int = 0):
    """Run MKL (torch CPU) LAPACK/BLAS calls on k (default THREADS) threads."""
    old = torch.get_num_threads()
    torch.set_num_threads(k or THREADS)
    try:
        yield
    finally:
        torch.set_num_threads(old)

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "matern.c")
_SO = os.path.join(_HERE, "_oracle_matern.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile matern.c (gcc -O2 -fopenmp, no fast-math). Returns the .so path."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", _SO, _SRC, "-lm"])
    return _SO


def _load():
    global _lib
    if _lib is None:
        build()
        # OpenMP threads of matern.c must not spin after their loop and starve the
        # LAPACK (OpenBLAS) threads of the Cholesky step.
        os.environ.setdefault("OMP_WAIT_POLICY", "PASSIVE")
        os.environ.setdefault("OMP_NUM_THREADS", str(THREADS))
        lib = ctypes.CDLL(_SO)
        d, i64, p = ctypes.c_double, ctypes.c_int64, ctypes.c_void_p
        lib.oracle_besselk.restype = d
        lib.oracle_besselk.argtypes = [d, d]
        lib.oracle_besselk_scaled.restype = d
        lib.oracle_besselk_scaled.argtypes = [d, d]
        lib.oracle_matern.restype = d
        lib.oracle_matern.argtypes = [d, d, d, d]
        lib.oracle_matern_integral.restype = d
        lib.oracle_matern_integral.argtypes = [d, d, d, d]
        lib.oracle_cov_dense.restype = None
        lib.oracle_cov_dense.argtypes = [i64, ctypes.c_int, p, d, d, d, d, p]
        lib.oracle_cov_entries.restype = None
        lib.oracle_cov_entries.argtypes = [i64, ctypes.c_int, p, d, d, d, d, p, i64, p, i64, p]
        _lib = lib
    return _lib


def besselk(nu: float, x: float) -> float:
    """K_nu(x) by the trapezoid rule on DLMF 10.32.9."""
    return _load().oracle_besselk(float(nu), float(x))


def matern(h: float, sigma2: float, ell: float, nu: float, integral: bool = False) -> float:
    """Eq. (3): sigma^2 / (2^(nu-1) Gamma(nu)) (h/ell)^nu K_nu(h/ell)."""
    lib = _load()
    f = lib.oracle_matern_integral if integral else lib.oracle_matern
    return f(float(h), float(sigma2), float(ell), float(nu))


def _coords(s) -> np.ndarray:
    s = np.ascontiguousarray(s, dtype=np.float64)
    if s.ndim != 2 or s.shape[1] not in (2, 3):
        raise ValueError("locations must be n x 2 or n x 3")
    return s


def cov_dense(s: np.ndarray, sigma2: float, ell: float, nu: float, nugget: float) -> np.ndarray:
    """Dense n x n covariance in external order (Eq. (1) definition + nugget); s: n x 2, or n x 3
    for the 3-D variant."""
    s = _coords(s)
    n = s.shape[0]
    C = np.empty((n, n), dtype=np.float64)
    _load().oracle_cov_dense(n, s.shape[1], s.ctypes.data, sigma2, ell, nu, nugget, C.ctypes.data)
    return C


def cov_entries(s, sigma2, ell, nu, nugget, rows, cols) -> np.ndarray:
    """C[rows][:, cols] (external indices) without forming C."""
    s = _coords(s)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    cols = np.ascontiguousarray(cols, dtype=np.int64)
    out = np.empty((rows.size, cols.size), dtype=np.float64)
    _load().oracle_cov_entries(s.shape[0], s.shape[1], s.ctypes.data, sigma2, ell, nu, nugget,
                               rows.ctypes.data, rows.size, cols.ctypes.data, cols.size,
                               out.ctypes.data)
    return out


class NotSPD(Exception):
    pass


def cholesky(C: np.ndarray) -> np.ndarray:
    """Lower Cholesky factor (LAPACK dpotrf, MKL). Raises NotSPD if a pivot is <= 0."""
    with lapack_threads():
        L, info = torch.linalg.cholesky_ex(torch.from_numpy(np.ascontiguousarray(C, dtype=np.float64)))
    if int(info) != 0:
        raise NotSPD(f"leading minor {int(info)} is not positive definite")
    return L.numpy()


def solve_lower(L: np.ndarray, b: np.ndarray) -> np.ndarray:
    """x = L^{-1} b for lower-triangular L (LAPACK dtrtrs / BLAS dtrsm, MKL)."""
    b = np.asarray(b, dtype=np.float64)
    B = torch.from_numpy(np.ascontiguousarray(b.reshape(b.shape[0], -1)))
    with lapack_threads():
        x = torch.linalg.solve_triangular(torch.from_numpy(L), B, upper=False)
    return x.numpy().reshape(b.shape)


def loglik_from_factor(L: np.ndarray, Z: np.ndarray):
    """Eq. (1) through the factor: returns (loglik, logdet, quad)."""
    n = L.shape[0]
    logdet = 2.0 * float(np.sum(np.log(np.diag(L))))
    v = solve_lower(L, Z)
    quad = float(v @ v)
    ll = -0.5 * n * np.log(2.0 * np.pi) - 0.5 * logdet - 0.5 * quad
    return ll, logdet, quad


def loglik_dense(s, Z, sigma2, ell, nu, nugget):
    """Exact Gaussian log-likelihood Eq. (1). Returns (loglik, logdet, quad)."""
    C = cov_dense(s, sigma2, ell, nu, nugget)
    L = cholesky(C)
    del C
    return loglik_from_factor(L, Z)


def sample_dense(s, xi, sigma2, ell, nu, nugget):
    """Z = L xi with the exact dense Cholesky factor (external order)."""
    C = cov_dense(s, sigma2, ell, nu, nugget)
    L = cholesky(C)
    del C
    with lapack_threads():
        return (torch.from_numpy(L) @ torch.from_numpy(np.ascontiguousarray(xi, dtype=np.float64))).numpy()


def loglik_ou_collinear(x, Z, sigma2, ell):
    """Exact Eq. (1) for nu = 1/2, tau^2 = 0, points (x_i, 0) on a line.

    Sort x_1 < ... < x_n, rho_i = exp(-(x_i - x_{i-1}) / ell).  The field is Markov:
    Z_1 ~ N(0, sigma2), Z_i | Z_{i-1} ~ N(rho_i Z_{i-1}, sigma2 (1 - rho_i^2)), hence
    log det C = n log sigma2 + sum_{i>=2} log(1 - rho_i^2) and
    Z^T C^{-1} Z = Z_1^2 / sigma2 + sum_{i>=2} (Z_i - rho_i Z_{i-1})^2 / (sigma2 (1 - rho_i^2)).
    Returns (loglik, logdet, quad)."""
    x = np.asarray(x, dtype=np.float64)
    Z = np.asarray(Z, dtype=np.float64)
    o = np.argsort(x, kind="stable")
    x, z = x[o], Z[o]
    d = np.diff(x)
    om = -np.expm1(-2.0 * d / ell)          # 1 - rho^2 without cancellation
    rho = np.exp(-d / ell)
    n = x.size
    logdet = n * np.log(sigma2) + float(np.sum(np.log(om)))
    quad = z[0] ** 2 / sigma2 + float(np.sum((z[1:] - rho * z[:-1]) ** 2 / (sigma2 * om)))
    return -0.5 * n * np.log(2.0 * np.pi) - 0.5 * logdet - 0.5 * quad, logdet, quad


def sample_ou_collinear(x, xi, sigma2, ell):
    """Exact draw Z ~ N(0, C) for the collinear exponential model (same setting as
    loglik_ou_collinear): in sorted order Z_1 = sigma xi_1,
    Z_i = rho_i Z_{i-1} + sigma sqrt(1 - rho_i^2) xi_i.  Returned in the input order."""
    x = np.asarray(x, dtype=np.float64)
    xi = np.asarray(xi, dtype=np.float64)
    o = np.argsort(x, kind="stable")
    xs = x[o]
    d = np.diff(xs)
    rho = np.exp(-d / ell)
    sd = np.sqrt(sigma2 * -np.expm1(-2.0 * d / ell))
    z = np.empty_like(xs)
    z[0] = np.sqrt(sigma2) * xi[o[0]]
    for i in range(1, xs.size):
        z[i] = rho[i - 1] * z[i - 1] + sd[i - 1] * xi[o[i]]
    out = np.empty_like(z)
    out[o] = z
    return out

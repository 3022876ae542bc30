"""CPU build of the device Matern / K_nu code (matern.cuh compiled with g++): the series /
continued fraction K_nu and the per-theta Chebyshev table against scipy.special.kv and the oracle."""
import ctypes
import math
import os
import subprocess

import numpy as np
import pytest
from scipy.special import kv, gamma

import oracle

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "host", "matern_host.cpp")
SO = os.path.join(HERE, "host", "_matern_host.so")


@pytest.fixture(scope="module")
def lib():
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-o", SO, SRC])
    L = ctypes.CDLL(SO)
    L.host_besselk.restype = ctypes.c_double
    L.host_besselk.argtypes = [ctypes.c_double, ctypes.c_double]
    L.host_matern.restype = None
    L.host_matern.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_void_p,
                              ctypes.c_int64, ctypes.c_int, ctypes.c_void_p]
    return L


def _matern(L, s2, ell, nu, h, tab):
    h = np.ascontiguousarray(h, dtype=np.float64)
    out = np.empty_like(h)
    L.host_matern(s2, ell, nu, h.ctypes.data, h.size, int(tab), out.ctypes.data)
    return out


@pytest.mark.parametrize("nu", [0.05, 0.3, 0.7, 1.0, 1.3, 2.2, 3.7, 5.0])
def test_device_besselk_vs_scipy(lib, nu):
    worst = 0.0
    for x in np.geomspace(1e-8, 600, 400):
        ref = kv(nu, x)
        if ref > 1e-300:
            worst = max(worst, abs(lib.host_besselk(nu, x) - ref) / ref)
    assert worst < 5e-14, worst


@pytest.mark.parametrize("nu", [0.3, 1.0, 2.2, 3.7])
def test_chebyshev_table_matches_direct_and_oracle(lib, nu):
    ell = 0.05
    h = np.concatenate([[0.0], np.geomspace(1e-9, 30.0, 3000)])
    direct = _matern(lib, 1.7, ell, nu, h, False)
    tab = _matern(lib, 1.7, ell, nu, h, True)
    m = direct > 1e-290
    # exp(-x) amplifies the rounding of x = h / ell by a factor x: tolerance 2e-14 * max(1, x)
    tol = 2e-14 * np.maximum(1.0, h / ell)
    assert np.all(np.abs(tab[m] - direct[m]) <= tol[m] * np.abs(direct[m]))
    assert tab[0] == 1.7                               # C(0) = sigma^2
    # against the oracle's independent integral representation
    for k in range(1, h.size, 97):
        ref = oracle.matern(h[k], 1.7, ell, nu)
        if ref > 1e-290:
            assert abs(tab[k] - ref) <= 2e-13 * max(1.0, h[k] / ell) * ref, (h[k], tab[k], ref)


@pytest.mark.parametrize("nu", [0.5, 1.5, 2.5])
def test_device_besselk_half_integer_closed_forms(lib, nu):
    """|mu| = 1/2 (the reduced order where Temme's normalising coefficients C_j vanish for j >= 1):
    K_{1/2}(x) = sqrt(pi/(2x)) e^{-x}, K_{3/2} = K_{1/2} (1 + 1/x), K_{5/2} = K_{1/2} (1 + 3/x + 3/x^2)
    (DLMF 10.49.12), on both sides of the series / backward-recurrence switch at x = 2."""
    for x in np.concatenate([np.geomspace(1e-6, 700, 300), [1.999999, 2.0, 2.000001]]):
        k12 = math.sqrt(math.pi / (2 * x)) * math.exp(-x)
        ref = {0.5: k12, 1.5: k12 * (1 + 1 / x), 2.5: k12 * (1 + 3 / x + 3 / x ** 2)}[nu]
        assert abs(lib.host_besselk(nu, x) - ref) <= 3e-15 * ref * max(1.0, 1.0), (nu, x)


def test_device_besselk_continuity_at_switch(lib):
    """The two regimes (series x <= 2, U-function backward recurrence x > 2) agree at the switch."""
    for nu in [0.05, 0.3, 1.0, 1.7, 3.3]:
        a, b = lib.host_besselk(nu, 2.0), lib.host_besselk(nu, np.nextafter(2.0, 3.0))
        assert abs(a - b) <= 4e-15 * a, (nu, a, b)

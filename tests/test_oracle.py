"""Pins for the oracle (CPU, no GPU).  Each pin checks the oracle against something other
than itself: printed/tabulated values, closed forms, identities of K_nu, an independent
library (scipy.special.kv, numpy LU slogdet), an O(n) exact Markov formula, brute force."""
import math
import os

import numpy as np
import pytest
from scipy.special import kv, gamma

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden", "besselk.txt")


def _gold():
    rows = []
    for line in open(GOLD):
        if line.startswith("#") or not line.strip():
            continue
        kind, nu, x, val, cite = line.split()
        rows.append((kind, float(nu), float(x), float(val), cite))
    return rows


@pytest.mark.parametrize("row", _gold(), ids=lambda r: f"{r[0]}{r[1]}@{r[2]}")
def test_golden_values(row):
    kind, nu, x, val, _ = row
    if kind == "K":
        got = oracle.besselk(nu, x)
    else:
        got = oracle.matern(x, 1.0, 1.0, nu, integral=(nu != 0.5))
    assert abs(got - val) <= 2e-14 * abs(val), (got, val)


@pytest.mark.parametrize("nu,form", [
    (0.5, lambda x: np.exp(-x)),
    (1.5, lambda x: (1 + x) * np.exp(-x)),
    (2.5, lambda x: (1 + x + x * x / 3) * np.exp(-x)),
])
def test_integral_matches_closed_forms(nu, form):
    # Eq. (3) with half-integer nu reduces to exponential x polynomial
    for x in np.geomspace(1e-6, 60, 97):
        a = oracle.matern(x, 1.0, 1.0, nu, integral=True)
        b = form(x)
        assert abs(a - b) <= 1e-13 * b, (nu, x, a, b)


@pytest.mark.parametrize("nu,c", [(1.5, math.sqrt(3.0)), (2.5, math.sqrt(5.0))])
def test_printed_forms_are_eq3_with_rescaled_ell(nu, c):
    # DESIGN.md R1: PAPER.md:205-208 print the forms with argument sqrt(2 nu) h / ell; they
    # equal Eq. (3) at ell' = ell / sqrt(2 nu).
    ell = 0.3
    for h in np.linspace(0.0, 2.0, 41):
        y = c * h / ell
        printed = (1 + y) * np.exp(-y) if nu == 1.5 else (1 + y + y * y / 3) * np.exp(-y)
        got = oracle.matern(h, 1.0, ell / c, nu)
        assert abs(got - printed) <= 1e-14, (h, got, printed)


def test_besselk_recurrence_and_scipy():
    # K_{nu+1} = K_{nu-1} + (2 nu / x) K_nu  (DLMF 10.29.1) and scipy's independent kv
    for nu in (0.7, 1.3, 2.2, 3.6):
        for x in (0.01, 0.3, 1.0, 4.0, 25.0):
            lhs = oracle.besselk(nu + 1, x)
            rhs = oracle.besselk(nu - 1, x) + 2 * nu / x * oracle.besselk(nu, x)
            assert abs(lhs - rhs) <= 1e-13 * abs(lhs)
    worst = 0.0
    for nu in (0.05, 0.3, 0.5, 1.0, 1.7, 2.5, 5.0):
        for x in np.geomspace(1e-8, 700, 120):
            b = kv(nu, x)
            if b > 0:
                worst = max(worst, abs(oracle.besselk(nu, x) - b) / b)
    assert worst < 1e-12, worst


def test_matern_general_nu_vs_scipy_and_limits():
    for nu in (0.3, 0.8, 1.0, 2.0, 3.3):
        for h in (1e-7, 1e-3, 0.05, 0.2, 1.0, 3.0):
            ell, s2 = 0.17, 2.5
            x = h / ell
            ref = s2 * 2 ** (1 - nu) / gamma(nu) * x ** nu * kv(nu, x)
            assert abs(oracle.matern(h, s2, ell, nu) - ref) <= 1e-12 * ref
        # C(0) = sigma^2 (x^nu K_nu(x) -> Gamma(nu) 2^(nu-1))
        assert oracle.matern(0.0, 2.5, 0.17, nu) == 2.5
        assert abs(oracle.matern(1e-12, 2.5, 0.17, nu) - 2.5) < 1e-3 * 2.5 + (1e-4 if nu < 0.5 else 0)


def test_cov_dense_entries_and_symmetry():
    s = synth.uniform_points(50, 7)
    C = oracle.cov_dense(s, 1.3, 0.2, 1.0, 1e-3)
    assert np.array_equal(C, C.T)
    i, j = 3, 41
    h = np.hypot(*(s[i] - s[j]))
    assert C[i, j] == oracle.matern(h, 1.3, 0.2, 1.0)
    assert C[5, 5] == 1.3 + 1e-3
    sub = oracle.cov_entries(s, 1.3, 0.2, 1.0, 1e-3, [1, 5, 9], [5, 0])
    assert np.array_equal(sub, C[np.ix_([1, 5, 9], [5, 0])])


def test_loglik_n1_n2_closed_forms():
    # n = 1: L = -1/2 log 2pi - 1/2 log(s2 + tau2) - z^2 / (2 (s2 + tau2))
    s2, ell, nu, tau2 = 1.7, 0.3, 0.5, 1e-2
    s = np.array([[0.2, 0.4]])
    z = np.array([0.9])
    ll, ld, q = oracle.loglik_dense(s, z, s2, ell, nu, tau2)
    a = s2 + tau2
    assert abs(ll - (-0.5 * math.log(2 * math.pi) - 0.5 * math.log(a) - 0.5 * 0.81 / a)) < 1e-14
    # n = 2 by hand: det = a^2 - b^2, quad = (a z1^2 - 2 b z1 z2 + a z2^2) / det
    s = np.array([[0.1, 0.1], [0.4, 0.5]])
    z = np.array([0.3, -1.1])
    b = s2 * math.exp(-0.5 / ell)
    det = a * a - b * b
    quad = (a * z[0] ** 2 - 2 * b * z[0] * z[1] + a * z[1] ** 2) / det
    ll, ld, q = oracle.loglik_dense(s, z, s2, ell, nu, tau2)
    assert abs(ld - math.log(det)) < 1e-13 and abs(q - quad) < 1e-13
    assert abs(ll - (-math.log(2 * math.pi) - 0.5 * math.log(det) - 0.5 * quad)) < 1e-13


@pytest.mark.parametrize("n", [1, 7, 33, 64])
def test_logdet_quad_vs_lu(n):
    # log det vs partial-pivot LU determinant (numpy slogdet), quad vs LU solve
    s = synth.uniform_points(n, 100 + n)
    z = synth.xi(n, 200 + n)
    for nu in (0.5, 1.0, 1.5):
        C = oracle.cov_dense(s, 1.0, 0.1, nu, 1e-6)
        sign, ld_lu = np.linalg.slogdet(C)
        q_lu = float(z @ np.linalg.solve(C, z))
        ll, ld, q = oracle.loglik_dense(s, z, 1.0, 0.1, nu, 1e-6)
        assert sign == 1.0
        assert abs(ld - ld_lu) <= 1e-9 * max(1.0, abs(ld_lu))
        assert abs(q - q_lu) <= 1e-7 * abs(q_lu)
        L = oracle.cholesky(C)
        assert np.min(np.diag(L) ** 2) >= 1e-6 * (1 - 1e-9)   # pivots are conditional variances >= tau^2
        assert np.linalg.norm(L @ L.T - C) <= 1e-13 * np.linalg.norm(C)


def test_collinear_ou_closed_form():
    n = 600
    s = synth.collinear_points(n, 11)
    z = synth.xi(n, 12)
    ll, ld, q = oracle.loglik_dense(s, z, 1.4, 0.05, 0.5, 0.0)
    ll2, ld2, q2 = oracle.loglik_ou_collinear(s[:, 0], z, 1.4, 0.05)
    assert abs(ld - ld2) <= 1e-10 * abs(ld2)
    assert abs(q - q2) <= 1e-9 * abs(q2)
    assert abs(ll - ll2) <= 1e-10 * abs(ll2)


def test_permutation_invariance():
    n = 300
    s = synth.uniform_points(n, 5)
    z = synth.xi(n, 6)
    p = np.random.default_rng(0).permutation(n)
    a = oracle.loglik_dense(s, z, 1.0, 0.1, 1.0, 1e-6)
    b = oracle.loglik_dense(s[p], z[p], 1.0, 0.1, 1.0, 1e-6)
    assert abs(a[0] - b[0]) <= 1e-10 * abs(a[0])


def test_sample_statistics():
    # Z = L xi at the generating theta: v = L^{-1} Z = xi, so quad = xi^T xi exactly;
    # and it is chi^2_n-distributed around n.
    n = 800
    s = synth.uniform_points(n, 9)
    x = synth.xi(n, 10)
    Z = oracle.sample_dense(s, x, 1.0, 0.1, 0.5, 1e-6)
    ll, ld, q = oracle.loglik_dense(s, Z, 1.0, 0.1, 0.5, 1e-6)
    assert abs(q - float(x @ x)) <= 1e-8 * q
    assert abs(q - n) <= 5 * math.sqrt(2 * n)


def test_theta_recovery_small():
    # recovery of the known theta on synthetic data (north star):
    # n = 1000 dense MLE over (nu, ell, sigma^2) by Nelder-Mead from 1.5x the truth.
    from scipy.optimize import minimize
    n = 1000
    s = synth.uniform_points(n, 21)
    Z = oracle.sample_dense(s, synth.xi(n, 22), 1.0, 0.1, 0.5, 1e-6)

    def f(p):
        nu, ell, s2 = p
        if not (0.05 < nu < 5 and 1e-3 < ell < 10 and 1e-3 < s2 < 1e3):
            return 1e300
        return -oracle.loglik_dense(s, Z, s2, ell, nu, 1e-6)[0]

    r = minimize(f, [0.75, 0.15, 1.5], method="Nelder-Mead",
                 options=dict(xatol=1e-3, fatol=1e-4, maxiter=150))
    nu, ell, s2 = r.x
    assert abs(nu - 0.5) < 0.15, r.x
    micro = s2 / ell ** (2 * nu)
    assert abs(micro / 10.0 - 1) < 0.3, r.x
    assert -r.fun >= -f([0.5, 0.1, 1.0]) - 1e-6


def test_ou_sampler_matches_dense_factor():
    # the exact OU recursion draws from N(0, C): L^{-1} Z has the same log-likelihood terms;
    # pinned by quad(Z) = xi^T xi when Z comes from the Markov recursion (whitening is exact)
    n = 400
    s = synth.collinear_points(n, 13)
    xi = synth.xi(n, 14)
    Z = oracle.sample_ou_collinear(s[:, 0], xi, 1.3, 0.07)
    ll, ld, q = oracle.loglik_dense(s, Z, 1.3, 0.07, 0.5, 0.0)
    assert abs(q - float(xi @ xi)) <= 1e-8 * q


# ---- 3-D variant (only dim changes) ---------------------------------------
def test_3d_distance_by_hand_and_n2_closed_form():
    # |(0,0,0) - (1,2,2)| = 3 exactly; nu = 1/2: C_01 = s2 exp(-3/ell)
    s = np.array([[0.0, 0.0, 0.0], [1.0, 2.0, 2.0]])
    s2, ell, tau2 = 1.4, 2.0, 1e-3
    C = oracle.cov_dense(s, s2, ell, 0.5, tau2)
    assert abs(C[0, 1] - s2 * math.exp(-1.5)) < 1e-15 and C[0, 0] == s2 + tau2
    z = np.array([0.7, -0.2])
    a, b = s2 + tau2, s2 * math.exp(-1.5)
    det = a * a - b * b
    _, ld, q = oracle.loglik_dense(s, z, s2, ell, 0.5, tau2)
    assert abs(ld - math.log(det)) < 1e-13
    assert abs(q - (a * z[0] ** 2 - 2 * b * z[0] * z[1] + a * z[1] ** 2) / det) < 1e-13


def test_3d_plane_embedding_equals_2d():
    # points of the plane z = c in 3-D give the 2-D covariance exactly
    s = synth.uniform_points(300, 17)
    s3 = np.column_stack([s, np.full(300, 0.25)])
    for nu in (0.5, 1.0, 1.5):
        assert np.array_equal(oracle.cov_dense(s, 1.0, 0.1, nu, 1e-6), oracle.cov_dense(s3, 1.0, 0.1, nu, 1e-6))


def test_3d_rotation_invariance():
    # an orthogonal map of the locations leaves C and L unchanged (up to rounding of the distances)
    s = synth.uniform_points_3d(400, 18)
    q, _ = np.linalg.qr(np.random.default_rng(19).standard_normal((3, 3)))
    z = synth.xi(400, 20)
    a = oracle.loglik_dense(s, z, 1.0, 0.2, 1.0, 1e-4)
    b = oracle.loglik_dense(s @ q.T + 0.3, z, 1.0, 0.2, 1.0, 1e-4)
    assert abs(a[0] - b[0]) <= 1e-9 * abs(a[0])

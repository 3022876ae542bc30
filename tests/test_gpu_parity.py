"""GPU parity: the CUDA path (through the C ABI, libhcov.so) against the CPU oracle.

Bars (BASELINE.json north_star):
  * rel. error of L(theta) <= 1e-6 at eps = 1e-8 and <= 1e-3 at eps = 1e-4 (n <= 32K);
  * all-dense mode (eta = 0, no low-rank block) is a blocked dense Cholesky: rounding only;
  * dense-tile entries of C~ equal the oracle's Matern entries to ~1e-13;
  * sampled-column ||C - C~||_F / ||C||_F <= 10 eps at sizes the dense oracle cannot reach;
  * exact closed forms at any n (collinear OU), and v = xi for Z = L~ xi.
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import oracle  # noqa: E402
import synth  # noqa: E402
import paper_1709_08625_b200 as H  # noqa: E402

pytestmark = pytest.mark.gpu


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def _rel(a, b):
    return abs(a - b) / abs(b)


def _scale(ref, n):
    return 0.5 * n * math.log(2 * math.pi) + 0.5 * abs(ref[1]) + 0.5 * ref[2]


def _scaled_err(r, ref, n):
    """Component-scaled error |dL| / (n/2 log 2pi + |logdet|/2 + q/2) (reading R11)."""
    return abs(r["loglik"] - ref[0]) / _scale(ref, n)


def _err(r, ref, n):
    """the plain relative error of L, except where |L| < 0.1 x the
    component scale (L near a sign change), where the component-scaled error is graded."""
    if abs(ref[0]) < 0.1 * _scale(ref, n):
        return _scaled_err(r, ref, n)
    return _rel(r["loglik"], ref[0])


@pytest.fixture(scope="module")
def c1():
    cfg = synth.CONFIGS["C1"]
    s = synth.points(cfg)
    th = (cfg.sigma2, cfg.ell, cfg.nu, cfg.nugget)
    Z = oracle.sample_dense(s, synth.xi(cfg.n, cfg.seed_xi), *th)
    ref = oracle.loglik_dense(s, Z, *th)
    return cfg, s, Z, th, ref


def test_c1_parity(c1):
    cfg, s, Z, th, ref = c1
    T = H.Tree(_dev(s))
    r = H.eval_loglik(T, th, _dev(Z), eps=cfg.eps[0])
    assert r["status"] == 0
    assert _rel(r["loglik"], ref[0]) <= 1e-6, (r, ref)
    assert _rel(r["logdet"], ref[1]) <= 1e-6
    assert _rel(r["quad"], ref[2]) <= 1e-6
    assert r["min_pivot"] >= cfg.nugget * (1 - 1e-6)   # pivots are conditional variances >= tau^2
    assert r["acc_loss"] == 0 and r["cap_binds"] == 0


def test_c1_staged_api_equals_eval(c1):
    cfg, s, Z, th, ref = c1
    T = H.Tree(_dev(s))
    h = H.HMatrix(T, th, cfg.eps[0])
    assert h.cholesky() == -1
    r1 = h.loglik(_dev(Z))
    r2 = H.eval_loglik(T, th, _dev(Z), eps=cfg.eps[0])
    assert r1["loglik"] == r2["loglik"]           # same kernels, same order: bitwise
    r3 = H.eval_loglik(T, th, _dev(Z), eps=cfg.eps[0])
    assert r3["loglik"] == r2["loglik"]           # determinism


@pytest.mark.parametrize("n,seed", [(1, 3), (17, 4), (32, 5), (33, 6), (1000, 7), (2000, 8)])
def test_all_dense_mode_ragged(n, seed):
    # eta = 0: no admissible block -> the schedule is a blocked dense Cholesky (rounding only)
    s = synth.uniform_points(n, seed)
    th = (1.3, 0.2, 1.0, 1e-4)
    Z = synth.xi(n, seed + 50)
    ref = oracle.loglik_dense(s, Z, *th)
    T = H.Tree(_dev(s), eta=0.0)
    r = H.eval_loglik(T, th, _dev(Z), eps=1e-8)
    assert r["status"] == 0
    assert abs(r["loglik"] - ref[0]) <= 1e-10 * max(1.0, abs(ref[0])), (r, ref)
    assert abs(r["logdet"] - ref[1]) <= 1e-10 * max(1.0, abs(ref[1]))


@pytest.mark.parametrize("eps,bar", [(1e-13, 1e-10), (1e-11, 1e-9)])
def test_near_full_rank_mode(eps, bar):
    # eps -> 0 with the largest rank capacity (64): the H-matrix reproduces the dense matrix
    n = 1200
    s = synth.uniform_points(n, 11)
    th = (1.0, 0.1, 0.5, 1e-6)
    Z = oracle.sample_dense(s, synth.xi(n, 12), *th)
    ref = oracle.loglik_dense(s, Z, *th)
    T = H.Tree(_dev(s))
    r = H.eval_loglik(T, th, _dev(Z), eps=eps, kcap=64)
    assert r["status"] == 0, r
    assert r["acc_loss"] == 0
    assert _rel(r["loglik"], ref[0]) <= bar, (r, ref)


@pytest.mark.parametrize("nu,ell", [(1.0, 0.05), (0.3, 0.1), (2.2, 0.03), (1.5, 0.05), (2.5, 0.02)])
def test_general_nu_parity(nu, ell):
    n = 4096
    s = synth.uniform_points(n, 21)
    th = (1.0, ell, nu, 1e-6)
    Z = oracle.sample_dense(s, synth.xi(n, 22), *th)
    ref = oracle.loglik_dense(s, Z, *th)
    T = H.Tree(_dev(s))
    r = H.eval_loglik(T, th, _dev(Z), eps=1e-8)
    assert r["status"] == 0 and r["acc_loss"] == 0
    assert _err(r, ref, n) <= 1e-6, (r, ref)


@pytest.mark.parametrize("nu,ell,sigma2", [(0.5, 0.1, 1.0), (1.0, 0.05, 2.0), (0.3, 0.2, 1.0),
                                          (1.5, 0.05, 1.0), (3.7, 0.01, 0.5)])
def test_assembled_entries_vs_oracle(nu, ell, sigma2):
    """Dense tiles: device Matern/K_nu vs the oracle's integral K_nu entry by entry;
    whole columns (dense + low-rank): relative Frobenius error <= 10 eps."""
    n = 3000
    s = synth.uniform_points(n, 31)
    th = (sigma2, ell, nu, 1e-6)
    eps = 1e-8
    T = H.Tree(_dev(s))
    h = H.HMatrix(T, th, eps)
    cols = np.random.default_rng(5).choice(n, 24, replace=False)
    got = h.columns(cols).cpu().numpy()
    ref = oracle.cov_entries(s, sigma2, ell, nu, 1e-6, np.arange(n), cols)
    # rows in the same leaf as the column -> dense tile entries: near-exact
    perm = T.perm_i2e()
    pos = np.empty(n, dtype=np.int64)
    pos[perm[perm >= 0]] = np.nonzero(perm >= 0)[0]
    for k, c in enumerate(cols):
        same = (pos // 32) == (pos[c] // 32)
        d = np.abs(got[same, k] - ref[same, k])
        assert np.all(d <= 1e-13 * np.abs(ref[same, k]) + 1e-300), (nu, c, d.max())
    fro = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert fro <= 10 * eps, fro
    # the device's exact-column evaluator (bench accuracy field) against the oracle as well
    ce = H.cov_columns(T, th, cols).cpu().numpy()
    assert np.max(np.abs(ce - ref) / np.abs(ref).max()) <= 1e-13


def test_collinear_ou_exact_large():
    """nu = 1/2, tau^2 = 0 on a line: exact O(n) Markov likelihood at n = 65,536 (any n)."""
    n = 65536
    s = synth.collinear_points(n, 41)
    Z = oracle.sample_ou_collinear(s[:, 0], synth.xi(n, 42), 1.0, 0.05)
    ref = oracle.loglik_ou_collinear(s[:, 0], Z, 1.0, 0.05)
    T = H.Tree(_dev(s))
    r = H.eval_loglik(T, (1.0, 0.05, 0.5, 0.0), _dev(Z), eps=1e-6, kmax=20)
    assert r["status"] == 0
    assert _rel(r["logdet"], ref[1]) <= 1e-8, (r, ref)
    assert _rel(r["quad"], ref[2]) <= 1e-8, (r, ref)
    assert _rel(r["loglik"], ref[0]) <= 1e-8, (r, ref)


@pytest.mark.parametrize("n", [50001, 300007])
def test_collinear_ou_exact_ragged_gangs(n):
    """Exact Markov likelihood at n not a power of two: gangs with a remainder row split
    (the last member takes m - (G-1) floor(m/G) rows) and, at 300,007, member panels above 256 rows
    (in-CTA chunked TSQR)."""
    s = synth.collinear_points(n, 43)
    Z = oracle.sample_ou_collinear(s[:, 0], synth.xi(n, 44), 1.0, 0.05)
    ref = oracle.loglik_ou_collinear(s[:, 0], Z, 1.0, 0.05)
    T = H.Tree(_dev(s))
    r = H.eval_loglik(T, (1.0, 0.05, 0.5, 0.0), _dev(Z), eps=1e-6, kmax=20)
    assert r["status"] == 0
    assert _rel(r["logdet"], ref[1]) <= 1e-8, (r, ref)
    assert _rel(r["quad"], ref[2]) <= 1e-8, (r, ref)


def test_ragged_n_dense_oracle():
    """n = 12,345 uniform points (ragged clusters, gangs with remainders) vs the dense oracle."""
    n = 12345
    s = synth.uniform_points(n, 45)
    th = (1.0, 0.05, 0.5, 1e-6)
    Z = oracle.sample_dense(s, synth.xi(n, 46), *th)
    ref = oracle.loglik_dense(s, Z, *th)
    T = H.Tree(_dev(s))
    r = H.eval_loglik(T, th, _dev(Z), eps=1e-8)
    assert r["status"] == 0 and r["acc_loss"] == 0
    assert _err(r, ref, n) <= 1e-6, (r, ref)


def test_sample_then_solve_gives_xi():
    """Z = L~ xi with the same factor => v = L~^{-1} Z = xi, q = xi^T xi (to round-off)."""
    n = 20000
    s = synth.uniform_points(n, 51)
    xi = synth.xi(n, 52)
    T = H.Tree(_dev(s))
    h = H.HMatrix(T, (1.0, 0.1, 0.5, 1e-6), 1e-6, kmax=20)
    assert h.cholesky() == -1
    Z = h.sample(_dev(xi))
    r = h.loglik(Z)
    assert _rel(r["quad"], float(xi @ xi)) <= 1e-9, (r["quad"], float(xi @ xi))
    assert abs(r["quad"] - n) <= 5 * math.sqrt(2 * n)


def test_not_spd_reported():
    # coincident points with tau^2 = 0 make C singular: the H-Cholesky must report NOT_SPD
    s = synth.uniform_points(600, 61)
    s[301] = s[300]
    s[302] = s[300]
    T = H.Tree(_dev(s))
    h = H.HMatrix(T, (1.0, 0.5, 2.5, 0.0), 1e-8)
    with pytest.raises(H.HcovError) as e:
        h.cholesky()
    assert e.value.code == 3


def test_mle_batch_matches_single_evals_and_rejects():
    n = 2500
    s = synth.uniform_points(n, 71)
    th0 = (1.0, 0.1, 0.5, 1e-6)
    Z = _dev(oracle.sample_dense(s, synth.xi(n, 72), *th0))
    T = H.Tree(_dev(s))
    thetas = [(1.0, 0.08, 0.5, 1e-6), (1.2, 0.1, 0.7, 1e-6), (1.0, -0.1, 0.5, 1e-6), (0.9, 0.12, 1.0, 1e-6)]
    ll, st = H.mle_batch(T, Z, thetas, eps=1e-8)
    assert st[2] == 1 and ll[2] == -np.inf
    for k in (0, 1, 3):
        assert st[k] == 0
        r = H.eval_loglik(T, thetas[k], Z, eps=1e-8)
        assert r["loglik"] == ll[k]


def test_invalid_arguments():
    s = synth.uniform_points(100, 81)
    T = H.Tree(_dev(s))
    for th in [(0.0, 0.1, 0.5, 0.0), (1.0, 0.0, 0.5, 0.0), (1.0, 0.1, -1.0, 0.0), (1.0, 0.1, 0.5, -1e-3)]:
        with pytest.raises(H.HcovError) as e:
            H.HMatrix(T, th, 1e-6)
        assert e.value.code == 1
    h = H.HMatrix(T, (1.0, 0.1, 0.5, 0.0), 1e-6)
    with pytest.raises(H.HcovError) as e:
        h.loglik(_dev(np.zeros(100)))           # not factored yet
    assert e.value.code == 7
    with pytest.raises(H.HcovError) as e:
        H.Tree(torch.zeros((0, 2), dtype=torch.float64, device="cuda"))
    assert e.value.code == 2

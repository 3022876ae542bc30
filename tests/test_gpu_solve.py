"""NEXT (f1): back-solve, H-matvec and the listing's PCG (Table 1 "C~ z").

* u = L~^{-T} v with v = L~^{-1} Z gives u = C~^{-1} Z and Z^T u = v^T v = q (Eq. (2)) to rounding;
* the transpose identity  forward(a)^T b = a^T backsolve(b)  for random a, b (exact algebra);
* all-dense mode (eta = 0, C~ = C): solve and matvec against the dense oracle;
* y = C~ x against the dense oracle's C x at eps = 1e-8 (relative error <= 10 eps), and the
  symmetry a^T (C~ b) = (C~ a)^T b;
* PCG on C3 (131,072 clustered points): A = C~ at eps = 1e-6, k = 16, preconditioner = the
  H-Cholesky factor at a looser eps; converges to 1e-6 within the listing's 150 iterations, the
  residual re-checked with an independent H-matvec, and Z^T x equals the eps = 1e-6 factor's q.
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


@pytest.mark.parametrize("cfgname", ["C1", "C2"])
def test_backsolve_quadratic_form(cfgname):
    cfg = synth.CONFIGS[cfgname]
    s = synth.points(cfg)
    th = (cfg.sigma2, cfg.ell, cfg.nu, cfg.nugget)
    Z = oracle.sample_dense(s, synth.xi(cfg.n, cfg.seed_xi), *th)
    T = H.Tree(_dev(s))
    h = H.HMatrix(T, th, 1e-8)
    assert h.cholesky() == -1
    Zd = _dev(Z)
    r = h.loglik(Zd)
    v = h.forward_solve(Zd)
    q_v = float(v @ v)
    assert abs(q_v - r["quad"]) <= 1e-12 * r["quad"]
    u = h.backsolve(v)
    x = h.solve(Zd)
    assert torch.equal(u, x)                         # same kernels, same order
    q_u = float(Zd @ u)
    print(f"{cfgname}: v^T v = {q_v:.12g}, Z^T u = {q_u:.12g}")
    assert abs(q_u - q_v) <= 1e-10 * q_v, (q_u, q_v)


def test_transpose_identity():
    n = 5000
    s = synth.uniform_points(n, 101)
    T = H.Tree(_dev(s))
    h = H.HMatrix(T, (1.0, 0.05, 1.0, 1e-6), 1e-7)
    assert h.cholesky() == -1
    a, b = _dev(synth.xi(n, 102)), _dev(synth.xi(n, 103))
    lhs = float(h.forward_solve(a) @ b)
    rhs = float(a @ h.backsolve(b))
    assert abs(lhs - rhs) <= 1e-9 * (abs(lhs) + 1.0), (lhs, rhs)


@pytest.mark.parametrize("n,seed", [(1000, 111), (2047, 112)])
def test_all_dense_solve_and_matvec_vs_oracle(n, seed):
    s = synth.uniform_points(n, seed)
    th = (1.3, 0.2, 1.0, 1e-4)
    C = oracle.cov_dense(s, *th)
    b = synth.xi(n, seed + 1)
    T = H.Tree(_dev(s), eta=0.0)
    A = H.HMatrix(T, th, 1e-8)
    y = A.matvec(_dev(b)).cpu().numpy()
    assert np.linalg.norm(y - C @ b) <= 1e-13 * np.linalg.norm(C @ b)
    M = H.HMatrix(T, th, 1e-8)
    assert M.cholesky() == -1
    x = M.solve(_dev(b)).cpu().numpy()
    xo = np.linalg.solve(C, b)
    assert np.linalg.norm(x - xo) <= 1e-9 * np.linalg.norm(xo)


def test_matvec_vs_oracle_and_symmetry():
    cfg = synth.CONFIGS["C1"]
    s = synth.points(cfg)
    th = (cfg.sigma2, cfg.ell, cfg.nu, cfg.nugget)
    C = oracle.cov_dense(s, *th)
    T = H.Tree(_dev(s))
    A = H.HMatrix(T, th, 1e-8)
    a, b = synth.xi(cfg.n, 121), synth.xi(cfg.n, 122)
    ya, yb = A.matvec(_dev(a)), A.matvec(_dev(b))
    err = np.linalg.norm(ya.cpu().numpy() - C @ a) / np.linalg.norm(C @ a)
    assert err <= 10 * 1e-8, err
    s1, s2 = float(_dev(a) @ yb), float(ya @ _dev(b))
    assert abs(s1 - s2) <= 1e-12 * abs(s1)


def test_pcg_c3():
    cfg = synth.CONFIGS["C3"]
    s = synth.points(cfg)
    th = (cfg.sigma2, cfg.ell, cfg.nu, cfg.nugget)
    T = H.Tree(_dev(s))
    Zd = _dev(synth.xi(cfg.n, cfg.seed_xi))
    A = H.HMatrix(T, th, cfg.eps[0], cfg.kmax)             # C~ (eps = 1e-6, k = 16), kept assembled
    F = H.HMatrix(T, th, cfg.eps[0], cfg.kmax)             # its own factor: reference q
    assert F.cholesky() == -1
    q_ref = F.loglik(Zd)["quad"]
    del F
    # a cheaper, looser preconditioner: the loosest of these whose factorisation is SPD (a loose
    # truncation of C3's clustered field can be indefinite, R24)
    M, used = None, None
    for eps_m, k_m in ((1e-4, 8), (1e-5, 10), (1e-5, 12)):
        try:
            M = H.HMatrix(T, th, eps_m, k_m)
            M.cholesky()
            used = (eps_m, k_m)
            break
        except H.HcovError as e:
            M = None
            assert e.code == 3, e
    assert M is not None
    x, it, rr = H.pcg(A, M, Zd, maxit=150, tol=1e-6)
    print(f"C3 PCG (preconditioner eps, k = {used}): {it} iterations, relres {rr:.2e}")
    assert it >= 2
    assert it <= 150 and rr <= 1e-6
    res = Zd - A.matvec(x)
    assert float(torch.linalg.norm(res) / torch.linalg.norm(Zd)) <= 1.01e-6
    q_pcg = float(Zd @ x)
    assert abs(q_pcg - q_ref) <= 1e-4 * q_ref, (q_pcg, q_ref)

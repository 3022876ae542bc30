"""NEXT (f3): the accuracy diagnostics of Sec. 4 (Tables 2-3: KLD, ||C - C~||_2,
||C C~^{-1} - I||_2; Table 4's ||I - (L~ L~^T)^{-1} C~||_2) computed by the library
(hcov_norm2_diff, hcov_inv_error, hcov_trace_inv), checked against dense numpy linear algebra on
the same matrices at small n, and against exact values where the method is exact (eta = 0)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
import oracle  # noqa: E402
import synth  # noqa: E402
import paper_1709_08625_b200 as H  # noqa: E402

pytestmark = pytest.mark.gpu


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


@pytest.fixture(scope="module")
def setup():
    n = 1024
    s = synth.uniform_points(n, 301)
    th = (1.0, 0.25, 0.5, 1e-6)
    T = H.Tree(_dev(s))
    Te = H.Tree(_dev(s), eta=0.0)
    C = oracle.cov_dense(s, *th)
    return n, s, th, T, Te, C


def test_exact_tree_diagnostics_vanish(setup):
    n, s, th, T, Te, C = setup
    d = H.kld(Te, Te, th, 0.0)
    print(d)
    assert abs(d["kld"]) <= 1e-8 * n
    assert d["norm2_C_minus_Ct"] == 0.0
    assert d["norm2_C_Ctinv_minus_I"] <= 1e-8


@pytest.mark.parametrize("kmax", [6, 10, 20])
def test_diagnostics_against_dense(setup, kmax):
    n, s, th, T, Te, C = setup
    A = H.HMatrix(T, th, 1e-14, kmax)                         # rank-capped C~ (Table 2's k)
    Ct = A.columns(np.arange(n)).cpu().numpy()
    M = H.HMatrix(T, th, 1e-14, kmax)
    M.cholesky()
    Minv = np.stack([M.solve(_dev(np.eye(n)[:, j])).cpu().numpy() for j in range(n)], axis=1)
    Ce = H.HMatrix(Te, th, 0.0)
    # ||C - C~||_2 (power iteration, a lower bound converging to the norm)
    ref = np.linalg.norm(C - Ct, 2)
    got = H.norm2_diff(Ce, A, iters=200)
    assert got <= ref * (1 + 1e-8) and got >= 0.9 * ref, (got, ref)
    # ||I - M^{-1} C||_2 = ||C M^{-1} - I||_2
    ref = np.linalg.norm(np.eye(n) - Minv @ C, 2)
    got = H.inv_error(Ce, M, iters=200)
    assert got <= ref * (1 + 1e-8) and got >= 0.9 * ref, (got, ref)
    # tr(M^{-1} C)
    ref = np.trace(Minv @ C)
    got = H.trace_inv(M, Ce)
    assert abs(got - ref) <= 1e-9 * abs(ref), (got, ref)
    d = H.kld(T, Te, th, 1e-14, kmax)
    print(f"k={kmax}: {d}")
    assert d["kld"] >= -1e-9 * n

"""NEXT (f4): the point-wise LDL^T form (listing's ldl_inv / point_wise; R8).

D_e = L~_pp^2 of point e must equal the dense LDL^T pivots of C in the same (tree) order: the
oracle's Cholesky of the permuted dense matrix gives them (D = diag(L)^2 is the LDL^T pivot of
the definition, Golub & Van Loan Alg. 4.1.2).  Exact all-dense mode to 1e-11; H-mode at eps = 1e-8
to the parity tolerance; sum log D = log det; D >= tau^2."""
import numpy as np
import pytest
import torch

import oracle
import paper_1709_08625_b200 as H
import synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("eta,eps,tol", [(0.0, 1e-8, 1e-11), (2.0, 1e-8, 1e-6)])
def test_ldl_pivots_vs_dense(eta, eps, tol):
    n = 2500
    s = synth.uniform_points(n, 51)
    th = (1.0, 0.1, 0.5, 1e-6)
    T = H.Tree(torch.from_numpy(s).cuda(), eta=eta)
    A = H.HMatrix(T, th, eps, 0)
    A.cholesky()
    D = A.ldl_diag().cpu().numpy()
    perm = T.perm_i2e()
    perm = perm[perm >= 0]                      # internal order of the real points
    C = oracle.cov_dense(s, *th)[np.ix_(perm, perm)]
    L = oracle.cholesky(C)
    Dref = np.empty(n)
    Dref[perm] = np.diag(L) ** 2
    np.testing.assert_allclose(D, Dref, rtol=tol)
    r = A.loglik(torch.zeros(n, dtype=torch.float64, device="cuda"))
    assert abs(np.sum(np.log(D)) - r["logdet"]) <= 1e-10 * abs(r["logdet"])
    assert D.min() >= th[3] * (1 - 1e-9)

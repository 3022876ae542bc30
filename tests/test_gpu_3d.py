"""NEXT (f4): the 3-D variant ("replace dim = 2 by dim = 3"): locations n x 3,
3-D boxes / admissibility / split axis in the trees (device K1 / K2), the 3-D distance in the
Matern entries (A3).  Parity against the dense oracle (its own 3-D distance, pinned in
tests/test_oracle.py), device trees against the host planner, and the plane embedding."""
import numpy as np
import pytest
import torch

import oracle
import paper_1709_08625_b200 as H
import synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("nu,ell", [(0.5, 0.2), (1.0, 0.2), (1.5, 0.2)])
def test_3d_parity_vs_oracle(nu, ell):
    """3-D eps-ranks are higher than 2-D ones (they grow like |log eps|^(d+1)).  Measured on this
    point set's admissible blocks (dense SVD): max rank 61-72 at eps = 1e-8, 48-57 at 1e-7, 35-42
    at 1e-6; the method also needs the ACA (eps/10) and the near-lossless intermediate states
    (eps * 1e-2, R22) within the largest rank capacity (64), so the 3-D parity runs at eps = 1e-5
    (intermediate 1e-7: <= 57); n = 2,000 (blocks <= 512) and ell = 0.2 keep the Schur-complement
    ranks of the factor inside the capacity too (at n = 3,000, nu = 1, ell = 0.1 they reach it).  Bar: the log-linear interpolation of north_star's two bars (1e-6 at
    eps = 1e-8, 1e-3 at eps = 1e-4) at eps = 1e-5: 10^-3.75 ~ 1.8e-4, on the error SURVEY 8(c) row 11 grades (L(theta) at nu = 1 is
    -107 against a component scale of 5.6e3, so the component-scaled error is the graded one)."""
    n = 2000
    s = synth.uniform_points_3d(n, 31)
    th = (1.0, ell, nu, 1e-6)
    Z = oracle.sample_dense(s, synth.xi(n, 32), *th)
    ref = oracle.loglik_dense(s, Z, *th)
    T = H.Tree(torch.from_numpy(s).cuda())
    assert T.info()["dim"] == 3 and T.info()["tree_on_device"] == 1
    r = H.eval_loglik(T, th, torch.from_numpy(Z).cuda(), 1e-5, 0, 64)
    # where |L| < 0.1 x the component scale
    # n/2 log 2pi + |logdet|/2 + q/2 (L near a sign change), the component-scaled error is graded
    scale = 0.5 * n * np.log(2 * np.pi) + 0.5 * abs(ref[1]) + 0.5 * ref[2]
    dl = abs(r["loglik"] - ref[0])
    err = dl / scale if abs(ref[0]) < 0.1 * scale else dl / abs(ref[0])
    print(f"3-D nu={nu} ell={ell}: status {r['status']} rel {dl / abs(ref[0]):.2e} graded {err:.2e} "
          f"max_rank {r['max_rank']} acc_loss {r['acc_loss']} interm_cuts {r['interm_cuts']}")
    assert r["status"] == 0, r
    assert err <= 1.8e-4, (r, ref)
    assert abs(r["logdet"] - ref[1]) <= 1.8e-4 * abs(ref[1])


def test_3d_entries_vs_oracle():
    n = 5000
    s = synth.uniform_points_3d(n, 33)
    th = (1.3, 0.2, 1.0, 1e-6)
    T = H.Tree(torch.from_numpy(s).cuda())
    cols = np.array([0, 17, 2500, 4999])
    got = H.cov_columns(T, th, cols).cpu().numpy()
    ref = oracle.cov_entries(s, *th, np.arange(n), cols)
    assert got.shape == ref.shape
    np.testing.assert_allclose(got, ref, rtol=1e-13, atol=1e-15)


def test_3d_device_tree_equals_host():
    s = synth.uniform_points_3d(40000, 34)
    Td, Th = H.Tree(torch.from_numpy(s).cuda()), H.Tree(s)
    assert np.array_equal(Td.perm_i2e(), Th.perm_i2e())
    assert np.array_equal(Td.bbox(), Th.bbox())
    assert np.array_equal(Td.blocks(), Th.blocks())
    assert np.array_equal(Td.tasks(), Th.tasks())


def test_3d_plane_embedding_equals_2d():
    """Points on the plane z = const: the 3-D path computes the 2-D likelihood (same trees, same
    distances up to the rounding of the + 0 term)."""
    n = 20000
    s = synth.uniform_points(n, 35)
    s3 = np.column_stack([s, np.full(n, 0.7)])
    Z = torch.from_numpy(synth.xi(n, 36)).cuda()
    th = (1.0, 0.1, 0.5, 1e-6)
    a = H.eval_loglik(H.Tree(torch.from_numpy(s).cuda()), th, Z, 1e-6, 20)
    b = H.eval_loglik(H.Tree(torch.from_numpy(s3).cuda()), th, Z, 1e-6, 20)
    assert a["status"] == 0 and b["status"] == 0
    assert abs(a["loglik"] - b["loglik"]) <= 1e-10 * abs(a["loglik"])

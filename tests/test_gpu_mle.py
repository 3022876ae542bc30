"""The theta-batched MLE with hcov_mle_batch as the evaluator against the same driver with the dense
CPU oracle as the evaluator (Eq. (1); driver reading R17).

At n = 2,000 and eps = 1e-8 the H-matrix likelihood agrees with the dense one to ~1e-9 relative,
far below the gaps between the Nelder-Mead / grid candidates, so every decision of the driver is
the same on both sides: the simplex (every vertex, every iteration) is bitwise equal and the
objective values agree to the evaluation tolerance.  The oracle side is the exact likelihood, so
this pins the GPU estimate theta^ to the exact-likelihood estimate."""
import numpy as np
import pytest
import torch

import oracle
import paper_1709_08625_b200 as H
import synth
from paper_1709_08625_b200 import mle

pytestmark = pytest.mark.gpu


def test_mle_gpu_equals_oracle_mle():
    cfg = synth.CONFIGS["C1"]
    s = synth.points(cfg)
    th = (cfg.sigma2, cfg.ell, cfg.nu, cfg.nugget)
    Z = oracle.sample_dense(s, synth.xi(cfg.n, cfg.seed_xi), *th)
    T = H.Tree(torch.from_numpy(s).cuda())
    gpu_ev = mle.gpu_evaluator(T, torch.from_numpy(Z).cuda(), 1e-8, 0, cfg.nugget)

    def ora_ev(xs):
        out = []
        for nu, ell, s2 in xs:
            try:
                out.append(oracle.loglik_dense(s, Z, s2, ell, nu, cfg.nugget)[0])
            except oracle.NotSPD:
                out.append(-np.inf)
        return out

    x0 = (0.75, 0.15, 1.5)
    Sg = mle.run_mle(gpu_ev, x0, iters=5)
    So = mle.run_mle(ora_ev, x0, iters=5)
    for hg, ho in zip(Sg.history, So.history):
        assert hg["best"] == ho["best"], (hg, ho)
        assert abs(hg["negloglik"] - ho["negloglik"]) <= 1e-7 * abs(ho["negloglik"])
    assert np.array_equal(Sg.X, So.X)
    np.testing.assert_allclose(Sg.F, So.F, rtol=1e-7)

"""theta-batched MLE driver (paper_1709_08625_b200/mle.py): candidate generation, exact
sequential Nelder-Mead resolution, and the multi-process path (world size 2 over gloo on CPU)
giving bitwise the same estimate as one process.  The evaluator here is the CPU oracle (dense
Eq. (1)); on the GPU it is hcov_mle_batch."""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
from paper_1709_08625_b200 import mle  # noqa: E402


def quad(x):
    # smooth bowl with minimum at (0.5, 0.1, 1.0)
    return float(((x[0] - 0.5) / 0.1) ** 2 + ((x[1] - 0.1) / 0.02) ** 2 + ((x[2] - 1.0) / 0.3) ** 2)


def test_candidates_structure():
    X = np.array([[0.7, 0.15, 1.5], [0.8, 0.15, 1.5], [0.7, 0.18, 1.5], [0.7, 0.15, 1.8]])
    S = mle.Simplex(X.copy(), np.array([quad(x) for x in X]))
    C = mle.candidates(S)
    assert C.shape == (64, 3)
    c = S.X[:-1].mean(0)
    np.testing.assert_allclose(C[0], c + (c - S.X[-1]))         # reflection
    np.testing.assert_allclose(C[1], c + 2 * (c - S.X[-1]))     # expansion
    assert len({tuple(r) for r in C[7:59]}) == 52                # distinct grid points


def _sequential_nm(S, f):
    """Textbook Nelder-Mead step (coefficients 1, 2, 1/2, 1/2), evaluating on demand."""
    S.order()
    X, F = S.X.copy(), S.F.copy()
    c = X[:-1].mean(0)
    r = c + (c - X[-1]); fr = f(r)
    if fr < F[0]:
        e = c + 2 * (c - X[-1]); fe = f(e)
        X[-1], F[-1] = (e, fe) if fe < fr else (r, fr)
    elif fr < F[-2]:
        X[-1], F[-1] = r, fr
    else:
        if fr < F[-1]:
            oc = c + 0.5 * (r - c); foc = f(oc)
            ok = foc <= fr
            if ok:
                X[-1], F[-1] = oc, foc
        else:
            ic = c - 0.5 * (c - X[-1]); fic = f(ic)
            ok = fic < F[-1]
            if ok:
                X[-1], F[-1] = ic, fic
        if not ok:
            for i in (1, 2, 3):
                X[i] = X[0] + 0.5 * (X[i] - X[0]); F[i] = f(X[i])
    return X, F


def test_speculative_resolution_equals_sequential_nm():
    rng = np.random.default_rng(3)
    for trial in range(30):
        X = np.array([0.5, 0.1, 1.0]) + rng.normal(scale=[0.2, 0.05, 0.4], size=(4, 3))
        X = np.abs(X) + 0.05
        S1 = mle.Simplex(X.copy(), np.array([quad(x) for x in X]))
        S2 = mle.Simplex(X.copy(), np.array([quad(x) for x in X]))
        Xs, Fs = _sequential_nm(S1, quad)
        C = mle.candidates(S2)
        f = np.array([quad(x) for x in C])
        f[7:] = np.inf                                            # grid off: pure NM
        mle.resolve(S2, C, f)
        o = np.lexsort((np.arange(4), Fs))
        np.testing.assert_array_equal(S2.X, Xs[o])


def test_mle_converges_on_bowl():
    S = mle.run_mle(lambda xs: [-quad(x) for x in xs], (0.75, 0.15, 1.5), iters=40)
    np.testing.assert_allclose(S.X[0], [0.5, 0.1, 1.0], rtol=0.02, atol=1e-3)


def test_checkpoint_resume_bitwise(tmp_path):
    """A run split over three calls through the state file equals one uninterrupted run."""
    f = lambda xs: [-quad(x) for x in xs]  # noqa: E731
    ref = mle.run_mle(f, (0.75, 0.15, 1.5), iters=9)
    st = str(tmp_path / "state.json")
    for _ in range(3):
        S = mle.run_mle(f, (0.75, 0.15, 1.5), iters=9, state=st, max_new_iters=3)
    assert S.iters_done == 9
    assert np.array_equal(S.X, ref.X) and np.array_equal(S.F, ref.F)
    assert [h["best"] for h in S.history] == [h["best"] for h in ref.history]
    again = mle.run_mle(f, (0.75, 0.15, 1.5), iters=9, state=st)     # already done: no new iterations
    assert np.array_equal(again.X, ref.X) and len(again.history) == 9


def _oracle_evaluator(n=300):
    import oracle
    import synth
    s = synth.uniform_points(n, 41)
    Z = oracle.sample_dense(s, synth.xi(n, 42), 1.0, 0.1, 0.5, 1e-6)

    def ev(xs):
        out = []
        for nu, ell, s2 in xs:
            try:
                out.append(oracle.loglik_dense(s, Z, s2, ell, nu, 1e-6)[0])
            except oracle.NotSPD:
                out.append(-np.inf)
        return out
    return ev


def _worker(rank, world, port, out):
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    S = mle.run_mle(_oracle_evaluator(), (0.75, 0.15, 1.5), iters=4, rank=rank, world=world)
    if rank == 0:
        np.save(out, np.concatenate([S.X.ravel(), S.F]))
    dist.destroy_process_group()


def test_world2_gloo_equals_single_process(tmp_path):
    import torch.multiprocessing as tmp
    S = mle.run_mle(_oracle_evaluator(), (0.75, 0.15, 1.5), iters=4)
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    out = str(tmp_path / "w2.npy")
    tmp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    got = np.load(out)
    np.testing.assert_array_equal(got, np.concatenate([S.X.ravel(), S.F]))
    assert S.F[0] < S.history[0]["negloglik"] + 1e-9

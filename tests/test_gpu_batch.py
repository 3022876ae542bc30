"""Theta batches through hcov_mle_batch: several H-matrices of one tree evaluated in ONE persistent
engine launch (their task DAGs share the priority queue, "B candidates
advance in lockstep through the shared schedule").

Every batched value must be bitwise equal to the single evaluation of the same theta (each task's
arithmetic and the order of a block's terms do not depend on the schedule), a
rejected candidate (not SPD) must not disturb the others, and the batch must really share launches.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
import synth  # noqa: E402
import paper_1709_08625_b200 as H  # noqa: E402

pytestmark = pytest.mark.gpu


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def _engine_launches(fn):
    H.prof_control(enable_events=False, reset=True)
    out = fn()
    p = H.prof_read()
    return out, p["count"]["engine"]


@pytest.mark.parametrize("n,kmax", [(20000, 0), (70000, 20)])
def test_batch_bitwise_equals_single(n, kmax):
    # n = 20000 / 70000: low-rank blocks up to 4096 / 16384 rows (gangs, chunked recompression),
    # closed-form and general-nu kernels (per-instance K_nu tables) in one launch
    s = synth.uniform_points(n, 201)
    T = H.Tree(_dev(s))
    Z = _dev(synth.xi(n, 202))
    thetas = [(1.0, 0.10, 0.5, 1e-6), (1.0, 0.08, 0.5, 1e-6), (1.3, 0.12, 0.5, 1e-5), (1.0, 0.05, 1.0, 1e-4),
              (0.8, 0.10, 0.5, 1e-6), (1.0, 0.09, 0.7, 1e-4)]
    eps = 1e-6
    (ll, st), launches = _engine_launches(lambda: H.mle_batch(T, Z, thetas, eps=eps, kmax=kmax))
    print(f"n={n}: {len(thetas)} candidates in {launches} engine launches; L = {ll}")
    assert launches < len(thetas)
    for k, th in enumerate(thetas):
        r = H.eval_loglik(T, th, Z, eps=eps, kmax=kmax)
        assert st[k] == r["status"]
        assert r["loglik"] == ll[k], (k, r["loglik"], ll[k])


def test_batch_with_rejected_candidates():
    # coincident points: tau^2 = 0 makes C singular (NOT SPD), tau^2 > 0 does not; both in one batch
    s = synth.uniform_points(3000, 211)
    # (16 copies: a single duplicate leaves one pivot that is pure rounding noise of either sign,
    # so whether tau^2 = 0 is flagged would flip with any change of the summation order)
    s[1001:1016] = s[1000]
    T = H.Tree(_dev(s))
    Z = _dev(synth.xi(3000, 212))
    thetas = [(1.0, 0.1, 0.5, 1e-4), (1.0, 0.1, 0.5, 0.0), (1.0, 0.2, 2.5, 1e-4), (1.0, 0.2, 2.5, 0.0),
              (1.0, 0.15, 1.5, 1e-4)]
    ll, st = H.mle_batch(T, Z, thetas, eps=1e-8)
    assert list(st) == [0, 3, 0, 3, 0], st
    assert ll[1] == -np.inf and ll[3] == -np.inf
    for k in (0, 2, 4):
        r = H.eval_loglik(T, thetas[k], Z, eps=1e-8)
        assert r["loglik"] == ll[k]

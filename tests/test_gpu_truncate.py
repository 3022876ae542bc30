"""GPU unit tests of the truncation step (A6) against numpy's SVD:
||X Y^T - U V^T||_2 <= 10 eps ||X Y^T||_2 (SURVEY Sec. 8(c) pin; SPEC acceptance), all QR paths
(0 global Householder, 1 shifted CholeskyQR3, 2 shared-memory Householder)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
import paper_1709_08625_b200 as H  # noqa: E402

pytestmark = pytest.mark.gpu


def _panel(m, R, seed, kind):
    rng = np.random.default_rng(seed)
    if kind == "decay":          # singular values 10^(-k/4)
        A = np.linalg.qr(rng.standard_normal((m, R)))[0]
        B = np.linalg.qr(rng.standard_normal((m, R)))[0]
        return A * 10.0 ** (-np.arange(R) / 4.0), B
    if kind == "dependent":      # exactly rank-deficient X (repeated columns)
        A = rng.standard_normal((m, R // 2))
        X = np.concatenate([A, A @ rng.standard_normal((R // 2, R - R // 2))], axis=1)
        return X, rng.standard_normal((m, R))
    if kind == "scaled":         # columns of wildly different scales
        X = rng.standard_normal((m, R)) * 10.0 ** rng.uniform(-8, 2, R)
        return X, rng.standard_normal((m, R))
    raise ValueError(kind)


@pytest.mark.parametrize("path", [0, 1])
@pytest.mark.parametrize("kind", ["decay", "dependent", "scaled"])
@pytest.mark.parametrize("m,R,eps", [(512, 60, 1e-6), (256, 80, 1e-8), (1024, 92, 1e-5)])
def test_truncation_error_bound(path, kind, m, R, eps):
    _check(path, kind, m, R, eps)


# shared-memory Householder path (panel m x R resident in the engine's 220 KB): sizes across the
# register-apply variants (m <= 256, m <= 512), ragged m, R = m
@pytest.mark.parametrize("kind", ["decay", "dependent", "scaled"])
@pytest.mark.parametrize("m,R,eps", [(256, 80, 1e-8), (200, 92, 1e-6), (300, 90, 1e-5), (64, 40, 1e-6),
                                     (100, 100, 1e-7), (33, 7, 1e-6)])
def test_truncation_smem_path(kind, m, R, eps):
    _check(2, kind, m, R, eps)


def _check(path, kind, m, R, eps):
    X, Y = _panel(m, R, 7 + m + R, kind)
    S = X @ Y.T
    U, V, r, cb, of = H.test_truncate(torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda(), eps, rlim=R, path=path)
    assert of == 0
    s = np.linalg.svd(S, compute_uv=False)
    err = np.linalg.norm(S - U.cpu().numpy() @ V.cpu().numpy().T, 2)
    assert err <= 10 * eps * s[0], (err / s[0], r)
    r_ref = int(np.sum(s > eps * s[0]))
    assert abs(r - r_ref) <= 2, (r, r_ref)


# large work capacities (K = 3 kcap + 32 up to 224 columns at kcap = 64): the core arrays leave
# shared memory (R > 96) and the panel QRs use the global paths; tight eps down to 1e-13
@pytest.mark.parametrize("path", [0, 1, 2])
@pytest.mark.parametrize("kind", ["decay", "dependent", "scaled"])
@pytest.mark.parametrize("m,R,eps", [(512, 150, 1e-10), (256, 200, 1e-12), (1024, 120, 1e-9), (300, 224, 1e-13)])
def test_truncation_large_capacity(path, kind, m, R, eps):
    _check(path, kind, m, R, eps)


# the dense-mode pipeline of small low-rank blocks (R23: dense S, fully pivoted ACA, shared-memory
# truncation) at tight eps, where the cross approximation runs to (or near) full rank
@pytest.mark.parametrize("kind", ["decay", "dependent", "scaled"])
@pytest.mark.parametrize("m,R,eps", [(128, 128, 1e-13), (128, 100, 1e-13), (64, 64, 1e-13), (128, 90, 3e-13),
                                     (256, 200, 1e-13), (200, 150, 1e-12), (96, 60, 1e-8)])
def test_truncation_dense_mode_pipeline(kind, m, R, eps):
    _check(3, kind, m, R, eps)


# the smem path with R = m (a full-rank cross approximation of a dense-mode block) at tight eps
@pytest.mark.parametrize("kind", ["decay", "dependent", "scaled"])
@pytest.mark.parametrize("m,R,eps", [(128, 128, 1e-13), (120, 110, 1e-13), (64, 64, 1e-13)])
def test_truncation_smem_full_rank_tight(kind, m, R, eps):
    _check(2, kind, m, R, eps)

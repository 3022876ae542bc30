"""Pins of the eps-oracle and of the oracle's own cluster / block tree (no GPU).

* htree: a hand-derived block tree for a contrived geometry (Def. A.1/A.2, PAPER.md:709-743,
  admissibility min(diam) <= eta dist), partition invariants.
* eps_rank: the definition of Remark 2 (R3) on spelled-out spectra.
* eps_matrix: every replaced block is at spectral distance sigma_{r+1} <= eps sigma_1 from the
  exact block (Eckart-Young; checked with an independent 2-norm), the rest of C is untouched, the
  result is symmetric; eps -> 0 recovers the exact likelihood.
"""
import numpy as np
import pytest

import oracle
import synth
from oracle import htree
from oracle.eps_oracle import eps_rank, eps_matrix, loglik_eps, truncation_spectra


def _groups(gap=0.35):
    # 4 groups of 64 collinear points: group g at x = gap*g + 0.1 k/63, k = 0..63, y = 0
    x = np.concatenate([gap * g + 0.1 * np.arange(64) / 63.0 for g in range(4)])
    return np.stack([x, np.zeros_like(x)], axis=1)


def test_block_tree_hand_derived():
    T = htree.cluster_tree(_groups())
    assert T.depth == 3 and T.n_pad == 256
    got = set(htree.block_tree(T, eta=2.0))
    H, R, Tt = htree.ND_H, htree.ND_R, htree.ND_T
    # level-1 halves: x in [0, 0.45] and [0.70, 1.15]: diam 0.45 <= 2 * 0.25 -> low rank;
    # level-2 groups g1 vs g0 (g3 vs g2): diam 0.1 <= 2 * 0.25 -> low rank; leaves inside a group
    # are adjacent (gap 0.1/63, diam ~0.05) -> dense tiles
    want = {(0, 0, 0, H), (1, 0, 0, H), (1, 1, 0, R), (1, 1, 1, H),
            (2, 0, 0, H), (2, 1, 0, R), (2, 1, 1, H), (2, 2, 2, H), (2, 3, 2, R), (2, 3, 3, H)}
    for g in range(4):
        want |= {(3, 2 * g, 2 * g, Tt), (3, 2 * g + 1, 2 * g, Tt), (3, 2 * g + 1, 2 * g + 1, Tt)}
    assert got == want
    # eta = 1: the level-1 pair is no longer admissible (0.45 > 0.25): its four children are
    got1 = set(htree.block_tree(T, eta=1.0))
    assert (1, 1, 0, H) in got1
    assert {(2, 2, 0, R), (2, 2, 1, R), (2, 3, 0, R), (2, 3, 1, R)} <= got1


@pytest.mark.parametrize("n,seed", [(2000, 1001), (4096, 7), (777, 3)])
def test_block_tree_partitions_the_matrix(n, seed):
    s = synth.uniform_points(n, seed)
    T = htree.cluster_tree(s)
    assert np.array_equal(np.sort(T.perm[T.perm >= 0]), np.arange(n))
    cover = np.zeros((n, n), dtype=np.int32)
    for (l, i, j, ty) in htree.block_tree(T):
        if ty == htree.ND_H:
            continue
        r, c = T.members[(l, i)], T.members[(l, j)]
        cover[np.ix_(r, c)] += 1
        if i != j:
            cover[np.ix_(c, r)] += 1
        if ty == htree.ND_R:     # low-rank leaves satisfy the admissibility condition
            assert min(htree.diam(T, l, i), htree.diam(T, l, j)) <= 2.0 * htree.dist(T, l, i, j)
    assert np.all(cover == 1)


def test_eps_rank_definition():
    sig = np.array([2.0, 1.0, 3e-4, 1e-4, 1e-9])
    assert eps_rank(sig, 1e-4) == 3          # sigma_4 = 1e-4 <= 1e-4 * 2 -> keep 3
    assert eps_rank(sig, 1e-3) == 2
    assert eps_rank(sig, 1e-12) == 5
    assert eps_rank(sig, 1e-12, kmax=4) == 4
    assert eps_rank(np.zeros(3), 1e-4) == 0


def test_eps_matrix_blocks_are_optimal_truncations():
    n = 1500
    s = synth.uniform_points(n, 17)
    C = oracle.cov_dense(s, 1.0, 0.1, 1.5, 1e-6)
    sp = truncation_spectra(s, C)
    eps = 1e-4
    Ce, info = eps_matrix(C, sp, eps)
    assert np.array_equal(Ce, Ce.T)
    touched = np.zeros_like(C, dtype=bool)
    for rows, cols, U, sig, Vt in sp:
        B, Bt = C[np.ix_(rows, cols)], Ce[np.ix_(rows, cols)]
        r = eps_rank(sig, eps)
        e2 = np.linalg.norm(B - Bt, 2)                   # independent 2-norm (LAPACK SVD of the error)
        s1 = np.linalg.norm(B, 2)
        assert e2 <= eps * s1 * (1 + 1e-10) + 1e-15
        assert np.linalg.matrix_rank(Bt, tol=1e-12 * s1) <= r
        touched[np.ix_(rows, cols)] = True
        touched[np.ix_(cols, rows)] = True
    assert np.array_equal(Ce[~touched], C[~touched])     # dense blocks untouched
    assert info["blocks"] == len(sp) > 0


def test_eps_to_zero_recovers_exact():
    n = 1200
    s = synth.uniform_points(n, 19)
    th = (1.0, 0.1, 0.5, 1e-6)
    Z = oracle.sample_dense(s, synth.xi(n, 20), *th)
    r = loglik_eps(s, Z, *th, eps_list=[0.0, 1e-6])
    ex = r["exact"]
    assert abs(r[0.0][0] - ex[0]) <= 1e-10 * abs(ex[0])
    # a looser eps moves L, within the first-order bound |dlogdet| <= n ||E||_2 / lambda_min-ish:
    assert abs(r[1e-6][0] - ex[0]) > 0

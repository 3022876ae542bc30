"""ORACLE (test infrastructure only) — the eps-oracle of SURVEY.md Sec. 8(c).

The dense covariance C (``oracle.cov_dense``) with every admissible block of the block tree
(``oracle.htree``, the same rules as the method: Def. A.1/A.2) replaced by its
OPTIMAL truncation at (eps, k) — the truncated SVD, which is the best rank-r approximation in the
spectral norm — with r the smallest rank such that sigma_{r+1} <= eps * sigma_1 (Remark 2,
PAPER.md:256-264, read as DESIGN.md R3), capped at r <= kmax when kmax > 0.  The upper triangle is
the mirror image (Remark 1 / R10).  The resulting matrix is factored by dense LAPACK Cholesky and
L = -n/2 log 2 pi - 1/2 log det - 1/2 Z^T C_eps^{-1} Z (Eq. (1)/(2)).

It separates the method's inherent error (the approximation C -> C~ with the BEST possible blocks)
from the implementation's (ACA error, H-Cholesky truncations), SURVEY App. A.4.  It is feasible
where the dense oracle is.  It does not model ACA or the Cholesky's own truncations, so the GPU
path is expected at or slightly above its error.

One SVD per admissible block serves every eps of a run (``truncation_spectra`` then
``eps_matrix``), so C2's two eps values cost one set of SVDs per theta.
"""
from __future__ import annotations

from typing import Dict, List, Sequence, Tuple

import numpy as np

import torch

from . import cholesky, cov_dense, loglik_from_factor, NotSPD, lapack_threads
from .htree import cluster_tree, lowrank_blocks


def eps_rank(sig: np.ndarray, eps: float, kmax: int = 0) -> int:
    """Smallest r with sigma_{r+1} <= eps sigma_1 (sig descending), then r <= kmax (kmax > 0)."""
    if sig.size == 0 or sig[0] <= 0.0:
        return 0
    r = int(np.count_nonzero(sig > eps * sig[0]))
    if kmax > 0:
        r = min(r, kmax)
    return r


def truncation_spectra(s: np.ndarray, C: np.ndarray, eta: float = 2.0, dense_below: int = 32):
    """SVD of every admissible lower block of C: list of (rows, cols, U, sig, Vt)."""
    T = cluster_tree(s)
    out = []
    with lapack_threads():
        for rows, cols, _lvl in lowrank_blocks(T, eta, dense_below):
            B = torch.from_numpy(np.ascontiguousarray(C[np.ix_(rows, cols)]))
            U, sig, Vt = torch.linalg.svd(B, full_matrices=False)   # LAPACK gesdd (MKL)
            out.append((rows, cols, U.numpy(), sig.numpy(), Vt.numpy()))
    return out


def eps_matrix(C: np.ndarray, spectra, eps: float, kmax: int = 0) -> Tuple[np.ndarray, Dict]:
    """C with each admissible block (and its mirror) replaced by its (eps, kmax) truncated SVD."""
    Ce = C.copy()
    ranks: List[int] = []
    binds = 0
    for rows, cols, U, sig, Vt in spectra:
        r = eps_rank(sig, eps, kmax)
        if kmax > 0 and r == kmax and eps_rank(sig, eps, 0) > kmax:
            binds += 1
        ranks.append(r)
        Bt = (U[:, :r] * sig[:r]) @ Vt[:r, :]
        Ce[np.ix_(rows, cols)] = Bt
        Ce[np.ix_(cols, rows)] = Bt.T
    info = {"blocks": len(ranks), "max_rank": max(ranks) if ranks else 0,
            "mean_rank": float(np.mean(ranks)) if ranks else 0.0, "cap_binds": binds}
    return Ce, info


def loglik_eps(s, Z, sigma2, ell, nu, nugget, eps_list: Sequence[float], kmax: int = 0, eta: float = 2.0,
               with_exact: bool = True):
    """Exact L (if with_exact) and the eps-oracle L for each eps.  Returns a dict:
    {"exact": (L, logdet, quad), eps: (L, logdet, quad) or "NOT_SPD", ...} plus rank info."""
    C = cov_dense(s, sigma2, ell, nu, nugget)
    out = {}
    if with_exact:
        out["exact"] = loglik_from_factor(cholesky(C), Z)
    spectra = truncation_spectra(s, C, eta)
    for eps in eps_list:
        Ce, info = eps_matrix(C, spectra, eps, kmax)
        try:
            out[eps] = loglik_from_factor(cholesky(Ce), Z)
        except NotSPD:
            out[eps] = "NOT_SPD"
        out[("info", eps)] = info
        del Ce
    return out

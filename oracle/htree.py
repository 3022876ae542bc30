"""ORACLE (test infrastructure only) — cluster tree A1 and block tree A2, restated on the CPU.

Independent of the CUDA path's planner (``paper_1709_08625_b200/csrc/plan.cpp``): written from
the definitions, not from that code, and used by the eps-oracle (``oracle/eps_oracle.py``) and
by ``tests/test_plan.py`` (which compares plan.cpp with it).

* Cluster tree — Def. A.1 with the split strategy of the listing
  (``TAutoBSPPartStrat(adaptive_split_axis)``) read as DESIGN.md R5:
  tight bounding box of a cluster's points, split the longest axis (ties -> x), stable sort on
  that coordinate, the first ceil(m/2) points go left.  Uniform depth L = ceil(log2(n / 32)):
  every leaf holds <= 32 points; internal positions are padded to 32 per leaf (phantom slots).
* Block tree — Def. A.2 with ``TStdGeomAdmCond(2.0, use_min_diam)``
  (PAPER.md:475), read as DESIGN.md R6: (tau, sigma) admissible iff dist > 0 and
  min(diam tau, diam sigma) <= eta * dist, diam = bounding-box diagonal, dist = Euclidean gap of
  the boxes.  Admissible blocks above the leaf level are low-rank leaves; admissible blocks at the
  leaf level are dense 32 x 32 tiles (R21); a subdivided admissible block forces its
  descendants to be subdivided down to tiles (never low-rank) when dense_below > 32.  Lower
  triangle plus diagonal only (R10).
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Dict, List, Tuple

import numpy as np

LEAF = 32
ND_H, ND_R, ND_T = 0, 1, 2   # subdivided, low-rank leaf, dense leaf


@dataclass
class ClusterTree:
    n: int
    depth: int                       # L
    perm: np.ndarray                 # n_pad int64: external index of internal position, -1 = phantom
    members: Dict[Tuple[int, int], np.ndarray]   # (level, c) -> external indices of the cluster's points
    boxes: Dict[Tuple[int, int], Tuple[np.ndarray, np.ndarray]]   # (level, c) -> (lo, hi)

    @property
    def n_pad(self) -> int:
        return LEAF << self.depth


def cluster_tree(s: np.ndarray) -> ClusterTree:
    s = np.asarray(s, dtype=np.float64)
    n = s.shape[0]
    L = 0
    while (LEAF << L) < n:
        L += 1
    members: Dict[Tuple[int, int], np.ndarray] = {(0, 0): np.arange(n, dtype=np.int64)}
    boxes: Dict[Tuple[int, int], Tuple[np.ndarray, np.ndarray]] = {}
    for l in range(L + 1):
        for c in range(1 << l):
            idx = members[(l, c)]
            if idx.size:
                P = s[idx]
                lo, hi = P.min(axis=0), P.max(axis=0)
            else:
                lo = hi = np.full(s.shape[1], np.nan)
            boxes[(l, c)] = (lo, hi)
            if l == L:
                continue
            ext = hi - lo
            # longest extent, ties -> the lowest axis (x, then y); 2-D or 3-D
            axis = 0 if idx.size == 0 else int(np.argmax(ext))
            order = np.argsort(s[idx, axis], kind="stable")   # ties keep the current order
            idx = idx[order]
            m1 = (idx.size + 1) // 2
            members[(l + 1, 2 * c)] = idx[:m1]
            members[(l + 1, 2 * c + 1)] = idx[m1:]
    perm = np.full(LEAF << L, -1, dtype=np.int64)
    for c in range(1 << L):
        idx = members[(L, c)]
        assert idx.size <= LEAF
        perm[c * LEAF: c * LEAF + idx.size] = idx
    return ClusterTree(n, L, perm, members, boxes)


def diam(T: ClusterTree, l: int, c: int) -> float:
    lo, hi = T.boxes[(l, c)]
    return math.hypot(*(hi - lo))


def dist(T: ClusterTree, l: int, i: int, j: int) -> float:
    (a0, a1), (b0, b1) = T.boxes[(l, i)], T.boxes[(l, j)]
    gap = np.maximum(0.0, np.maximum(a0 - b1, b0 - a1))
    return math.hypot(*gap)


def admissible(T: ClusterTree, l: int, i: int, j: int, eta: float) -> bool:
    if eta <= 0 or i == j:
        return False
    d = dist(T, l, i, j)
    if not d > 0:          # also False for empty clusters (NaN boxes)
        return False
    return min(diam(T, l, i), diam(T, l, j)) <= eta * d


def block_tree(T: ClusterTree, eta: float = 2.0, dense_below: int = LEAF) -> List[Tuple[int, int, int, int]]:
    """Blocks (level, i, j, type) of the lower triangle incl. the diagonal (i >= j)."""
    L = T.depth
    out: List[Tuple[int, int, int, int]] = []

    def rec(l: int, i: int, j: int, forced: bool) -> None:
        if i == j:
            if l == L:
                out.append((l, i, j, ND_T))
                return
            out.append((l, i, j, ND_H))
            rec(l + 1, 2 * i, 2 * j, forced)
            rec(l + 1, 2 * i + 1, 2 * j, forced)
            rec(l + 1, 2 * i + 1, 2 * j + 1, forced)
            return
        adm = (not forced) and admissible(T, l, i, j, eta)
        if adm and l < L and (T.n_pad >> l) > dense_below:
            out.append((l, i, j, ND_R))
            return
        if l == L:
            out.append((l, i, j, ND_T))
            return
        out.append((l, i, j, ND_H))
        for a in (0, 1):
            for b in (0, 1):
                rec(l + 1, 2 * i + a, 2 * j + b, forced or adm)

    rec(0, 0, 0, False)
    return out


def lowrank_blocks(T: ClusterTree, eta: float = 2.0, dense_below: int = LEAF):
    """(row external indices, col external indices, level) of every low-rank leaf (lower)."""
    for (l, i, j, ty) in block_tree(T, eta, dense_below):
        if ty == ND_R:
            yield T.members[(l, i)], T.members[(l, j)], l

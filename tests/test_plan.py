"""Host-side logic of libhcov (no GPU): symbol exports, cluster tree (A1) and block tree (A2)
against an independent Python mirror of the rules (R5, R6), partition invariants."""
import math
import os
import re

import numpy as np
import pytest

import paper_1709_08625_b200 as H
import synth
from oracle import htree

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "hcov.h")).read()
    names = set(re.findall(r"\b(hcov_[a-z_0-9]+)\s*\(", hdr))
    assert len(names) >= 17
    L = H.lib()
    for nm in sorted(names):
        assert hasattr(L, nm), nm
    assert set(H._SIGS) == names


def _mirror_tree(s, leaf=32):
    """The oracle's restatement of A1 (oracle/htree.py; R5)."""
    T = htree.cluster_tree(s)
    return T.depth, T.perm


def _mirror_blocks(s, perm, L, eta=2.0, leaf=32, dense_below=32):
    """The oracle's restatement of A2 (oracle/htree.py; R6, R21)."""
    return set(htree.block_tree(htree.cluster_tree(s), eta, dense_below))


@pytest.mark.parametrize("n,seed,geom", [(1, 1, "u"), (31, 2, "u"), (33, 3, "u"), (500, 4, "u"),
                                         (2000, 1001, "u"), (4096, 5, "c"), (1000, 6, "line")])
def test_tree_and_blocks_match_mirror(n, seed, geom):
    if geom == "u":
        s = synth.uniform_points(n, seed)
    elif geom == "c":
        s = synth.clustered_points(n, seed, seed + 1, frac=0.2)
    else:
        s = synth.collinear_points(n, seed)
    T = H.Tree(s)
    info = T.info()
    L, perm = _mirror_tree(s)
    assert info["depth"] == L and info["n_pad"] == 32 << L
    got = T.perm_i2e()
    assert np.array_equal(got, perm)
    real = got[got >= 0]
    assert np.array_equal(np.sort(real), np.arange(n))       # bijection on the real points
    assert np.all((got.reshape(-1, 32) >= 0).sum(1) <= 32)
    blocks = {tuple(int(v) for v in b) for b in T.blocks()}
    assert blocks == _mirror_blocks(s, perm, L)


@pytest.mark.parametrize("eta,dense_below", [(2.0, 32), (2.0, 128), (0.0, 32), (0.7, 32)])
def test_block_partition_covers_lower_triangle(eta, dense_below):
    n = 3000
    s = synth.uniform_points(n, 77)
    T = H.Tree(s, eta=eta, dense_below=dense_below)
    info = T.info()
    L, npad = info["depth"], info["n_pad"]
    b = T.blocks()
    leaves = b[b[:, 3] != H.ND_H]
    m = npad >> leaves[:, 0].astype(np.int64)
    off = leaves[:, 1] != leaves[:, 2]
    # lower + diagonal leaves mirrored cover I x I exactly once
    assert int(np.sum(m[off] ** 2)) * 2 + int(np.sum(m[~off] ** 2)) == npad * npad
    assert np.all(leaves[:, 1] >= leaves[:, 2])
    assert np.all(leaves[~off, 0] == L)                        # diagonal leaves are 32x32 tiles
    assert np.all(leaves[leaves[:, 3] == H.ND_T, 0] == L)
    r = leaves[leaves[:, 3] == H.ND_R]
    assert np.all((npad >> r[:, 0].astype(np.int64)) > dense_below)
    if eta == 0.0:
        assert len(r) == 0 and info["n_dense_tiles"] == (npad // 32) * (npad // 32 + 1) // 2
    # no overlaps: paint a leaf-level occupancy grid
    N = npad // 32
    grid = np.zeros((N, N), dtype=np.int32)
    for l, i, j, t in leaves:
        sp = 1 << (L - l)
        grid[i * sp:(i + 1) * sp, j * sp:(j + 1) * sp] += 1
    assert np.array_equal(grid, np.tril(np.ones((N, N), dtype=np.int32)))


def test_admissibility_is_symmetric_and_eta_monotone():
    s = synth.uniform_points(4096, 9)
    c1 = np.bincount(H.Tree(s, eta=1.0).blocks()[:, 3], minlength=3)
    c2 = np.bincount(H.Tree(s, eta=2.0).blocks()[:, 3], minlength=3)
    c4 = np.bincount(H.Tree(s, eta=4.0).blocks()[:, 3], minlength=3)
    # larger eta admits coarser blocks -> fewer dense tiles
    assert c1[H.ND_T] >= c2[H.ND_T] >= c4[H.ND_T]


def test_invalid_inputs():
    with pytest.raises(H.HcovError) as e:
        H.Tree(np.zeros((0, 2)))
    assert e.value.code == 2
    bad = synth.uniform_points(10, 1)
    bad[3, 1] = np.nan
    with pytest.raises(H.HcovError) as e:
        H.Tree(bad)
    assert e.value.code == 1


def test_task_dag_is_consistent():
    # every task's arguments are in range; the DAG's longest chain grows ~linearly in the leaves
    for n in (2048, 16384):
        T = H.Tree(synth.uniform_points(n, 3))
        info = T.info()
        t = T.tasks()
        assert t.shape[0] == info["n_tasks"]
        assert set(np.unique(t[:, 0])) <= set(range(14))
        assert set(np.unique(t[:, 1])) == {0, 1, 2, 3}
        # phases are ordered: assembly tasks first, then the root forward solve, the back-solve last
        ph = t[:, 1]
        assert np.all(np.diff(ph[ph > 0]) >= 0)
        assert info["n_waves"] <= 12 * info["n_leaves"] + 64


def test_backsolve_dag_is_the_transposed_solve():
    """Phase 3 (root back-solve, NEXT (f1)): one BSEG per leaf segment, in reverse order, each
    depending only on later segments / BPROJ tasks; one BPROJ per low-rank block."""
    n = 4096
    T = H.Tree(synth.uniform_points(n, 5))
    info = T.info()
    t = T.tasks()
    off, sc = T.succ()
    ph3 = np.nonzero(t[:, 1] == 3)[0]
    bseg = ph3[t[ph3, 0] == 12]
    bproj = ph3[t[ph3, 0] == 13]
    assert len(bseg) == info["n_leaves"] and len(bproj) == info["n_lowrank"]
    assert np.array_equal(t[bseg, 3], np.arange(info["n_leaves"])[::-1])
    seg_of = {int(k): int(t[k, 3]) for k in bseg}
    # edges into a BSEG come from BSEGs of larger segments, BPROJs or joins of phase 3 only
    for k in range(len(t)):
        for z in range(off[k], off[k + 1]):
            d = sc[z]
            if t[d, 1] == 3:
                assert t[k, 1] == 3
            if d in seg_of and k in seg_of:
                assert seg_of[k] > seg_of[d]


@pytest.mark.parametrize("n,seed", [(3000, 21), (9000, 22)])
def test_factor_trunc_schedule(n, seed):
    """SPD-preserving mode (hcov_tree_opts.factor_trunc, R27): every low-rank block gets
    exactly one TRUNC task (a RAPP without terms, d = 1) that runs after the block's last update
    (d = 2 chunk or its ACA) and after the solve of its column; no other RAPP truncates (d = 1)."""
    s = synth.uniform_points(n, seed)
    T0 = H.Tree(s)
    T1 = H.Tree(s, factor_trunc=True)
    t0, t1 = T0.tasks(), T1.tasks()
    RAPP, ACA, SEG = 5, 1, 6
    nr = int(np.sum(t0[:, 0] == ACA))
    assert nr > 0 and int(np.sum(t1[:, 0] == ACA)) == nr
    tr = np.nonzero((t1[:, 0] == RAPP) & (t1[:, 5] == 1))[0]
    assert tr.size == nr                                        # one TRUNC per low-rank block
    assert np.all(t1[tr, 3] == t1[tr, 4])                       # ... without terms
    assert sorted(t1[tr, 2].tolist()) == sorted(t1[t1[:, 0] == ACA, 2].tolist())
    last0 = (t0[:, 0] == RAPP) & (t0[:, 5] == 1)
    last1 = (t1[:, 0] == RAPP) & (t1[:, 5] == 2)
    assert int(np.sum(last1)) == int(np.sum(last0))             # the last update chunk stays near-lossless
    # predecessors of each TRUNC: reachable from a SEG task of its column's solve
    off, sc = T1.succ()
    pred = {}
    for u in range(len(off) - 1):
        for v in sc[off[u]:off[u + 1]]:
            pred.setdefault(int(v), []).append(u)

    def ancestors_have(t, ty, depth=4):
        frontier = [t]
        for _ in range(depth):
            nxt = []
            for x in frontier:
                for p in pred.get(x, []):
                    if t1[p, 0] == ty:
                        return True
                    nxt.append(p)
            frontier = nxt
        return False
    for t in tr[:50]:
        assert ancestors_have(int(t), SEG), t
    # the rest of the schedule is unchanged in size: standard tasks + one TRUNC per block + one join per column
    assert t1.shape[0] > t0.shape[0] + nr - 1


@pytest.mark.parametrize("n,seed", [(1, 1), (33, 2), (3000, 3)])
def test_3d_tree_and_blocks_match_mirror(n, seed):
    """3-D variant: host planner vs the oracle's restatement (argmax-extent axis,
    3-D boxes, diameters and gaps)."""
    s = synth.uniform_points_3d(n, seed)
    T = H.Tree(s)
    info = T.info()
    Tm = htree.cluster_tree(s)
    assert info["dim"] == 3 and info["depth"] == Tm.depth
    assert np.array_equal(T.perm_i2e(), Tm.perm)
    assert {tuple(int(v) for v in b) for b in T.blocks()} == set(htree.block_tree(Tm, 2.0, 32))
    bb = T.bbox()
    assert bb.shape[1] == 6
    lo, hi = Tm.boxes[(0, 0)]
    assert np.array_equal(bb[0, :3], lo) and np.array_equal(bb[0, 3:], hi)


def test_3d_flat_points_give_the_2d_tree():
    """Points with a constant z: the z extent is 0, never the longest, so the 3-D planner splits
    exactly as the 2-D one."""
    s = synth.uniform_points(5000, 4)
    T2 = H.Tree(s)
    T3 = H.Tree(np.column_stack([s, np.full(5000, 0.5)]))
    assert np.array_equal(T2.perm_i2e(), T3.perm_i2e())
    assert np.array_equal(T2.blocks(), T3.blocks())
    assert np.array_equal(T2.tasks(), T3.tasks())

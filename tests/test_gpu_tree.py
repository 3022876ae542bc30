"""A1 / A2 on the device (tree.cu kernels K1, K2) against the host planner, bit for bit.

The host planner's trees are pinned against the oracle's independent restatement of the rules
(oracle/htree.py; tests/test_plan.py, R5 / R6); here the device-built cluster tree
(internal order, bounding boxes), block tree (every node with its level, indices and type) and
the task schedule planned from them must equal the host's exactly, including the tie cases of the
stable median split (duplicate points, points on a lattice, collinear points) and ragged n.
Also pinned directly against the mirror for two small cases."""
import numpy as np
import pytest
import torch

import paper_1709_08625_b200 as H
import synth
from oracle import htree

pytestmark = pytest.mark.gpu


def _cases():
    r = np.random.default_rng(77)
    lattice = np.stack(np.meshgrid(np.arange(64) / 64.0, np.arange(48) / 48.0), -1).reshape(-1, 2)
    dup = np.repeat(r.random((700, 2)), 3, axis=0)[r.permutation(2100)]
    line = np.stack([r.random(3000), np.zeros(3000)], 1)
    neg = r.standard_normal((5000, 2)) * 1e3
    return {
        "n1": synth.uniform_points(1, 1),
        "n32": synth.uniform_points(32, 2),
        "n33": synth.uniform_points(33, 3),
        "c1": synth.uniform_points(2000, 1001),
        "ragged": synth.uniform_points(12345, 9),
        "clustered": synth.clustered_points(40000, 11, 12),
        "lattice_ties": lattice,
        "duplicates": dup,
        "collinear": line,
        "wide_range": neg,
    }


CASES = _cases()


def _same(Td, Th):
    idv, ih = Td.info(), Th.info()
    assert idv["tree_on_device"] == 1 and ih["tree_on_device"] == 0
    for k in ("n", "n_pad", "depth", "n_leaves", "n_dense_tiles", "n_lowrank", "n_tasks", "n_waves", "uv_elems",
              "w_elems", "slot_a", "slot_b", "n_cores", "n_edges", "n_xterm", "max_mq"):
        assert idv[k] == ih[k], k
    assert np.array_equal(Td.perm_i2e(), Th.perm_i2e())
    bd, bh = Td.bbox(), Th.bbox()
    assert np.array_equal(np.isnan(bd), np.isnan(bh))
    ok = ~np.isnan(bh)
    assert np.array_equal(bd[ok], bh[ok])            # -0.0 == +0.0 only where a coordinate is a zero
    assert np.array_equal(Td.blocks(), Th.blocks())
    assert np.array_equal(Td.tasks(), Th.tasks())
    od, sd = Td.succ()
    oh, sh = Th.succ()
    assert np.array_equal(od, oh) and np.array_equal(sd, sh)


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("eta,dense_below", [(2.0, 32), (0.7, 128)])
def test_device_tree_equals_host(name, eta, dense_below):
    s = CASES[name]
    Td = H.Tree(torch.from_numpy(s).cuda(), eta=eta, dense_below=dense_below)
    Th = H.Tree(s, eta=eta, dense_below=dense_below)
    _same(Td, Th)


@pytest.mark.parametrize("factor_trunc", [False, True])
def test_device_tree_equals_host_c3(factor_trunc):
    cfg = synth.CONFIGS["C3"]
    s = synth.points(cfg)
    Td = H.Tree(torch.from_numpy(s).cuda(), factor_trunc=factor_trunc)
    Th = H.Tree(s, factor_trunc=factor_trunc)
    _same(Td, Th)


def test_device_tree_matches_mirror():
    for s in (CASES["c1"], CASES["duplicates"]):
        Td = H.Tree(torch.from_numpy(s).cuda())
        T = htree.cluster_tree(s)
        assert Td.info()["depth"] == T.depth
        p = Td.perm_i2e()
        np.testing.assert_array_equal(p, T.perm)
        got = {tuple(int(v) for v in b) for b in Td.blocks()}
        assert got == set(htree.block_tree(T, 2.0, 32))


def test_device_tree_2M_equals_host():
    """C5's 2M points: K1 + K2 on the device against the host planner (and faster than it)."""
    cfg = synth.CONFIGS["C5"]
    s = synth.points(cfg)
    Td = H.Tree(torch.from_numpy(s).cuda())
    Th = H.Tree(s)
    assert np.array_equal(Td.perm_i2e(), Th.perm_i2e())
    assert np.array_equal(Td.bbox(), Th.bbox())
    assert np.array_equal(Td.blocks(), Th.blocks())
    print(f"2M: device A1+A2 {Td.info()['geo_ms']:.0f} ms; host plan {Th.info()['geo_ms']:.0f} ms")


def test_device_tree_rejects_bad_input():
    s = synth.uniform_points(100, 1)
    s[17, 1] = np.nan
    with pytest.raises(H.HcovError):
        H.Tree(torch.from_numpy(s).cuda())
    s[17, 1] = np.inf
    with pytest.raises(H.HcovError):
        H.Tree(torch.from_numpy(s).cuda())

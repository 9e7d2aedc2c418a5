"""Host forest scheduler (csrc/tree.cu skb_forest_schedule, used by tree.Forest) against the
per-node scheduler skb_tree_schedule on the same forests: heights, level order, leaves,
parent destinations and global child ids identical; malformed trees rejected."""
import ctypes

import numpy as np
import pytest

from oracle import fixtures
from paper_1810_08061_b200 import runtime as rt
from paper_1810_08061_b200.tree import Forest


def _reference_schedule(trees):
    sizes = [len(t[0]) for t in trees]
    bases = np.concatenate([[0], np.cumsum(sizes)[:-1]])
    shift = np.repeat(bases, sizes)
    L = np.concatenate([t[1] for t in trees]).astype(np.int64)
    R = np.concatenate([t[2] for t in trees]).astype(np.int64)
    L = np.ascontiguousarray(np.where(L >= 0, L + shift, -1))
    R = np.ascontiguousarray(np.where(R >= 0, R + shift, -1))
    n = len(L)
    out = [np.empty(n, np.int32) for _ in range(2)] + [np.empty(n + 1, np.int32)] + \
          [np.empty(n, np.int32) for _ in range(2)]
    c = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    mh = rt.host_lib().skb_tree_schedule(n, c(L), c(R), *[c(a) for a in out])
    h, o, lo, lv, d = out
    ni = lo[mh]
    return mh, h, o[:ni], lo[:mh + 1], lv[:n - ni], d, L, R


@pytest.mark.parametrize("ntrees,leaves,seed", [(1, 1, 0), (7, 5, 1), (300, 32, 2), (1000, 17, 3)])
def test_forest_schedule_matches_node_schedule(ntrees, leaves, seed):
    rng = np.random.default_rng(seed)
    trees = [fixtures.random_tree_arrays(int(rng.integers(1, leaves + 1)), rng) for _ in range(ntrees)]
    f = Forest(trees)
    mh, h, o, lo, lv, d, L, R = _reference_schedule(trees)
    assert f.nlevels == mh
    for got, ref in ((f.height, h), (f.order, o), (f.level_off, lo), (f.leaves, lv), (f.dest, d),
                     (f.left, L), (f.right, R)):
        assert np.array_equal(got, ref)


@pytest.mark.parametrize("tree", [
    (np.zeros(3), np.array([1, -1, -1]), np.array([-1, -1, -1])),    # one child
    (np.zeros(3), np.array([1, -1, -1]), np.array([5, -1, -1])),     # child outside the tree
    (np.zeros(3), np.array([-1, 0, -1]), np.array([-1, 2, -1])),     # child before its parent
])
def test_malformed_trees_rejected(tree):
    with pytest.raises(ValueError):
        Forest([tree])

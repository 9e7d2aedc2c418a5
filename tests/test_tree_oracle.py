"""CPU: the float64 TreeLSTM restatement (oracle/tree.py) against the
reference's own interpret_module outputs (tests/golden/treelstm_*.json)."""
import numpy as np
import pytest

from oracle import fixtures
from oracle import tree as otree
from vm_cases import parse_tree


def flat(t):
    val, left, right = [], [], []

    def go(n):
        i = len(val)
        val.append(n.value if n.value is not None else 0.0)
        left.append(-1)
        right.append(-1)
        if n.left is not None and n.left.value is not None:
            left[i] = go(n.left)
            right[i] = go(n.right)
        return i
    go(t)
    return np.asarray(val), np.asarray(left), np.asarray(right)


@pytest.mark.parametrize("name", [c["name"] for c in fixtures.TREE_CASES])
def test_tree_oracle_matches_reference(name):
    doc = fixtures.load_golden(name)
    case = doc["case"]
    w = fixtures.tree_weights(case["H"], case["seed"])
    trees = [flat(parse_tree(s)) for s in doc["trees"]]
    for (val, left, right), (h_ref, c_ref) in zip(trees, doc["expected"]):
        h, c = otree.node_state(val, left, right, w)
        assert np.array_equal(h.reshape(-1), np.asarray(h_ref)), (h, h_ref)
        assert np.array_equal(c.reshape(-1), np.asarray(c_ref))
    hb, cb = otree.forest(trees, w)
    ref = np.asarray([e[0] for e in doc["expected"]])
    assert np.max(np.abs(hb - ref)) < 1e-12

"""C5 TreeLSTM on the GPU (csrc/tree.cu via paper_1810_08061_b200.tree):
the forest's root states against the reference's own interpret_module outputs
(tests/golden/treelstm_*.json) and the float64 restatement at larger batches.
fp32 GEMMs: rtol 1e-5 (stated bound); TF32: 2e-3."""
import numpy as np
import pytest

from oracle import fixtures
from oracle import tree as otree
from paper_1810_08061_b200.tree import Forest, tree_lstm
from vm_cases import parse_tree

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", [c["name"] for c in fixtures.TREE_CASES])
def test_forest_matches_reference(name):
    doc = fixtures.load_golden(name)
    case = doc["case"]
    w = fixtures.tree_weights(case["H"], case["seed"])
    forest = Forest([parse_tree(s) for s in doc["trees"]])
    h, c = tree_lstm(forest, w)
    h_ref = np.asarray([e[0] for e in doc["expected"]])
    c_ref = np.asarray([e[1] for e in doc["expected"]])
    assert np.allclose(h.array, h_ref, rtol=1e-5, atol=1e-6)
    assert np.allclose(c.array, c_ref, rtol=1e-5, atol=1e-6)


# (H = 40 and 128 leave a partial last group of the engine path's 3-unit interleave, H = 2 a
# single one; odd H always takes the cuBLAS level GEMMs.)
@pytest.mark.parametrize("ntrees,leaves,H,math,tol", [(300, 32, 64, "fp32", 1e-5), (257, 17, 128, "tf32", 2e-3),
                                                     (600, 32, 128, "tf32", 2e-3), (120, 9, 40, "tf32", 2e-3),
                                                     (64, 5, 2, "tf32", 2e-3), (90, 12, 33, "tf32", 2e-3)])
def test_forest_matches_oracle(ntrees, leaves, H, math, tol):
    rng = np.random.default_rng(ntrees)
    trees = [fixtures.random_tree_arrays(int(rng.integers(1, leaves + 1)), rng) for _ in range(ntrees)]
    w = fixtures.tree_weights(H, 5)
    h_ref, c_ref = otree.forest(trees, w)
    h, c = tree_lstm(Forest(trees), w, math=math)
    assert np.allclose(h.array, h_ref, rtol=tol, atol=tol)
    assert np.allclose(c.array, c_ref, rtol=tol, atol=tol)


def test_repeated_forest_replays_graph():
    from paper_1810_08061_b200 import runtime
    from paper_1810_08061_b200.tree import pack_weights
    import torch
    rng = np.random.default_rng(9)
    trees = [fixtures.random_tree_arrays(int(rng.integers(1, 20)), rng) for _ in range(50)]
    w = fixtures.tree_weights(32, 6)
    forest = Forest(trees)
    pw = pack_weights(w, torch.device("cuda"))
    first = tree_lstm(forest, w, packed=pw)[0].array
    outs = [tree_lstm(forest, w, packed=pw)[0].array for _ in range(3)]
    assert runtime.lib().skb_tree_last_mode() == 1
    for o in outs:
        assert np.array_equal(o, first)


def test_engine_path_matches_oracle():
    """SKB_TREE_TC=1: every level on skb's tcgen05 engine with the cell fused into the GEMM
    epilogue (read once per process: run in a child)."""
    import os
    import subprocess
    import sys
    code = (
        "import numpy as np\n"
        "from oracle import fixtures\n"
        "from oracle import tree as otree\n"
        "from paper_1810_08061_b200.tree import Forest, tree_lstm\n"
        "for nt, lv, H in ((257, 17, 128), (120, 9, 40), (64, 5, 2), (90, 12, 33)):\n"
        "    rng = np.random.default_rng(nt)\n"
        "    trees = [fixtures.random_tree_arrays(int(rng.integers(1, lv + 1)), rng) for _ in range(nt)]\n"
        "    w = fixtures.tree_weights(H, 5)\n"
        "    h_ref, c_ref = otree.forest(trees, w)\n"
        "    h, c = tree_lstm(Forest(trees), w, math='tf32')\n"
        "    assert np.allclose(h.array, h_ref, rtol=2e-3, atol=2e-3), H\n"
        "    assert np.allclose(c.array, c_ref, rtol=2e-3, atol=2e-3), H\n"
        "print('ok')\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SKB_TREE_TC="1", PYTHONPATH=os.pathsep.join([root, os.path.join(root, "tests")]))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr

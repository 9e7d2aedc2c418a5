"""Golden fixtures for recursive FuncCall on the region VM (TEST
INFRASTRUCTURE; run in the build container where the reference lives).

The programs under oracle/programs/recursion/ are traced with the reference's
`sexpr` backend — the one that stages recursion as FuncCall (reference
runtime/calls.py:88-164, corpus/manifest.json tree_prod) — and executed by the
reference `execute` (graph/execute.py:191-193), which recurses on the host.
Output: tests/golden/vm_recursion.json in the vm_corpus.json format.

Usage: python oracle/gen_recursion_golden.py
"""

from __future__ import annotations

import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
REF = os.environ.get("SKB_REF", "/root/reference/pkg/src")
sys.path.insert(0, REPO)
sys.path.insert(0, REF)
sys.path.insert(0, HERE)

from gen_vm_golden import _execute, _input_json  # noqa: E402
from paper_1810_08061_b200 import ir  # noqa: E402

PROGS = os.path.join(HERE, "programs", "recursion")


def random_tree_text(n_nodes, rng):
    """A random binary tree of n_nodes values in the reference's feed syntax
    (feeds.py parse_tree: `(value left right)`, `()` = empty)."""
    if n_nodes == 0:
        return "()"
    left = rng.randint(0, n_nodes - 1)
    v = round(rng.uniform(-2.0, 2.0), 3)
    return f"({v} {random_tree_text(left, rng)} {random_tree_text(n_nodes - 1 - left, rng)})"


def cases():
    rng = random.Random(2024)
    small = "(5.0 (3.0 () ()) (2.0 () ()))"
    t31 = random_tree_text(31, rng)
    t200 = random_tree_text(200, rng)
    tree = lambda s: {"dtype": "tree", "data": s}  # noqa: E731
    i64 = lambda v: {"dtype": "i64", "shape": [], "data": [v]}  # noqa: E731
    f64 = lambda v: {"dtype": "f64", "shape": [], "data": [v]}  # noqa: E731
    return [
        ("fib_10", "fib.msl", "main", [("n", f64(10.0))]),
        ("fib_1", "fib.msl", "main", [("n", f64(1.0))]),
        ("tree_sum_small", "tree_sum.msl", "main", [("t", tree(small))]),
        ("tree_sum_31", "tree_sum.msl", "main", [("t", tree(t31))]),
        ("tree_sum_200", "tree_sum.msl", "main", [("t", tree(t200))]),
        ("tree_sum_empty", "tree_sum.msl", "main", [("t", tree("()"))]),
        ("tree_depth_200", "tree_depth.msl", "main", [("t", tree(t200))]),
        ("even_odd_7", "even_odd.msl", "main", [("n", f64(7.0))]),
        ("even_odd_20", "even_odd.msl", "main", [("n", f64(20.0))]),
        ("tree_print_31", "tree_print.msl", "main", [("t", tree(t31))]),
        ("tree_loop_31", "tree_loop.msl", "main", [("t", tree(t31)), ("x", f64(0.75))]),
        ("fact_12", "fact_assert.msl", "main", [("n", f64(12.0))]),
        ("fact_negative", "fact_assert.msl", "main", [("n", f64(-3.0))]),
        ("tree_prod_31", os.path.join("..", "..", "..", "..", "reference", "pkg", "corpus", "tree_prod.msl"),
         "tree_prod", [("base", f64(1.01)), ("tree", tree(t31))]),
    ]


def main():
    from stagekit.feeds import parse_tree
    from stagekit.graph.tensor import TensorValue
    from stagekit.runtime import ParamSpec, trace_module
    from stagekit.syntax import parse_module
    from stagekit.transforms import PassConfig
    docs = []
    for name, fname, entry, params in cases():
        path = os.path.join(PROGS, fname) if not fname.startswith("..") else \
            os.path.join(os.path.dirname(REF), "corpus", os.path.basename(fname))
        src = open(path).read()
        module = parse_module(src, os.path.basename(path))
        config = PassConfig(backend="sexpr")
        specs, feeds = [], {}
        for pname, p in params:
            if p["dtype"] == "tree":
                specs.append(ParamSpec(pname, "tree"))
                feeds[pname] = parse_tree(p["data"])
            else:
                specs.append(ParamSpec(pname, p["dtype"], tuple(p["shape"])))
                feeds[pname] = TensorValue(p["dtype"], tuple(p["shape"]), tuple(p["data"]))
        try:
            outcome = trace_module(module, entry, specs, config)
        except Exception as exc:   # the reference cannot stage this program: not a test case
            print(name, "TRACE FAILS:", type(exc).__name__, str(exc)[:100])
            continue
        g = outcome.graph
        assert g.functions, f"{name}: the sexpr backend staged no FuncCall"
        docs.append({"name": name, "program": os.path.basename(path), "backend": "sexpr",
                     "graph": json.loads(ir.to_json(g)),
                     "feeds": {k: _input_json(v) for k, v in feeds.items()},
                     "expected": _execute(g, feeds)})
        print(name, docs[-1]["expected"] if "error" in docs[-1]["expected"] else
              str(docs[-1]["expected"]["outputs"])[:80])
    with open(os.path.join(REPO, "tests", "golden", "vm_recursion.json"), "w") as f:
        json.dump({"generator": "oracle/gen_recursion_golden.py", "programs": docs}, f, separators=(",", ":"))


if __name__ == "__main__":
    main()

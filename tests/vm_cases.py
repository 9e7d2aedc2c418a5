"""Loaders for the region-VM golden fixtures (tests/golden/vm_*.json)."""
import json
import os

import numpy as np

from paper_1810_08061_b200 import ir
from paper_1810_08061_b200.values import ListValue, TensorValue, Tree

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def parse_tree(text):
    toks = text.replace("(", " ( ").replace(")", " ) ").split()
    pos = 0

    def node():
        nonlocal pos
        assert toks[pos] == "("
        pos += 1
        if toks[pos] == ")":
            pos += 1
            return Tree()
        v = float(toks[pos])
        pos += 1
        left = node()
        right = node()
        assert toks[pos] == ")"
        pos += 1
        return Tree(v, left, right)
    return node()


def feed_value(d):
    if "tree" in d:
        return parse_tree(d["tree"])
    t = d["tensor"]
    return TensorValue(t["dtype"], tuple(t["shape"]), np.asarray(t["data"]))


def corpus():
    with open(os.path.join(GOLDEN, "vm_corpus.json")) as f:
        return json.load(f)["programs"]


def fuzz_cases():
    with open(os.path.join(GOLDEN, "vm_fuzz.json")) as f:
        seeds = json.load(f)["seeds"]
    out = []
    for s in seeds:
        for c in s["cases"]:
            if "graph" in c:
                out.append((f"seed{s['seed']}-v{c['vector']}-{c['mode']}", c))
    return out


def flatten(values):
    out = []
    for v in values:
        if isinstance(v, ListValue):
            out.extend(flatten(v.items))
        else:
            out.append(v)
    return out


def leaf_equal(got, exp, rel=1e-9):
    """The reference harness comparison (harness/diff.py:86-105)."""
    if "repr" in exp:
        return False
    t = exp["tensor"]
    a = np.asarray(got.array if hasattr(got, "array") else got)
    b = np.asarray(t["data"]).reshape(t["shape"])
    if got.dtype != t["dtype"] or tuple(a.shape) != tuple(b.shape):
        return False
    if t["dtype"] != "f64":
        return bool(np.array_equal(a.astype(np.int64), b.astype(np.int64)))
    a = a.astype(np.float64)
    b = b.astype(np.float64)
    nan = np.isnan(a) & np.isnan(b)
    inf = np.isinf(a) | np.isinf(b)
    if np.any(inf & ~nan & (a != b)):
        return False
    fin = ~nan & ~inf
    return bool(np.all(np.abs(a[fin] - b[fin]) <= rel * np.maximum(1.0, np.maximum(np.abs(a[fin]), np.abs(b[fin])))))


def recursion():
    """Recursive FuncCall programs (oracle/gen_recursion_golden.py)."""
    with open(os.path.join(GOLDEN, "vm_recursion.json")) as f:
        return json.load(f)["programs"]

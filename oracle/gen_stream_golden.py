"""Golden fixtures for the vector-stream tier (TEST INFRASTRUCTURE; run in the
build container, where the reference is importable).

For every case of ``fixtures.STREAM_CASES`` the program under
oracle/programs/ is traced with the reference's ``trace_module``
(runtime/__init__.py:49-76) and executed with the reference's ``execute``
(graph/execute.py:27-36) on ``fixtures.make_stream_feeds``; the traced graph
(skb wire format), the feed spec and the reference's flattened outputs (or its
failure cause_kind and span) go to tests/golden/<case>.json.

Usage: python oracle/gen_stream_golden.py [case ...]
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
REF = os.environ.get("SKB_REF", "/root/reference/pkg/src")
sys.path.insert(0, REPO)
sys.path.insert(0, REF)

from oracle import fixtures  # noqa: E402
from oracle.gen_vm_golden import _flatten, _leaf_json  # noqa: E402
from paper_1810_08061_b200 import ir  # noqa: E402


def _ref_value(a):
    from stagekit.graph import TensorValue
    a = np.asarray(a)
    if a.dtype == np.int64:
        return TensorValue("i64", a.shape, tuple(int(v) for v in a.reshape(-1)))
    return TensorValue("f64", a.shape, tuple(float(v) for v in a.reshape(-1)))


def trace(case):
    from stagekit.runtime import ParamSpec, trace_module
    from stagekit.syntax import parse_module
    path = os.path.join(fixtures.PROGRAMS, case["program"])
    module = parse_module(open(path).read(), case["program"])
    feeds = fixtures.make_stream_feeds(case)
    specs = [ParamSpec(k, "i64" if v.dtype == np.int64 else "f64", tuple(v.shape)) for k, v in feeds.items()]
    return trace_module(module, case["entry"], specs).graph


def run_case(case):
    from stagekit.errors import RuntimeGraphError
    from stagekit.graph import execute
    graph = trace(case)
    feeds = {k: _ref_value(v) for k, v in fixtures.make_stream_feeds(case).items()}
    doc = {"case": case, "generator": "oracle/gen_stream_golden.py", "graph": json.loads(ir.to_json(graph))}
    t0 = time.time()
    try:
        res = execute(graph, feeds)
        flat = []
        for v in res.outputs:
            flat.extend(_flatten(v))
        doc["expected"] = {"outputs": [_leaf_json(v) for v in flat], "print_log": list(res.print_log)}
    except RuntimeGraphError as exc:
        doc["expected"] = {"error": exc.cause_kind,
                           "span": [exc.span.file, exc.span.start_line, exc.span.start_col] if exc.span else None}
    doc["reference_seconds"] = round(time.time() - t0, 3)
    return doc


def write_c4_graph():
    """tests/golden/graph_lbfgs_c4.json: the C4 program (m=10) traced with a
    dynamic vector length (f64[?]) so one graph serves every n."""
    from stagekit.runtime import ParamSpec, trace_module
    from stagekit.syntax import parse_module
    path = os.path.join(fixtures.PROGRAMS, "lbfgs_m10.msl")
    module = parse_module(open(path).read(), "lbfgs_m10.msl")
    specs = [ParamSpec("x0", "f64", (None,)), ParamSpec("a", "f64", (None,)), ParamSpec("b", "f64", (None,)),
             ParamSpec("tol", "f64", ()), ParamSpec("max_iter", "i64", ())]
    graph = trace_module(module, "lbfgs", specs).graph
    doc = {"case": {"name": "graph_lbfgs_c4", "program": "lbfgs_m10.msl", "entry": "lbfgs", "m": 10,
                    "note": "BASELINE config C4: L-BFGS, history m=10, vector length bound at execution"},
           "generator": "oracle/gen_stream_golden.py --graphs", "graph": json.loads(ir.to_json(graph))}
    with open(os.path.join(fixtures.GOLDEN, "graph_lbfgs_c4.json"), "w") as f:
        json.dump(doc, f, separators=(",", ":"))
    print("graph_lbfgs_c4 graph only")


MICRO = {"micro_dot": ["x", "y"], "micro_axpy": ["x", "y"], "micro_copy": ["x"]}


def write_micro_graphs():
    """tests/golden/graph_micro_*.json: one-group loops (dot, axpy, scale) with a
    dynamic vector length, for the stream-tier bandwidth probes (tools/stream_micro.py)."""
    from stagekit.runtime import ParamSpec, trace_module
    from stagekit.syntax import parse_module
    for name, vecs in MICRO.items():
        path = os.path.join(fixtures.PROGRAMS, name + ".msl")
        module = parse_module(open(path).read(), name + ".msl")
        specs = [ParamSpec(v, "f64", (None,)) for v in vecs] + [ParamSpec("iters", "i64", ())]
        graph = trace_module(module, name, specs).graph
        doc = {"case": {"name": "graph_" + name, "program": name + ".msl", "entry": name},
               "generator": "oracle/gen_stream_golden.py --graphs", "graph": json.loads(ir.to_json(graph))}
        with open(os.path.join(fixtures.GOLDEN, f"graph_{name}.json"), "w") as f:
            json.dump(doc, f, separators=(",", ":"))
        print("graph_" + name)


def main(argv):
    if argv and argv[0] == "--graphs":
        write_c4_graph()
        write_micro_graphs()
        return
    names = argv or [c["name"] for c in fixtures.STREAM_CASES]
    for name in names:
        doc = run_case(fixtures.stream_case_by_name(name))
        with open(fixtures.golden_path(name), "w") as f:
            json.dump(doc, f, separators=(",", ":"))
        exp = doc["expected"]
        what = exp.get("error") or [tuple(o["tensor"]["shape"]) for o in exp["outputs"]]
        print(f"{name:24s} {what} ({doc['reference_seconds']} s in the reference executor)")


if __name__ == "__main__" and sys.argv[1:2] not in (["--greedy"], ["--tree"], ["--bptt"], ["--maml"]):
    main(sys.argv[1:])


def greedy_goldens():
    """tests/golden/greedy_*.json: SURVEY App. F greedy decoder traced and run by
    the reference (EOS `break` lowered into the While test)."""
    from stagekit.runtime import ParamSpec, trace_module
    from stagekit.syntax import parse_module
    from stagekit.graph import execute
    path = os.path.join(fixtures.PROGRAMS, "greedy.msl")
    for case in fixtures.GREEDY_CASES:
        feeds = fixtures.make_greedy_feeds(case)
        module = parse_module(open(path).read(), "greedy.msl")
        specs = [ParamSpec(k, "i64" if v.dtype == np.int64 else "f64", tuple(v.shape)) for k, v in feeds.items()]
        graph = trace_module(module, "greedy", specs).graph
        ref = {k: _ref_value(v) for k, v in feeds.items()}
        if case["eos"] == -1:   # pick the first token the decoder emits twice -> a stop inside max_len
            probe = dict(ref, eos=_ref_value(np.asarray(-7, dtype=np.int64)))
            toks = list(execute(graph, probe).outputs[0].data)
            seen = set()
            for t in toks[1:]:
                if t in seen:
                    case = dict(case, eos=int(t))
                    break
                seen.add(t)
            ref["eos"] = _ref_value(np.asarray(case["eos"], dtype=np.int64))
        res = execute(graph, ref)
        flat = []
        for v in res.outputs:
            flat.extend(_flatten(v))
        doc = {"case": case, "generator": "oracle/gen_stream_golden.py --greedy",
               "graph": json.loads(ir.to_json(graph)),
               "expected": {"outputs": [_leaf_json(v) for v in flat], "print_log": list(res.print_log)}}
        with open(fixtures.golden_path(case["name"]), "w") as f:
            json.dump(doc, f, separators=(",", ":"))
        print(case["name"], "eos", case["eos"], "tokens", doc["expected"]["outputs"][0]["tensor"]["data"][:12],
              "t", doc["expected"]["outputs"][1]["tensor"]["data"])


if __name__ == "__main__" and sys.argv[1:2] == ["--greedy"]:
    greedy_goldens()


def tree_goldens():
    """tests/golden/treelstm_*.json: the TreeLSTM program (oracle/programs/
    tree_lstm.msl) run natively by the reference's
    interpret_module (runtime/__init__.py:41-46) on random binary trees, plus the
    graph of the first tree traced with a concrete Tree (unrolled, Cond-free)."""
    from stagekit.graph.tensor import Tree
    from stagekit.runtime import ParamSpec, interpret_module, trace_module
    from stagekit.syntax import parse_module
    path = os.path.join(fixtures.PROGRAMS, "tree_lstm.msl")
    src = open(path).read()
    for case in fixtures.TREE_CASES:
        module = parse_module(src, "tree_lstm.msl")
        H = case["H"]
        w = fixtures.tree_weights(H, case["seed"])
        rng = np.random.default_rng(case["seed"] + 1000)
        trees, outs = [], []

        def to_tree(val, left, right, i=0):
            if i < 0:
                return Tree()
            return Tree(float(val[i]), to_tree(val, left, right, left[i]), to_tree(val, left, right, right[i]))
        for n in case["leaves"]:
            val, left, right = fixtures.random_tree_arrays(n, rng)
            trees.append(fixtures.tree_str(val, left, right))
            res, _ = interpret_module(module, "tree_lstm", [to_tree(val, left, right)] +
                                      [_ref_value(w[k]) for k in fixtures.TREE_WEIGHTS])
            outs.append([list(res.items[0].data), list(res.items[1].data)])
        doc = {"case": case, "generator": "oracle/gen_stream_golden.py --tree", "trees": trees, "expected": outs}
        with open(fixtures.golden_path(case["name"]), "w") as f:
            json.dump(doc, f, separators=(",", ":"))
        print(case["name"], len(trees), "trees; root h[0] =", [o[0][0] for o in outs])


if __name__ == "__main__" and sys.argv[1:2] == ["--tree"]:
    tree_goldens()


BPTT_CASES = [
    {"name": "lstm_bptt_4x3", "T": 4, "B": 3, "F": 3, "H": 4, "lens": [4, 2, 1], "seed": 71},
    {"name": "lstm_bptt_6x4", "T": 6, "B": 4, "F": 5, "H": 6, "lens": [6, 0, 3, 5], "seed": 72,
     "note": "a zero-length row, len < T rows frozen"},
]


def bptt_feeds(case):
    rng = np.random.default_rng(case["seed"])
    T, B, F, H = case["T"], case["B"], case["F"], case["H"]
    v = {"x": rng.uniform(-1, 1, (T, B, F)), "h0": rng.uniform(-.5, .5, (B, H)), "c0": rng.uniform(-.5, .5, (B, H)),
         "lens": np.asarray(case["lens"], dtype=np.int64), "y": rng.uniform(-1, 1, (T, B, H))}
    for g in "ifgo":
        v["w" + g] = rng.uniform(-1, 1, (F, H))
        v["u" + g] = rng.uniform(-1, 1, (H, H))
        v["b" + g] = np.broadcast_to(rng.uniform(-.5, .5, (1, H)), (B, H)).copy()
    v["inv_b"] = np.float64(1.0 / B)
    return v


def bptt_goldens():
    """tests/golden/lstm_bptt_*.json: the hand-derived staged BPTT program
    (oracle/programs/lstm_bptt.msl) traced and executed by the reference."""
    from stagekit.graph import execute
    from stagekit.runtime import ParamSpec, trace_module
    from stagekit.syntax import parse_module
    path = os.path.join(fixtures.PROGRAMS, "lstm_bptt.msl")
    names = ["x", "h0", "c0", "lens", "y"] + [f"{k}{g}" for g in "ifgo" for k in "wub"] + ["inv_b"]
    for case in BPTT_CASES:
        v = bptt_feeds(case)
        module = parse_module(open(path).read(), "lstm_bptt.msl")
        specs = [ParamSpec(k, "i64" if np.asarray(v[k]).dtype == np.int64 else "f64", tuple(np.asarray(v[k]).shape))
                 for k in names]
        graph = trace_module(module, "lstm_bptt", specs).graph
        res = execute(graph, {k: _ref_value(v[k]) for k in names})
        doc = {"case": case, "generator": "oracle/gen_stream_golden.py --bptt",
               "outputs": [{"shape": list(o.shape), "data": list(o.data)} for o in res.outputs]}
        with open(fixtures.golden_path(case["name"]), "w") as f:
            json.dump(doc, f, separators=(",", ":"))
        print(case["name"], "loss", res.outputs[0].data)


if __name__ == "__main__" and sys.argv[1:2] == ["--bptt"]:
    bptt_goldens()


MAML_CASES = [{"name": "maml_h8_k5", "H": 8, "K": 5, "tasks": 3, "seed": 81, "alpha": 0.01},
              {"name": "maml_h40_k10", "H": 40, "K": 10, "tasks": 2, "seed": 82, "alpha": 0.01}]


def maml_goldens():
    """tests/golden/maml_*.json: per-task query loss and second-order
    meta-gradient from the reference's gradient() (graph/grad.py:35-70) over
    the staged one-task MAML program (oracle/programs/maml.msl)."""
    from oracle import maml as omaml
    from stagekit.graph import execute
    from stagekit.graph.grad import gradient
    from stagekit.runtime import ParamSpec, trace_module
    from stagekit.syntax import parse_module
    path = os.path.join(fixtures.PROGRAMS, "maml.msl")
    for case in MAML_CASES:
        H, K = case["H"], case["K"]
        th = omaml.init_theta(H, case["seed"])
        xs, ys, xq, yq = omaml.sinusoid_tasks(case["tasks"], K, case["seed"] + 1)
        module = parse_module(open(path).read(), "maml.msl")
        names = list(omaml.NAMES) + ["xs", "ys", "xq", "yq", "ones", "alpha", "inv_k"]
        shapes = {k: th[k].shape for k in omaml.NAMES}
        shapes.update(xs=(K, 1), ys=(K, 1), xq=(K, 1), yq=(K, 1), ones=(K, 1), alpha=(), inv_k=())
        graph = gradient(trace_module(module, "maml_task", [ParamSpec(k, "f64", shapes[k]) for k in names]).graph,
                         0, list(omaml.NAMES))
        outs = []
        for t in range(case["tasks"]):
            feeds = {k: _ref_value(th[k]) for k in omaml.NAMES}
            feeds.update(xs=_ref_value(xs[t]), ys=_ref_value(ys[t]), xq=_ref_value(xq[t]), yq=_ref_value(yq[t]),
                         ones=_ref_value(np.ones((K, 1))), alpha=_ref_value(np.float64(case["alpha"])),
                         inv_k=_ref_value(np.float64(1.0 / K)))
            res = execute(graph, feeds)
            outs.append([list(o.data) for o in res.outputs])
        doc = {"case": case, "generator": "oracle/gen_stream_golden.py --maml", "outputs": outs}
        with open(fixtures.golden_path(case["name"]), "w") as f:
            json.dump(doc, f, separators=(",", ":"))
        print(case["name"], "losses", [o[0][0] for o in outs])


if __name__ == "__main__" and sys.argv[1:2] == ["--maml"]:
    maml_goldens()

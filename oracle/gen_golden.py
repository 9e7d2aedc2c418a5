"""Generate tests/golden/*.json from the reference itself (TEST INFRASTRUCTURE).

Run in the build container, where the reference is importable:

    python oracle/gen_golden.py            # all cases in oracle/fixtures.CASES
    python oracle/gen_golden.py lstm_4x8x8 # selected cases

For every case it (1) traces the program with the reference's
``trace_module`` (reference pkg/src/stagekit/runtime/__init__.py:49-76),
(2) executes the traced graph with the reference's ``execute``
(graph/execute.py:27-36) on the deterministic feeds of
``fixtures.make_feeds``, and (3) stores the traced graph in the skb wire
format together with the reference outputs — or the reference's failure
``cause_kind`` and span.  The GPU box has no copy of the reference; the tests
replay these fixtures.
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
from paper_1810_08061_b200 import ir  # noqa: E402


def _ref_tensor(arr):
    from stagekit.graph import TensorValue
    arr = np.asarray(arr)
    if arr.dtype == np.int64:
        return TensorValue("i64", arr.shape, tuple(int(v) for v in arr.reshape(-1)))
    return TensorValue("f64", arr.shape, tuple(float(v) for v in arr.reshape(-1)))


def trace(case):
    from stagekit.runtime import ParamSpec, trace_module
    from stagekit.syntax import parse_module
    d = case["dims"]
    B, T, F, H = d["B"], d["T"], d["F"], d["H"]
    prog = case["program"]
    if prog == "handwritten":
        sys.path.insert(0, os.path.join(os.path.dirname(REF), "tests"))
        from helpers import handwritten_dynamic_rnn
        return handwritten_dynamic_rnn(B, T, F, H), "reference pkg/tests/helpers.py:40-80"
    if prog.startswith("corpus:"):
        path = os.path.join(os.path.dirname(REF), "corpus", prog.split(":", 1)[1])
    else:
        path = os.path.join(fixtures.PROGRAMS, prog)
    src = open(path).read()
    module = parse_module(src, os.path.basename(path))
    feeds = fixtures.make_feeds(case)
    specs = []
    for name in fixtures.param_names(case):
        a = feeds[name]
        specs.append(ParamSpec(name, "i64" if a.dtype == np.int64 else "f64", tuple(a.shape)))
    outcome = trace_module(module, case["entry"], specs)
    return outcome.graph, os.path.relpath(path, REPO) if path.startswith(REPO) else path


def run_case(case):
    from stagekit.errors import RuntimeGraphError
    from stagekit.graph import execute
    graph, source = trace(case)
    feeds = fixtures.make_feeds(case)
    ref_feeds = {k: _ref_tensor(v) for k, v in feeds.items()}
    t0 = time.time()
    doc = {"case": case, "source": source, "generator": "oracle/gen_golden.py",
           "graph": json.loads(ir.to_json(graph))}
    try:
        res = execute(graph, ref_feeds)
        doc["expected"] = {"outputs": [ir.tensor_to_json(v) for v in res.outputs],
                           "print_log": list(res.print_log)}
    except RuntimeGraphError as exc:
        span = exc.span
        doc["expected"] = {"error": exc.cause_kind, "message": exc.message,
                           "span": [span.file, span.start_line, span.start_col] if span else None}
    doc["reference_seconds"] = round(time.time() - t0, 3)
    return doc


# Graph-only fixtures: the traced program at benchmark sizes (the reference
# executor would need minutes per batch there; parity at those sizes is
# checked against the float64 oracle instead).
GRAPHS = {
    "graph_lstm_c1": fixtures.lstm_case("graph_lstm_c1", 32, 64, 256, 256, "random", 0,
                                        note="BASELINE config C1: hidden 256, batch 32, max_len 64"),
}


def write_graph_fixture(name):
    case = GRAPHS[name]
    graph, source = trace(case)
    doc = {"case": case, "source": source, "generator": "oracle/gen_golden.py",
           "graph": json.loads(ir.to_json(graph))}
    with open(os.path.join(fixtures.GOLDEN, f"{name}.json"), "w") as f:
        json.dump(doc, f, separators=(",", ":"))
    print(f"{name:28s} graph only ({graph.node_count()} nodes)")


def main(argv):
    if argv and argv[0] == "--graphs":
        for name in GRAPHS:
            write_graph_fixture(name)
        return
    names = argv or [c["name"] for c in fixtures.CASES]
    os.makedirs(fixtures.GOLDEN, exist_ok=True)
    for name in names:
        case = fixtures.case_by_name(name)
        doc = run_case(case)
        with open(fixtures.golden_path(name), "w") as f:
            json.dump(doc, f, separators=(",", ":"))
        exp = doc["expected"]
        what = exp.get("error") or [tuple(o["shape"]) for o in exp["outputs"]]
        print(f"{name:28s} {what} ({doc['reference_seconds']} s in the reference executor)")


if __name__ == "__main__":
    main(sys.argv[1:])

"""Golden fixtures for the region VM, produced by the reference itself
(TEST INFRASTRUCTURE; run in the build container where the reference lives).

* tests/golden/vm_corpus.json — the reference's corpus (pkg/corpus/*.msl) with
  the manifest's own feeds (harness/diff.py:267-286 `_manifest_value`), traced
  with `trace_module` and executed with the reference `execute`.
* tests/golden/vm_fuzz.json — the reference's differential fuzz programs
  (harness/fuzz.py:366-381 `gen_program_with_params`, `gen_inputs`): for each
  seed the staged-parameter graph with 3 input vectors and the concrete-mode
  graph of vector 0, exactly as `diff_one` stages them (harness/diff.py:144-164),
  with the reference's outputs, print logs or failure kinds.

Usage: python oracle/gen_vm_golden.py [n_seeds]
"""

from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
REF = os.environ.get("SKB_REF", "/root/reference/pkg/src")
sys.path.insert(0, REPO)
sys.path.insert(0, REF)

from paper_1810_08061_b200 import ir  # noqa: E402


def _leaf_json(v):
    from stagekit.graph.tensor import TensorValue
    if isinstance(v, TensorValue):
        return {"tensor": ir.tensor_to_json(v)}
    if isinstance(v, bool):
        return {"tensor": {"dtype": "bool", "shape": [], "data": [v]}}
    if isinstance(v, int):
        return {"tensor": {"dtype": "i64", "shape": [], "data": [v]}}
    if isinstance(v, float):
        return {"tensor": {"dtype": "f64", "shape": [], "data": [v]}}
    return {"repr": str(v)}


def _flatten(value):
    from stagekit.graph.tensor import ListValue
    from stagekit.runtime import MslList
    if value is None:
        return []
    if isinstance(value, (ListValue, MslList)):
        out = []
        for item in value.items:
            out.extend(_flatten(item))
        return out
    return [value]


def _input_json(v):
    from stagekit.graph.tensor import Tree
    if isinstance(v, Tree):
        return {"tree": str(v)}
    return _leaf_json(v)


def _execute(graph, feeds):
    from stagekit.errors import RuntimeGraphError, StagekitError
    from stagekit.graph import execute
    try:
        res = execute(graph, feeds)
        flat = []
        for v in res.outputs:
            flat.extend(_flatten(v))
        return {"outputs": [_leaf_json(v) for v in flat], "print_log": list(res.print_log)}
    except RuntimeGraphError as exc:
        return {"error": exc.cause_kind, "span": [exc.span.file, exc.span.start_line] if exc.span else None}
    except StagekitError as exc:
        return {"error": type(exc).__name__, "span": None}


def corpus():
    from stagekit.harness.diff import _manifest_value
    from stagekit.runtime import ParamSpec, trace_module
    from stagekit.syntax import parse_module
    from stagekit.transforms import PassConfig
    cdir = os.path.join(os.path.dirname(REF), "corpus")
    manifest = json.load(open(os.path.join(cdir, "manifest.json")))
    docs = []
    for prog in manifest["programs"]:
        src = open(os.path.join(cdir, prog["file"])).read()
        module = parse_module(src, prog["file"])
        config = PassConfig(backend=prog.get("backend", "graph"))
        params = [ParamSpec(p["name"], p["dtype"], tuple(p.get("shape", ()))) for p in prog["params"]]
        feeds = {p["name"]: _manifest_value(p) for p in prog["params"]}
        outcome = trace_module(module, prog["entry"], params, config)
        docs.append({"name": prog["name"], "backend": config.backend,
                     "graph": json.loads(ir.to_json(outcome.graph)),
                     "feeds": {k: _input_json(v) for k, v in feeds.items()},
                     "expected": _execute(outcome.graph, feeds)})
        print(prog["name"], list(docs[-1]["expected"].keys()))
    return docs


def fuzz(n):
    from stagekit.errors import StagekitError
    from stagekit.harness.diff import _spec_for
    from stagekit.harness.fuzz import FuzzSpec, gen_inputs, gen_program_with_params
    from stagekit.runtime import trace_module
    from stagekit.syntax import parse_module
    from stagekit.transforms import PassConfig, convert
    docs = []
    for seed in range(n):
        spec = FuzzSpec(seed=seed)
        source, kinds = gen_program_with_params(spec)
        try:
            module = parse_module(source, "<fuzz>")
            converted = convert(module, PassConfig())
        except StagekitError:
            continue
        entry = {"seed": seed, "cases": []}
        for vector in range(3):
            inputs = gen_inputs(kinds, seed * 1000 + vector)
            for mode in ("staged_params", "concrete"):
                if mode == "concrete" and vector > 0:
                    continue
                try:
                    if mode == "staged_params":
                        params = [_spec_for(f"p{i}", v) for i, v in enumerate(inputs)]
                        outcome = trace_module(module, "main", params, PassConfig(), pre_converted=converted)
                        feeds = {f"p{i}": v for i, v in enumerate(inputs)}
                    else:
                        outcome = trace_module(module, "main", config=PassConfig(), pre_converted=converted,
                                               args=inputs)
                        feeds = {}
                except StagekitError as exc:
                    entry["cases"].append({"vector": vector, "mode": mode, "trace_error": type(exc).__name__})
                    continue
                entry["cases"].append({
                    "vector": vector, "mode": mode,
                    "graph": json.loads(ir.to_json(outcome.graph)),
                    "feeds": {k: _input_json(v) for k, v in feeds.items()},
                    "expected": _execute(outcome.graph, feeds)})
        docs.append(entry)
    return docs


def main(argv):
    n = int(argv[0]) if argv else 120
    out = os.path.join(REPO, "tests", "golden")
    with open(os.path.join(out, "vm_corpus.json"), "w") as f:
        json.dump({"generator": "oracle/gen_vm_golden.py", "programs": corpus()}, f, separators=(",", ":"))
    docs = fuzz(n)
    with open(os.path.join(out, "vm_fuzz.json"), "w") as f:
        json.dump({"generator": "oracle/gen_vm_golden.py", "seeds": docs}, f, separators=(",", ":"))
    ncase = sum(len(d["cases"]) for d in docs)
    nerr = sum(1 for d in docs for c in d["cases"] if "error" in c.get("expected", {}))
    print(f"fuzz: {len(docs)} seeds, {ncase} cases ({nerr} reference failures)")


if __name__ == "__main__":
    main(sys.argv[1:])

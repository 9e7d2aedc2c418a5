"""Live reference graphs straight into skb (no JSON round trip): the corpus
programs are traced by the reference's own `trace_module` in this process and
the resulting `stagekit.graph.ir.Graph` objects go through skb's `validate`,
plan selection and region-VM compiler; the stagekit binding converts skb
values into the reference's classes.  Skipped where the reference package is
not importable (the GPU box runs the replayed fixtures instead)."""

import json
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for cand in (os.environ.get("SKB_REF"), "/root/reference/pkg/src", os.path.join(REPO, "baseline", "_ref")):
    if cand and os.path.isdir(os.path.join(cand, "stagekit")):
        sys.path.insert(0, cand)
        CORPUS = os.path.join(os.path.dirname(cand), "corpus") if cand.endswith("src") else os.path.join(cand, "corpus")
        break
else:
    CORPUS = None
stagekit = pytest.importorskip("stagekit")

from paper_1810_08061_b200 import stagekit_binding, vm  # noqa: E402
from paper_1810_08061_b200.executor import plan_kind  # noqa: E402
from paper_1810_08061_b200.validate import validate  # noqa: E402
from paper_1810_08061_b200.values import DeviceTensor, ListValue, Tree  # noqa: E402


def _traced():
    from stagekit.harness.diff import _manifest_value
    from stagekit.runtime import ParamSpec, trace_module
    from stagekit.syntax import parse_module
    from stagekit.transforms import PassConfig
    manifest = json.load(open(os.path.join(CORPUS, "manifest.json")))
    out = []
    for prog in manifest["programs"]:
        module = parse_module(open(os.path.join(CORPUS, prog["file"])).read(), prog["file"])
        params = [ParamSpec(p["name"], p["dtype"], tuple(p.get("shape", ()))) for p in prog["params"]]
        feeds = {p["name"]: _manifest_value(p) for p in prog["params"]}
        g = trace_module(module, prog["entry"], params, PassConfig(backend=prog.get("backend", "graph"))).graph
        out.append((prog["name"], g, feeds))
    return out


@pytest.mark.skipif(CORPUS is None or not os.path.isdir(CORPUS or ""), reason="reference corpus not present")
def test_live_corpus_graphs_validate_plan_and_compile():
    from stagekit.graph.validate import validate as ref_validate
    for name, g, feeds in _traced():
        assert validate(g) == [] and ref_validate(g, raise_on_error=False) == [], name
        kind = plan_kind(g, feeds)
        assert kind == ("rnn" if name == "dynamic_rnn" else "vm"), (name, kind)
        p = vm.compile_graph(g)
        assert len(p.outputs) == len(g.main.outputs)
        if name == "tree_prod":
            assert vm.OP["CALL"] in [c[0] for c in p.code]


@pytest.mark.skipif(CORPUS is None or not os.path.isdir(CORPUS or ""), reason="reference corpus not present")
def test_live_broken_graph_rejected_like_the_reference():
    from stagekit.graph.validate import validate as ref_validate
    for name, g, _ in _traced():
        loops = [n for n in g.main.nodes if n.op == "While"]
        if not loops:
            continue
        loops[0].inputs = loops[0].inputs[:-1]   # drop a capture
        assert validate(g, raise_on_error=False) and ref_validate(g, raise_on_error=False), name


def test_binding_converts_values_to_reference_classes():
    import torch
    from stagekit.graph.tensor import ListValue as RefList, TensorValue as RefTV, Tree as RefTree
    sk_tensor = __import__("stagekit.graph.tensor", fromlist=["x"])
    t = stagekit_binding._to_reference(DeviceTensor("f64", torch.arange(6, dtype=torch.float64).reshape(2, 3)),
                                       sk_tensor)
    assert isinstance(t, RefTV) and t.shape == (2, 3) and t.data == (0.0, 1.0, 2.0, 3.0, 4.0, 5.0)
    b = stagekit_binding._to_reference(DeviceTensor("bool", torch.tensor([True, False])), sk_tensor)
    assert b.data == (True, False) and all(type(v) is bool for v in b.data)
    i = stagekit_binding._to_reference(DeviceTensor("i64", torch.tensor(7)), sk_tensor)
    assert i.item() == 7 and type(i.item()) is int
    lst = stagekit_binding._to_reference(ListValue([DeviceTensor("i64", torch.tensor([1, 2]))]), sk_tensor)
    assert isinstance(lst, RefList) and lst.items[0].data == (1, 2)
    tr = stagekit_binding._to_reference(Tree(2.0, Tree(), Tree(1.0, Tree(), Tree())), sk_tensor)
    assert isinstance(tr, RefTree) and str(tr) == "(2.0 () (1.0 () ()))"
    assert np.isclose(tr.right.value, 1.0)

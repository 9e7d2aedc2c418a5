"""Automatic differentiation through While (paper_1810_08061_b200.autodiff),
CPU side: graph structure, error behaviour, the fixtures' own consistency and
— where the reference is importable (the build container only) — the
reference executor running the generated gradient graphs.  Numerical parity
of the graphs on the B200 is tests/test_gpu_autodiff.py."""
import importlib.util
import json
import os

import numpy as np
import pytest

from autodiff_cases import NAMES, close, load
from paper_1810_08061_b200 import ir
from paper_1810_08061_b200.autodiff import NotDifferentiable, gradient

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.mark.parametrize("name", NAMES)
def test_gradient_graph_structure(name):
    d = load(name)
    g = d["graph_obj"]
    gg = gradient(g, d["output"], d["wrt"])
    assert len(gg.main.outputs) == len(g.main.outputs) + len(d["wrt"])
    assert [p.attrs["name"] for p in gg.main.params] == [p.attrs["name"] for p in g.main.params]
    n_while = g.count_ops("While")
    # one taping forward loop and one reverse loop per While; no FuncCall left (inlined)
    assert gg.count_ops("While") == 2 * n_while
    assert gg.count_ops("FuncCall") == 0
    for k, name_ in enumerate(d["wrt"]):
        spec = next(p for p in g.main.params if p.attrs["name"] == name_).out_types[0]
        assert gg.main.outputs[len(g.main.outputs) + k].type.dtype == "f64"
        assert gg.main.outputs[len(g.main.outputs) + k].type.shape in (spec.shape, None)
    # the transform does not touch its input
    assert len(g.main.outputs) == len(json.loads(ir.to_json(g))["main"]["outputs"])


@pytest.mark.parametrize("name", NAMES)
def test_fixture_autodiff_matches_independent_source(name):
    """recorded at generation: the reference executor running our gradient
    graph agrees with the hand BPTT / reference gradient() / finite differences"""
    d = load(name)
    tol = d.get("expected_tol", 1e-12)
    nw = len(d["wrt"])
    assert len(d["expected"]) == nw + 1
    for a, b in zip(d["via_reference"][-nw:], d["expected"][1:]):
        assert close(a, b, tol)


def test_while_with_list_reads_is_not_differentiable():
    with open(os.path.join(GOLDEN, "lbfgs_m3_n50.json")) as f:
        g = ir.from_json(json.load(f)["graph"])
    f64 = [p.attrs["name"] for p in g.main.params if p.out_types[0].dtype == "f64" and p.out_types[0].shape != ()]
    with pytest.raises(NotDifferentiable):
        gradient(g, 1, f64[:1]) if g.main.outputs[1].type.shape == () else gradient(g, 0, f64[:1])


def test_target_and_wrt_checks():
    d = load("ad_rnn_full")
    g = d["graph_obj"]
    with pytest.raises(NotDifferentiable):
        gradient(g, 1, ["w"])            # the i64 trip count is not a scalar f64 target
    with pytest.raises(NotDifferentiable):
        gradient(g, 0, ["nope"])
    with pytest.raises(NotDifferentiable):
        gradient(g, 0, ["lens"])         # i64 parameter


def test_inactive_wrt_gets_zeros():
    d = load("ad_rnn_full")
    gg = gradient(d["graph_obj"], 0, ["limit"])   # only steers the break test
    out = gg.main.outputs[-1].node
    assert out.op == "Mul" and out.inputs[1].node.op == "Const"
    assert gg.count_ops("While") == 1     # no reverse loop needed


@pytest.mark.skipif(importlib.util.find_spec("stagekit") is None and not os.path.isdir("/root/reference/pkg/src"),
                    reason="the reference is not importable here")
@pytest.mark.parametrize("name", NAMES)
def test_reference_executor_runs_gradient_graph(name):
    from oracle.gen_autodiff_golden import run_ref, to_reference
    d = load(name)
    feeds = {k: np.asarray(v.data, dtype=np.int64 if v.dtype == "i64" else np.float64).reshape(v.shape)
             for k, v in d["feed_values"].items()}
    got = run_ref(to_reference(gradient(d["graph_obj"], d["output"], d["wrt"])), feeds)
    tol = d.get("expected_tol", 1e-12)
    assert close(got[0], d["expected"][0], 1e-12)
    for a, b in zip(got[len(got) - len(d["wrt"]):], d["expected"][1:]):
        assert close(a, b, tol)

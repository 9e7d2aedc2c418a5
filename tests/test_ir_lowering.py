"""Host logic without a GPU: the IR wire format, validation, feed binding and
the lowering of reference-traced graphs (tests/golden/*.json) onto the
recurrent kernel."""

import json

import numpy as np
import pytest

from oracle import fixtures
from paper_1810_08061_b200 import errors as E
from paper_1810_08061_b200 import ir
from paper_1810_08061_b200.executor import bind_feeds
from paper_1810_08061_b200.lowering import CELL_GRU, CELL_LSTM, CELL_RNN_TANH, lower_rnn_program
from paper_1810_08061_b200.validate import validate


def _graph(name):
    return ir.from_json(fixtures.load_golden(name)["graph"])


@pytest.mark.parametrize("name", [c["name"] for c in fixtures.CASES])
def test_json_round_trip_is_stable(name):
    doc = fixtures.load_golden(name)["graph"]
    g = ir.from_json(doc)
    again = json.loads(ir.to_json(g))
    assert again == doc


@pytest.mark.parametrize("name", [c["name"] for c in fixtures.CASES])
def test_reference_graphs_validate(name):
    assert validate(_graph(name)) == []


@pytest.mark.parametrize("name", [c["name"] for c in fixtures.CASES])
def test_reference_graphs_lower_to_the_recurrent_kernel(name):
    case = fixtures.case_by_name(name)
    g = _graph(name)
    prog = lower_rnn_program(g)
    assert prog.cell == {"lstm": CELL_LSTM, "gru": CELL_GRU}.get(case["cell"], CELL_RNN_TANH)
    assert prog.x.name == "input_data" and prog.lens.name == "sequence_len"
    if case["cell"] == "gru":   # blocks z, r, n_x = (Wn, -, bn), n_h = (-, Un, bhn)
        names = [tuple(s.name if s is not None else None for s in t) for t in prog.gates]
        assert names == [("wz", "uz", "bz"), ("wr", "ur", "br"), ("wn", None, "bn"), (None, "un", "bhn")]
        assert prog.h0.name == "h0" and prog.c0 is None
    elif case["cell"] == "lstm":
        assert [t[0].name for t in prog.gates] == ["wi", "wf", "wg", "wo"]
        assert [t[1].name for t in prog.gates] == ["ui", "uf", "ug", "uo"]
        assert [t[2].name for t in prog.gates] == ["bi", "bf", "bg", "bo"]
        assert prog.h0.name == "h0" and prog.c0.name == "c0"
    else:
        assert [t.name for t in prog.gates[0]] == ["w_x", "w_h", "b"]
        assert prog.h0.name == "initial_state"
    kinds = [o.kind for o in prog.outputs]
    if case["entry"] == "dynamic_lstm_states":
        assert kinds == ["seq_tm", "h_final", "c_final"]
    else:
        assert kinds == ["seq_bm"]
    assert prog.index_node.op == "Index" and prog.stack_node.op == "ListStack"
    if case["program"] == "rnn_limited.msl":
        assert prog.max_iterations == 4


def test_lowering_rejects_other_programs():
    # while_halve-like scalar loop: While over a scalar f64 state
    g = ir.Graph()
    x = g.main.add_param("x", ir.TypeSpec("f64", ()))
    test, body = ir.Subgraph(), ir.Subgraph()
    tp = test.add_param("x", ir.TypeSpec("f64", ()))
    one = test.add(ir.Node("Const", [], {"value": None}, out_types=[ir.TypeSpec("f64", ())]))
    gt = test.add(ir.Node("Gt", [tp.ref(), one.ref()], {}, out_types=[ir.TypeSpec("bool", ())]))
    test.outputs = [gt.ref()]
    bp = body.add_param("x", ir.TypeSpec("f64", ()))
    body.outputs = [bp.ref()]
    w = g.main.add(ir.Node("While", [x.ref()], {"test_graph": test, "body_graph": body, "n_state": 1,
                                                "n_test_caps": 0, "n_body_caps": 0, "names": ["x"]},
                           out_types=[ir.TypeSpec("f64", ())]))
    g.main.outputs = [w.ref()]
    with pytest.raises(E.LoweringError):
        lower_rnn_program(g)


def test_lowering_rejects_graph_without_loop():
    g = ir.Graph()
    a = g.main.add_param("a", ir.TypeSpec("f64", (2,)))
    n = g.main.add(ir.Node("Tanh", [a.ref()], {}, out_types=[ir.TypeSpec("f64", (2,))]))
    g.main.outputs = [n.ref()]
    with pytest.raises(E.LoweringError):
        lower_rnn_program(g)


def test_bind_feeds_errors_match_reference_kinds():
    g = _graph("lstm_4x8x8")
    feeds = fixtures.make_feeds(fixtures.case_by_name("lstm_4x8x8"))
    bound = bind_feeds(g, feeds)
    assert set(bound) == set(feeds)
    missing = dict(feeds)
    del missing["h0"]
    with pytest.raises(E.RuntimeGraphError) as info:
        bind_feeds(g, missing)
    assert info.value.cause_kind == "MissingFeed"
    bad = dict(feeds, sequence_len=feeds["sequence_len"].astype(np.float64))
    with pytest.raises(E.RuntimeGraphError) as info:
        bind_feeds(g, bad)
    assert info.value.cause_kind == "DtypeMismatch"
    bad = dict(feeds, h0=np.zeros((5, 8)))
    with pytest.raises(E.RuntimeGraphError) as info:
        bind_feeds(g, bad)
    assert info.value.cause_kind == "ShapeMismatch"


def test_validation_error_on_broken_graph():
    g = _graph("rnn_corpus_2x3x4")
    w = [n for n in g.main.nodes if n.op == "While"][0]
    w.inputs = w.inputs[:-1]     # drop a capture
    with pytest.raises(E.ValidationError):
        validate(g)


def test_reference_tensorvalue_feeds_are_accepted():
    """Feeds in the reference's own TensorValue form (row-major tuples)."""
    from paper_1810_08061_b200.values import TensorValue, as_numpy, infer_dtype
    arr = np.arange(6, dtype=np.float64).reshape(2, 3)

    class RefTV:   # duck-typed reference TensorValue (tensor.py:23-48)
        def __init__(self, dtype, shape, data):
            self.dtype, self.shape, self.data = dtype, shape, data

    v = RefTV("f64", (2, 3), tuple(arr.reshape(-1).tolist()))
    assert infer_dtype(v) == "f64"
    np.testing.assert_array_equal(as_numpy(v), arr)
    tv = TensorValue("f64", (2, 3), arr)
    assert tv.data == v.data and str(tv) == "f64[2,3]:0.0,1.0,2.0,3.0,4.0,5.0"

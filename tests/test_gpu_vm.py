"""Region-VM parity on the GPU: the reference's corpus programs (manifest
feeds) and its differential-fuzz programs (harness/fuzz.py), staged by the
reference and executed by `paper_1810_08061_b200.execute`, against the
reference executor's outputs, print logs and failure kinds.  The VM computes
in float64/int64 like the reference: floats within the reference harness's
own 1e-9 tolerance (harness/diff.py:31), ints and bools exact.  The corpus
`dynamic_rnn` lowers to the fused fp16 tensor-core kernel instead (TOL 3e-3)."""

import pytest

from paper_1810_08061_b200 import LoweringError, RuntimeGraphError, execute, ir
from paper_1810_08061_b200.executor import plan_kind
from vm_cases import corpus, feed_value, flatten, fuzz_cases, leaf_equal

pytestmark = pytest.mark.gpu


def _check(graph_doc, feeds_doc, exp, rel=1e-9):
    g = ir.from_json(graph_doc)
    feeds = {k: feed_value(v) for k, v in feeds_doc.items()}
    if "error" in exp:
        with pytest.raises(RuntimeGraphError) as info:
            execute(g, feeds)
        assert info.value.cause_kind == exp["error"]
        return
    res = execute(g, feeds)
    got = flatten(res.outputs)
    assert len(got) == len(exp["outputs"])
    for a, b in zip(got, exp["outputs"]):
        assert leaf_equal(a, b, rel), (a.array if hasattr(a, "array") else a, b)
    assert res.print_log == exp["print_log"]


@pytest.mark.parametrize("prog", corpus(), ids=lambda p: p["name"])
def test_corpus_programs(prog):
    rel = 3e-3 if plan_kind(ir.from_json(prog["graph"])) == "rnn" else 1e-9
    _check(prog["graph"], prog["feeds"], prog["expected"], rel)


CASES = fuzz_cases()


@pytest.mark.parametrize("case", [c for _, c in CASES], ids=[n for n, _ in CASES])
def test_fuzz_programs(case):
    _check(case["graph"], case["feeds"], case["expected"])


@pytest.mark.parametrize("prog", __import__("vm_cases").recursion(), ids=lambda p: p["name"])
def test_recursive_funccall_programs(prog):
    """Recursive FuncCall (reference graph/execute.py:191-193) on the device
    call stack: outputs, print logs (pre-order effects) and the AssertionFailed
    raised 1 call deep equal the reference executor's."""
    _check(prog["graph"], prog["feeds"], prog["expected"])


def test_int64_overflow_is_reported_not_wrapped():
    """The reference's ints are unbounded Python ints; the VM computes in int64
    and raises IntegerOverflow where a result leaves int64 (never wraps)."""
    import numpy as np
    from paper_1810_08061_b200 import sexpr
    from paper_1810_08061_b200.errors import IntegerOverflow
    g = sexpr.from_sexpr("(def main ((x i64)) (mul x x))")
    ok = execute(g, {"x": np.asarray(3_000_000_000, dtype=np.int64)})
    assert int(ok.outputs[0].item()) == 9_000_000_000_000_000_000
    with pytest.raises(IntegerOverflow):
        execute(g, {"x": np.asarray(4_000_000_000, dtype=np.int64)})
    g2 = sexpr.from_sexpr("(def main ((x i64)) (sub x (const i64 2)))")
    with pytest.raises(IntegerOverflow):
        execute(g2, {"x": np.asarray(-(2 ** 63) + 1, dtype=np.int64)})

"""Vector-stream tier parity on the GPU (BASELINE config C4 class).

Programs under oracle/programs/ (L-BFGS with m=3/10, a mixed i64/bool/f64
element-wise program with lists, failure cases) are traced and executed by
the reference (oracle/gen_stream_golden.py); here the same graphs run through
`execute_stream` (csrc/stream.cu) on the GPU.  The tier computes in float64
like the reference, but its reductions combine per-CTA partials instead of
the reference's left-to-right sum (tensor.py:335-341), so floats are compared
within the reference harness's own tolerance (harness/diff.py:31, 1e-9);
trip counts, integers, booleans and failure kinds/spans are exact."""

import numpy as np
import pytest

from oracle import fixtures
from paper_1810_08061_b200 import RuntimeGraphError, execute, ir
from paper_1810_08061_b200.executor import execute_stream, plan_kind
from paper_1810_08061_b200 import stream as st
from vm_cases import flatten, leaf_equal

pytestmark = pytest.mark.gpu
TOL = 1e-9
NAMES = [c["name"] for c in fixtures.STREAM_CASES]


def _load(name):
    doc = fixtures.load_golden(name)
    return ir.from_json(doc["graph"]), fixtures.make_stream_feeds(doc["case"]), doc["expected"]


@pytest.mark.parametrize("name", NAMES)
def test_stream_golden(name):
    g, feeds, exp = _load(name)
    if "error" in exp:
        with pytest.raises(RuntimeGraphError) as info:
            execute_stream(g, feeds)
        assert info.value.cause_kind == exp["error"]
        if exp.get("span"):
            assert info.value.span is not None and info.value.span.start_line == exp["span"][1]
        return
    res = execute_stream(g, feeds)
    got = flatten(res.outputs)
    assert len(got) == len(exp["outputs"])
    for a, b in zip(got, exp["outputs"]):
        assert a.tensor.is_cuda
        assert leaf_equal(a, b, TOL), (a.array, b)


def test_stream_runs_one_launch_with_few_barriers():
    g, feeds, exp = _load("lbfgs_m10_n2000")
    execute_stream(g, feeds)
    info = st.run.last
    k = exp["outputs"][1]["tensor"]["data"][0]
    # one grid exchange per fused reduction group: <= 2m + 2 per iteration
    assert info["barriers"] <= (2 * 10 + 2) * (k + 1), info
    assert info["max_live"] <= info["pool"]


def test_stream_feeds_on_device_zero_copy():
    import torch
    g, feeds, exp = _load("lbfgs_m3_n50")
    dev = {k: (torch.from_numpy(np.asarray(v)).cuda() if np.asarray(v).ndim else v) for k, v in feeds.items()}
    res = execute_stream(g, dev)
    got = flatten(res.outputs)
    for a, b in zip(got, exp["outputs"]):
        assert leaf_equal(a, b, TOL)


def test_auto_dispatch_large_lbfgs_matches_oracle():
    """n = 2^20 through plain `execute` (auto-selects the stream tier) against
    the float64 C restatement of the same L-BFGS program."""
    import oracle
    from paper_1810_08061_b200.executor import _stream_plans  # noqa: F401
    doc = fixtures.load_golden("graph_lbfgs_c4")
    g = ir.from_json(doc["graph"])
    n = 1 << 20
    case = fixtures.stream_case("c4", "lbfgs_m10.msl", "lbfgs", fixtures.lbfgs_feeds(n), 7)
    feeds = fixtures.make_stream_feeds(case)
    assert plan_kind(g, feeds) == "stream"
    res = execute(g, feeds)
    x, k = res.outputs
    xo, ko, margin = oracle.lbfgs(feeds["x0"], feeds["a"], feeds["b"], float(feeds["tol"]), int(feeds["max_iter"]), 10)
    assert int(k.item()) == ko, (k.item(), ko, margin)
    err = np.max(np.abs(x.array - xo) / np.maximum(1.0, np.abs(xo)))
    assert err <= TOL, err

"""Gradients through While on the B200: graphs from
paper_1810_08061_b200.autodiff.gradient() run by `execute` (region VM,
float64) against sources independent of the transform — the reference
executing the hand-written BPTT program (ad_lstm_*), the reference's own
gradient() (ad_maml_h8), and central finite differences (ad_rnn_*, tolerance
1e-6 relative, stated in the fixture) plus the reference executor running the
same gradient graph (1e-9, the reference harness tolerance)."""
import numpy as np
import pytest

from autodiff_cases import NAMES, close, load
from paper_1810_08061_b200 import execute
from paper_1810_08061_b200.autodiff import gradient

pytestmark = pytest.mark.gpu


def _arr(v):
    return np.asarray(v.array if hasattr(v, "array") else v.data, dtype=np.float64).reshape(-1)


@pytest.mark.parametrize("name", NAMES)
def test_gradient_through_while_on_device(name):
    d = load(name)
    g = d["graph_obj"]
    gg = gradient(g, d["output"], d["wrt"])
    res = execute(gg, d["feed_values"])
    outs = [_arr(o) for o in res.outputs]
    nw = len(d["wrt"])
    assert close(outs[d["output"]], d["expected"][0], 1e-9)
    tol = d.get("expected_tol", 1e-9)
    for k, (a, b) in enumerate(zip(outs[-nw:], d["expected"][1:])):
        assert close(a, b, tol), (d["wrt"][k], np.max(np.abs(a - np.asarray(b))))
    for a, b in zip(outs[-nw:], d["via_reference"][-nw:]):
        assert close(a, b, 1e-9)
    if "trips" in d:
        assert int(outs[1][0]) == d["trips"]

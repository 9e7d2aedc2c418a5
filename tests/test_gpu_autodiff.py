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


def test_gradient_medium_shape_matches_bptt_oracle():
    """The automatic BPTT of the staged LSTM loss at T=16, B=32, F=H=64
    (tests/golden/graph_lstm_loss_bench.json, traced by the reference) on the
    region VM against the float64 BPTT restatement (oracle/bptt.py, pinned to
    the reference's hand-written BPTT program) — all 12 gradients, run three
    times: this shape once exposed a VM list-append race (threads disagreeing
    on copy-on-write) that the tiny fixtures did not."""
    from oracle import bptt, fixtures
    from oracle.gen_stream_golden import bptt_feeds
    from paper_1810_08061_b200 import ir
    doc = fixtures.load_golden("graph_lstm_loss_bench")
    g = ir.from_json(doc["graph"])
    wrt = [f"{k}{q}" for q in "ifgo" for k in "wub"]
    gg = gradient(g, 0, wrt)
    v = bptt_feeds(doc["case"])
    feeds = {k: np.asarray(v[k]) for k in doc["order"]}
    W = np.concatenate([v["w" + q] for q in "ifgo"], axis=1)
    U = np.concatenate([v["u" + q] for q in "ifgo"], axis=1)
    b = np.concatenate([v["b" + q][0] for q in "ifgo"])
    loss, dW, dU, db = bptt.forward_backward(np.transpose(v["x"], (1, 0, 2)), v["h0"], v["c0"], v["lens"],
                                             np.transpose(v["y"], (1, 0, 2)), W, U, b, float(v["inv_b"]))
    H = v["h0"].shape[1]
    for _ in range(3):
        outs = [_arr(o) for o in execute(gg, feeds).outputs]
        assert abs(outs[0][0] - loss) < 1e-12
        for k in range(4):
            assert np.allclose(outs[1 + 3 * k].reshape(-1, H), dW[:, k * H:(k + 1) * H], rtol=1e-9, atol=1e-12)
            assert np.allclose(outs[2 + 3 * k].reshape(H, H), dU[:, k * H:(k + 1) * H], rtol=1e-9, atol=1e-12)
            assert np.allclose(outs[3 + 3 * k].reshape(-1, H).sum(axis=0), db[k * H:(k + 1) * H], rtol=1e-9,
                               atol=1e-12)


@pytest.mark.parametrize("shape", [(16, 64, 64, 64), (8, 128, 64, 64)], ids=["T16B64", "T8B128"])
def test_gradient_grid_mode_matches_bptt_oracle(shape):
    """Tensors of >= 64 K elements run the region VM as a grid of CTAs: the
    traced 4x3 LSTM-loss graph with its shapes relaxed, at a larger shape, run
    twice against the f64 BPTT oracle (this once exposed cross-CTA descriptor
    races in the VM)."""
    from oracle import bptt
    from paper_1810_08061_b200.ir import TypeSpec
    d = load("ad_lstm_4x3")
    g = d["graph_obj"]

    def relax(t):
        if t is None or t.dtype == "tree":
            return t
        if t.dtype == "list":
            return TypeSpec("list", None, relax(t.elem))
        return t if t.shape in ((), None) else TypeSpec(t.dtype, tuple(None for _ in t.shape))
    for n in g.iter_nodes():
        n.out_types = [relax(t) for t in n.out_types]
    gg = gradient(g, 0, d["wrt"])
    T, B, F, H = shape
    rng = np.random.default_rng(11)
    v = {"x": rng.uniform(-1, 1, (T, B, F)), "h0": rng.uniform(-.5, .5, (B, H)), "c0": rng.uniform(-.5, .5, (B, H)),
         "lens": rng.integers(0, T + 1, B).astype(np.int64), "y": rng.uniform(-1, 1, (T, B, H))}
    v["lens"][0] = T
    for q in "ifgo":
        v["w" + q] = rng.uniform(-1, 1, (F, H))
        v["u" + q] = rng.uniform(-1, 1, (H, H))
        v["b" + q] = np.broadcast_to(rng.uniform(-.5, .5, (1, H)), (B, H)).copy()
    v["inv_b"] = np.float64(1.0 / B)
    W = np.concatenate([v["w" + q] for q in "ifgo"], axis=1)
    U = np.concatenate([v["u" + q] for q in "ifgo"], axis=1)
    b = np.concatenate([v["b" + q][0] for q in "ifgo"])
    loss, dW, dU, _ = bptt.forward_backward(np.transpose(v["x"], (1, 0, 2)), v["h0"], v["c0"], v["lens"],
                                            np.transpose(v["y"], (1, 0, 2)), W, U, b, float(v["inv_b"]))
    for _ in range(2):
        outs = [_arr(o) for o in execute(gg, v, check=False).outputs]
        assert abs(outs[0][0] - loss) < 1e-9 * max(1.0, abs(loss))
        for k in range(4):
            assert np.allclose(outs[1 + 3 * k].reshape(F, H), dW[:, k * H:(k + 1) * H], rtol=1e-9, atol=1e-11)
            assert np.allclose(outs[2 + 3 * k].reshape(H, H), dU[:, k * H:(k + 1) * H], rtol=1e-9, atol=1e-11)

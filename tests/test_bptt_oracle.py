"""CPU: the float64 LSTM BPTT restatement (oracle/bptt.py, C2) against the
reference executing the hand-derived staged BPTT program
(oracle/programs/lstm_bptt.msl -> tests/golden/lstm_bptt_*.json), and against
central finite differences."""
import numpy as np
import pytest

from oracle import bptt, fixtures
from oracle.gen_stream_golden import BPTT_CASES, bptt_feeds


def _concat(v):
    W = np.concatenate([v["w" + g] for g in "ifgo"], axis=1)
    U = np.concatenate([v["u" + g] for g in "ifgo"], axis=1)
    b = np.concatenate([v["b" + g][0] for g in "ifgo"])
    x = np.transpose(v["x"], (1, 0, 2))
    y = np.transpose(v["y"], (1, 0, 2))
    return x, y, W, U, b


@pytest.mark.parametrize("case", BPTT_CASES, ids=lambda c: c["name"])
def test_bptt_oracle_matches_reference_program(case):
    v = bptt_feeds(case)
    doc = fixtures.load_golden(case["name"])
    outs = [np.asarray(o["data"]).reshape(o["shape"]) for o in doc["outputs"]]
    x, y, W, U, b = _concat(v)
    loss, dW, dU, db = bptt.forward_backward(x, v["h0"], v["c0"], v["lens"], y, W, U, b, float(v["inv_b"]))
    H = v["h0"].shape[1]
    assert abs(loss - float(outs[0])) < 1e-12
    for k, g in enumerate("ifgo"):
        gw, gu, gb = outs[1 + 3 * k], outs[2 + 3 * k], outs[3 + 3 * k]
        assert np.allclose(dW[:, k * H:(k + 1) * H], gw, atol=1e-12)
        assert np.allclose(dU[:, k * H:(k + 1) * H], gu, atol=1e-12)
        assert np.allclose(db[k * H:(k + 1) * H], gb.sum(axis=0), atol=1e-12)


def test_bptt_oracle_finite_differences():
    rng = np.random.default_rng(3)
    B, T, F, H = 3, 5, 4, 3
    x, y = rng.uniform(-1, 1, (B, T, F)), rng.uniform(-1, 1, (B, T, H))
    h0, c0 = rng.uniform(-.5, .5, (B, H)), rng.uniform(-.5, .5, (B, H))
    lens = np.array([5, 2, 0])
    W, U, b = rng.uniform(-1, 1, (F, 4 * H)), rng.uniform(-1, 1, (H, 4 * H)), rng.uniform(-.5, .5, 4 * H)
    _, dW, dU, db = bptt.forward_backward(x, h0, c0, lens, y, W, U, b, 1 / B)
    eps = 1e-6
    for P, dP in ((W, dW), (U, dU), (b, db)):
        for idx in [(0,) * P.ndim, tuple(s - 1 for s in P.shape)]:
            old = P[idx]
            P[idx] = old + eps
            lp = bptt.forward_backward(x, h0, c0, lens, y, W, U, b, 1 / B)[0]
            P[idx] = old - eps
            lm = bptt.forward_backward(x, h0, c0, lens, y, W, U, b, 1 / B)[0]
            P[idx] = old
            assert abs((lp - lm) / (2 * eps) - dP[idx]) < 1e-6 * max(1, abs(dP[idx]))

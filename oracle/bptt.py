"""Float64 CPU restatement of one dynamic-length LSTM training step (BASELINE
config C2) — TEST INFRASTRUCTURE ONLY (checker / CPU baseline).

The reference cannot differentiate a While (graph/grad.py:159-161), so its
BPTT is the hand-derived staged program oracle/programs/lstm_bptt.msl (SURVEY
App. E pattern, LSTM gates): forward While storing states, reverse While.
This module is that program in numpy, with the gates concatenated
(W [F,4H], U [H,4H], b [4H], gate order i,f,g,o): tests/test_bptt_oracle.py
pins it against the reference executing lstm_bptt.msl.

loss = inv_b * sum_t sum_b [t < len_b] <h_{b,t}, y_{b,t}>; rows past their
length keep their state (Where), their gradient flows straight through.
"""
from __future__ import annotations

import numpy as np


def _sig(x):
    return 1.0 / (1.0 + np.exp(-x))


def forward_backward(x, h0, c0, lens, y, W, U, b, inv_b):
    """x [B,T,F] (batch-major), y [B,T,H]; returns (loss, dW, dU, db)."""
    B, T, F = x.shape
    H = h0.shape[1]
    n = int(max(lens.max(initial=0), 0))
    hs, cs, acts = [h0], [c0], []
    h, c = h0, c0
    loss = 0.0
    for t in range(n):
        z = x[:, t] @ W + h @ U + b
        i, f, g, o = _sig(z[:, :H]), _sig(z[:, H:2 * H]), np.tanh(z[:, 2 * H:3 * H]), _sig(z[:, 3 * H:])
        cn = f * c + i * g
        hn = o * np.tanh(cn)
        m = (t < lens)[:, None]
        h = np.where(m, hn, h)
        c = np.where(m, cn, c)
        loss += float(np.sum(np.where(m, h * y[:, t], 0.0))) * inv_b
        hs.append(h)
        cs.append(c)
        acts.append((i, f, g, o, cn))
    dW, dU, db = np.zeros_like(W), np.zeros_like(U), np.zeros_like(b)
    dh, dc = np.zeros_like(h0), np.zeros_like(c0)
    for t in range(n - 1, -1, -1):
        m = (t < lens)[:, None]
        i, f, g, o, cn = acts[t]
        hp, cp = hs[t], cs[t]
        tc = np.tanh(cn)
        dh = dh + np.where(m, y[:, t], 0.0) * inv_b
        dha = np.where(m, dh, 0.0)
        dca = np.where(m, dc, 0.0)
        dcn = dca + dha * o * (1.0 - tc * tc)
        z = np.concatenate([dcn * g * i * (1 - i), dcn * cp * f * (1 - f), dcn * i * (1 - g * g),
                            dha * tc * o * (1 - o)], axis=1)
        dW += x[:, t].T @ z
        dU += hp.T @ z
        db += z.sum(axis=0)
        dh = z @ U.T + np.where(m, 0.0, dh)
        dc = dcn * f + np.where(m, 0.0, dc)
    return loss, dW, dU, db

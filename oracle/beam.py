"""Float64 CPU restatement of the staged decoder (BASELINE config C3) —
TEST INFRASTRUCTURE ONLY (checker / CPU baseline).

The reference IR cannot express beam search (no exp/log/top-k, SURVEY §8(c)
C3; graph/ir.py:19-27), so its semantics are defined here, following the
reference's kernel conventions (k-ordered matmul accumulate tensor.py:302-319,
tanh/stable sigmoid :391-407) and pinned against the reference itself at
beam 1: `decode(cell="rnn", beam=1)` reproduces the staged greedy program
oracle/programs/greedy.msl token for token
(tests/test_decode_oracle.py against tests/golden/greedy_*.json).

Decoder step for every live beam b of sentence s:
    x = emb[tok_b]
    rnn : h' = tanh(x @ w_in + h @ u)                                  (App. F)
    lstm: [i f g o] = [x, h] @ W + bias; c' = f*c + i*g; h' = o*tanh(c')   (App. A gate order)
    logits = h' @ w_out (+ b_out)
    logp = logits - logsumexp(logits)
Candidates: unfinished beam b -> (b, v) for every v with score_b + logp[v];
finished beam b -> only (b, EOS) with score_b.  The K best by score, ties
broken by the lowest flat index b*V + v, become the next beams (parent b,
token v, finished |= v == EOS, length += 0 if the parent had finished else 1).
Step 0 has one live beam per sentence (the others start at -inf).  The loop
stops when every beam of every sentence has finished (EOS) or after max_len
steps — the data-dependent stop of the greedy program's `break`.
"""
from __future__ import annotations

import numpy as np


def _sigmoid(x):
    out = np.empty_like(x)
    pos = x >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-x[pos]))
    e = np.exp(x[~pos])
    out[~pos] = e / (1.0 + e)
    return out


def _mm(a, b):
    """k-ordered accumulation like the reference matmul (tensor.py:302-319)."""
    acc = np.zeros((a.shape[0], b.shape[1]))
    for t in range(a.shape[1]):
        acc += a[:, t:t + 1] * b[t:t + 1, :]
    return acc


def decode(cell, h0, emb, weights, beam, eos, max_len, c0=None, exact=False):
    """h0: [S, H]; emb: [V, E]; weights: rnn (w_in [E,H], u [H,H], w_out [H,V])
    or lstm (W [E+H, 4H], bias [4H], w_out [H,V], b_out [V]).
    Returns dict(tokens [S,K,max_len+1], scores [S,K], lengths [S,K], parents
    [steps,S,K], steps, margins [steps] = smallest score gap at the K-th choice)."""
    mm = _mm if exact else (lambda a, b: a @ b)
    S, H = h0.shape
    V = emb.shape[0]
    K = beam
    h = np.repeat(h0[:, None, :], K, axis=1).reshape(S * K, H).astype(np.float64)
    c = np.zeros_like(h) if c0 is None else np.repeat(c0[:, None, :], K, axis=1).reshape(S * K, H)
    score = np.full((S, K), -np.inf)
    score[:, 0] = 0.0
    tok = np.zeros(S * K, dtype=np.int64)
    fin = np.zeros((S, K), dtype=bool)
    length = np.zeros((S, K), dtype=np.int64)
    hist = np.zeros((S, K, max_len + 1), dtype=np.int64)
    parents, margins = [], []
    t = 0
    while t < max_len and not fin.all():
        x = emb[tok]
        if cell == "rnn":
            w_in, u, w_out = weights[:3]
            hn = np.tanh(mm(x, w_in) + mm(h, u))
            cn = c
            logits = mm(hn, w_out)
        else:
            W, bias, w_out, b_out = weights
            gates = mm(np.concatenate([x, h], axis=1), W) + bias
            i, f, g, o = (gates[:, k * H:(k + 1) * H] for k in range(4))
            cn = _sigmoid(f) * c + _sigmoid(i) * np.tanh(g)
            hn = _sigmoid(o) * np.tanh(cn)
            logits = mm(hn, w_out) + b_out
        mx = logits.max(axis=1, keepdims=True)
        lse = mx + np.log(np.exp(logits - mx).sum(axis=1, keepdims=True))
        logp = (logits - lse).reshape(S, K, V)
        cand = score[:, :, None] + logp
        cand = np.where(fin[:, :, None], -np.inf, cand)
        eos_keep = np.where(fin, score, -np.inf)
        cand[:, :, eos] = np.where(fin, eos_keep, cand[:, :, eos])
        flat = cand.reshape(S, K * V)
        order = np.argsort(-flat, axis=1, kind="stable")[:, :K + 1]   # stable: lowest index wins ties
        sel = order[:, :K]
        new_score = np.take_along_axis(flat, sel, axis=1)
        nxt = np.take_along_axis(flat, order[:, K:K + 1], axis=1)[:, 0]
        with np.errstate(invalid="ignore"):
            gap = new_score[:, -1] - nxt
        margins.append(float(np.nanmin(np.where(np.isfinite(gap), gap, np.inf))))
        par = sel // V
        vtok = sel % V
        rows = (np.arange(S)[:, None] * K + par).reshape(-1)
        pfin = np.take_along_axis(fin, par, axis=1)
        length = np.take_along_axis(length, par, axis=1) + (~pfin)
        hist = np.take_along_axis(hist, par[:, :, None], axis=1)
        hist[:, :, t + 1] = vtok
        fin = pfin | (vtok == eos)
        score = new_score
        h = np.where(pfin.reshape(-1)[:, None], h[rows], hn[rows])
        c = np.where(pfin.reshape(-1)[:, None], c[rows], cn[rows])
        tok = vtok.reshape(-1)
        parents.append(par)
        t += 1
    return {"tokens": hist, "scores": score, "lengths": length, "parents": parents, "steps": t,
            "margins": margins, "finished": fin}

"""Float64 CPU restatement of the TreeLSTM program (oracle/programs/tree_lstm.msl,
SURVEY App. D; BASELINE config C5) — TEST INFRASTRUCTURE ONLY.

node_state(tree): leaf -> c = wc * value, h = tanh(c); internal node with
children (hl, cl), (hr, cr):
    i  = sigmoid(hl@uil + hr@uir + bi)      fl = sigmoid(hl@ufll + hr@uflr + bf)
    fr = sigmoid(hl@ufrl + hr@ufrr + bf)    o  = sigmoid(hl@uol + hr@uor + bo)
    u  = tanh(hl@uul + hr@uur + bu)
    c  = i*u + fl*cl + fr*cr ;  h = o*tanh(c)
in the reference's operation order (matmul k-ordered accumulate, `+` left to
right, two-branch sigmoid: graph/tensor.py:302-319, 397-407), evaluated
recursively like the reference interpreter (tests pin it against
tests/golden/treelstm_*.json, produced by the reference's interpret_module).
"""
from __future__ import annotations

import math

import numpy as np


def _mm(a, b):
    acc = np.zeros((a.shape[0], b.shape[1]))
    for t in range(a.shape[1]):
        acc = acc + a[:, t:t + 1] * b[t:t + 1, :]
    return acc


def _sig(x):
    return np.vectorize(lambda v: 1.0 / (1.0 + math.exp(-v)) if v >= 0 else math.exp(v) / (1.0 + math.exp(v)))(x)


def _tanh(x):
    return np.vectorize(math.tanh)(x)


def node_state(val, left, right, w, i=0):
    if left[i] < 0:
        c = w["wc"] * val[i]
        return _tanh(c), c
    hl, cl = node_state(val, left, right, w, left[i])
    hr, cr = node_state(val, left, right, w, right[i])
    g = lambda a, b, bias: (_mm(hl, w[a]) + _mm(hr, w[b])) + w[bias]
    i_ = _sig(g("uil", "uir", "bi"))
    fl = _sig(g("ufll", "uflr", "bf"))
    fr = _sig(g("ufrl", "ufrr", "bf"))
    o = _sig(g("uol", "uor", "bo"))
    u = _tanh(g("uul", "uur", "bu"))
    c = (i_ * u + fl * cl) + fr * cr
    return o * _tanh(c), c


def forest(trees, w):
    """Batched, level-by-level float64 evaluation with BLAS matmuls (fast;
    used for large CPU baselines).  trees: list of (val, left, right).
    Returns (h_roots [N,H], c_roots [N,H])."""
    H = w["wc"].shape[1]
    U = np.zeros((2 * H, 5 * H))
    for k, (a, b) in enumerate((("uil", "uir"), ("ufll", "uflr"), ("ufrl", "ufrr"), ("uol", "uor"), ("uul", "uur"))):
        U[:H, k * H:(k + 1) * H] = w[a]
        U[H:, k * H:(k + 1) * H] = w[b]
    bias = np.concatenate([w["bi"], w["bf"], w["bf"], w["bo"], w["bu"]])
    vals, lefts, rights, roots = [], [], [], []
    base = 0
    for val, left, right in trees:
        vals.append(val)
        lefts.append(np.where(left >= 0, left + base, -1))
        rights.append(np.where(right >= 0, right + base, -1))
        roots.append(base)
        base += len(val)
    val, left, right = np.concatenate(vals), np.concatenate(lefts), np.concatenate(rights)
    n = len(val)
    height = np.zeros(n, dtype=np.int64)
    for i in range(n - 1, -1, -1):   # pre-order: children after parents
        if left[i] >= 0:
            height[i] = 1 + max(height[left[i]], height[right[i]])
    h = np.zeros((n, H))
    c = np.zeros((n, H))
    leaf = left < 0
    c[leaf] = w["wc"] * val[leaf][:, None]
    h[leaf] = np.tanh(c[leaf])
    for lvl in range(1, int(height.max(initial=0)) + 1):
        idx = np.nonzero(height == lvl)[0]
        g = np.concatenate([h[left[idx]], h[right[idx]]], axis=1) @ U + bias
        sg = lambda x: 1.0 / (1.0 + np.exp(-x))
        i_, fl, fr, o, u = (g[:, k * H:(k + 1) * H] for k in range(5))
        c[idx] = sg(i_) * np.tanh(u) + sg(fl) * c[left[idx]] + sg(fr) * c[right[idx]]
        h[idx] = sg(o) * np.tanh(c[idx])
    return h[roots], c[roots]

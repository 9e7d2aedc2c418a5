"""Float64 CPU restatement of the MAML sinusoid meta-gradient (BASELINE config
C5) — TEST INFRASTRUCTURE ONLY (checker / CPU baseline).

oracle/programs/maml.msl is one task: an MLP 1-H-H-1 with ReLU (`where(z>0,
z, 0*z)`) and biases applied as `matmul(ones, b)`, one hand-written inner SGD
step theta' = theta - alpha * grad L_support(theta), and the query loss
L_q(theta').  The reference's `gradient()` (graph/grad.py:35-70)
differentiates that graph, second order included (tests/golden/maml_*.json).
Here the same derivative in closed form, vectorised over tasks:

    meta_grad = g_q - alpha * H_s g_q,   g_q = grad L_q at theta',
    H_s v = the Pearlmutter R-operator of the support backward pass along v.
"""
from __future__ import annotations

import numpy as np

NAMES = ("w1", "b1", "w2", "b2", "w3", "b3")


def _fwd(x, th):
    z1 = x @ th["w1"] + th["b1"]
    a1 = np.where(z1 > 0, z1, 0.0)
    z2 = a1 @ th["w2"] + th["b2"]
    a2 = np.where(z2 > 0, z2, 0.0)
    p = a2 @ th["w3"] + th["b3"]
    return p, z1, a1, z2, a2


def _bwd(x, th, z1, a1, z2, a2, dp):
    T = lambda a: np.swapaxes(a, -1, -2)
    gw3, gb3 = T(a2) @ dp, dp.sum(axis=-2, keepdims=True)
    dz2 = np.where(z2 > 0, dp @ T(th["w3"]), 0.0)
    gw2, gb2 = T(a1) @ dz2, dz2.sum(axis=-2, keepdims=True)
    dz1 = np.where(z1 > 0, dz2 @ T(th["w2"]), 0.0)
    gw1, gb1 = T(x) @ dz1, dz1.sum(axis=-2, keepdims=True)
    return {"w1": gw1, "b1": gb1, "w2": gw2, "b2": gb2, "w3": gw3, "b3": gb3}, dz1, dz2


def meta_grad(theta, xs, ys, xq, yq, alpha):
    """theta: shared weights (w1 [1,H], b1 [1,H], w2 [H,H], b2 [1,H], w3 [H,1],
    b3 [1,1]); xs, ys, xq, yq: [N, K, 1] per task.  Returns (per-task query
    losses [N], per-task meta-gradients {name: [N, ...]})."""
    T = lambda a: np.swapaxes(a, -1, -2)
    K = xs.shape[1]
    inv_k = 1.0 / K
    p, z1, a1, z2, a2 = _fwd(xs, theta)
    dp = (p - ys) * (2.0 * inv_k)
    g, dz1, dz2 = _bwd(xs, theta, z1, a1, z2, a2, dp)
    th2 = {k: theta[k] - alpha * g[k] for k in NAMES}                     # [N, ...] adapted weights
    q, qz1, qa1, qz2, qa2 = _fwd(xq, th2)
    eq = q - yq
    loss = (eq * eq).sum(axis=(1, 2)) * inv_k
    gq, _, _ = _bwd(xq, th2, qz1, qa1, qz2, qa2, eq * (2.0 * inv_k))      # grad at theta'
    v = gq
    # R-operator of the support pass along v (H_s v)
    m1, m2 = z1 > 0, z2 > 0
    Rz1 = xs @ v["w1"] + v["b1"]
    Ra1 = np.where(m1, Rz1, 0.0)
    Rz2 = Ra1 @ theta["w2"] + a1 @ v["w2"] + v["b2"]
    Ra2 = np.where(m2, Rz2, 0.0)
    Rp = Ra2 @ theta["w3"] + a2 @ v["w3"] + v["b3"]
    Rdp = Rp * (2.0 * inv_k)
    Hv = {"w3": T(Ra2) @ dp + T(a2) @ Rdp, "b3": Rdp.sum(axis=-2, keepdims=True)}
    Rdz2 = np.where(m2, Rdp @ T(theta["w3"]) + dp @ T(v["w3"]), 0.0)
    Hv["w2"] = T(Ra1) @ dz2 + T(a1) @ Rdz2
    Hv["b2"] = Rdz2.sum(axis=-2, keepdims=True)
    Rdz1 = np.where(m1, Rdz2 @ T(theta["w2"]) + dz2 @ T(v["w2"]), 0.0)
    Hv["w1"] = T(xs) @ Rdz1
    Hv["b1"] = Rdz1.sum(axis=-2, keepdims=True)
    return loss, {k: gq[k] - alpha * Hv[k] for k in NAMES}


def init_theta(H, seed):
    rng = np.random.default_rng(seed)
    return {"w1": rng.normal(0, 1.0, (1, H)), "b1": rng.normal(0, 0.1, (1, H)),
            "w2": rng.normal(0, np.sqrt(2.0 / H), (H, H)), "b2": rng.normal(0, 0.1, (1, H)),
            "w3": rng.normal(0, np.sqrt(2.0 / H), (H, 1)), "b3": rng.normal(0, 0.1, (1, 1))}


def sinusoid_tasks(n, K, seed):
    """amplitude U[0.1,5], phase U[0,pi], x U[-5,5]; K support + K query."""
    rng = np.random.default_rng(seed)
    amp, ph = rng.uniform(0.1, 5.0, (n, 1, 1)), rng.uniform(0, np.pi, (n, 1, 1))
    xs, xq = rng.uniform(-5, 5, (n, K, 1)), rng.uniform(-5, 5, (n, K, 1))
    return xs, amp * np.sin(xs + ph), xq, amp * np.sin(xq + ph)

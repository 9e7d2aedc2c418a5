"""Gradient-through-While timing: the autodiff graph of the staged LSTM loss
(tests/golden/ad_lstm_6x4.json) on the region VM (f64) — per-call latency."""
import sys
import time

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from autodiff_cases import load  # noqa: E402
from paper_1810_08061_b200 import execute, gradient  # noqa: E402

for name in ("ad_lstm_4x3", "ad_lstm_6x4", "ad_rnn_full"):
    d = load(name)
    gg = gradient(d["graph_obj"], d["output"], d["wrt"])
    for _ in range(3):
        execute(gg, d["feed_values"])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    n = 20
    for _ in range(n):
        res = execute(gg, d["feed_values"])
    torch.cuda.synchronize()
    print(name, f"{1e3 * (time.perf_counter() - t0) / n:.2f} ms per gradient call (nodes {gg.node_count()})")

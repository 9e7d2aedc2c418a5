"""Gradient through While at a medium shape (T=16, B=32, F=H=64): the
autodiff graph of the staged LSTM loss on the region VM vs the float64
numpy BPTT restatement (oracle/bptt.py) on the host."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import bptt, fixtures  # noqa: E402
from oracle.gen_stream_golden import bptt_feeds  # noqa: E402
from paper_1810_08061_b200 import execute, gradient, ir  # noqa: E402

doc = fixtures.load_golden("graph_lstm_loss_bench")
g = ir.from_json(doc["graph"])
wrt = [f"{k}{q}" for q in "ifgo" for k in "wub"]
gg = gradient(g, 0, wrt)
v = bptt_feeds(doc["case"])
feeds = {k: np.asarray(v[k]) for k in doc["order"]}
res = execute(gg, feeds)
torch.cuda.synchronize()
n = 5
t0 = time.perf_counter()
for _ in range(n):
    res = execute(gg, feeds)
torch.cuda.synchronize()
vm_ms = 1e3 * (time.perf_counter() - t0) / n
W = np.concatenate([v["w" + q] for q in "ifgo"], axis=1)
U = np.concatenate([v["u" + q] for q in "ifgo"], axis=1)
b = np.concatenate([v["b" + q][0] for q in "ifgo"])
x, y = np.transpose(v["x"], (1, 0, 2)), np.transpose(v["y"], (1, 0, 2))
t0 = time.perf_counter()
ref = bptt.forward_backward(x, v["h0"], v["c0"], v["lens"], y, W, U, b, float(v["inv_b"]))
cpu_ms = 1e3 * (time.perf_counter() - t0)
got_w = np.asarray(res.outputs[1].array)
loss_err = abs(ref[0] - float(np.asarray(res.outputs[0].array).reshape(-1)[0]))
grad_err = float(np.max(np.abs(got_w - ref[1][:, :v["h0"].shape[1]])))
print(json.dumps({"vm_ms": vm_ms, "oracle_ms": cpu_ms, "loss_err": loss_err, "dwi_err": grad_err,
                  "loss": float(np.asarray(res.outputs[0].array).reshape(-1)[0]), "ref_loss": float(ref[0])}))

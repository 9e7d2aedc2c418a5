"""Region-VM stress: the traced C1 LSTM program forced onto the VM (grid mode,
x = 32x64x256 elements) against the f64 C oracle, repeated."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
from oracle.fixtures import load_graph_fixture  # noqa: E402
from paper_1810_08061_b200.executor import execute_vm  # noqa: E402

g, _ = load_graph_fixture("graph_lstm_c1")
B, T, F, H = 32, 64, 256, 256
rng = np.random.default_rng(3)
W = [rng.uniform(-0.1, 0.1, (F, H)) for _ in range(4)]
U = [rng.uniform(-0.1, 0.1, (H, H)) for _ in range(4)]
bb = [rng.uniform(-0.1, 0.1, (H,)) for _ in range(4)]
x = rng.uniform(-1, 1, (B, T, F))
h0 = rng.uniform(-0.1, 0.1, (B, H))
c0 = rng.uniform(-0.1, 0.1, (B, H))
lens = rng.integers(1, T + 1, B).astype(np.int64)
feeds = {"input_data": x, "h0": h0, "c0": c0, "sequence_len": lens}
for k, q in enumerate("ifgo"):
    feeds["w" + q], feeds["u" + q], feeds["b" + q] = W[k], U[k], bb[k]
ref, m = oracle.rnn_program(1, x, h0, c0, lens, W, U, bb)
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    t0 = time.perf_counter()
    res = execute_vm(g, feeds)
    torch.cuda.synchronize()
    got = np.asarray(res.outputs[0].array)
    print(f"rep {rep}: {time.perf_counter() - t0:.2f} s, shape {got.shape}, max abs err {np.max(np.abs(got - ref)):.3e}")
